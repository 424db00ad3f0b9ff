"""Fused BN kernels in isolation (CUDA-graph timed) over the models' layer shapes:
achieved GB/s against the minimal traffic (fwd: read z + write y; bwd: read dy, z, y + write dx)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2103_16898_b200 import kernels as K
from scripts.gemm_micro import timeit

for rows, C in [(524288, 32), (524288, 64), (131072, 64), (131072, 128), (32768, 256), (8192, 512)]:
    z = torch.randn(rows, C, device="cuda").bfloat16()
    y = torch.empty_like(z)
    dy = torch.randn(rows, C, device="cuda").bfloat16()
    dx = torch.empty_like(z)
    g, b = torch.rand(C, device="cuda") + 0.5, torch.randn(C, device="cuda") * 0.1
    mean, rstd, dg, db = (torch.empty(C, device="cuda") for _ in range(4))
    ws = K.bn_workspace(rows, C)
    f = lambda: K.bn_forward(z, rows, C, C, ws, mean, rstd, g, b, y, C)  # noqa: E731
    ms_f = timeit(f)
    bwd = lambda: K.bn_backward(dy, C, z, C, rows, C, mean, rstd, g, b, ws, dg, db, y=y, ycs=C, dx=dx, dxcs=C)  # noqa
    ms_b = timeit(bwd)
    mb = rows * C * 2 / 1e6
    print(f"rows {rows:7d} C {C:4d} ({mb:6.1f} MB/tensor): fwd {ms_f * 1e3:7.1f} us {4 * mb / ms_f / 1e3:7.0f} GB/s(min) | "
          f"bwd {ms_b * 1e3:7.1f} us {8 * mb / ms_b / 1e3:7.0f} GB/s(min)")
