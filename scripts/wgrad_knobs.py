"""WGRAD shapes of ResNet-18 / small CNN in isolation (graph-timed)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2103_16898_b200 import kernels as K
from scripts.gemm_micro import timeit

for (n, h, cin, cout, k, s, p) in [(512, 32, 64, 64, 3, 1, 1), (512, 16, 128, 128, 3, 1, 1), (512, 8, 256, 256, 3, 1, 1),
                                   (512, 32, 32, 32, 3, 1, 1), (512, 32, 8, 32, 3, 1, 1), (512, 32, 8, 64, 3, 1, 1)]:
    x = torch.randn(n, h, h, cin, device="cuda").bfloat16()
    oh = (h + 2 * p - k) // s + 1
    dy = torch.randn(n, oh, oh, cout, device="cuda").bfloat16()
    part = torch.empty(148 * cout * k * k * cin, device="cuda")
    ms = timeit(lambda: K.conv2d_wgrad_partials(dy, x, k, k, s, p, part=part.view(148, cout, k * k * cin)))
    fl = 2 * n * oh * oh * cout * k * k * cin
    print(f"wgrad {n}x{h}x{h} {cin}->{cout} k{k}: {ms * 1e3:7.1f} us {fl / ms / 1e9:7.1f} TF/s")
