"""Isolate what bounds the halo conv: time ResNet-18 stage shapes with the engine's debug
knobs (CVB_GEMM_DBG=1 skips the MMAs, =2 skips the TMA loads; results invalid then)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2103_16898_b200 import kernels as K
from scripts.gemm_micro import timeit

for (n, h, cin, cout) in [(512, 32, 64, 64), (512, 16, 128, 128), (512, 8, 256, 256), (512, 4, 512, 512)]:
    x = torch.randn(n, h, h, cin, device="cuda").bfloat16()
    w = torch.randn(cout, 3, 3, cin, device="cuda").bfloat16()
    y = torch.empty(n, h, h, cout, device="cuda", dtype=torch.bfloat16)
    fl = 2 * n * h * h * cout * 9 * cin
    ms = timeit(lambda: K.conv2d_fwd(x, w, 1, 1, out=y))
    ms2 = timeit(lambda: K.conv2d_fwd(x, w, 1, 1, out=y, accumulate=True))
    print(f"{n}x{h}x{h} {cin}->{cout}: fwd {ms*1e3:7.1f} us {fl/ms/1e9:6.1f} TF/s | accumulate {ms2*1e3:7.1f} us")
