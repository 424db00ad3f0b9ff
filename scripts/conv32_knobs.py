"""32-channel-group convs (small CNN conv2, DenseNet 1x1 with cin = 32 mod 64) in isolation."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2103_16898_b200 import kernels as K
from scripts.gemm_micro import timeit

for (n, h, cin, cout, k, p) in [(512, 32, 32, 32, 3, 1), (512, 16, 32, 64, 3, 1), (128, 56, 96, 128, 1, 0),
                                (128, 28, 160, 128, 1, 0), (128, 14, 480, 128, 1, 0)]:
    x = torch.randn(n, h, h, cin, device="cuda").bfloat16()
    w = torch.randn(cout, k, k, cin, device="cuda").bfloat16()
    y = torch.empty(n, h, h, cout, device="cuda", dtype=torch.bfloat16)
    ms = timeit(lambda: K.conv2d_fwd(x, w, 1, p, out=y))
    fl = 2 * n * h * h * cout * k * k * cin
    print(f"conv {n}x{h}x{h} {cin}->{cout} k{k}: {ms * 1e3:7.1f} us {fl / ms / 1e9:7.1f} TF/s")
