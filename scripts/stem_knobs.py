"""Stem conv (3 channels padded to 8) forward: small CNN (->32) and ResNet-18 (->64) shapes."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2103_16898_b200 import kernels as K
from scripts.gemm_micro import timeit

for cout in (32, 64):
    x = torch.randn(512, 32, 32, 8, device="cuda").bfloat16()
    w = torch.randn(cout, 3, 3, 8, device="cuda").bfloat16()
    y = torch.empty(512, 32, 32, cout, device="cuda", dtype=torch.bfloat16)
    ms = timeit(lambda: K.conv2d_fwd(x, w, 1, 1, out=y))
    print(f"stem 512x32x32 8->{cout}: {ms * 1e3:7.1f} us  {(x.numel() + y.numel()) * 2 / ms / 1e6:7.1f} GB/s")
