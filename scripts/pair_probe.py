"""Device time of the ResNet-18 (batch 512) gathered convs: forward and stride-1 dgrad shapes,
CUDA events over 20 back-to-back launches.  Run with CVB_GEMM_PAIR=0/1 (CTA pair off/on) and
CVB_KB_PAIR=0/1 to compare the plans."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2103_16898_b200 import kernels as K  # noqa: E402

SHAPES = [  # n, h, w, cin, cout, k, s, p
    (512, 32, 32, 64, 128, 1, 2, 0), (512, 16, 16, 128, 256, 1, 2, 0), (512, 8, 8, 256, 512, 1, 2, 0),   # downsample
    (512, 32, 32, 8, 64, 3, 1, 1), (512, 32, 32, 64, 64, 3, 1, 1),                                   # ResNet-18 stem, stage 1 (halo)
    (512, 32, 32, 8, 32, 3, 1, 1), (512, 32, 32, 32, 32, 3, 1, 1), (512, 16, 16, 32, 64, 3, 1, 1),   # small CNN (halo)
    (512, 16, 16, 64, 64, 3, 1, 1),
    (512, 16, 16, 128, 128, 3, 1, 1), (512, 32, 32, 64, 128, 3, 2, 1), (512, 32, 32, 64, 128, 1, 2, 0),
    (512, 8, 8, 256, 256, 3, 1, 1), (512, 16, 16, 128, 256, 3, 2, 1),
    (512, 4, 4, 512, 512, 3, 1, 1), (512, 8, 8, 256, 512, 3, 2, 1),
]
tag = f"pair={os.environ.get('CVB_GEMM_PAIR', '1')}/{os.environ.get('CVB_GEMM_PAIR_HALO', '1')} kbpair={os.environ.get('CVB_KB_PAIR', 'auto')}"
for (n, h, w, cin, cout, k, s, p) in SHAPES:
    x = torch.randn(n, h, w, cin, device="cuda").to(torch.bfloat16)
    wt = (torch.randn(cout, k, k, cin, device="cuda") / (k * k * cin) ** 0.5).to(torch.bfloat16)
    y = K.conv2d_fwd(x, wt, s, p)
    ref = torch.nn.functional.conv2d(x.permute(0, 3, 1, 2).float(), wt.permute(0, 3, 1, 2).float(), stride=s, padding=p)
    err = (y.float() - ref.permute(0, 2, 3, 1)).abs().max().item() / (ref.abs().max().item() + 1e-6)
    for _ in range(3):
        K.conv2d_fwd(x, wt, s, p, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        K.conv2d_fwd(x, wt, s, p, out=y)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1000
    oh, ow = y.shape[1], y.shape[2]
    fl = 2.0 * n * oh * ow * cout * k * k * cin
    print(f"{tag} conv {cin}->{cout} k{k} s{s} {h}x{w}: {us:7.1f} us  {fl / us / 1e6:7.1f} TF/s  relerr {err:.1e}")
