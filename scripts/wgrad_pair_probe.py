"""Device time of the ResNet-18 (batch 512) weight-gradient GEMMs (split-K partials, reduction
excluded), CUDA events over 20 launches.  CVB_GEMM_PAIR_WGRAD=0/1 compares the CTA-pair plan."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2103_16898_b200 import kernels as K  # noqa: E402

SHAPES = [  # n, h, w, cin, cout, k, s, p
    (512, 16, 16, 128, 128, 3, 1, 1), (512, 8, 8, 256, 256, 3, 1, 1), (512, 16, 16, 128, 256, 3, 2, 1),
    (512, 4, 4, 512, 512, 3, 1, 1), (512, 8, 8, 256, 512, 3, 2, 1), (512, 16, 16, 128, 256, 1, 2, 0),
    (128, 56, 56, 128, 32, 3, 1, 1), (128, 28, 28, 128, 32, 3, 1, 1),   # DenseNet conv2
    (512, 32, 32, 32, 32, 3, 1, 1), (512, 16, 16, 32, 64, 3, 1, 1), (512, 16, 16, 64, 64, 3, 1, 1),   # small CNN
    (512, 32, 32, 8, 32, 3, 1, 1), (512, 32, 32, 8, 64, 3, 1, 1),   # stems (8 = 3 padded channels)
]
tag = f"wgrad pair={os.environ.get('CVB_GEMM_PAIR_WGRAD', '1')} grp={0 if os.environ.get('CVB_NO_WGRAD_HALO_GROUPS') else 1}"
for (n, h, w, cin, cout, k, s, p) in SHAPES:
    oh, ow = K.conv_out_hw(h, w, k, s, p)
    x = torch.randn(n, h, w, cin, device="cuda").to(torch.bfloat16)
    dy = torch.randn(n, oh, ow, cout, device="cuda").to(torch.bfloat16)
    part, used = K.conv2d_wgrad_partials(dy, x, k, k, s, p)
    got = part[:used].sum(0)
    xr = x.permute(0, 3, 1, 2).float().requires_grad_(False)
    ref = torch.nn.grad.conv2d_weight(xr, (cout, cin, k, k), dy.permute(0, 3, 1, 2).float(), stride=s, padding=p)
    ref = ref.permute(0, 2, 3, 1).reshape(cout, -1)
    err = (got - ref).abs().max().item() / (ref.abs().max().item() + 1e-6)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        K.conv2d_wgrad_partials(dy, x, k, k, s, p, part=part)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1000
    fl = 2.0 * n * oh * ow * cout * k * k * cin
    print(f"{tag} wgrad {cin}->{cout} k{k} s{s} {h}x{w}: splits {used:3d} {us:7.1f} us  {fl / us / 1e6:7.1f} TF/s  relerr {err:.1e}")
