"""Every tcgen05 launch of the small-CNN step in isolation (graph-timed, warm): forward, wgrad
(split-K partials) and dgrad convs of the four conv layers at batch 512, with achieved TF/s
and the HBM-traffic floor (inputs + output once) for comparison."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2103_16898_b200 import kernels as K
from scripts.gemm_micro import timeit

B = 512
LAYERS = [("conv1", 32, 8, 32, 3), ("conv2", 32, 32, 32, 3), ("conv3", 16, 32, 64, 3), ("conv4", 16, 64, 64, 3)]
HBM = 7.0e12
tot = 0.0
for name, h, cin, cout, k in LAYERS:
    x = torch.randn(B, h, h, cin, device="cuda").bfloat16()
    w = torch.randn(cout, k, k, cin, device="cuda").bfloat16() * 0.1
    dy = torch.randn(B, h, h, cout, device="cuda").bfloat16()
    y = torch.empty(B, h, h, cout, device="cuda", dtype=torch.bfloat16)
    dx = torch.empty(B, h, h, cin, device="cuda", dtype=torch.bfloat16)
    wt = torch.randn(cin, k, k, cout, device="cuda").bfloat16() * 0.1
    fl = 2 * B * h * h * cout * k * k * (3 if name == "conv1" else cin)
    part = [None]

    def wg():
        part[0] = K.conv2d_wgrad_partials(dy, x, k, k, 1, 1)

    cases = [("fwd", lambda: K.conv2d_fwd(x, w, 1, 1, out=y), (x.numel() + y.numel()) * 2),
             ("wgrad", wg, (x.numel() + dy.numel()) * 2)]
    if name != "conv1":
        cases.append(("dgrad", lambda: K.conv2d_fwd(dy, wt, 1, 1, out=dx), (dy.numel() + dx.numel()) * 2))
    for what, fn, nb in cases:
        ms = timeit(fn)
        tot += ms
        extra = ""
        if what == "wgrad":
            p, used = part[0]
            extra = f" splits={used}"
        print(f"{name} {what:5s}: {ms * 1e3:7.1f} us  {fl / ms / 1e9:6.1f} TF/s  hbm floor {nb / HBM * 1e6:5.1f} us{extra}")
print(f"total {tot * 1e3:.1f} us")
