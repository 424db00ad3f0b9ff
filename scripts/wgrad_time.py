"""Time the ResNet-18 / small-CNN weight-gradient shapes (CUDA graph, warm)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2103_16898_b200 import kernels as K  # noqa: E402
from scripts.gemm_micro import timeit  # noqa: E402

for (n, h, cin, cout) in [(512, 32, 64, 64), (512, 16, 64, 64), (512, 16, 128, 128), (512, 8, 256, 256),
                          (512, 4, 512, 512)]:
    x = torch.randn(n, h, h, cin, device="cuda").bfloat16()
    dy = torch.randn(n, h, h, cout, device="cuda").bfloat16()
    part = torch.empty(148, cout, 9 * cin, device="cuda", dtype=torch.float32)
    fl = 2 * n * h * h * cout * 9 * cin
    ms = timeit(lambda: K.conv2d_wgrad_partials(dy, x, 3, 3, 1, 1, part=part))
    print(f"wgrad {n}x{h}x{h} {cin}->{cout}: {ms * 1e3:7.1f} us {fl / ms / 1e9:6.1f} TF/s", flush=True)
