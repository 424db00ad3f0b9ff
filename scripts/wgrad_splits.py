import sys
sys.path.insert(0, '.')
import torch
from paper_2103_16898_b200 import kernels as K
from scripts.gemm_micro import timeit
B = 512
for (h, cin, cout) in [(32, 8, 32), (32, 32, 32), (16, 32, 64), (16, 64, 64)]:
    x = torch.randn(B, h, h, cin, device="cuda").bfloat16()
    dy = torch.randn(B, h, h, cout, device="cuda").bfloat16()
    for ms in (148, 96, 74, 48, 37, 24):
        ms_t = timeit(lambda: K.conv2d_wgrad_partials(dy, x, 3, 3, 1, 1, max_splits=ms))
        p, used = K.conv2d_wgrad_partials(dy, x, 3, 3, 1, 1, max_splits=ms)
        print(f"cin {cin} cout {cout} h {h}: max_splits {ms:3d} used {used:3d}: {ms_t*1e3:6.1f} us")
