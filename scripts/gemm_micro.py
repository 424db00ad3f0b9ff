"""Micro-benchmarks of the tcgen05 engine on isolated shapes (CUDA events, warm)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2103_16898_b200 import kernels as K


def timeit(fn, n=20):
    """Device time per call: n calls captured in one CUDA graph (host-side argument
    preparation is outside the measurement, as in the training step's graph replay)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def dense(M, N, Kd, am=0, bm=0, splits=1):
    a = torch.randn(M, Kd, device="cuda").bfloat16() if am == 0 else torch.randn(Kd, M, device="cuda").bfloat16()
    b = torch.randn(N, Kd, device="cuda").bfloat16() if bm == 0 else torch.randn(Kd, N, device="cuda").bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16) if splits == 1 else None
    ms = timeit(lambda: K.gemm(a, b, M, N, Kd, am, bm, out=out, splits=splits))
    print(f"dense M{M} N{N} K{Kd} am{am} bm{bm} s{splits}: {ms * 1e3:8.1f} us  {2 * M * N * Kd / ms / 1e9:7.1f} TF/s")


def conv(n, h, cin, cout, k, s, p):
    x = torch.randn(n, h, h, cin, device="cuda").bfloat16()
    w = torch.randn(cout, k, k, cin, device="cuda").bfloat16()
    oh = (h + 2 * p - k) // s + 1
    y = torch.empty(n, oh, oh, cout, device="cuda", dtype=torch.bfloat16)
    ms = timeit(lambda: K.conv2d_fwd(x, w, s, p, out=y))
    fl = 2 * n * oh * oh * cout * k * k * cin
    print(f"conv n{n} {h}x{h} {cin}->{cout} k{k}s{s}: {ms * 1e3:8.1f} us  {fl / ms / 1e9:7.1f} TF/s  "
          f"{(x.numel() + y.numel()) * 2 / ms / 1e6:7.1f} GB/s")
    dy = torch.randn(n, oh, oh, cout, device="cuda").bfloat16()
    part = torch.empty(148 * cout * k * k * cin, device="cuda")
    ms = timeit(lambda: K.conv2d_wgrad_partials(dy, x, k, k, s, p, part=part.view(148, cout, k * k * cin)))
    print(f"  wgrad: {ms * 1e3:8.1f} us  {fl / ms / 1e9:7.1f} TF/s")


if __name__ == "__main__":
    dense(8192, 256, 8192)
    dense(8192, 128, 8192)
    dense(4096, 4096, 4096)
    dense(512, 256, 4096)
    dense(512, 256, 4096, splits=8)
    conv(512, 32, 32, 32, 3, 1, 1)
    conv(512, 16, 64, 64, 3, 1, 1)
    conv(512, 32, 64, 64, 3, 1, 1)
    conv(256, 8, 256, 256, 3, 1, 1)
