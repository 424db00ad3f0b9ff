"""Device time of single conv launches captured in a CUDA graph (no host launch overhead):
DenseNet dense-layer shapes by default.  usage: graph_conv_probe.py [dense|r18]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2103_16898_b200 import kernels as K  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "dense"
if which == "dense":
    SHAPES = [(128, 56, 56, cin, 128, 1, 1, 0) for cin in (64, 128, 256)] + [(128, 56, 56, 128, 32, 3, 1, 1)]
    SHAPES += [(128, 28, 28, cin, 128, 1, 1, 0) for cin in (128, 256, 512)] + [(128, 28, 28, 128, 32, 3, 1, 1)]
    SHAPES += [(128, 14, 14, 512, 128, 1, 1, 0), (128, 14, 14, 128, 32, 3, 1, 1), (128, 7, 7, 128, 32, 3, 1, 1)]
else:
    SHAPES = [(512, 32, 32, 8, 64, 3, 1, 1), (512, 32, 32, 64, 64, 3, 1, 1), (512, 16, 16, 128, 128, 3, 1, 1),
              (512, 32, 32, 64, 128, 1, 2, 0)]
for (n, h, w, cin, cout, k, s, p) in SHAPES:
    x = torch.randn(n, h, w, cin, device="cuda").to(torch.bfloat16)
    wt = (torch.randn(cout, k, k, cin, device="cuda") / (k * k * cin) ** 0.5).to(torch.bfloat16)
    y = K.conv2d_fwd(x, wt, s, p)
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            for _ in range(10):
                K.conv2d_fwd(x, wt, s, p, out=y)
    torch.cuda.current_stream().wait_stream(st)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 50 * 1000
    oh, ow = y.shape[1], y.shape[2]
    fl = 2.0 * n * oh * ow * cout * k * k * cin
    mb = (x.numel() + y.numel()) * 2 / 1e6
    print(f"conv {cin}->{cout} k{k} s{s} {h}x{w} n{n}: {us:7.1f} us  {fl / us / 1e6:7.1f} TF/s  "
          f"{mb / us:5.2f} TB/s (x+y {mb:.0f} MB)")
