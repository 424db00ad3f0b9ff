"""Phase timeline of one fused BN backward launch (CVB_BN_TRACE=1) at the small-CNN / ResNet
layer sizes: per-CTA globaltimer stamps at start / pass-1 done / partials / barrier 1 /
finalise / barrier 2 / end (medians over CTAs, us from the earliest start)."""
import ctypes
import os
import sys
from pathlib import Path

os.environ["CVB_BN_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2103_16898_b200 import _lib, kernels as K  # noqa: E402

L = _lib.load()
L.cvb_bn_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
names = ["start", "pass1", "partials", "barrier1", "finalise", "barrier2", "end"]
for rows, C in [(524288, 32), (131072, 64), (8192, 512), (524288, 64)]:
    z = torch.randn(rows, C, device="cuda").bfloat16()
    dy = torch.randn(rows, C, device="cuda").bfloat16()
    dx = torch.empty_like(z)
    g, b = torch.rand(C, device="cuda") + 0.5, torch.randn(C, device="cuda") * 0.1
    mean, rstd = z.float().mean(0), 1 / z.float().std(0)
    dg, db = torch.empty(C, device="cuda"), torch.empty(C, device="cuda")
    ws = K.bn_workspace(rows, C)
    for _ in range(5):
        K.bn_backward(dy, C, z, C, rows, C, mean, rstd, g, b, ws, dg, db, relu=True, dx=dx, dxcs=C)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        K.bn_backward(dy, C, z, C, rows, C, mean, rstd, g, b, ws, dg, db, relu=True, dx=dx, dxcs=C)
    e1.record()
    torch.cuda.synchronize()
    grid = 296
    buf = np.zeros(8 * grid, dtype=np.int64)
    assert L.cvb_bn_debug_trace(buf.ctypes.data, grid) == 0
    t = buf.reshape(grid, 8)[:, :7].astype(np.float64)
    t = t[t[:, 0] > 0]
    rel = (t - t[:, 0].min()) / 1000.0
    print(f"rows {rows} C {C} ({e0.elapsed_time(e1) / 10 * 1000:.1f} us/launch): " +
          " | ".join(f"{n} {np.median(rel[:, k]):.2f}/{rel[:, k].max():.2f}" for k, n in enumerate(names)))
