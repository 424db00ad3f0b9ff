"""Phase timeline of one fused BN forward launch (CVB_BN_TRACE=1): per-CTA globaltimer stamps at
start / pass-1 done / partials written / barrier 1 / finalise done / barrier 2 / end."""
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
for rows, C in [(8192, 512), (32768, 256), (131072, 64), (524288, 64)]:
    z = torch.randn(rows, C, device="cuda").bfloat16()
    y = torch.empty_like(z)
    g, b = torch.rand(C, device="cuda") + 0.5, torch.randn(C, device="cuda") * 0.1
    mean, rstd = torch.empty(C, device="cuda"), torch.empty(C, device="cuda")
    ws = K.bn_workspace(rows, C)
    for _ in range(5):
        K.bn_forward(z, rows, C, C, ws, mean, rstd, g, b, y, C)
    torch.cuda.synchronize()
    grid = 296
    buf = np.zeros(8 * grid, dtype=np.int64)
    assert L.cvb_bn_debug_trace(buf.ctypes.data, grid) == 0
    t = buf.reshape(grid, 8)[:, :7].astype(np.float64)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1000.0
    print(f"rows {rows} C {C}: " + " | ".join(f"{n} med {np.median(rel[:, k]):.2f} max {rel[:, k].max():.2f}"
                                           for k, n in enumerate(names)) + " (us)")
