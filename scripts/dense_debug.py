"""Per-tensor gradient difference: DenseNet deferred BN input gradient vs per-layer accumulation."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2103_16898_b200 import nets  # noqa: E402
from tests import cnn_parity as P  # noqa: E402

rec = P.make_records(8, 11, c=1, h=224, w=224, classes=2)
x, lab = P.gpu_inputs(rec, P.loader.MEDICAL)
gs = []
for accum in (False, True):
    if accum:
        os.environ["CVB_DENSE_ACCUM"] = "1"
    net = nets.make_model("densenet121", seed=3).build(8)
    net.fwd_bwd(x, lab)
    torch.cuda.synchronize()
    gs.append({k: v.clone() for k, v in net.ps.g.items()})
    names = [s[0] for s in net.ps.specs]
a, b = gs
bad = 0
for k in reversed(names):
    d = ((a[k] - b[k]).norm() / b[k].norm().clamp_min(1e-30)).item()
    if d > 1e-6:
        bad += 1
        if bad < 12:
            print(f"{k:60s} {d:.3e}  |g| {b[k].norm().item():.3e}")
print("tensors differing:", bad, "of", len(names))
