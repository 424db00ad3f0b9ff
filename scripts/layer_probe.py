"""Per-launch device time of one eager training step (CUDA events around every launch).

usage: layer_probe.py MODEL [BATCH] [OUT.json]   -- prints the launches sorted by time with
their achieved TF/s (GEMMs) or GB/s (memory-bound kernels), and the graph-replay step time.
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2103_16898_b200 import kernels as K
from paper_2103_16898_b200 import loader, nets
from tests.cnn_parity import gpu_inputs, make_records

model = sys.argv[1] if len(sys.argv) > 1 else "small_cnn"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 512
out = sys.argv[3] if len(sys.argv) > 3 else None
net = nets.make_model(model, seed=0).build(batch)
spec = loader.MEDICAL if model == "densenet121" else loader.CIFAR
rec = make_records(batch, 3, c=spec["c"], h=spec["h"], w=spec["w"], classes=net.num_classes)
x, lab = gpu_inputs(rec, spec)
for _ in range(3):
    net.step(x, lab)
torch.cuda.synchronize()
# graph step time
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    net.step(x, lab)
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    net.step(x, lab)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 20
e0.record()
for _ in range(n):
    g.replay()
e1.record()
torch.cuda.synchronize()
graph_ms = e0.elapsed_time(e1) / n
# instrumented eager step
K.REC.timing, K.REC.records = True, []
net.step(x, lab)
torch.cuda.synchronize()
K.REC.timing = False
rows = K.REC.per_launch()
tot = sum(r[2] for r in rows)
if out:
    Path(out).write_text(json.dumps({"model": model, "batch": batch, "graph_ms": graph_ms,
                                     "launches": [list(r) for r in rows]}, indent=0))
print(f"{model} b{batch}: graph {graph_ms:.3f} ms/step ({batch / graph_ms * 1e3:,.0f} img/s); "
      f"instrumented sum {tot:.3f} ms over {len(rows)} launches")
kinds = {}
for site, kind, ms, fl, nb in rows:
    k = kinds.setdefault(kind, [0, 0.0, 0, 0])
    k[0] += 1
    k[1] += ms
    k[2] += fl
    k[3] += nb
for kind, (c, ms, fl, nb) in sorted(kinds.items(), key=lambda kv: -kv[1][1]):
    rate = f"{fl / ms / 1e9:7.1f} TF/s" if fl else f"{nb / ms / 1e6:7.1f} GB/s"
    print(f"  {kind:10s} {c:4d} launches {ms:8.3f} ms {ms / tot * 100:5.1f}%  {rate}")
print("top launches:")
for i, (site, kind, ms, fl, nb) in sorted(enumerate(rows), key=lambda r: -r[1][2])[:40]:
    rate = f"{fl / ms / 1e9:7.1f} TF/s" if fl else f"{nb / ms / 1e6:7.1f} GB/s"
    print(f"  #{i:3d} {ms * 1e3:8.1f} us {rate}  {kind:9s} {site}  flops={fl:.3g} bytes={nb:.3g}")
