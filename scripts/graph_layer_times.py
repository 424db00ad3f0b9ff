"""In-graph device time of every launch of one kernel class in a training step.

usage: graph_layer_times.py MODEL [BATCH] [CLASS]   (CLASS default umma_gemm)

For launch j of the class, the step is captured as a CUDA graph in which every other launch is
a no-op (kernels.ONLY_CLASSES + ONLY_INDEX) and the graph is replayed 20x under CUDA events: the
launch's time inside a graph, warm, without launch gaps.  The eager instrumented step (REC)
supplies each launch's call site and algorithmic flops / bytes.
"""
import sys
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2103_16898_b200 import kernels as K  # noqa: E402
from paper_2103_16898_b200 import loader, nets  # noqa: E402
from tests.cnn_parity import gpu_inputs, make_records  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 512
kind = sys.argv[3] if len(sys.argv) > 3 else "umma_gemm"
net = nets.make_model(model, seed=0).build(batch)
spec = loader.MEDICAL if model == "densenet121" else loader.CIFAR
rec = make_records(batch, 3, c=spec["c"], h=spec["h"], w=spec["w"], classes=net.num_classes)
x, lab = gpu_inputs(rec, spec)
for _ in range(3):
    net.step(x, lab)
torch.cuda.synchronize()
K.REC.timing, K.REC.records = True, []
net.step(x, lab)
torch.cuda.synchronize()
K.REC.timing = False
rows = [r for r in K.REC.per_launch() if r[1] == kind]


def graph_ms(reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            net.step(x, lab)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


warnings.filterwarnings("ignore", message="The CUDA Graph is empty")
K.ONLY_CLASSES = {kind}
K.ONLY_INDEX = -1
K.ONLY_SEEN.clear()
base = graph_ms()            # every launch filtered out: the empty step's cost
names = list(K.ONLY_SEEN)
n = len(names)
print(f"{model} b{batch} class {kind}: {n} launch calls (REC rows {len(rows)}), empty graph {base * 1e3:.1f} us")
tot = 0.0
for j in range(n):
    K.ONLY_INDEX = j
    K.ONLY_SEEN.clear()
    ms = graph_ms() - base
    tot += ms
    site, fl, nb = (rows[j][0], rows[j][3], rows[j][4]) if len(rows) == n else ("?", 0, 0)
    rate = f"{fl / ms / 1e9:7.1f} TF/s" if fl and ms > 0 else (f"{nb / ms / 1e6:7.1f} GB/s" if nb and ms > 0 else "")
    print(f"  #{j:3d} {ms * 1e3:8.1f} us {rate:>13s}  {names[j]:28s} {site}")
K.ONLY_CLASSES, K.ONLY_INDEX = None, None
print(f"sum {tot:.3f} ms")
