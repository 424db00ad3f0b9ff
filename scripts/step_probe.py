"""Quick device-time probe of one training step (eager and CUDA-graph replay)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2103_16898_b200 import nets
from tests.cnn_parity import gpu_inputs, make_records
from paper_2103_16898_b200 import loader

model = sys.argv[1] if len(sys.argv) > 1 else "small_cnn"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 512
net = nets.make_model(model, seed=0).build(batch)
spec = loader.MEDICAL if model == "densenet121" else loader.CIFAR
rec = make_records(batch, 3, c=spec["c"], h=spec["h"], w=spec["w"], classes=net.num_classes)
x, lab = gpu_inputs(rec, spec)
for _ in range(3):
    net.step(x, lab)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 20
e0.record()
for _ in range(n):
    net.step(x, lab)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print(f"{model} b{batch} eager: {ms:.3f} ms/step  {batch / ms * 1e3:,.0f} img/s  loss {net.loss.item():.4f}")
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
e0.record()
for _ in range(n):
    g.replay()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print(f"{model} b{batch} graph: {ms:.3f} ms/step  {batch / ms * 1e3:,.0f} img/s  loss {net.loss.item():.4f}")
