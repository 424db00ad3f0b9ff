"""Layer-by-layer comparison of the SmallCNN step against the CPU restatement (debug aid)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import torch.nn.functional as F

from oracle.cnn_ref import RefTrainer, normalise_records
from paper_2103_16898_b200 import loader, nets
from tests.cnn_parity import gpu_inputs, make_records, rel

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
net = nets.make_model("small_cnn", seed=0).build(B)
ref = RefTrainer("small_cnn", net.ps.state_cpu())
rec = make_records(B, 0)
x, lab = gpu_inputs(rec, loader.CIFAR)
xr, labr = normalise_records(torch.from_numpy(rec), 3, 32, 32, (0.5,) * 3, (0.25,) * 3)
print("input", rel(x[..., :3].float().cpu().permute(0, 3, 1, 2), xr))

# oracle forward with retained intermediates
m = ref.model
acts = {}
a = m.conv_bn(xr, "conv1", 1, 1, cin_real=3); a.retain_grad(); acts["a1"] = a
a = m.conv_bn(a, "conv2", 1, 1); a.retain_grad(); acts["a2"] = a
p1 = F.max_pool2d(a, 2); p1.retain_grad(); acts["p1"] = p1
a = m.conv_bn(p1, "conv3", 1, 1); a.retain_grad(); acts["a3"] = a
a = m.conv_bn(a, "conv4", 1, 1); a.retain_grad(); acts["a4"] = a
p2 = F.max_pool2d(a, 2); p2.retain_grad(); acts["p2"] = p2
flat = m.R.rb(p2.permute(0, 2, 3, 1).reshape(B, -1))
h = m.linear(flat, "fc1", 256, relu=True); h.retain_grad(); acts["h"] = h
logits = m.linear(h, "fc2", 10, out_f32=True); logits.retain_grad(); acts["logits"] = logits
loss = F.cross_entropy(m.R.rbg(logits), labr)
loss.backward()

net.forward(x)
net.loss_and_grad(lab)
net.backward(x)
torch.cuda.synchronize()
print("loss", loss.item(), net.loss.item())
nchw = lambda t: t.float().cpu().permute(0, 3, 1, 2)  # noqa: E731
pairs = [("a1", net.a1), ("a2", net.a2), ("p1", net.p1), ("a3", net.a3), ("a4", net.a4), ("p2", net.p2)]
for name, g in pairs:
    print(f"fwd {name:6s} {rel(nchw(g), acts[name].detach()):.3e}")
print(f"fwd h      {rel(net.h.float().cpu(), acts['h'].detach()):.3e}")
print(f"fwd logits {rel(net.logits[:, :10].cpu(), acts['logits'].detach()):.3e}")
print(f"bwd dlogit {rel(net.dlogits[:, :10].float().cpu(), acts['logits'].grad.bfloat16().float()):.3e}")
hm = (acts["h"].detach() > 0).float()
print(f"bwd dh     {rel(net.dh.float().cpu(), acts['h'].grad.bfloat16().float() * hm):.3e}  (masked)")
# isolate the GEMMs with torch on the GPU copies
W2 = net.ps.b["fc2.w"].float()
dh_t = (net.dlogits.float() @ W2).bfloat16().float() * (net.h.float() > 0).float()
print(f"gemm dh vs torch(gpu operands) {rel(net.dh.float(), dh_t):.3e}")
W1 = net.ps.b["fc1.w"].float()
dp2_t = (net.dh.float() @ W1)
print(f"gemm dp2 vs torch(gpu operands) {rel(net.dp2.view(B, -1).float(), dp2_t):.3e}")
gw1 = net.dh.float().t() @ net.p2.view(B, -1).float()
print(f"gemm dW1 vs torch(gpu operands) {rel(net.ps.g['fc1.w'], gw1):.3e}")
print("dh nonzero frac", (net.dh != 0).float().mean().item(), "ref", (acts['h'].grad * hm != 0).float().mean().item())
bw = [("p2", net.dp2), ("a4", net.da4), ("a3", net.da3), ("p1", net.dp1), ("a2", net.da2), ("a1", net.da1)]
for name, g in bw:
    print(f"bwd d{name:5s} {rel(nchw(g), acts[name].grad):.3e}")
for k, p in m.params.items():
    print(f"grad {k:14s} {rel(net.ps.g[k.replace('__', '.')].cpu(), p.grad):.3e}")
