"""Fused classifier head (csrc/head.cu, K.head_train) vs a torch fp32 reference of the same op
on identical bf16 inputs, and vs the unfused gemm/softmax/col_sum launches inside a model step.

Tolerances: logits/row losses are fp32 sums of bf16 products (accumulation order differs from
torch: 1e-5 relative); dlogits are bf16-rounded (one bf16 ulp where a rounding boundary falls
between the two fp32 values); dx is a bf16 output (4e-3 relative); dW, db, colsum(dx) are fp32
sums over the batch (1e-4 relative, driven by the dlogits ulp flips)."""
import pytest
import torch
import torch.nn.functional as F

from paper_2103_16898_b200 import kernels as K
from paper_2103_16898_b200 import nets

pytestmark = pytest.mark.gpu
dev = "cuda"


def rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-12)).item()


def run_head(B, fin, C, relu, gb=None, ldx=None):
    g = torch.Generator(device=dev).manual_seed(B * 7 + fin + C)
    ldx = ldx or fin
    xs = torch.randn(B, ldx, device=dev, generator=g)
    if relu:
        xs = xs.clamp_min(0)
    x = xs.bfloat16()
    w = torch.zeros(16, fin, device=dev)
    w[:C] = torch.randn(C, fin, device=dev, generator=g) / fin ** 0.5
    w = w.bfloat16()
    bias = torch.zeros(16, device=dev)
    bias[:C] = torch.randn(C, device=dev, generator=g) * 0.1
    lab = torch.randint(0, C, (B,), device=dev, generator=g, dtype=torch.int32)
    scale = 1.0 / (gb or B)
    out = dict(logits=torch.empty(B, 16, device=dev), dlogits=torch.empty(B, 16, device=dev, dtype=torch.bfloat16),
               row_loss=torch.empty(B, device=dev), loss=torch.empty(1, device=dev),
               dw=torch.empty(16, fin, device=dev), db=torch.empty(16, device=dev),
               dx=torch.empty(B, fin, device=dev, dtype=torch.bfloat16), dprev=torch.empty(fin, device=dev))
    part = torch.empty(K.head_workspace_floats(B, fin), device=dev)
    K.head_train(x[:, :fin] if ldx == fin else x, w, bias, lab, B, C, scale, out["logits"], out["dlogits"],
                 out["row_loss"], out["loss"], out["dw"], out["db"], part, dx=out["dx"], relu_mask=relu,
                 dprev_b=out["dprev"])
    torch.cuda.synchronize()
    return x[:, :fin].float(), w.float(), bias, lab.long(), scale, out


@pytest.mark.parametrize("B,fin,C,relu,ldx", [(512, 256, 10, True, None), (512, 512, 10, False, None),
                                              (128, 1024, 14, False, None), (1000, 256, 16, True, None),
                                              (7, 256, 2, False, None), (4096, 512, 10, False, None),
                                              (512, 256, 10, True, 512)])
def test_head_train_vs_torch(B, fin, C, relu, ldx):
    x, w, bias, lab, scale, o = run_head(B, fin, C, relu, ldx=ldx)
    logits = x @ w.t() + bias
    assert rel(o["logits"], logits) < 1e-5
    assert torch.all(o["logits"][:, C:] == 0)
    lr = logits[:, :C].clone().requires_grad_(True)
    rows = F.cross_entropy(lr, lab, reduction="none")
    assert rel(o["row_loss"], rows) < 1e-5
    assert abs(o["loss"].item() - rows.mean().item()) < 1e-5 * max(1.0, abs(rows.mean().item()))
    (rows.sum() * scale).backward()
    dl = lr.grad
    # bf16 rounding of dlogits: at most one ulp apart from the bf16 rounding of torch's value
    dk = o["dlogits"].float()[:, :C]
    assert torch.all(o["dlogits"][:, C:] == 0)
    assert torch.all((dk - dl.bfloat16().float()).abs() <= dl.abs() * 2 ** -7 + 1e-30)
    # backward from the kernel's own (bf16) dlogits: the op is dx = dl W, dW = dl^T x
    dlb = o["dlogits"].float()
    dx = dlb @ w
    if relu:
        dx = dx * (x > 0)
    assert rel(o["dx"], dx) < 4e-3
    assert rel(o["dw"], dlb.t() @ x) < 1e-4
    assert rel(o["db"], dlb.sum(0)) < 1e-4
    assert rel(o["dprev"], o["dx"].float().sum(0)) < 1e-5


def test_head_train_deterministic():
    a = run_head(4096, 256, 10, True)[-1]
    b = run_head(4096, 256, 10, True)[-1]
    for k in a:
        assert torch.equal(a[k], b[k]), k


def test_head_train_rejects_bad_shapes():
    x = torch.zeros(8, 100, device=dev, dtype=torch.bfloat16)
    w = torch.zeros(16, 100, device=dev, dtype=torch.bfloat16)
    f = lambda *s: torch.zeros(*s, device=dev)  # noqa: E731
    with pytest.raises(RuntimeError):
        K.head_train(x, w, f(16), torch.zeros(8, device=dev, dtype=torch.int32), 8, 10, 0.125, f(8, 16),
                     f(8, 16).bfloat16(), f(8), f(1), f(16, 100), f(16), f(10000))


@pytest.mark.parametrize("model,batch", [("small_cnn", 256), ("resnet18", 64)])
def test_fused_head_matches_unfused_step(model, batch):
    from tests.cnn_parity import gpu_inputs, make_records
    from paper_2103_16898_b200 import loader
    a = nets.make_model(model, seed=3).build(batch)
    b = nets.make_model(model, seed=3).build(batch)
    assert a.fused_head
    b.fused_head = False
    rec = make_records(batch, 5, c=3, h=32, w=32, classes=a.num_classes)
    x, lab = gpu_inputs(rec, loader.CIFAR)
    # one forward+backward: same loss, logits, gradients (bf16 rounding flips of dlogits / dx
    # propagate through the backward, hence 2e-3 on the gradient vector)
    a.fwd_bwd(x, lab)
    b.fwd_bwd(x, lab)
    torch.cuda.synchronize()
    assert abs(a.loss.item() - b.loss.item()) < 1e-5 * max(1.0, abs(b.loss.item()))
    assert rel(a.logits, b.logits) < 1e-5
    assert rel(a.ps.g32, b.ps.g32) < 2e-3
    # and the loss curves of a few full steps agree
    for _ in range(3):
        a.step(x, lab)
        b.step(x, lab)
    torch.cuda.synchronize()
    assert abs(a.loss.item() - b.loss.item()) < 1e-2 * max(1.0, abs(b.loss.item()))


@pytest.mark.parametrize("model,batch", [("small_cnn", 128), ("resnet18", 32)])
def test_wgrad_side_stream_overlap_is_bit_exact(model, batch, monkeypatch):
    """Weight gradients on the side stream (single GPU) == the serial order, bit for bit."""
    from tests.cnn_parity import gpu_inputs, make_records
    from paper_2103_16898_b200 import loader
    a = nets.make_model(model, seed=5).build(batch)
    b = nets.make_model(model, seed=5).build(batch)
    rec = make_records(batch, 9, c=3, h=32, w=32, classes=a.num_classes)
    x, lab = gpu_inputs(rec, loader.CIFAR)
    monkeypatch.setattr(nets, "_NO_OVERLAP", False)
    a.fwd_bwd(x, lab)
    assert a.ps.side is None and a._side is not None   # the side stream was used and joined
    monkeypatch.setattr(nets, "_NO_OVERLAP", True)
    b.fwd_bwd(x, lab)
    torch.cuda.synchronize()
    assert torch.equal(a.ps.g32, b.ps.g32)
    assert torch.equal(a.loss, b.loss)
