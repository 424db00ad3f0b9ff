"""Shared CNN parity harness: GPU training steps vs the CPU restatement (oracle/cnn_ref.py).

Tolerances (stated in DESIGN.md), bf16-emulating oracle (same rounding points as the GPU):
  step-0 loss                     |dL| <= 1e-3 * max(1, |L|)
  later losses (curve overlay)    |dL| <= 5e-2 * max(1, |L|)
  step-0 full gradient vector     cosine >= 0.99
  step-0 conv/FC weight grads     ||g_gpu - g_ref|| <= GRAD_TOL[model] * ||g_ref||
  all weights after the steps     ||w_gpu - w_ref|| <= 1e-2 * ||w_ref||  (whole vector)
Why per-tensor gradient bounds are loose: fp32 summation-order noise (TMEM vs CPU blocking)
flips a few bf16 roundings per layer and a flipped near-zero pre-activation toggles its ReLU
mask, moving a whole gradient element (batch 32: ~3 of 8192 FC1 units, ~5% norm).  After
one Adam step (every weight moves by ~lr) the two runs are different trajectories, so only
the loss curve is compared.  Kernel parity on identical inputs is tight
(tests/test_umma_gpu.py, tests/test_nn_kernels_gpu.py).
Plain fp32 oracle (bf16 vs fp32): per-step loss within 2e-2 relative.
"""
from __future__ import annotations

import numpy as np
import torch

from oracle.cnn_ref import RefTrainer, normalise_records
from paper_2103_16898_b200 import loader, nets

LOSS_TOL = 1e-3
CURVE_TOL = 2e-2
# Adam's first steps move every weight by ~lr; at the paper's lr=1e-3 the loss jumps from
# 2.3 to ~3.8 on these synthetic batches, which turns rounding noise into trajectory
# divergence.  Parity of the multi-step update is therefore checked at lr=1e-4 (same code
# path; lr is a kernel argument); the bench and the loss-decrease test use 1e-3.
PARITY_LR = 1e-4
# deep BN/ReLU stacks amplify the flips: 17 layers (ResNet-18) -> cos 0.97, 121 layers at
# batch 8 (DenseNet-121) -> cos 0.86; the layer compositions themselves are checked on
# identical inputs in tests/test_blocks_gpu.py (<= 5% per gradient).
COS_MIN = {"small_cnn": 0.99, "resnet18": 0.95, "densenet121": 0.80}
GRAD_TOL = {"small_cnn": 0.15, "resnet18": 0.40, "densenet121": 0.80}
W_TOL = 1e-2
FP32_LOSS_TOL = 2e-2


def make_records(n, seed, c=3, h=32, w=32, classes=10):
    """Learnable synthetic records: per-class template + noise."""
    rng = np.random.default_rng(seed)
    templ = np.random.default_rng(0).normal(size=(classes, c * h * w))
    labels = rng.integers(0, classes, size=n)
    px = np.clip(np.round(128 + 40 * templ[labels] + 30 * rng.normal(size=(n, c * h * w))), 0, 255).astype(np.uint8)
    return np.concatenate([labels.astype(np.uint8)[:, None], px], axis=1)


def gpu_inputs(rec: np.ndarray, spec):
    pt = torch.from_numpy(rec.reshape(-1).copy()).cuda()
    x, lab = loader.decode_records(pt, rec.shape[0], spec["c"], spec["h"], spec["w"], spec["mean"], spec["std"])
    return x, lab


def rel(a, b):
    return (a - b).norm().item() / max(b.norm().item(), 1e-12)


def run_parity(model="small_cnn", batch=32, steps=3, seed=0, emulate=True, lr=PARITY_LR):
    spec = loader.MEDICAL if model == "densenet121" else loader.CIFAR
    classes = 2 if model == "densenet121" else 10
    net = nets.make_model(model, seed=seed).build(batch)
    net.lr = lr
    state0 = net.ps.state_cpu()
    ref = RefTrainer(model, state0, emulate_bf16=emulate, lr=lr)
    report = []
    for s in range(steps):
        rec = make_records(batch, seed * 100 + s, c=spec["c"], h=spec["h"], w=spec["w"], classes=classes)
        x, lab = gpu_inputs(rec, spec)
        xr, labr = normalise_records(torch.from_numpy(rec), spec["c"], spec["h"], spec["w"], spec["mean"],
                                     spec["std"], emulate_bf16=emulate)
        loss_gpu = float(net.step(x, lab).item())
        g_gpu = {k: v.detach().cpu() for k, v in net.ps.g.items()}
        loss_ref, g_ref = ref.step(xr, labr)
        grads = {}
        va, vb = [], []
        for k, gr in g_ref.items():
            name = k.replace("__", ".")
            grads[name] = rel(g_gpu[name].float(), gr.float())
            va.append(g_gpu[name].float().reshape(-1))
            vb.append(gr.float().reshape(-1))
        va, vb = torch.cat(va), torch.cat(vb)
        cos = float(torch.dot(va, vb) / (va.norm() * vb.norm()).clamp_min(1e-30))
        report.append(dict(step=s, loss_gpu=loss_gpu, loss_ref=loss_ref, grads=grads, cos=cos))
    w_gpu = net.ps.state_cpu()
    w_ref = ref.state()
    a = torch.cat([w_gpu[k].reshape(-1) for k in w_ref])
    b = torch.cat([w_ref[k].reshape(-1) for k in w_ref])
    return report, rel(a, b)


def check(report, wrel, model):
    r0 = report[0]
    assert abs(r0["loss_gpu"] - r0["loss_ref"]) <= LOSS_TOL * max(1.0, abs(r0["loss_ref"])), r0
    assert r0["cos"] >= COS_MIN[model], r0["cos"]
    bad = {k: v for k, v in r0["grads"].items() if k.endswith(".w") and v > GRAD_TOL[model]}
    assert not bad, bad
    for r in report[1:]:
        assert abs(r["loss_gpu"] - r["loss_ref"]) <= CURVE_TOL * max(1.0, abs(r["loss_ref"])), r
    assert wrel <= W_TOL, wrel


# ---- mask-matched, teacher-forced per-step parity ------------------------------------------
# Every step starts the oracle from the GPU's pre-step weights and Adam moments, and the
# oracle's ReLU masks and max-pool arg-max positions are the GPU's own (read back from the
# GPU's stored activations after its step).  What remains is pure arithmetic noise (fp32
# summation order, bf16 rounding of a different fp32 sum), so each step's loss, EVERY
# per-tensor gradient and every updated weight tensor are held to tight relative bounds:
FORCED_LOSS_TOL = 1e-3      # |dL| <= 1e-3 * max(1, |L|)
# ||g_gpu - g_ref|| <= tol * ||g_ref|| for EVERY parameter tensor (conv/FC weights, BN gamma/beta).
# Measured maxima (B200, seeds below): small CNN 7.3e-3 (batch 64) / 3.9e-3 (batch 512);
# ResNet-18 1.55e-2 at batch 512 -- what is left is bf16 re-rounding of slightly different fp32
# sums through 17 BN/ReLU layers (the masks are matched).  Round 1 allowed 15% / 40%.
FORCED_GRAD_TOL = {"small_cnn": 1e-2, "resnet18": 2.5e-2}
# Adam applied to the GPU's own gradient (torch.optim.Adam semantics, fp32) reproduces the GPU's
# updated weights to fp32 rounding: the optimiser kernel itself, per tensor.
ADAM_SAME_GRAD_TOL = 1e-5
# The updated weights vs the oracle's own step (its gradient), whole parameter vector: Adam's
# first steps move every weight by ~lr whatever the gradient's size, so a near-zero gradient
# element whose sign differs moves by 2 lr -- bounded relative to the weights, not per element.
FORCED_W_TOL = {"small_cnn": 5e-3, "resnet18": 1e-2}   # measured: ResNet-18 batch 512 5.4e-3


def _nchw(t):
    return t.detach().float().cpu().permute(0, 3, 1, 2).contiguous()


def pool2_argmax(x_nchw):
    """First arg-max (window order (0,0),(0,1),(1,0),(1,1)) of every 2x2/stride-2 window, the
    tie rule of csrc/nn.cu maxpool2_bwd."""
    n, c, h, w = x_nchw.shape
    win = x_nchw.reshape(n, c, h // 2, 2, w // 2, 2).permute(0, 1, 2, 4, 3, 5).reshape(n, c, h // 2, w // 2, 4)
    return win.argmax(dim=-1)


def gpu_forcing(net, model):
    """(ReLU masks, pool arg-max) of the GPU's last forward, keyed by oracle site names."""
    if model == "small_cnn":
        acts = {"conv1": net.a1, "conv2": net.a2, "conv3": net.a3, "conv4": net.a4}
        masks = {k: (_nchw(v) > 0).float() for k, v in acts.items()}
        masks["fc1"] = (net.h.detach().float().cpu() > 0).float()
        return masks, {"pool1": pool2_argmax(_nchw(net.a2)), "pool2": pool2_argmax(_nchw(net.a4))}
    if model == "resnet18":
        masks = {"stem": (_nchw(net.x0) > 0).float()}
        for i, (b, o) in enumerate(zip(net.blocks, net.outs)):
            nm = f"layer{i // 2 + 1}.{i % 2}"
            masks[f"{nm}.conv1"] = (_nchw(b.o1) > 0).float()
            masks[f"{nm}.conv2"] = (_nchw(o) > 0).float()
        return masks, {}
    raise ValueError(f"no mask matching for {model}")


def _moment_views(ps, buf):
    return {name: buf[ps.offsets[name]:ps.offsets[name] + int(np.prod(shape))].view(shape).detach().cpu().clone()
            for name, shape, _ in ps.specs}


def _adam_same_grad(ps, w_pre, m_pre, v_pre, step, lr, g):
    """torch.optim.Adam (b 0.9/0.999, eps 1e-8) on CPU from the pre-step state with gradient g."""
    out = {}
    for name, shape, _ in ps.specs:
        p = torch.nn.Parameter(w_pre[name].clone().float())
        opt = torch.optim.Adam([p], lr=lr, betas=(0.9, 0.999), eps=1e-8, foreach=False)
        if step > 0:
            opt.state[p] = {"step": torch.tensor(float(step)), "exp_avg": m_pre[name].clone(),
                            "exp_avg_sq": v_pre[name].clone()}
        p.grad = g[name].clone().float()
        opt.step()
        out[name] = p.detach()
    return out


def run_forced(model="small_cnn", batch=64, steps=3, seed=0, lr=1e-3):
    """Per step: dict(loss_gpu, loss_ref, grads={param: rel err}, adam={param: rel err of the GPU
    update vs Adam on the GPU's own gradient}, wvec=whole-vector rel err vs the oracle's step)."""
    spec = loader.CIFAR
    net = nets.make_model(model, seed=seed).build(batch)
    net.lr = lr
    ref = RefTrainer(model, net.ps.state_cpu(), emulate_bf16=True, lr=lr)
    out = []
    for s in range(steps):
        rec = make_records(batch, seed * 100 + s, c=spec["c"], h=spec["h"], w=spec["w"])
        x, lab = gpu_inputs(rec, spec)
        xr, labr = normalise_records(torch.from_numpy(rec), spec["c"], spec["h"], spec["w"], spec["mean"],
                                     spec["std"], emulate_bf16=True)
        k = int(net.ps.step_dev.item())
        w_pre = net.ps.state_cpu()
        m_pre, v_pre = _moment_views(net.ps, net.ps.m), _moment_views(net.ps, net.ps.v)
        ref.load(w_pre, m_pre, v_pre, step=k)
        loss_gpu = float(net.step(x, lab).item())
        torch.cuda.synchronize()
        ref.model.force(*gpu_forcing(net, model))
        loss_ref, g_ref = ref.step(xr, labr)
        w_gpu, w_ref = net.ps.state_cpu(), ref.state()
        g_gpu = {name: net.ps.g[name].detach().float().cpu() for name, _, _ in net.ps.specs}
        w_same = _adam_same_grad(net.ps, w_pre, m_pre, v_pre, k, lr, g_gpu)
        grads, adam = {}, {}
        for key, gr in g_ref.items():
            name = key.replace("__", ".")
            grads[name] = rel(g_gpu[name], gr.float())
            adam[name] = rel(w_gpu[name].float(), w_same[name])
        a = torch.cat([w_gpu[k_].reshape(-1).float() for k_ in w_ref])
        b = torch.cat([w_ref[k_].reshape(-1).float() for k_ in w_ref])
        out.append(dict(loss_gpu=loss_gpu, loss_ref=loss_ref, grads=grads, adam=adam, wvec=rel(a, b)))
    return out


def check_forced(out, model):
    for s, r in enumerate(out):
        assert abs(r["loss_gpu"] - r["loss_ref"]) <= FORCED_LOSS_TOL * max(1.0, abs(r["loss_ref"])), (s, r)
        bad = {k: v for k, v in r["grads"].items() if v > FORCED_GRAD_TOL[model]}
        assert not bad, (s, bad)
        bad = {k: v for k, v in r["adam"].items() if v > ADAM_SAME_GRAD_TOL}
        assert not bad, (s, bad)
        assert r["wvec"] <= FORCED_W_TOL[model], (s, r["wvec"])


# Free-running overlay at the paper's lr 1e-3, 20 Adam steps, no forcing:
# both runs are their own trajectories (Adam turns rounding noise in tiny gradients into full
# lr-sized moves), so the loss curves are compared with an absolute-or-relative bound.
# Measured: max |dL| / max(1, |L|) = 0.085 over 20 steps (small CNN, batch 64), final weights 4.7e-2.
FREE_CURVE_TOL = 0.1
FREE_W_TOL = 0.1


def one_step_check(batch=16, model="small_cnn"):
    report, wrel = run_parity(model, batch=batch, steps=2)
    check(report, wrel, model)
