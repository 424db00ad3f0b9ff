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


def one_step_check(batch=16, model="small_cnn"):
    report, wrel = run_parity(model, batch=batch, steps=2)
    check(report, wrel, model)
