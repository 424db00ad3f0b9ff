"""CNN training-step parity on the B200 vs the CPU restatement (tolerances: tests/cnn_parity.py)."""
import pytest
import torch

from tests import cnn_parity as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("model,batch", [("small_cnn", 32), ("small_cnn", 64), ("resnet18", 16), ("densenet121", 8)])
def test_train_steps_match_bf16_emulating_oracle(model, batch):
    report, wrel = P.run_parity(model, batch=batch, steps=3)
    P.check(report, wrel, model)


def test_loss_curve_vs_fp32_oracle():
    report, _ = P.run_parity("small_cnn", batch=64, steps=5, emulate=False)
    for r in report:
        assert abs(r["loss_gpu"] - r["loss_ref"]) <= P.FP32_LOSS_TOL * max(1.0, abs(r["loss_ref"])), r


def test_loss_decreases():
    from paper_2103_16898_b200 import nets

    net = nets.make_model("small_cnn", seed=1).build(128)
    rec = P.make_records(128, 5)
    x, lab = P.gpu_inputs(rec, P.loader.CIFAR)
    losses = [float(net.step(x, lab).item()) for _ in range(30)]
    assert losses[-1] < 0.5 * losses[0], losses


def test_configs1_full_batch_loss_curve():
    """BASELINE configs[1] at its own size: small CNN, batch 512, fp32 accumulate -- the GPU
    loss curve over 4 steps tracks the CPU restatement (bf16-emulating oracle: tolerances of
    tests/cnn_parity.py; plain fp32 oracle: 2e-2 relative per step)."""
    report, wrel = P.run_parity("small_cnn", batch=512, steps=4)
    P.check(report, wrel, "small_cnn")
    report32, _ = P.run_parity("small_cnn", batch=512, steps=4, emulate=False)
    for r in report32:
        assert abs(r["loss_gpu"] - r["loss_ref"]) <= P.FP32_LOSS_TOL * max(1.0, abs(r["loss_ref"])), r


@pytest.mark.parametrize("model,batch,steps", [("small_cnn", 64, 3), ("small_cnn", 512, 3), ("resnet18", 512, 1)])
def test_mask_matched_per_step_parity(model, batch, steps):
    """Teacher-forced, mask-matched steps at the paper's lr 1e-3: per-step loss <= 1e-3, every
    per-tensor gradient within FORCED_GRAD_TOL, the GPU Adam == torch Adam on the same gradient,
    updated weights within FORCED_W_TOL of the oracle's step (tests/cnn_parity.py)."""
    P.check_forced(P.run_forced(model, batch=batch, steps=steps), model)


def test_free_running_20_steps_lr_1e3():
    report, wrel = P.run_parity("small_cnn", batch=64, steps=20, lr=1e-3)
    for r in report:
        assert abs(r["loss_gpu"] - r["loss_ref"]) <= P.FREE_CURVE_TOL * max(1.0, abs(r["loss_ref"])), r
    assert report[-1]["loss_gpu"] < 0.2 * report[0]["loss_gpu"]        # both actually learn
    assert wrel <= P.FREE_W_TOL, wrel


@pytest.mark.timeout(1800)
def test_densenet_batch128_step0():
    """configs[3]'s batch (128): the step-0 loss and full-gradient direction vs the oracle."""
    report, _ = P.run_parity("densenet121", batch=128, steps=1)
    r = report[0]
    assert abs(r["loss_gpu"] - r["loss_ref"]) <= P.LOSS_TOL * max(1.0, abs(r["loss_ref"])), r
    assert r["cos"] >= P.COS_MIN["densenet121"], r["cos"]


def test_records_to_nhwc_bit_exact_vs_oracle():
    """The GPU record decode (csrc/loader.cu and the fused K1b kernel's arithmetic) == the
    oracle's normalise_records, bit for bit, CIFAR and medical shapes."""
    from oracle.cnn_ref import normalise_records

    for spec, classes in ((P.loader.CIFAR, 10), (P.loader.MEDICAL, 2)):
        rec = P.make_records(64 if spec is P.loader.CIFAR else 8, 3, c=spec["c"], h=spec["h"], w=spec["w"],
                             classes=classes)
        x, lab = P.gpu_inputs(rec, spec)
        xr, labr = normalise_records(torch.from_numpy(rec), spec["c"], spec["h"], spec["w"], spec["mean"],
                                     spec["std"], emulate_bf16=True)
        got = x[..., :spec["c"]].float().cpu().permute(0, 3, 1, 2)
        assert torch.equal(got.view(torch.int32), xr.contiguous().view(torch.int32))
        assert torch.equal(lab.long().cpu(), labr)


def test_fused_decrypt_decode_bit_exact_vs_oracle():
    """The fused decrypt-and-normalise kernel (K1b, gcm_kernel<open, decode>) on a shard sealed by
    the reference's AES-GCM (cryptography.AESGCM, crypto.py:262) == oracle normalise_records."""
    from cryptography.hazmat.primitives.ciphers.aead import AESGCM

    from oracle.cnn_ref import normalise_records
    from paper_2103_16898_b200.crypto import GcmContext

    spec = P.loader.CIFAR
    rec = P.make_records(96, 11)
    key, nonce, aad = bytes(range(32)), bytes(range(12)), b"training-data\x00shard-00000.bin"
    blob = AESGCM(key).encrypt(nonce, rec.tobytes(), aad)
    ctx = GcmContext(key)
    ct = torch.frombuffer(bytearray(blob), dtype=torch.uint8).cuda()
    aad_d = torch.frombuffer(bytearray(aad), dtype=torch.uint8).cuda()
    tile = torch.zeros(96, 32, 32, 8, dtype=torch.bfloat16, device="cuda")
    lab = torch.empty(96, dtype=torch.int32, device="cuda")
    work = ctx.new_workspace()
    ctx.open_records_device(nonce, aad_d, ct, tile, lab, work, spec)
    assert ctx.status_ok(work)
    xr, labr = normalise_records(torch.from_numpy(rec), 3, 32, 32, spec["mean"], spec["std"], emulate_bf16=True)
    got = tile[..., :3].float().cpu().permute(0, 3, 1, 2).contiguous()
    assert torch.equal(got.view(torch.int32), xr.contiguous().view(torch.int32))
    assert torch.equal(lab.long().cpu(), labr)
    assert torch.count_nonzero(tile[..., 3:]) == 0


def test_densenet_deferred_bn_gradient_matches_accumulating_form(monkeypatch):
    """DenseNet's deferred BN input gradient (statistics pass per layer + one gather per channel
    range, csrc/bn_fused.cu bn_gather_dx) reproduces the per-layer fp32-accumulating form: same
    terms, same order, same (uncontracted) roundings -> bit-identical gradients."""
    from paper_2103_16898_b200 import nets

    rec = P.make_records(8, 11, c=1, h=224, w=224, classes=2)
    x, lab = P.gpu_inputs(rec, P.loader.MEDICAL)
    grads = []
    # default (deferred gradient, slice statistics merged into the next BN's launch), then the
    # per-layer accumulating backward, then a separate slice-statistics launch as well
    for env in (None, "CVB_DENSE_ACCUM", "CVB_DENSE_SLICE_STATS"):
        if env:
            monkeypatch.setenv(env, "1")
        net = nets.make_model("densenet121", seed=3).build(8)
        assert net.deferred == (env is None) and net.merge_stats == (env != "CVB_DENSE_SLICE_STATS")
        net.fwd_bwd(x, lab)
        torch.cuda.synchronize()
        grads.append(net.ps.g32.clone())
    a = grads[0]
    assert torch.isfinite(a).all()
    for b in grads[1:]:
        assert torch.equal(a, b), ((a - b).norm() / b.norm()).item()
