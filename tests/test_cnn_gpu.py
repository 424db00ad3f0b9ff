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
