"""GPU reference trainer: bit-exact against DEMO_MODEL_SHA256 and the oracle
(mirrors pkg/tests/test_workload.py:26-65)."""
import hashlib
import json

import numpy as np
import pytest

from oracle import ref
from paper_2103_16898_b200 import workload

pytestmark = pytest.mark.gpu
DEMO_MODEL_SHA256 = "7e799c1f44492be596de4727ead2d0a9877d2699a12e88ebcf20b9a6f514607c"


def test_demo_fixture_digest(golden):
    params = json.loads((golden / "demo_params.json").read_text())
    model = workload.run_training(params, (golden / "demo_dataset.csv").read_text())
    assert hashlib.sha256(model).hexdigest() == DEMO_MODEL_SHA256


def test_same_inputs_twice_identical():
    params = {"learning_rate": 0.2, "epochs": 25}
    csv = "1.0,2.0,1\n-1.0,-2.0,0\n0.5,0.1,1\n"
    assert workload.run_training(params, csv) == workload.run_training(params, csv)


def test_model_actually_separates():
    csv = "\n".join([f"{x},{x+0.5},1" for x in (1.0, 1.5, 2.0, 2.5)] +
                    [f"{x},{x-0.5},0" for x in (-1.0, -1.5, -2.0, -2.5)])
    w, b = workload.deserialize_model(workload.run_training({"learning_rate": 0.5, "epochs": 200}, csv))
    assert workload.predict(w, b, [2.0, 2.5]) > 0.5
    assert workload.predict(w, b, [-2.0, -2.5]) < 0.5


@pytest.mark.parametrize("n,f,epochs", [(1, 1, 3), (257, 3, 5), (1000, 3072, 2), (64, 50176, 1)])
def test_exact_mode_matches_oracle_bitwise(n, f, epochs):
    rng = np.random.default_rng(n + f)
    X = np.round(rng.random((n, f)), 4)
    y = (rng.random(n) > 0.5).astype(np.float64)
    w0, b0 = ref.logistic_train(X, y, 0.1, epochs)
    w1, b1 = workload.train_arrays(X, y, 0.1, epochs, exact=True)
    assert np.array_equal(w0.view(np.uint64), w1.view(np.uint64)) and b0 == b1


def test_fast_mode_within_tolerance():
    rng = np.random.default_rng(1)
    X = np.round(rng.random((5000, 3072)), 4)
    y = (rng.random(5000) > 0.5).astype(np.float64)
    w0, b0 = ref.logistic_train(X, y, 0.1, 3)
    w1, b1 = workload.train_arrays(X, y, 0.1, 3, exact=False)
    assert np.max(np.abs(w1 - w0)) <= 1e-9 * max(1.0, np.max(np.abs(w0)))
    assert abs(b1 - b0) <= 1e-9 * max(1.0, abs(b0))


def test_reference_api_drop_in():
    """install() routes covault.workload.run_training to the GPU; golden digest holds."""
    cw = pytest.importorskip("covault.workload")
    import covault.crypto as cc
    import covault.volume as cv
    from paper_2103_16898_b200 import install

    saved = (cw.run_training, cc.aead_open, cc.aead_seal, cv.aead_open, cv.aead_seal)
    try:
        install()
        assert cw.run_training is workload.run_training
        golden = __import__("pathlib").Path(__file__).parent / "golden"
        params = json.loads((golden / "demo_params.json").read_text())
        model = cw.run_training(params, (golden / "demo_dataset.csv").read_text())
        assert hashlib.sha256(model).hexdigest() == DEMO_MODEL_SHA256
        # the reference Volume now decrypts through the GPU AEAD
        key = cc.SymmetricKey(bytes(range(32)))
        vol = cv.Volume.open(golden / "volume_demo")
        assert vol.get(key, "dataset.csv") == (golden / "demo_dataset.csv").read_bytes()
    finally:
        cw.run_training, cc.aead_open, cc.aead_seal, cv.aead_open, cv.aead_seal = saved
