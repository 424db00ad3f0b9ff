"""Pin the CPU oracle before trusting it (runs without a GPU).

The oracle (oracle/gcm_ref.c, oracle/logistic_ref.c) is checked against:
  * FIPS-197 appendix C.3 (AES-256 single block),
  * the GCM spec AES-256 test cases 13-16 and seeded vectors sealed by the reference's own
    covault.crypto.aead_seal (tests/golden/gcm_vectors.json, tests/golden/make_golden.py),
  * DEMO_MODEL_SHA256 of the reference trainer (pkg/tests/test_workload.py:23),
  * the reference-format volume sealed by covault.volume.Volume.put (tests/golden/volume_demo).
"""
import hashlib
import json

import numpy as np
import pytest

from oracle import ref
from paper_2103_16898_b200 import workload
from paper_2103_16898_b200.volume import Volume, aad_for

DEMO_MODEL_SHA256 = "7e799c1f44492be596de4727ead2d0a9877d2699a12e88ebcf20b9a6f514607c"


def test_fips197_c3():
    key = bytes(range(32))
    assert ref.aes256_block(key, bytes.fromhex("00112233445566778899aabbccddeeff")).hex() == \
        "8ea2b7ca516745bfeafc49904b496089"


def test_gcm_vectors_seal_and_open(gcm_vectors):
    for v in gcm_vectors:
        key, iv, aad, pt = (bytes.fromhex(v[k]) for k in ("key", "iv", "aad", "pt"))
        blob = bytes.fromhex(v["ct"] + v["tag"])
        assert ref.gcm_seal(key, iv, aad, pt) == blob, v["name"]
        assert ref.gcm_open(key, iv, aad, blob) == pt, v["name"]


def test_gcm_every_bit_flip_fails():
    # mirrors pkg/tests/test_crypto.py:129-136
    key, iv = bytes(range(32)), bytes(12)
    blob = ref.gcm_seal(key, iv, b"aad", b"thirty-two bytes of plaintext!!!")
    for bit in range(len(blob) * 8):
        m = bytearray(blob)
        m[bit // 8] ^= 1 << (bit % 8)
        with pytest.raises(ref.OracleAuthFailure):
            ref.gcm_open(key, iv, b"aad", bytes(m))


def test_gcm_matches_reference_library_random():
    cryptography = pytest.importorskip("cryptography.hazmat.primitives.ciphers.aead")
    rng = np.random.default_rng(5)
    for n in [0, 1, 16, 17, 1023, 5000]:
        key, iv = rng.bytes(32), rng.bytes(12)
        aad, pt = rng.bytes(int(rng.integers(0, 50))), rng.bytes(n)
        assert ref.gcm_seal(key, iv, aad, pt) == cryptography.AESGCM(key).encrypt(iv, pt, aad)


def test_logistic_oracle_reproduces_demo_digest(golden):
    params = json.loads((golden / "demo_params.json").read_text())
    X, y = workload.parse_dataset_arrays((golden / "demo_dataset.csv").read_text())
    w, b = ref.logistic_train(X, y, params["learning_rate"], params["epochs"])
    assert hashlib.sha256(workload.serialize_model(list(w), b)).hexdigest() == DEMO_MODEL_SHA256


def test_logistic_oracle_matches_reference_trainer_random():
    cw = pytest.importorskip("covault.workload")
    rng = np.random.default_rng(11)
    X = np.round(rng.normal(size=(37, 5)), 4)
    y = (rng.random(37) > 0.5).astype(float)
    csv = "\n".join(",".join(repr(float(v)) for v in row) + f",{int(l)}" for row, l in zip(X, y))
    want = cw.run_training({"learning_rate": 0.3, "epochs": 17}, csv)
    Xp, yp = workload.parse_dataset_arrays(csv)
    w, b = ref.logistic_train(Xp, yp, 0.3, 17)
    assert workload.serialize_model(list(w), b) == want


def test_golden_volume_opens_with_oracle(golden):
    meta = json.loads((golden / "volume_demo.json").read_text())
    vol = Volume.open(golden / "volume_demo")
    key = bytes.fromhex(meta["key"])
    for path in vol.paths():
        e = vol.entry(path)
        pt = ref.gcm_open(key, e.nonce, aad_for(vol.volume_name, path), vol.read_blob(path))
        assert hashlib.sha256(pt).hexdigest() == meta["plaintext_sha256"][path]


def test_parse_dataset_mirrors_reference():
    # pkg/tests/test_workload.py:55-65
    with pytest.raises(workload.WorkloadError):
        workload.parse_dataset("only-one-field\n")
    with pytest.raises(workload.WorkloadError):
        workload.parse_dataset("")
    with pytest.raises(workload.WorkloadError):
        workload.parse_dataset("1,2,0\n1,2,3,0\n")
    assert workload.parse_dataset("# header\n\n1,2,1\n# tail\n") == [([1.0, 2.0], 1.0)]


def test_model_serialization_round_trip():
    w, b = [0.25, -1.5, 3.0], 0.125
    assert workload.deserialize_model(workload.serialize_model(w, b)) == (w, b)


def test_shard_rows_partitions_in_order():
    from paper_2103_16898_b200.workload import shard_rows

    for n in (0, 1, 5, 60, 2001):
        for world in (1, 2, 3, 8):
            blocks = [shard_rows(n, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))
            assert max(h - l for l, h in blocks) - min(h - l for l, h in blocks) <= 1


def test_standalone_model_format_matches_reference():
    """The standalone restatements of serialize/deserialize/predict (used without covault)
    produce exactly the reference's bytes and values (workload.py:74-93)."""
    import pytest

    cw = pytest.importorskip("covault.workload")
    w, b = [0.5, -1.25, 3.0e-7], -0.125
    assert workload._serialize_model(w, b) == cw.serialize_model(w, b)
    assert workload._deserialize_model(cw.serialize_model(w, b)) == cw.deserialize_model(cw.serialize_model(w, b))
    for x in ([1.0, 2.0, 3.0], [-4.0, 0.0, 1e9]):
        assert workload._predict(w, b, x) == cw.predict(w, b, x)
