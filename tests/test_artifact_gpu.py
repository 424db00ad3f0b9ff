"""The B200 workload artifact run by the reference's own attestation harness
(covault.runtime.attested_workload_run -> TeeSimulator.launch -> stdin key injection),
mirroring pkg/tests/test_workload.py:68-176 with the GPU trainer inside the "enclave"."""
import hashlib
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
cv = pytest.importorskip("covault")

from covault.crypto import SigningKey, hash_bytes  # noqa: E402
from covault.manager import PolicyManager  # noqa: E402
from covault.policy import KeyGrant, SecurityPolicy, VolumeDecl, sign_policy  # noqa: E402
from covault.runtime import attested_workload_run, owner_fetch_keys  # noqa: E402
from covault.tee import TeeSimulator, measure_code, pack_tree  # noqa: E402
from covault.volume import Volume  # noqa: E402

from paper_2103_16898_b200.workload_main import make_artifact  # noqa: E402

DEMO = "7e799c1f44492be596de4727ead2d0a9877d2699a12e88ebcf20b9a6f514607c"


def _policy(name, sk, meas, volumes=(), grants=(), exec_command="python train.py"):
    return sign_policy(SecurityPolicy(name=name, exec=exec_command, code_measurement=meas,
                                      volumes=tuple(VolumeDecl(n, d) for n, d in volumes),
                                      key_grants=tuple(KeyGrant(v, g) for v, g in grants),
                                      platform_requirement=None, creator_public_key=sk.public_key, version=1), sk)


def _lab(tmp_path, golden, data_files, params):
    tee = TeeSimulator(base_dir=tmp_path / "work")
    manager = PolicyManager(tmp_path / "store", tee.attestation_public_key)
    artifact = pack_tree(make_artifact(tmp_path / "artifact"))
    alice, bob = SigningKey.generate(), SigningKey.generate()
    manager.upsert_policy(_policy("alice/data", alice, hash_bytes(b"placeholder"),
                                  volumes=[("training-data", "input")], grants=[("training-data", "bob/trainer")]))
    manager.upsert_policy(_policy("bob/trainer", bob, measure_code(artifact).digest,
                                  volumes=[("trainer-code", "input"), ("model", "output")]))
    _, ak = owner_fetch_keys(manager, "alice/data", alice)
    _, bk = owner_fetch_keys(manager, "bob/trainer", bob)
    refs = {"data": "alice/data/training-data", "code": "bob/trainer/trainer-code", "model": "bob/trainer/model"}
    vols = {refs["data"]: tmp_path / "v/data", refs["code"]: tmp_path / "v/code", refs["model"]: tmp_path / "v/model"}
    dv = Volume.create(vols[refs["data"]], "training-data", ak[refs["data"]])
    for name, blob in data_files.items():
        dv.put(ak[refs["data"]], name, blob)
    Volume.create(vols[refs["code"]], "trainer-code", bk[refs["code"]]).put(bk[refs["code"]], "params.json", params)
    roles = {"training-data": refs["data"], "trainer-code": refs["code"], "model-output": refs["model"]}
    return tee, manager, artifact, vols, roles, bob, refs


def _run(tee, manager, artifact, vols, roles, policy="bob/trainer"):
    return attested_workload_run(manager, tee, policy, artifact, {r: str(p) for r, p in vols.items()}, roles=roles,
                                 timeout=600)


def test_logistic_demo_through_attested_run(tmp_path, golden):
    lab = _lab(tmp_path, golden, {"dataset.csv": (golden / "demo_dataset.csv").read_bytes()},
               (golden / "demo_params.json").read_bytes())
    tee, manager, artifact, vols, roles, bob, refs = lab
    run = _run(tee, manager, artifact, vols, roles)
    assert run.provisioned and run.exit_code == 0, run.handle.diagnostics() if run.handle else run.reject_reason
    _, bk = owner_fetch_keys(manager, "bob/trainer", bob)
    model = Volume.open(vols[refs["model"]]).get(bk[refs["model"]], "model.bin")
    assert hashlib.sha256(model).hexdigest() == DEMO


def _shards(n_shards, batch, seed=0):
    from tests.cnn_parity import make_records

    return {f"shard-{i:05d}.bin": make_records(batch, seed + i).tobytes() for i in range(n_shards)}


def test_cnn_training_through_attested_run(tmp_path, golden):
    params = json.dumps({"model": "small_cnn", "epochs": 2, "batch_size": 32}).encode()
    tee, manager, artifact, vols, roles, bob, refs = _lab(tmp_path, golden, _shards(3, 32), params)
    run = _run(tee, manager, artifact, vols, roles)
    assert run.provisioned and run.exit_code == 0, run.handle.diagnostics() if run.handle else run.reject_reason
    _, bk = owner_fetch_keys(manager, "bob/trainer", bob)
    model = Volume.open(vols[refs["model"]]).get(bk[refs["model"]], "model.bin")
    from paper_2103_16898_b200.trainer import deserialize_cnn_model

    header, params_out = deserialize_cnn_model(model)
    assert header["model"] == "SmallCNN" and header["logical_params"] == 1117162
    assert all(np.isfinite(v).all() for v in params_out.values())


def test_tampered_shard_exits_4_without_output(tmp_path, golden):
    params = json.dumps({"model": "small_cnn", "epochs": 1, "batch_size": 16}).encode()
    tee, manager, artifact, vols, roles, bob, refs = _lab(tmp_path, golden, _shards(2, 16), params)
    d = vols[refs["data"]]
    entry = json.loads((d / "manifest.json").read_text())["entries"][1]
    blob = d / entry["ciphertext_hash"]
    raw = bytearray(blob.read_bytes())
    raw[1000] ^= 1
    blob.write_bytes(bytes(raw))
    run = _run(tee, manager, artifact, vols, roles)
    assert run.provisioned and run.exit_code == 4
    assert not (vols[refs["model"]] / "manifest.json").exists()


def test_missing_data_key_exits_3(tmp_path, golden):
    tee, manager, artifact, vols, roles, bob, refs = _lab(
        tmp_path, golden, {"dataset.csv": (golden / "demo_dataset.csv").read_bytes()},
        (golden / "demo_params.json").read_bytes())
    solo = SigningKey.generate()
    manager.upsert_policy(_policy("bob/solo", solo, measure_code(artifact).digest,
                                  volumes=[("trainer-code", "input"), ("model", "output")]))
    vols2 = dict(vols)
    vols2["bob/solo/trainer-code"] = tmp_path / "v/solo-code"
    vols2["bob/solo/model"] = tmp_path / "v/solo-model"
    roles2 = {"training-data": refs["data"], "trainer-code": "bob/solo/trainer-code",
              "model-output": "bob/solo/model"}
    run = _run(tee, manager, artifact, vols2, roles2, policy="bob/solo")
    assert run.provisioned and run.exit_code == 3
    assert not (tmp_path / "v/solo-model").exists()


def _tamper(vols, refs, index):
    d = vols[refs["data"]]
    entry = json.loads((d / "manifest.json").read_text())["entries"][index]
    blob = d / entry["ciphertext_hash"]
    raw = bytearray(blob.read_bytes())
    raw[1000] ^= 1
    blob.write_bytes(bytes(raw))


def test_two_rank_cnn_training_through_attested_run(tmp_path, golden):
    """world_size 2 (two spawned ranks sharing the one B200 over gloo): the artifact trains
    data-parallel and seals one model."""
    params = json.dumps({"model": "small_cnn", "epochs": 1, "batch_size": 16, "world_size": 2,
                         "backend": "gloo"}).encode()
    tee, manager, artifact, vols, roles, bob, refs = _lab(tmp_path, golden, _shards(4, 16), params)
    run = _run(tee, manager, artifact, vols, roles)
    assert run.provisioned and run.exit_code == 0, run.handle.diagnostics() if run.handle else run.reject_reason
    _, bk = owner_fetch_keys(manager, "bob/trainer", bob)
    from paper_2103_16898_b200.trainer import deserialize_cnn_model

    header, _ = deserialize_cnn_model(Volume.open(vols[refs["model"]]).get(bk[refs["model"]], "model.bin"))
    assert header["model"] == "SmallCNN"


def test_two_rank_tampered_shard_on_rank1_exits_4_without_output(tmp_path, golden):
    """A shard of rank 1 fails its tag: the verdict travels with the gradient all-reduce, both
    ranks stop, the workload exits 4 and no model.bin is sealed (train.py:44-46)."""
    params = json.dumps({"model": "small_cnn", "epochs": 1, "batch_size": 16, "world_size": 2,
                         "backend": "gloo"}).encode()
    tee, manager, artifact, vols, roles, bob, refs = _lab(tmp_path, golden, _shards(4, 16), params)
    names = sorted(json.loads((vols[refs["data"]] / "manifest.json").read_text())["entries"],
                   key=lambda e: e["path"])
    idx = [e["path"] for e in names].index("shard-00003.bin")        # rank 1 owns shards 1 and 3
    _tamper(vols, refs, idx)
    run = _run(tee, manager, artifact, vols, roles)
    assert run.provisioned and run.exit_code == 4
    assert not (vols[refs["model"]] / "manifest.json").exists()
