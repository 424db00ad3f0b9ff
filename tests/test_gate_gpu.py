"""SURVEY 8(f) rows 2-3 on the GPU: tree sealing (volume.py:239-258) and the trusted-boot
gate's re-encryption copy (gate.py:186-190) with the AES-GCM work on the device.  Source is
the reference-written golden volume (tests/golden/volume_demo, sealed by covault.volume.Volume.put);
the destination is checked by the CPU oracle (oracle/gcm_ref.c), not by the GPU code."""
import hashlib
import json
import shutil

import pytest

from oracle import ref
from paper_2103_16898_b200.crypto import AuthenticationFailure
from paper_2103_16898_b200.volume import Volume, aad_for, gate_copy, seal_tree, unseal_tree

pytestmark = pytest.mark.gpu
DEST_KEY = bytes(range(100, 132))


def test_gate_copy_reencrypts_reference_volume(golden, tmp_path):
    meta = json.loads((golden / "volume_demo.json").read_text())
    src = Volume.open(golden / "volume_demo")
    dst = Volume.create(tmp_path / "dest", "trained-inputs", DEST_KEY)
    report = gate_copy(src, bytes.fromhex(meta["key"]), dst, DEST_KEY)
    assert {p: d for p, d, _ in report} == meta["plaintext_sha256"]
    dst = Volume.open(tmp_path / "dest")
    assert dst.verify() == []
    for path, digest, n in report:
        e = dst.entry(path)
        pt = ref.gcm_open(DEST_KEY, e.nonce, aad_for("trained-inputs", path), dst.read_blob(path))   # oracle
        assert pt is not None and len(pt) == n and hashlib.sha256(pt).hexdigest() == digest


def test_gate_copy_rejects_tampered_source(golden, tmp_path):
    meta = json.loads((golden / "volume_demo.json").read_text())
    shutil.copytree(golden / "volume_demo", tmp_path / "src")
    src = Volume.open(tmp_path / "src")
    victim = src.paths()[-1]
    bp = src.blob_path(victim)
    b = bytearray(bp.read_bytes())
    b[len(b) // 2] ^= 0x10
    bp.write_bytes(bytes(b))
    dst = Volume.create(tmp_path / "dest", "trained-inputs", DEST_KEY)
    with pytest.raises(AuthenticationFailure):
        gate_copy(src, bytes.fromhex(meta["key"]), dst, DEST_KEY)
    assert victim not in Volume.open(tmp_path / "dest").paths()


def test_seal_tree_unseal_tree_roundtrip(tmp_path):
    srcdir = tmp_path / "tree"
    (srcdir / "a" / "b").mkdir(parents=True)
    files = {"x.bin": bytes(range(256)) * 41, "a/empty": b"", "a/b/c.txt": b"hello covault\n"}
    for rel, data in files.items():
        (srcdir / rel).write_bytes(data)
    key = bytes(range(32))
    vol = Volume.create(tmp_path / "vol", "tree-volume", key)
    assert seal_tree(vol, key, srcdir) == 3
    for rel, data in files.items():      # oracle opens what the GPU sealed
        e = vol.entry(rel)
        assert ref.gcm_open(key, e.nonce, aad_for("tree-volume", rel), vol.read_blob(rel)) == data
    out = tmp_path / "out"
    assert unseal_tree(Volume.open(tmp_path / "vol"), key, out) == 3
    for rel, data in files.items():
        assert (out / rel).read_bytes() == data


def _platform():
    sim = pytest.importorskip("covault.platform_sim")
    p = sim.SimulatedPlatform()
    p.boot(b"gate kernel", "quiet ima=on")
    p.load_file("usr/sbin/loader", b"loader", signed=True)
    return p


def _gate_config(tmp_path, platform, dest):
    from covault.gate import GateConfig

    return GateConfig(source_path=tmp_path / "source", source_policy="a", source_volume="src", dest_path=dest,
                      dest_policy="c", dest_volume="dst", gate_policy="g",
                      tpm_root_certs=(platform.root_certificate,), expected_pcrs=platform.expected_pcrs())


def test_device_gate_run_accepts_and_reports_plaintext_digests(tmp_path):
    """gate.gate_run (installed over covault.gate.gate_run) on a reference-written source:
    accepted, report digests = SHA-256 of the plaintexts, destination readable by the reference."""
    from covault.crypto import SymmetricKey
    from covault.volume import Volume as RefVolume

    from paper_2103_16898_b200.gate import gate_run

    platform = _platform()
    sk, dk = SymmetricKey.generate(), SymmetricKey.generate()
    src = RefVolume.create(tmp_path / "source", "src", sk)
    contents = {f"data/f{i}.bin": (f"payload {i} ".encode() * (i * 300 + 1)) for i in range(4)}
    contents["empty"] = b""
    for p, d in contents.items():
        src.put(sk, p, d)
    res = gate_run(_gate_config(tmp_path, platform, tmp_path / "dest"), platform.device, platform.device.log, sk, dk)
    assert res.accepted and res.exit_code == 0
    assert {p: (h, n) for p, h, n in res.report.files} == {
        p: (hashlib.sha256(d).hexdigest(), len(d)) for p, d in contents.items()}
    out = RefVolume.open(tmp_path / "dest")
    assert out.verify() == [] and {p: out.get(dk, p) for p in out.paths()} == contents


def test_device_gate_crash_at_every_file_leaves_no_destination(tmp_path, monkeypatch):
    """The reference's crash-atomicity property (pkg/tests/test_gate.py:144-188) against the
    device gate's own write path: a crash in the k-th destination write leaves nothing."""
    from covault.crypto import SymmetricKey
    from covault.volume import Volume as RefVolume

    from paper_2103_16898_b200.gate import gate_run

    platform = _platform()
    sk, dk = SymmetricKey.generate(), SymmetricKey.generate()
    src = RefVolume.create(tmp_path / "source", "src", sk)
    for i in range(4):
        src.put(sk, f"f{i}", bytes([i]) * (1000 * i + 7))
    real = Volume.put_sealed
    for crash_after in range(4):
        calls = {"n": 0}

        def crashing(self, *a, _lim=crash_after, _c=calls, **kw):
            if _c["n"] >= _lim:
                raise OSError("injected crash mid-copy")
            _c["n"] += 1
            return real(self, *a, **kw)

        monkeypatch.setattr(Volume, "put_sealed", crashing)
        dest = tmp_path / f"dest-{crash_after}"
        with pytest.raises(OSError):
            gate_run(_gate_config(tmp_path, platform, dest), platform.device, platform.device.log, sk, dk)
        monkeypatch.setattr(Volume, "put_sealed", real)
        assert not dest.exists() and not list(tmp_path.glob(f"dest-{crash_after}.*"))


def test_device_gate_rejects_corrupt_source(tmp_path):
    from covault.crypto import SymmetricKey
    from covault.volume import Volume as RefVolume

    from paper_2103_16898_b200.gate import gate_run

    platform = _platform()
    sk, dk = SymmetricKey.generate(), SymmetricKey.generate()
    src = RefVolume.create(tmp_path / "source", "src", sk)
    src.put(sk, "a", b"x" * 5000)
    blob = tmp_path / "source" / src._entries["a"].ciphertext_hash.hex
    raw = bytearray(blob.read_bytes())
    raw[7] ^= 1
    blob.write_bytes(bytes(raw))
    res = gate_run(_gate_config(tmp_path, platform, tmp_path / "dest"), platform.device, platform.device.log, sk, dk)
    assert not res.accepted and res.reason == "volume_auth_failure" and res.exit_code == 8
    assert not (tmp_path / "dest").exists()


def test_volume_put_names_blobs_by_device_sha256(tmp_path):
    key = bytes(range(32))
    vol = Volume.create(tmp_path / "v", "vv", key)
    for i in range(5):
        vol.put(key, f"p{i}", bytes(range(i * 17 % 256)) * i)
    for p in vol.paths():
        assert hashlib.sha256(vol.read_blob(p)).hexdigest() == vol.entry(p).ciphertext_hash
    assert vol.verify() == []
    victim = vol.blob_path("p3")
    b = bytearray(victim.read_bytes())
    b[0] ^= 1
    victim.write_bytes(bytes(b))
    assert vol.verify() == [("hash_mismatch", "p3")]
