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
