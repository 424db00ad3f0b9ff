"""GPU AES-256-GCM parity: bit-exact against the oracle, the golden vectors and the
reference's own tests' properties (pkg/tests/test_crypto.py:123-154, test_volume.py)."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import ref
from paper_2103_16898_b200 import crypto
from paper_2103_16898_b200.volume import Volume, aad_for

pytestmark = pytest.mark.gpu


def test_golden_vectors(gcm_vectors):
    for v in gcm_vectors:
        key, iv, aad, pt = (bytes.fromhex(v[k]) for k in ("key", "iv", "aad", "pt"))
        blob = bytes.fromhex(v["ct"] + v["tag"])
        assert crypto.aead_seal(key, iv, aad, pt) == blob, v["name"]
        assert crypto.aead_open(key, iv, aad, blob) == pt, v["name"]


@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 4095, 1 << 20, (1 << 20) + 3, 3073 * 512])
@pytest.mark.parametrize("alen", [0, 1, 13, 64, 200])
def test_random_lengths_match_oracle(n, alen):
    rng = np.random.default_rng(n * 7 + alen)
    key, iv, aad, pt = rng.bytes(32), rng.bytes(12), rng.bytes(alen), rng.bytes(n)
    blob = ref.gcm_seal(key, iv, aad, pt)
    assert crypto.aead_seal(key, iv, aad, pt) == blob
    assert crypto.aead_open(key, iv, aad, blob) == pt


def test_every_ciphertext_bit_flip_fails():
    key, nonce = crypto.SymmetricKey.generate(), crypto.fresh_nonce()
    ct = crypto.aead_seal(key, nonce, b"aad", b"thirty-two bytes of plaintext!!!")
    for bit in range(len(ct) * 8):
        m = bytearray(ct)
        m[bit // 8] ^= 1 << (bit % 8)
        with pytest.raises(crypto.AuthenticationFailure):
            crypto.aead_open(key, nonce, b"aad", bytes(m))


def test_aad_nonce_key_binding():
    key = crypto.SymmetricKey.generate()
    ct = crypto.aead_seal(key, b"\x00" * 12, b"volume/path", b"data")
    with pytest.raises(crypto.AuthenticationFailure):
        crypto.aead_open(key, b"\x00" * 12, b"volume/other", ct)
    with pytest.raises(crypto.AuthenticationFailure):
        crypto.aead_open(key, b"\x01" + b"\x00" * 11, b"volume/path", ct)
    with pytest.raises(crypto.AuthenticationFailure):
        crypto.aead_open(crypto.SymmetricKey.generate(), b"\x00" * 12, b"volume/path", ct)
    with pytest.raises(crypto.AuthenticationFailure):
        crypto.aead_open(key, b"\x00" * 12, b"volume/path", ct[:10])
    with pytest.raises(crypto.DecodeError):
        crypto.aead_open(key, b"\x00" * 11, b"", ct)


def test_open_seal_identity_many():
    rng = np.random.default_rng(3)
    for _ in range(50):
        key, nonce = rng.bytes(32), rng.bytes(12)
        pt, aad = rng.bytes(int(rng.integers(0, 513))), rng.bytes(int(rng.integers(0, 65)))
        assert crypto.aead_open(key, nonce, aad, crypto.aead_seal(key, nonce, aad, pt)) == pt


def test_large_message_tag_and_tamper_at_end():
    # 64 MiB + 5: many Horner iterations per thread and a partial final block
    rng = np.random.default_rng(9)
    key, iv = rng.bytes(32), rng.bytes(12)
    pt = rng.integers(0, 256, size=(64 << 20) + 5, dtype=np.uint8).tobytes()
    from cryptography.hazmat.primitives.ciphers.aead import AESGCM

    blob = AESGCM(key).encrypt(iv, pt, b"x")
    assert crypto.aead_open(key, iv, b"x", blob) == pt
    m = bytearray(blob)
    m[len(pt) - 1] ^= 0x80
    with pytest.raises(crypto.AuthenticationFailure):
        crypto.aead_open(key, iv, b"x", bytes(m))


@pytest.mark.parametrize("extra", [-1, 0, 17])
@pytest.mark.parametrize("alen", [0, 13, 200])
def test_multi_pass_messages_around_pass_boundaries(extra, alen):
    """Messages of two and three passes (one pass = 148 SMs x 1024 threads x 16 B): the GHASH
    digit tables, the folded AES round 1 and the per-thread round-2 lookups of the fixed counter
    byte are only used here; seal and open both bit-exact against `cryptography`."""
    from cryptography.hazmat.primitives.ciphers.aead import AESGCM

    import torch

    per_pass = torch.cuda.get_device_properties(0).multi_processor_count * 1024 * 16
    rng = np.random.default_rng(alen * 7 + extra + 3)
    key, iv, aad = rng.bytes(32), rng.bytes(12), rng.bytes(alen)
    for passes in (2, 3):
        pt = rng.integers(0, 256, size=passes * per_pass + extra, dtype=np.uint8).tobytes()
        blob = AESGCM(key).encrypt(iv, pt, aad)
        assert crypto.aead_seal(key, iv, aad, pt) == blob
        assert crypto.aead_open(key, iv, aad, blob) == pt
        bad = bytearray(blob)
        bad[-1] ^= 1
        with pytest.raises(crypto.AuthenticationFailure):
            crypto.aead_open(key, iv, aad, bytes(bad))


def test_device_open_poisons_on_failure():
    import torch

    key, iv = bytes(range(32)), bytes(12)
    pt = os.urandom(100_000)
    blob = ref.gcm_seal(key, iv, b"", pt)
    ctx = crypto.GcmContext(key)
    dev = torch.tensor(list(blob), dtype=torch.uint8, device="cuda")
    out = torch.empty(len(pt), dtype=torch.uint8, device="cuda")
    work = ctx.new_workspace()
    ctx.open_device(iv, None, dev, out, work)
    assert crypto.GcmContext.status_ok(work)
    assert bytes(out.cpu().numpy()) == pt
    dev[5] ^= 1
    work = ctx.new_workspace()
    ctx.open_device(iv, None, dev, out, work)
    assert not crypto.GcmContext.status_ok(work)
    assert int(out.count_nonzero().item()) == 0


def test_golden_reference_volume(golden):
    meta = json.loads((golden / "volume_demo.json").read_text())
    key = crypto.SymmetricKey.from_hex(meta["key"])
    vol = Volume.open(golden / "volume_demo")
    for path in vol.paths():
        assert hashlib.sha256(vol.get(key, path)).hexdigest() == meta["plaintext_sha256"][path]
    ctx = crypto.GcmContext(key)
    shard, _ = vol.get_device(ctx, "shard-00000.bin")
    assert hashlib.sha256(bytes(shard.cpu().numpy())).hexdigest() == meta["plaintext_sha256"]["shard-00000.bin"]


def test_volume_round_trip_and_reference_interop(tmp_path):
    cv = pytest.importorskip("covault.volume")
    cc = pytest.importorskip("covault.crypto")
    key = crypto.SymmetricKey.generate()
    vol = Volume.create(tmp_path / "v", "testvol", key)
    vol.put(key, "dir/file.bin", b"payload bytes")
    vol.put(key, "empty", b"")
    # the reference reads what the GPU wrote, and vice versa
    rkey = cc.SymmetricKey(key.reveal_bytes())
    rvol = cv.Volume.open(tmp_path / "v")
    assert rvol.get(rkey, "dir/file.bin") == b"payload bytes"
    assert rvol.get(rkey, "empty") == b""
    assert rvol.verify() == []
    rvol.put(rkey, "ref.bin", b"written by the reference")
    assert Volume.open(tmp_path / "v").get(key, "ref.bin") == b"written by the reference"


@pytest.mark.parametrize("c,h,w,nrec", [(3, 32, 32, 37), (1, 224, 224, 3), (3, 32, 32, 1), (1, 224, 224, 128)])
def test_fused_decrypt_normalise_matches_two_kernel_path(c, h, w, nrec):
    """K1b: cvb_gcm_open_records_dev (one kernel) == GCM open + records_to_nhwc, bit for bit,
    and a tampered shard leaves an all-zero tile and labels."""
    import numpy as np
    import torch

    from paper_2103_16898_b200.loader import decode_records, record_bytes

    spec = dict(c=c, h=h, w=w, mean=(0.5,) * c, std=(0.25,) * c)
    rb = record_bytes(c, h, w)
    rng = np.random.default_rng(nrec + c)
    pt = rng.integers(0, 256, size=nrec * rb, dtype=np.uint8).tobytes()
    key, iv, aad = bytes(range(32)), bytes(range(12)), b"training-data\x00shard-x.bin"
    blob = ref.gcm_seal(key, iv, aad, pt)
    ctx = crypto.GcmContext(key)
    dev = torch.frombuffer(bytearray(blob), dtype=torch.uint8).cuda()
    aad_dev = torch.frombuffer(bytearray(aad), dtype=torch.uint8).cuda()
    out = torch.empty(len(pt), dtype=torch.uint8, device="cuda")
    work = ctx.new_workspace()
    ctx.open_device(iv, aad_dev, dev, out, work)
    x_ref, lab_ref = decode_records(out, nrec, c, h, w, spec["mean"], spec["std"])
    tile = torch.zeros(nrec, h, w, 8, dtype=torch.bfloat16, device="cuda")
    labels = torch.empty(nrec, dtype=torch.int32, device="cuda")
    work2 = ctx.new_workspace()
    ctx.open_records_device(iv, aad_dev, dev, tile, labels, work2, spec)
    assert crypto.GcmContext.status_ok(work2)
    assert torch.equal(tile, x_ref) and torch.equal(labels, lab_ref)
    dev[len(pt) // 2] ^= 0x40
    ctx.open_records_device(iv, aad_dev, dev, tile, labels, work2, spec)
    assert not crypto.GcmContext.status_ok(work2)
    assert int(tile.count_nonzero()) == 0 and int(labels.count_nonzero()) == 0
