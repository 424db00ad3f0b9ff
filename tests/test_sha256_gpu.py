"""GPU SHA-256 (csrc/sha256.cu) bit-exact against hashlib (the reference's hash_bytes,
crypto.py:91-93) and the FIPS 180-2 known answers; batched and device-resident forms."""
import hashlib
import os

import pytest
import torch

from paper_2103_16898_b200 import crypto

pytestmark = pytest.mark.gpu

KAT = {  # FIPS 180-2 appendix B + the reference's EMPTY_SHA256 (pkg/tests/test_crypto.py:31)
    b"": "e3b0c44298fc1c149afbf4c8996fb92427ae41e4649b934ca495991b7852b855",
    b"abc": "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad",
    b"abcdbcdecdefdefgefghfghighijhijkijkljklmklmnlmnomnopnopq":
        "248d6a61d20638b8e5c026930c3e6039a33ce45964ff2167f6ecedd419db06c1",
    b"a" * 1_000_000: "cdc76e5c9914fb9281a1c7e284d73e67f1809a48a497200e046d39ccc7112cd0",
}


def test_known_answers():
    got = crypto.sha256_many(list(KAT))
    assert [g.hex() for g in got] == list(KAT.values())


def test_every_padding_boundary_and_random_lengths():
    rng = torch.Generator().manual_seed(0)
    lens = list(range(0, 200)) + [255, 256, 511, 512, 4095, 4096, 65535, 65536, 1 << 20]
    lens += [int(x) for x in torch.randint(0, 300_000, (40,), generator=rng)]
    msgs = [os.urandom(n) for n in lens]
    got = crypto.sha256_many(msgs)
    assert got == [hashlib.sha256(m).digest() for m in msgs]


def test_device_arena_unaligned_offsets():
    msgs = [os.urandom(n) for n in (0, 1, 3, 55, 56, 63, 64, 65, 119, 120, 1000, 70_001)]
    arena = b"".join(msgs)
    offs = [0]
    for m in msgs:
        offs.append(offs[-1] + len(m))
    data = torch.frombuffer(bytearray(arena), dtype=torch.uint8).cuda()
    off = torch.tensor(offs, dtype=torch.int64, device="cuda")
    dig = crypto.sha256_device(data, off).cpu().numpy()
    assert [bytes(d) for d in dig] == [hashlib.sha256(m).digest() for m in msgs]


def test_many_messages_one_launch():
    msgs = [os.urandom(37 * (i % 50)) for i in range(5000)]
    assert crypto.sha256_many(msgs) == [hashlib.sha256(m).digest() for m in msgs]


def test_span_form_separate_allocations():
    msgs = [os.urandom(n) for n in (0, 9, 64, 100_000)]
    ts = [torch.frombuffer(bytearray(m), dtype=torch.uint8).cuda() if m else torch.empty(0, dtype=torch.uint8,
                                                                                          device="cuda") for m in msgs]
    dig = crypto.sha256_tensors(ts).cpu().numpy()
    assert [bytes(d) for d in dig] == [hashlib.sha256(m).digest() for m in msgs]
