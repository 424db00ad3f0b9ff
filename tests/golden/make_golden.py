"""Regenerate the committed golden fixtures (run in the build container, where the reference
is importable from /root/reference or baseline/_ref).  Never run on the GPU box.

Outputs (all small, committed):
  gcm_vectors.json     GCM-spec AES-256 test cases 13-16 (McGrew & Viega, typed in and
                       cross-checked here against the reference's own AESGCM) + seeded
                       vectors sealed by covault.crypto.aead_seal (crypto.py:258-262)
  demo_params.json     copy of pkg/scenarios/assets/trainer_code/params.json
  demo_dataset.csv     copy of pkg/scenarios/assets/training_data/dataset.csv
  volume_demo/         a reference-format volume written by covault.volume.Volume.put
                       (volume.py:161-183) under key bytes(range(32)): dataset.csv,
                       params.json and shard-00000.bin (24 CIFAR-shaped records)
  volume_demo.json     key hex, expected plaintext SHA-256 per path, model digest
"""
from __future__ import annotations

import hashlib
import json
import random
import shutil
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

from covault.crypto import SymmetricKey, aead_seal  # noqa: E402
from covault.volume import Volume  # noqa: E402
from covault.workload import run_training  # noqa: E402
from cryptography.hazmat.primitives.ciphers.aead import AESGCM  # noqa: E402

SPEC_CASES = [
    dict(name="gcm-spec-tc13", key="00" * 32, iv="00" * 12, aad="", pt="", ct="",
         tag="530f8afbc74536b9a963b4f1c4cb738b"),
    dict(name="gcm-spec-tc14", key="00" * 32, iv="00" * 12, aad="", pt="00" * 16,
         ct="cea7403d4d606b6e074ec5d3baf39d18", tag="d0d1c8a799996bf0265b98b5d48ab919"),
    dict(name="gcm-spec-tc15", key="feffe9928665731c6d6a8f9467308308feffe9928665731c6d6a8f9467308308",
         iv="cafebabefacedbaddecaf888", aad="",
         pt="d9313225f88406e5a55909c5aff5269a86a7a9531534f7da2e4c303d8a318a72"
            "1c3c0c95956809532fcf0e2449a6b525b16aedf5aa0de657ba637b391aafd255",
         ct="522dc1f099567d07f47f37a32a84427d643a8cdcbfe5c0c97598a2bd2555d1aa"
            "8cb08e48590dbb3da7b08b1056828838c5f61e6393ba7a0abcc9f662898015ad",
         tag="b094dac5d93471bdec1a502270e3cc6c"),
    dict(name="gcm-spec-tc16", key="feffe9928665731c6d6a8f9467308308feffe9928665731c6d6a8f9467308308",
         iv="cafebabefacedbaddecaf888", aad="feedfacedeadbeeffeedfacedeadbeefabaddad2",
         pt="d9313225f88406e5a55909c5aff5269a86a7a9531534f7da2e4c303d8a318a72"
            "1c3c0c95956809532fcf0e2449a6b525b16aedf5aa0de657ba637b39",
         ct="522dc1f099567d07f47f37a32a84427d643a8cdcbfe5c0c97598a2bd2555d1aa"
            "8cb08e48590dbb3da7b08b1056828838c5f61e6393ba7a0abcc9f662",
         tag="76fc6ece0f4e1768cddf8853bb2d551b"),
]


def make_records(n: int, seed: int, c: int = 3, h: int = 32, w: int = 32, classes: int = 10) -> bytes:
    rng = random.Random(seed)
    out = bytearray()
    for _ in range(n):
        out.append(rng.randrange(classes))
        out += bytes(rng.randrange(256) for _ in range(c * h * w))
    return bytes(out)


def main() -> None:
    vectors = []
    for case in SPEC_CASES:
        k, iv, a, p = (bytes.fromhex(case[x]) for x in ("key", "iv", "aad", "pt"))
        blob = AESGCM(k).encrypt(iv, p, a)
        assert blob.hex() == case["ct"] + case["tag"], case["name"]
        vectors.append(case)
    rng = random.Random(2103_16898)
    lengths = [0, 1, 15, 16, 17, 31, 32, 33, 255, 256, 257, 1000, 3073, 4095, 4096, 4097]
    aads = [0, 1, 13, 16, 17, 64, 200]
    for i, n in enumerate(lengths):
        for j, alen in enumerate(aads[(i % 3)::3]):
            key = SymmetricKey(bytes(rng.randrange(256) for _ in range(32)))
            iv = bytes(rng.randrange(256) for _ in range(12))
            aad = bytes(rng.randrange(256) for _ in range(alen))
            pt = bytes(rng.randrange(256) for _ in range(n))
            blob = aead_seal(key, iv, aad, pt)   # the reference's own AEAD (crypto.py:258-262)
            vectors.append(dict(name=f"ref-aead-{n}-{alen}", key=key.reveal_hex(), iv=iv.hex(), aad=aad.hex(),
                                pt=pt.hex(), ct=blob[:-16].hex(), tag=blob[-16:].hex()))
    (HERE / "gcm_vectors.json").write_text(json.dumps(vectors, indent=0) + "\n")

    shutil.copy(REF / "scenarios/assets/trainer_code/params.json", HERE / "demo_params.json")
    shutil.copy(REF / "scenarios/assets/training_data/dataset.csv", HERE / "demo_dataset.csv")
    params = json.loads((HERE / "demo_params.json").read_text())
    csv_text = (HERE / "demo_dataset.csv").read_text()
    digest = hashlib.sha256(run_training(params, csv_text)).hexdigest()
    assert digest == "7e799c1f44492be596de4727ead2d0a9877d2699a12e88ebcf20b9a6f514607c"

    vdir = HERE / "volume_demo"
    shutil.rmtree(vdir, ignore_errors=True)
    key = SymmetricKey(bytes(range(32)))
    vol = Volume.create(vdir, "training-data", key)
    files = {
        "dataset.csv": (HERE / "demo_dataset.csv").read_bytes(),
        "params.json": (HERE / "demo_params.json").read_bytes(),
        "shard-00000.bin": make_records(24, seed=7),
    }
    for path, data in files.items():
        vol.put(key, path, data)
    meta = {
        "key": key.reveal_hex(),
        "volume_name": "training-data",
        "plaintext_sha256": {p: hashlib.sha256(d).hexdigest() for p, d in files.items()},
        "demo_model_sha256": digest,
        "shard_records": 24, "record_bytes": 3073,
    }
    (HERE / "volume_demo.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
    print(f"wrote {len(vectors)} vectors, volume with {len(files)} files")


if __name__ == "__main__":
    main()
