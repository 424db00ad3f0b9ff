"""BASELINE configs[4]: decrypt-bound sweep -- encrypted dataset throughput through the
AES-GCM open kernel, 1..64 GB resident in HBM as 1 GiB shards (each its own GCM message,
like one sealed volume file), vs the HBM roofline.  Parity: shard 0 is sealed by the
reference's AEAD library (cryptography/OpenSSL) and must open bit-exactly; every shard's tag
is checked.  Prints one JSON line per size."""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2103_16898_b200 import crypto

GIB = 1 << 30


def main():
    sizes = [int(s) for s in (sys.argv[1:] or ["1", "2", "4", "8", "16", "32", "64"])]
    key = bytes(range(32))
    ctx = crypto.GcmContext(key)
    peaks = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text()) \
        if (Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").exists() else {"hbm_gbs": 6650.0}
    hbm = peaks["hbm_gbs"]
    # shard 0: sealed on the CPU by the reference's AEAD library, checked bit-exactly
    from cryptography.hazmat.primitives.ciphers.aead import AESGCM

    g = torch.Generator(device="cuda").manual_seed(3)
    pt0 = torch.randint(0, 256, (GIB,), dtype=torch.uint8, device="cuda", generator=g)
    aad0 = b"training-data\x00shard-00000.bin"
    nonce0 = bytes(12)
    t0 = time.perf_counter()
    ref_blob = AESGCM(key).encrypt(nonce0, pt0.cpu().numpy().tobytes(), aad0)
    cpu_s = time.perf_counter() - t0
    blob0 = torch.frombuffer(bytearray(ref_blob), dtype=torch.uint8).cuda()
    max_n = max(sizes)
    free = torch.cuda.mem_get_info()[0]
    max_n = min(max_n, int(free * 0.9 // (GIB + 16)) - 2)
    blobs = [blob0]
    aad_dev = torch.frombuffer(bytearray(aad0), dtype=torch.uint8).cuda()
    work = ctx.new_workspace()
    for i in range(1, max_n):
        b = torch.empty(GIB + 16, dtype=torch.uint8, device="cuda")
        ctx.seal_device(i.to_bytes(12, "big"), aad_dev, pt0, b, work)   # distinct nonce per shard
        blobs.append(b)
    out = torch.empty(GIB, dtype=torch.uint8, device="cuda")
    works = [ctx.new_workspace() for _ in range(len(blobs))]
    ctx.open_device(nonce0, aad_dev, blobs[0], out, works[0])
    torch.cuda.synchronize()
    assert crypto.GcmContext.status_ok(works[0]) and torch.equal(out, pt0), "shard 0 parity failed"
    for n in sizes:
        n = min(n, len(blobs))
        for i in range(n):   # warm
            ctx.open_device((i or 0).to_bytes(12, "big") if i else nonce0, aad_dev, blobs[i], out, works[i])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(n):
            ctx.open_device(i.to_bytes(12, "big") if i else nonce0, aad_dev, blobs[i], out, works[i])
        e1.record()
        torch.cuda.synchronize()
        ok = all(crypto.GcmContext.status_ok(works[i]) for i in range(n))
        ms = e0.elapsed_time(e1)
        pt_gbs = n * GIB / ms / 1e6
        alg = n * (2 * GIB + 16) / ms / 1e6
        print(json.dumps({"config": "decrypt sweep (configs[4])", "gb": n * GIB / 1e9, "shards": n,
                          "ms": ms, "plaintext_GBps": pt_gbs, "algorithmic_GBps": alg, "hbm_peak_GBps": hbm,
                          "frac_of_hbm": alg / hbm, "all_tags_ok": ok,
                          "cpu_reference_1GiB_seal_s": cpu_s}), flush=True)


if __name__ == "__main__":
    main()
