"""BASELINE configs[4]: decrypt-bound sweep -- encrypted dataset throughput through the
AES-GCM open kernel, 1..64 GB resident in HBM as 1 GiB shards (each its own GCM message,
like one sealed volume file), vs the HBM roofline.

Parity: EVERY shard is sealed on the host by the reference's AEAD library (cryptography ->
OpenSSL AES-256-GCM, what covault.crypto.aead_seal calls, crypto.py:258-262) with its own
nonce and AAD, and after the timed runs every shard is opened again and compared bit for
bit with its plaintext (regenerated from its seed).  CPU baseline: the reference's open
(AESGCM.decrypt, crypto.py:265-272) of the same shards on 1 thread and on every host core
(threads; OpenSSL releases the GIL).  Prints one JSON line per size, then a summary line."""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2103_16898_b200 import crypto  # noqa: E402

GIB = 1 << 30
KEY = bytes(range(32))


def plaintext(i):
    g = torch.Generator(device="cuda").manual_seed(3 + i)
    return torch.randint(0, 256, (GIB,), dtype=torch.uint8, device="cuda", generator=g)


def aad_of(i):
    return f"training-data\x00shard-{i:05d}.bin".encode()


def main():
    from cryptography.hazmat.primitives.ciphers.aead import AESGCM

    sizes = [int(s) for s in (sys.argv[1:] or ["1", "2", "4", "8", "16", "32", "64"])]
    root = Path(__file__).resolve().parent.parent
    peaks = json.loads((root / "MEASURED_PEAKS.json").read_text()) if (root / "MEASURED_PEAKS.json").exists() \
        else {"hbm_gbs": 6550.0}
    hbm = peaks["hbm_gbs"]
    free = torch.cuda.mem_get_info()[0]
    max_n = min(max(sizes), int(free * 0.92 // (GIB + 16)) - 3)
    aes = AESGCM(KEY)
    cores = len(os.sched_getaffinity(0))
    nthr = max(1, min(8, cores))          # bounded host memory: nthr GiB plaintext + ciphertext in flight

    def seal(i):
        pt = plaintext(i).cpu().numpy().tobytes()
        return aes.encrypt(i.to_bytes(12, "big"), pt, aad_of(i))

    t0 = time.perf_counter()
    blobs = []
    with ThreadPoolExecutor(nthr) as ex:
        for blob in ex.map(seal, range(max_n)):
            blobs.append(torch.frombuffer(bytearray(blob), dtype=torch.uint8).cuda())
            del blob
    seal_s = time.perf_counter() - t0
    ctx = crypto.GcmContext(KEY)
    aads = [torch.frombuffer(bytearray(aad_of(i)), dtype=torch.uint8).cuda() for i in range(max_n)]
    out = torch.empty(GIB, dtype=torch.uint8, device="cuda")
    works = [ctx.new_workspace() for _ in range(max_n)]
    nonces = [i.to_bytes(12, "big") for i in range(max_n)]
    results = []
    for n in sizes:
        n = min(n, max_n)
        for i in range(n):   # warm
            works[i].zero_()
            ctx.open_device(nonces[i], aads[i], blobs[i], out, works[i])
        torch.cuda.synchronize()
        for w in works[:n]:
            w.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(n):
            ctx.open_device(nonces[i], aads[i], blobs[i], out, works[i])
        e1.record()
        torch.cuda.synchronize()
        ok = all(crypto.GcmContext.status_ok(works[i]) for i in range(n))
        ms = e0.elapsed_time(e1)
        alg = n * (2 * GIB + 16) / ms / 1e6
        r = {"config": "decrypt sweep (configs[4])", "gb": n * GIB / 1e9, "shards": n, "ms": ms,
             "plaintext_GBps": n * GIB / ms / 1e6, "algorithmic_GBps": alg, "hbm_peak_GBps": hbm,
             "frac_of_hbm": alg / hbm, "all_tags_ok": ok}
        results.append(r)
        print(json.dumps(r), flush=True)
    # bit-exactness of every shard against its plaintext
    exact = True
    for i in range(max_n):
        works[i].zero_()
        ctx.open_device(nonces[i], aads[i], blobs[i], out, works[i])
        exact = exact and crypto.GcmContext.status_ok(works[i]) and torch.equal(out, plaintext(i))
    # CPU baseline: the reference's open of k shards, 1 thread and every core
    k = min(max_n, max(2, cores))
    host = [bytes(blobs[i].cpu().numpy()) for i in range(k)]

    def open_(i):
        return len(aes.decrypt(nonces[i], host[i], aad_of(i)))

    t0 = time.perf_counter()
    for i in range(2):
        open_(i)
    cpu1 = 2 * GIB / (time.perf_counter() - t0) / 1e9
    t0 = time.perf_counter()
    with ThreadPoolExecutor(cores) as ex:
        list(ex.map(open_, range(k)))
    cpun = k * GIB / (time.perf_counter() - t0) / 1e9
    print(json.dumps({"summary": "decrypt sweep", "shards_sealed_by": "cryptography AESGCM (OpenSSL), host, every shard",
                      "every_shard_bit_exact": bool(exact), "host_seal_s": seal_s,
                      "cpu_open_GBps_1_thread": cpu1, "cpu_open_GBps_all_cores": cpun, "cpu_cores": cores,
                      "best_gpu_plaintext_GBps": max(r["plaintext_GBps"] for r in results)}), flush=True)


if __name__ == "__main__":
    main()
