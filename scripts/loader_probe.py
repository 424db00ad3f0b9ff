"""Fused decrypt-and-normalise (K1b) vs GCM open + records_to_nhwc on one 512-record CIFAR shard
and one 128-record medical shard (warm, back-to-back launches, CUDA events)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from oracle import ref
from paper_2103_16898_b200 import crypto
from paper_2103_16898_b200.loader import CIFAR, MEDICAL, decode_records, record_bytes

for spec, nrec in ((CIFAR, 512), (MEDICAL, 128)):
    rb = record_bytes(spec["c"], spec["h"], spec["w"])
    pt = np.random.default_rng(0).integers(0, 256, size=nrec * rb, dtype=np.uint8).tobytes()
    key, iv, aad = bytes(range(32)), bytes(12), b"training-data\x00s.bin"
    blob = torch.frombuffer(bytearray(ref.gcm_seal(key, iv, aad, pt)), dtype=torch.uint8).cuda()
    aad_d = torch.frombuffer(bytearray(aad), dtype=torch.uint8).cuda()
    ctx = crypto.GcmContext(key)
    work = ctx.new_workspace()
    out = torch.empty(len(pt), dtype=torch.uint8, device="cuda")
    tile = torch.zeros(nrec, spec["h"], spec["w"], 8, dtype=torch.bfloat16, device="cuda")
    lab = torch.empty(nrec, dtype=torch.int32, device="cuda")

    def two():
        ctx.open_device(iv, aad_d, blob, out, work)
        decode_records(out, nrec, spec["c"], spec["h"], spec["w"], spec["mean"], spec["std"], out=tile, labels=lab)

    def fused():
        ctx.open_records_device(iv, aad_d, blob, tile, lab, work, spec)

    for name, f in (("two-kernel", two), ("fused", fused)):
        for _ in range(5):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            f()
        e1.record()
        torch.cuda.synchronize()
        print(f"{spec['c']}x{spec['h']}x{spec['w']} x{nrec} {name:10s}: {e0.elapsed_time(e1) / 50 * 1e3:7.1f} us")
