"""One fused decrypt-and-normalise of a 512-record CIFAR shard (for ncu)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from oracle import ref
from paper_2103_16898_b200 import crypto
from paper_2103_16898_b200.loader import CIFAR, record_bytes

nrec = 512
rb = record_bytes(3, 32, 32)
pt = np.random.default_rng(0).integers(0, 256, size=nrec * rb, dtype=np.uint8).tobytes()
key, iv, aad = bytes(range(32)), bytes(12), b"training-data\x00s.bin"
blob = torch.frombuffer(bytearray(ref.gcm_seal(key, iv, aad, pt)), dtype=torch.uint8).cuda()
aad_d = torch.frombuffer(bytearray(aad), dtype=torch.uint8).cuda()
ctx = crypto.GcmContext(key)
work = ctx.new_workspace()
tile = torch.zeros(nrec, 32, 32, 8, dtype=torch.bfloat16, device="cuda")
lab = torch.empty(nrec, dtype=torch.int32, device="cuda")
for _ in range(4):
    ctx.open_records_device(iv, aad_d, blob, tile, lab, work, CIFAR)
torch.cuda.synchronize()
print("ok", crypto.GcmContext.status_ok(work))
