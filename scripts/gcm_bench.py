"""Quick GCM kernel throughput probe (CUDA events, device-resident buffers)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2103_16898_b200 import crypto

ctx = crypto.GcmContext(bytes(range(32)))
iv = bytes(12)
for mb in [1, 16, 256, 1024]:
    n = mb << 20
    pt = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
    blob = torch.empty(n + 16, dtype=torch.uint8, device="cuda")
    out = torch.empty(n, dtype=torch.uint8, device="cuda")
    work = ctx.new_workspace()
    ctx.seal_device(iv, None, pt, blob, work)
    for _ in range(3):
        ctx.open_device(iv, None, blob, out, work)
    torch.cuda.synchronize()
    assert ctx.status_ok(work) and torch.equal(out, pt)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(3, min(50, 2048 // mb))
    e0.record()
    for _ in range(reps):
        ctx.open_device(iv, None, blob, out, work)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"open {mb:5d} MiB: {ms:8.3f} ms  {n/ms/1e6:8.1f} GB/s plaintext  {(2*n+16)/ms/1e6:8.1f} GB/s algorithmic")
