"""One AES-256-GCM open of MiB (argv[1], default 256) for ncu (--set full of gcm_kernel)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2103_16898_b200 import crypto

mb = int(sys.argv[1]) if len(sys.argv) > 1 else 256
n = mb << 20
ctx = crypto.GcmContext(bytes(range(32)))
pt = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
blob = torch.empty(n + 16, dtype=torch.uint8, device="cuda")
out = torch.empty(n, dtype=torch.uint8, device="cuda")
work = ctx.new_workspace()
ctx.seal_device(bytes(12), None, pt, blob, work)
ctx.open_device(bytes(12), None, blob, out, work)
torch.cuda.synchronize()
assert ctx.status_ok(work) and torch.equal(out, pt)
print("ok")
