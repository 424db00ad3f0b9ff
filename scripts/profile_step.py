"""One eager training step inside cudaProfilerStart/Stop for ncu (--profile-from-start off)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2103_16898_b200.loader import CIFAR
from paper_2103_16898_b200.trainer import EncryptedTrainer

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import make_shards  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "small_cnn"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 512
from paper_2103_16898_b200.loader import MEDICAL  # noqa: E402

spec = MEDICAL if model == "densenet121" else CIFAR
key = bytes(range(32))
tr = EncryptedTrainer(model, key, batch=B, spec=spec)
sh = make_shards(2, B, 1, key, spec)
ct = [torch.frombuffer(bytearray(s[3]), dtype=torch.uint8).cuda() for s in sh]
aad = [torch.frombuffer(bytearray(s[2]), dtype=torch.uint8).cuda() for s in sh]
for i in range(3):
    tr.step_resident(ct[i % 2], sh[i % 2][1], aad[i % 2], B)
torch.cuda.synchronize()
torch.cuda.profiler.start()
tr.step_resident(ct[0], sh[0][1], aad[0], B)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("loss", tr.net.loss.item())
