"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck): one eager training
step of a model at a small batch, plus the AES-GCM open/seal/decode, SHA-256, CSV parse and
reference-trainer kernels on small inputs.  usage: sanitize_step.py {cnn MODEL BATCH | crypto}"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

what = sys.argv[1]
if what == "cnn":
    from bench import make_shards
    from paper_2103_16898_b200.loader import CIFAR
    from paper_2103_16898_b200.trainer import EncryptedTrainer

    model, B = sys.argv[2], int(sys.argv[3])
    key = bytes(range(32))
    tr = EncryptedTrainer(model, key, batch=B, spec=CIFAR)
    sh = make_shards(2, B, 1, key, CIFAR)
    ct = [torch.frombuffer(bytearray(s[3]), dtype=torch.uint8).cuda() for s in sh]
    aad = [torch.frombuffer(bytearray(s[2]), dtype=torch.uint8).cuda() for s in sh]
    for i in range(2):
        tr.step_resident(ct[i % 2], sh[i % 2][1], aad[i % 2], B)
    torch.cuda.synchronize()
    tr.check_status(include_pending=True)
    print("cnn ok", float(tr.net.loss.item()))
else:
    import os

    import numpy as np

    from paper_2103_16898_b200 import crypto, workload

    key, nonce, aad = bytes(range(32)), bytes(12), b"v\x00p"
    for n in (0, 1, 100, 70_000, 3 * 2**20 + 5):   # the last one runs two passes (GHASH tables)
        pt = os.urandom(n)
        assert crypto.aead_open(key, nonce, aad, crypto.aead_seal(key, nonce, aad, pt)) == pt
    assert len(crypto.sha256_many([b"", b"abc", os.urandom(5000)])) == 3
    X, y = workload.parse_dataset_device("1.5,2,1\n# c\n3,4e-3,0\n")
    tr = workload.LogisticTrainer(X, y, exact=True)
    tr.train(0.1, 2)
    tr2 = workload.LogisticTrainer(torch.from_numpy(np.random.rand(300, 70)).cuda(),
                                   torch.from_numpy((np.random.rand(300) > .5) * 1.0).cuda(), exact=False)
    tr2.train(0.1, 2)
    torch.cuda.synchronize()
    print("crypto/csv/logistic ok")
