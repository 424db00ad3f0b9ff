"""Encrypted-training step for the CNN configs: sealed shards -> GPU decrypt -> train.

This is the B200 form of the reference's trainer contract (train.py:23-53 ->
workload.run_training, /root/reference/pkg/src/covault/workload.py:48-71): the dataset is
read from a reference-format encrypted volume (volume.py), every shard is authenticated
(AES-256-GCM tag) on the device before its records reach training, and the model is sealed
back into an output volume (``serialize_cnn_model`` / ``seal_model``).

Data parallelism (weak scaling): one process per GPU, each rank opens its own shards
(round-robin by index), trains on a fixed per-rank batch, gradients are all-reduced in
buckets over NCCL (sum; the loss gradient is pre-scaled by 1/global_batch), BN statistics
are per rank (DDP default).
"""
from __future__ import annotations

import json
import struct

import numpy as np
import torch

from . import kernels as K
from .crypto import AuthenticationFailure, GcmContext
from .loader import CIFAR, ShardLoader, decode_records, record_bytes
from .nets import make_model

CNN_MAGIC = b"CVC1"


class GradAllReduce:
    """Bucketed NCCL all-reduce of the flat fp32 gradient buffer (~bucket_mb per bucket,
    issued back to front so the last layers' bucket goes first)."""

    def __init__(self, g32: torch.Tensor, bucket_mb: float = 25.0, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        n = g32.numel()
        per = max(1, int(bucket_mb * (1 << 20) / 4))
        self.buckets = [g32[max(0, e - per):e] for e in range(n, 0, -per)]

    def __call__(self, g32=None):
        works = [self.dist.all_reduce(b, op=self.dist.ReduceOp.SUM, group=self.group, async_op=True)
                 for b in self.buckets]
        for w in works:
            w.wait()


class EncryptedTrainer:
    def __init__(self, model="small_cnn", key: bytes = bytes(range(32)), batch=512, spec=CIFAR, seed=0,
                 world=1, rank=0, max_shard_bytes=None, lr=1e-3, force_allreduce=False):
        self.spec, self.batch, self.world, self.rank = spec, batch, world, rank
        self.net = make_model(model, seed=seed).build(batch, global_batch=batch * world)
        self.net.lr = lr
        self.ctx = GcmContext(key)
        rec = record_bytes(spec["c"], spec["h"], spec["w"])
        self.loader = ShardLoader(self.ctx, max_shard_bytes or batch * rec, batch, spec)
        self.allreduce = GradAllReduce(self.net.ps.g32) if (world > 1 or force_allreduce) else None
        self.graph = None
        self.status_host = torch.zeros(8, dtype=torch.int32).pin_memory()
        self.loss_host = torch.zeros(1, dtype=torch.float32).pin_memory()

    # -- the step ------------------------------------------------------------------------
    def _train_body(self):
        x, lab = self.loader.x[:self.batch], self.loader.labels[:self.batch]
        net = self.net
        net.forward(x)
        net.loss_and_grad(lab)
        net.backward(x)

    def _opt_body(self):
        self.net.optimizer_step()

    def capture(self):
        """Capture forward+backward and the optimiser into CUDA graphs (the NCCL all-reduce,
        when distributed, runs between the two)."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(2):   # warm-up on a side stream, as torch requires before capture
                self._train_body()
        torch.cuda.current_stream().wait_stream(s)
        self.g_train, self.g_opt = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.g_train):
            self._train_body()
        with torch.cuda.graph(self.g_opt):
            self._opt_body()
        self.graph = True
        self.net.ps.step_dev.zero_()

    def _run_train(self):
        if self.graph:
            self.g_train.replay()
            if self.allreduce is not None:
                self.allreduce()
            self.g_opt.replay()
        else:
            self._train_body()
            if self.allreduce is not None:
                self.allreduce()
            self._opt_body()

    def step_resident(self, ct_dev: torch.Tensor, nonce: bytes, aad_dev: torch.Tensor, nrec: int):
        """Ciphertext already in HBM: GCM open + decode + train.  Returns the device loss."""
        self.ctx.open_device(nonce, aad_dev, ct_dev, self.loader.pt, self.loader.work)
        s = self.spec
        decode_records(self.loader.pt, nrec, s["c"], s["h"], s["w"], s["mean"], s["std"], out=self.loader.x,
                       labels=self.loader.labels)
        self._run_train()
        return self.net.loss

    def step_host(self, blob_host: torch.Tensor, nonce: bytes, aad: bytes, nrec: int):
        """End-to-end step from pinned host ciphertext: H2D, decrypt, train, D2H of loss+status."""
        self.loader.stage(blob_host, aad)
        self.step_resident(self.loader.ct[:self.loader.n], nonce, self.loader.aad[:self.loader.aad_len], nrec)
        self.loss_host.copy_(self.net.loss, non_blocking=True)
        self.status_host[:1].copy_(self.loader.work[4:5], non_blocking=True)
        return self.loss_host

    def check_status(self):
        """Raise if the last shard's tag failed (its plaintext was zeroed on the device)."""
        torch.cuda.current_stream().synchronize()
        if int(self.status_host[0]) != 0:
            raise AuthenticationFailure("training shard failed authentication")


# ---- model sealing (the CVM1 format cannot hold CNN weights) ----------
def serialize_cnn_model(net) -> bytes:
    """b"CVC1" | u32 BE header length | canonical JSON header | fp32 LE parameters."""
    ps = net.ps
    header = {"model": type(net).__name__, "params": [[n, list(s)] for n, s, _ in ps.specs],
              "logical_params": ps.logical}
    hb = json.dumps(header, sort_keys=True, separators=(",", ":")).encode()
    blobs = [ps.p[n].detach().float().cpu().numpy().astype("<f4").tobytes() for n, _, _ in ps.specs]
    return CNN_MAGIC + struct.pack(">I", len(hb)) + hb + b"".join(blobs)


def deserialize_cnn_model(data: bytes):
    if not data.startswith(CNN_MAGIC):
        raise ValueError("bad model magic")
    (hl,) = struct.unpack_from(">I", data, 4)
    header = json.loads(data[8:8 + hl])
    off, out = 8 + hl, {}
    for name, shape in header["params"]:
        n = int(np.prod(shape))
        out[name] = np.frombuffer(data, dtype="<f4", count=n, offset=off).reshape(shape)
        off += 4 * n
    return header, out
