"""Decrypt-and-normalise loader: sealed record shards -> verified input tiles in HBM.

Replaces the reference's data path Volume.get(...) -> bytes.decode -> parse_dataset
(/root/reference/pkg/src/covault/volume.py:185-197, workload.py:24-41) for the binary
record payload (CIFAR-10 binary layout: 1 label byte + C*H*W CHW pixel bytes per record).

Per shard: ciphertext (host, pinned) -> H2D -> GCM open kernel (bit-exact AES-256-GCM,
tag verified on device) -> record decoder kernel -> NHWC-8 bf16 tile + int32 labels.
Security contract kept from the reference: a shard's plaintext is never consumed before its
tag verdict is known (``ShardLoader.next`` checks the device status word of the shard it
hands out; on a mismatch the plaintext was already zeroed on-stream and
AuthenticationFailure is raised -- volume.py:186 "never partial").
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from .crypto import AuthenticationFailure, GcmContext
from .volume import Volume, aad_for

CIFAR = dict(c=3, h=32, w=32, mean=(0.5, 0.5, 0.5), std=(0.25, 0.25, 0.25))
MEDICAL = dict(c=1, h=224, w=224, mean=(0.5,), std=(0.25,))


def record_bytes(c, h, w):
    return 1 + c * h * w


def decode_records(pt_dev: torch.Tensor, nrec: int, c: int, h: int, w: int, mean, std, out=None, labels=None,
                   dtype=torch.bfloat16):
    """Verified plaintext records (uint8 CUDA tensor) -> (NHWC-8 tile, int32 labels)."""
    lib = _lib.load()
    if out is None:
        out = torch.empty(nrec, h, w, 8, dtype=dtype, device=pt_dev.device)
    if labels is None:
        labels = torch.empty(nrec, dtype=torch.int32, device=pt_dev.device)
    m = (ctypes.c_float * 8)(*mean)
    s = (ctypes.c_float * 8)(*std)
    rc = lib.cvb_records_to_nhwc(pt_dev.data_ptr(), nrec, record_bytes(c, h, w), c, h, w, m, s,
                                 0 if dtype == torch.bfloat16 else 1, out.data_ptr(), labels.data_ptr(),
                                 _lib.stream_ptr())
    _lib.check(rc, "records_to_nhwc")
    return out, labels



def _pinned(b: bytes) -> torch.Tensor:
    """bytes -> page-locked uint8 tensor.  An H2D copy from pageable memory is staged
    synchronously by the driver (and can wait on the copy stream's pending work); from
    page-locked memory it is a true async DMA.  torch's caching host allocator keeps the
    block alive until the copy that reads it has completed."""
    t = torch.empty(len(b), dtype=torch.uint8, pin_memory=True)
    if len(b):
        t.numpy()[:] = memoryview(b)
    return t

class ShardSet:
    """Sealed shards of one volume, held as pinned host ciphertext (the e2e input)."""

    def __init__(self, volume: Volume, paths, spec=CIFAR):
        self.volume, self.paths, self.spec = volume, list(paths), spec
        self.rec = record_bytes(spec["c"], spec["h"], spec["w"])
        self.blobs, self.nonces, self.aads, self.nrec = [], [], [], []
        for p in self.paths:
            e = volume.entry(p)
            blob = volume.read_blob(p)
            if (len(blob) - 16) % self.rec:
                raise ValueError(f"{p}: plaintext length is not a whole number of records")
            host = torch.frombuffer(bytearray(blob), dtype=torch.uint8).pin_memory()
            self.blobs.append(host)
            self.nonces.append(e.nonce)
            self.aads.append(aad_for(volume.volume_name, p))
            self.nrec.append((len(blob) - 16) // self.rec)


class ShardLoader:
    """Device pipeline for one shard at a time (buffers reused; graph-capture friendly)."""

    def __init__(self, ctx: GcmContext, max_shard_bytes: int, max_records: int, spec=CIFAR, device="cuda"):
        self.ctx, self.spec = ctx, spec
        self.ct = torch.empty(max_shard_bytes + 16, dtype=torch.uint8, device=device)
        self.pt = torch.empty(max_shard_bytes, dtype=torch.uint8, device=device)
        self.aad = torch.zeros(256, dtype=torch.uint8, device=device)
        self.work = ctx.new_workspace(device)
        # zeroed once: the fused loader never writes the pad channels (3..7 / 1..7)
        self.x = torch.zeros(max_records, spec["h"], spec["w"], 8, dtype=torch.bfloat16, device=device)
        self.labels = torch.empty(max_records, dtype=torch.int32, device=device)

    def stage(self, blob_host: torch.Tensor, aad: bytes):
        """H2D copy of one sealed shard (async on the current stream)."""
        n = blob_host.numel()
        self.ct[:n].copy_(blob_host, non_blocking=True)
        self.aad[:len(aad)].copy_(_pinned(aad), non_blocking=True)
        self.n, self.aad_len = n, len(aad)

    # -- double-buffered host->device staging (the e2e path overlaps the next shard's H2D
    #    with this step's decrypt + training) ------------------------------------------------
    def prefetch(self, blob_host: torch.Tensor, aad: bytes):
        """Start the H2D copy of the NEXT shard on a copy stream into the spare buffer."""
        if not hasattr(self, "ct_next"):
            self.ct_next = torch.empty_like(self.ct)
            self.aad_next = torch.zeros_like(self.aad)
            self.copy_stream = torch.cuda.Stream()
            self.copy_done = torch.cuda.Event()
            self.buf_free = torch.cuda.Event()
            self.buf_free.record()
        n = blob_host.numel()
        self.copy_stream.wait_event(self.buf_free)       # the spare buffer's last reader is done
        with torch.cuda.stream(self.copy_stream):
            self.ct_next[:n].copy_(blob_host, non_blocking=True)
            self.aad_next[:len(aad)].copy_(_pinned(aad), non_blocking=True)
        self.copy_done.record(self.copy_stream)
        self.next_n, self.next_aad_len = n, len(aad)
        self.next_src = blob_host.data_ptr()

    def take_prefetched(self):
        """Swap the prefetched shard in (the compute stream waits for its copy); returns
        (ciphertext view, aad view)."""
        torch.cuda.current_stream().wait_event(self.copy_done)
        self.ct, self.ct_next = self.ct_next, self.ct
        self.aad, self.aad_next = self.aad_next, self.aad
        self.n, self.aad_len = self.next_n, self.next_aad_len
        self.next_n, self.next_src = None, None
        return self.ct[:self.n], self.aad[:self.aad_len]

    def release_spare(self):
        """Record that the compute stream is done with the (now spare) previous buffer."""
        if hasattr(self, "buf_free"):
            self.buf_free.record()

    def decrypt_decode(self, nonce: bytes, nrec: int):
        """Fused GCM open + record decode (one kernel), stream-ordered, no host sync."""
        self.ctx.open_records_device(nonce, self.aad[:self.aad_len], self.ct[:self.n], self.x, self.labels,
                                     self.work, self.spec)
        return self.x[:nrec], self.labels[:nrec]

    def verify(self):
        """Host check of the tag verdict of the last decrypted shard (synchronises)."""
        if int(self.work[4].item()) != 0:
            raise AuthenticationFailure("AEAD authentication failed for training shard")
