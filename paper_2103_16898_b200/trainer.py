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
import os
import struct
import warnings

import numpy as np

import torch

from . import kernels as K
from .crypto import AuthenticationFailure, GcmContext
from .loader import CIFAR, ShardLoader, decode_records, record_bytes
from .nets import make_model

CNN_MAGIC = b"CVC1"



_NO_PREFETCH = os.environ.get("CVB_NO_DECRYPT_PREFETCH", "0") not in ("", "0")

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


class OverlappedGradAllReduce:
    """Bucketed SUM all-reduce of the flat fp32 gradient buffer, overlapped with backward.

    Buckets are contiguous ranges of the flat buffer, built back to front (the order backward
    produces gradients), ~bucket_mb each.  Backward reports finished parameters through
    ParamStore.grad_ready; as soon as every parameter of the next bucket is final the bucket's
    all-reduce is launched on a side stream (after an event on the compute stream), so NCCL
    traffic over NVLink overlaps the remaining dgrad/wgrad kernels.  Buckets launch strictly in
    order (identical on every rank).  finish() launches the rest and joins the side stream.

    CUDA graphs: a `segment` callback, when set, is invoked at each bucket boundary instead of
    launching; EncryptedTrainer.capture uses it to split the captured backward into graph
    segments, and replays them with the bucket all-reduces issued between segments (NCCL stays
    outside the captured graphs).
    """

    def __init__(self, ps, bucket_mb: float | None = None, group=None):
        import torch.distributed as dist

        self.dist, self.group, self.ps = dist, group, ps
        if bucket_mb is None:   # <= 25 MB, and at least ~4 buckets so small models overlap too
            bucket_mb = min(25.0, ps.total * 4 / (1 << 20) / 4)
        per = max(1, int(bucket_mb * (1 << 20) / 4))
        self.buckets = []           # (lo, hi, names) flat ranges, back to front
        names, lo, hi = [], None, None
        order = sorted(ps.offsets.items(), key=lambda kv: -kv[1])
        ends = {}
        prev = ps.g32.numel()        # the first bucket also carries the verdict slot past ps.total
        for name, off in order:      # each parameter owns [off, next parameter's offset)
            ends[name] = prev
            prev = off
        for name, off in order:
            if hi is None:
                hi = ends[name]
            names.append(name)
            lo = off
            if hi - lo >= per:
                self.buckets.append((lo, hi, frozenset(names)))
                names, hi = [], None
        if names:
            self.buckets.append((0, hi, frozenset(names)))
        self.side = torch.cuda.Stream() if ps.g32.is_cuda else None
        self.segment = None
        self.reset()

    def reset(self):
        self.ready, self.next, self.works = set(), 0, []

    def __call__(self, names):
        self.ready.update(names)
        done = []
        while self.next < len(self.buckets) and self.buckets[self.next][2] <= self.ready:
            done.append(self.next)
            self.next += 1
        if done:
            self._launch(done)

    def launch_bucket(self, i):
        lo, hi, _ = self.buckets[i]
        view = self.ps.g32[lo:hi]
        if self.side is None:
            self.works.append(self.dist.all_reduce(view, op=self.dist.ReduceOp.SUM, group=self.group, async_op=True))
            return
        # the bucket's gradients come from the compute stream and, with the wgrad overlap on,
        # from the wgrad side stream: the collective waits for both
        cur = torch.cuda.current_stream()
        self.side.wait_stream(cur)
        wg = self.ps.side
        if wg is not None and wg != cur:
            self.side.wait_stream(wg)
        with torch.cuda.stream(self.side):
            self.dist.all_reduce(view, op=self.dist.ReduceOp.SUM, group=self.group)

    def _launch(self, idx):
        if self.segment is not None:
            self.segment(idx)
        else:
            for i in idx:
                self.launch_bucket(i)

    def finish(self):
        if self.next < len(self.buckets):
            self._launch(list(range(self.next, len(self.buckets))))
            self.next = len(self.buckets)
        self.join()

    def join(self):
        for w in self.works:
            w.wait()
        self.works = []
        if self.side is not None:
            torch.cuda.current_stream().wait_stream(self.side)


class EncryptedTrainer:
    def __init__(self, model="small_cnn", key: bytes = bytes(range(32)), batch=512, spec=CIFAR, seed=0,
                 world=1, rank=0, max_shard_bytes=None, lr=1e-3, force_allreduce=False, graph_collectives=None):
        self.spec, self.batch, self.world, self.rank = spec, batch, world, rank
        self.net = make_model(model, seed=seed).build(batch, global_batch=batch * world)
        self.net.lr = lr
        self.ctx = GcmContext(key)
        rec = record_bytes(spec["c"], spec["h"], spec["w"])
        self.loader = ShardLoader(self.ctx, max_shard_bytes or batch * rec, batch, spec)
        self.allreduce = None
        if world > 1 or force_allreduce:
            self.allreduce = OverlappedGradAllReduce(self.net.ps)
            self.net.ps.grad_hook = self.allreduce
        # NCCL collectives are capturable: the whole step (backward + bucket all-reduces on the
        # side stream + optimiser) is then ONE graph replay with no host issue between buckets,
        # and the wgrad side-stream overlap stays on.  gloo is not: its steps are captured as
        # segments cut at bucket boundaries, the all-reduces issued between segment replays.
        if graph_collectives is None:
            graph_collectives = False
            if self.allreduce is not None:
                import torch.distributed as dist

                graph_collectives = dist.is_initialized() and dist.get_backend() == "nccl"
        self.graph_collectives = bool(graph_collectives) and self.allreduce is not None
        self.net.ps.overlap_with_hook = self.graph_collectives
        self.graph = None
        # sticky run verdict: every shard opened through self.ctx ORs its tag verdict into this
        # word; each step snapshots it into the gradient buffer's verdict slot (summed over
        # ranks by the gradient all-reduce), and Adam skips the update when the slot is non-zero
        self.verdict = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.ctx.set_verdict(self.verdict)
        self.status_host = torch.zeros(8, dtype=torch.int32).pin_memory()
        self.verdict_host = torch.zeros(1, dtype=torch.float32).pin_memory()
        self.loss_host = torch.zeros(1, dtype=torch.float32).pin_memory()

    # -- the step ------------------------------------------------------------------------
    def _train_body(self):
        x, lab = self.loader.x[:self.batch], self.loader.labels[:self.batch]
        net = self.net
        if self.allreduce is not None:
            self.allreduce.reset()
        K.verdict_snapshot(self.verdict, net.ps.verdict_slot)   # no decrypt is in flight here
        net.fwd_bwd(x, lab)

    def _opt_body(self):
        self.net.optimizer_step()

    def capture(self):
        """Capture the step into CUDA graphs.  Single GPU: forward+backward and the optimiser.
        Data parallel: the backward is split into segments at gradient-bucket boundaries; at
        replay each bucket's NCCL all-reduce is issued (side stream) right after the segment
        that finishes it, so communication overlaps the rest of the backward."""
        ar = self.allreduce
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(2):   # warm-up on a side stream, as torch requires before capture
                self._train_body()
                if ar is not None:
                    ar.finish()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        pool = torch.cuda.graph_pool_handle()
        if self.graph_collectives:
            # one graph: forward, backward with the bucket all-reduces issued from the grad-ready
            # hooks on the collective side stream as buckets complete, the join, the optimiser
            self.segments, self.tail_from = [], len(ar.buckets)
            self.g_train = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                self.g_train.capture_begin(pool=pool)
                self._train_body()
                ar.finish()
                self.g_train.capture_end()
            self.g_opt = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.g_opt, pool=pool):
                self._opt_body()
            torch.cuda.current_stream().wait_stream(s)
            self.graph = True
            self.net.ps.step_dev.zero_()
            return
        self.segments = []
        cur = [torch.cuda.CUDAGraph()]
        if ar is not None:
            def cut(idx):
                cur[0].capture_end()
                self.segments.append((cur[0], idx))
                cur[0] = torch.cuda.CUDAGraph()
                cur[0].capture_begin(pool=pool)
            ar.segment = cut
        with torch.cuda.stream(s), warnings.catch_warnings():
            warnings.filterwarnings("ignore", message="The CUDA Graph is empty")   # tail after the last bucket
            cur[0].capture_begin(pool=pool)
            self._train_body()
            cur[0].capture_end()
        self.g_train = cur[0]
        if ar is not None:
            ar.segment = None
            self.tail_from = ar.next
        self.g_opt = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.g_opt, pool=pool):
            self._opt_body()
        torch.cuda.current_stream().wait_stream(s)
        self.graph = True
        self.net.ps.step_dev.zero_()

    def _run_train(self, after_train=None):
        """after_train: host callback issued between the forward/backward and the optimiser
        (the e2e path's D2H of loss + verdict, whose latency then hides behind the optimiser)."""
        ar = self.allreduce
        if self.graph:
            for g, idx in self.segments:
                g.replay()
                for i in idx:
                    ar.launch_bucket(i)
            self.g_train.replay()
            if ar is not None and not self.graph_collectives:
                for i in range(self.tail_from, len(ar.buckets)):
                    ar.launch_bucket(i)
                ar.join()
            if after_train is not None:
                after_train()
            self.g_opt.replay()
        else:
            self._train_body()
            if ar is not None:
                ar.finish()
            if after_train is not None:
                after_train()
            self._opt_body()

    def step_resident(self, ct_dev: torch.Tensor, nonce: bytes, aad_dev: torch.Tensor, nrec: int,
                      after_train=None, next_shard=None):
        """Ciphertext already in HBM: GCM open + decode + train.  Returns the device loss.

        ``next_shard = (ct_dev, nonce, aad_dev)`` of the following step: with a captured step its
        decrypt is issued on a side stream as soon as this step's forward/backward no longer
        needs the input tile, so it runs beside the optimiser; the next call with that shard
        then skips its decrypt.  Each shard's tag verdict lands in its own work buffer."""
        main = torch.cuda.current_stream()
        d2h = getattr(self, "d2h_done", None)
        if d2h is not None:   # the previous step's D2H has read the loss and the verdict
            main.wait_event(d2h)
        key = (ct_dev.data_ptr(), ct_dev.numel(), bytes(nonce))
        pend = getattr(self, "_pend", None)
        if pend is not None:
            main.wait_event(self._pend_ev)   # the prefetched decrypt has written the tile
            self._pend = None
        if pend is not None and pend[0] == key:
            self._wcur = pend[1]
        else:
            # fused decrypt-and-normalise: ciphertext -> bf16 tile + labels, tag checked on the device
            self._wcur = self._wnext()
            self.ctx.open_records_device(nonce, aad_dev, ct_dev, self.loader.x, self.loader.labels,
                                         self._works[self._wcur], self.spec)

        def after():
            if after_train is not None:
                after_train()
            if next_shard is not None and self.graph and not _NO_PREFETCH:
                self._prefetch_decrypt(*next_shard)

        self._run_train(after)
        return self.net.loss

    @property
    def _works(self):
        if getattr(self, "_work_pair", None) is None:
            self._work_pair = [self.loader.work, self.ctx.new_workspace(self.loader.work.device)]
        return self._work_pair

    def _wnext(self):
        return (getattr(self, "_wcur", 1) + 1) % 2

    def _prefetch_decrypt(self, ct_dev, nonce, aad_dev, wait_event=None):
        """Decrypt the next shard into the input tile on the decrypt stream (after this step's
        backward: the tile's last readers are done)."""
        if getattr(self, "dstream", None) is None:
            self.dstream = torch.cuda.Stream()
            self._pend_ev = torch.cuda.Event()
        self.dstream.wait_stream(torch.cuda.current_stream())
        if wait_event is not None:
            self.dstream.wait_event(wait_event)
        w = self._wnext()
        with torch.cuda.stream(self.dstream):
            self.ctx.open_records_device(nonce, aad_dev, ct_dev, self.loader.x, self.loader.labels, self._works[w],
                                         self.spec)
        self._pend_ev.record(self.dstream)
        self._pend = ((ct_dev.data_ptr(), ct_dev.numel(), bytes(nonce)), w)

    def _issue_d2h(self):
        """D2H of the step's loss and run verdict on a side stream (after forward/backward and
        the gradient exchange: with data parallelism the verdict slot is the sum over ranks)."""
        if getattr(self, "d2h_stream", None) is None:
            self.d2h_stream = torch.cuda.Stream()
            self.d2h_done = torch.cuda.Event()
        self.d2h_stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.d2h_stream):
            self.loss_host.copy_(self.net.loss, non_blocking=True)
            self.verdict_host.copy_(self.net.ps.verdict_slot, non_blocking=True)
        self.d2h_done.record(self.d2h_stream)

    def step_host(self, blob_host: torch.Tensor, nonce: bytes, aad: bytes, nrec: int, next_blob=None,
                  next_aad: bytes | None = None, next_nonce: bytes | None = None):
        """End-to-end step from pinned host ciphertext: H2D, decrypt, train, D2H of loss+status.

        With ``next_blob``/``next_aad`` (the following shard) the next H2D copy is issued on a
        copy stream while this step computes, and the next call consumes it (double buffering);
        the result of each step is identical either way."""
        ld = self.loader
        if getattr(ld, "next_src", None) == blob_host.data_ptr() and ld.next_n == blob_host.numel():
            ct, aad_dev = ld.take_prefetched()     # copied during the previous step
        else:
            ld.stage(blob_host, aad)
            ct, aad_dev = ld.ct[:ld.n], ld.aad[:ld.aad_len]
        if next_blob is not None:
            ld.prefetch(next_blob, next_aad)
        after = self._issue_d2h
        if next_blob is not None and next_nonce is not None and self.graph and not _NO_PREFETCH:
            # also decrypt the next shard beside this step's optimiser, once its H2D copy is in
            def after():
                self._issue_d2h()
                self._prefetch_decrypt(ld.ct_next[:ld.next_n], next_nonce, ld.aad_next[:ld.next_aad_len],
                                       wait_event=ld.copy_done)
        self.step_resident(ct, nonce, aad_dev, nrec, after_train=after)
        ld.release_spare()
        return self.loss_host

    def check_status(self, include_pending: bool = False):
        """Raise if any shard trained so far -- on any rank -- failed authentication.

        The device already kept every failed shard out of training (its tile was zeroed and
        the optimiser skipped that step and every later one); this surfaces the verdict on
        the host.  It reads the verdict slot of the last step, which the gradient all-reduce
        summed over ranks, so every rank raises at the same step.  ``include_pending`` also
        reads this rank's sticky word, which additionally covers a shard already decrypted
        ahead but not trained on yet (the final check before a model is sealed)."""
        torch.cuda.current_stream().synchronize()
        if getattr(self, "d2h_done", None) is not None:
            self.d2h_done.synchronize()
        bad = float(self.net.ps.verdict_slot.item()) != 0.0
        if include_pending:
            bad = bad or int(self.verdict.item()) != 0
        if bad:
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
