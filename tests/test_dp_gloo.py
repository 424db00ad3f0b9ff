"""Data-parallel plumbing on CPU with the gloo backend (world size 2, 127.0.0.1).

Covers trainer.GradAllReduce (bucketed SUM all-reduce of the flat fp32 gradient buffer) and
the weak-scaling gradient convention the GPU step uses: each rank scales its loss gradient
by 1/global_batch, so the all-reduced SUM equals the full-batch mean gradient.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _worker_allreduce(rank, world, port, q):
    from paper_2103_16898_b200.trainer import GradAllReduce

    _init(rank, world, port)
    g = torch.arange(10_000, dtype=torch.float32) * (rank + 1)
    ar = GradAllReduce(g, bucket_mb=0.01)       # ~2.6k floats per bucket -> 4 buckets
    nb = len(ar.buckets)
    ar()
    q.put((rank, nb, float(g.sum()), float(g[123])))
    dist.destroy_process_group()


def _worker_convention(rank, world, port, q):
    _init(rank, world, port)
    torch.manual_seed(0)
    X = torch.randn(16, 5)
    y = torch.randint(0, 3, (16,))
    W = torch.randn(3, 5, requires_grad=True)
    B = X.shape[0]
    lo, hi = rank * B // world, (rank + 1) * B // world
    loss = torch.nn.functional.cross_entropy(X[lo:hi] @ W.t(), y[lo:hi], reduction="sum") / B
    loss.backward()
    from paper_2103_16898_b200.trainer import GradAllReduce

    g = W.grad.reshape(-1).clone()
    GradAllReduce(g)()
    Wf = W.detach().clone().requires_grad_(True)
    torch.nn.functional.cross_entropy(X @ Wf.t(), y).backward()
    q.put((rank, float((g - Wf.grad.reshape(-1)).abs().max())))
    dist.destroy_process_group()


class _FakeStore:
    """The ParamStore fields the overlapped all-reduce uses (flat fp32 grads, offsets)."""

    def __init__(self, sizes, rank):
        self.offsets, off = {}, 0
        for i, n in enumerate(sizes):
            self.offsets[f"p{i}"] = off
            off += (n + 63) // 64 * 64
        self.total = off
        self.g32 = torch.zeros(off)
        for i, n in enumerate(sizes):
            o = self.offsets[f"p{i}"]
            self.g32[o:o + n] = (i + 1) * (rank + 1)


def _worker_overlapped(rank, world, port, q):
    from paper_2103_16898_b200.trainer import OverlappedGradAllReduce

    _init(rank, world, port)
    sizes = [3000, 64, 64, 5000, 10, 10, 20000, 256]
    ps = _FakeStore(sizes, rank)
    ar = OverlappedGradAllReduce(ps, bucket_mb=0.02)     # ~5k floats per bucket
    launched = []
    ar.segment = None
    orig = ar.launch_bucket
    ar.launch_bucket = lambda i: (launched.append(i), orig(i))   # noqa: E731
    # backward reports parameters last-to-first, two at a time (like conv W then BN G/B)
    names = [f"p{i}" for i in range(len(sizes))][::-1]
    progress = []
    for k in range(0, len(names), 2):
        ar(names[k:k + 2])
        progress.append(list(launched))
    ar.finish()
    ok = all(float(ps.g32[ps.offsets[f"p{i}"]]) == (i + 1) * 3 for i in range(len(sizes)))
    q.put((rank, len(ar.buckets), launched, progress, ok))
    dist.destroy_process_group()


def _run(target, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out)


@pytest.mark.timeout(300)
def test_bucketed_allreduce_sums_every_bucket():
    out = _run(_worker_allreduce)
    want_sum = float(torch.arange(10_000, dtype=torch.float32).sum() * 3)
    for rank, nb, s, v in out:
        assert nb >= 4
        assert abs(s - want_sum) / want_sum < 1e-6
        assert v == 123 * 3


@pytest.mark.timeout(300)
def test_weak_scaling_gradient_convention():
    for rank, err in _run(_worker_convention):
        assert err < 1e-6


@pytest.mark.timeout(300)
def test_overlapped_allreduce_launches_buckets_as_backward_finishes_them():
    """Buckets are contiguous back-to-front ranges; each launches as soon as backward has
    reported all of its parameters (before backward ends), in order, and every parameter is
    summed over the ranks exactly once."""
    for rank, nb, launched, progress, ok in _run(_worker_overlapped):
        assert ok
        assert launched == list(range(nb)) and nb >= 3
        assert progress[0] != [] and len(progress[-2]) < nb    # launches overlap the "backward"
