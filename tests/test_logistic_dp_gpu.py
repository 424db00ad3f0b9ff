"""Data-parallel reference trainer: rows sharded in contiguous blocks, one
SUM all-reduce of the F+1 gradient sums per epoch, identical update on every rank.

Reference loop: /root/reference/pkg/src/covault/workload.py:57-70.  At world size 1 the
device-resident trainer is the bit-exact reference schedule; at world size 2 (two gloo ranks
sharing the one B200) it is within 1e-9 relative of the single-rank fp64 result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import ref

pytestmark = pytest.mark.gpu


def _data(n=3000, f=3072, seed=11):
    rng = np.random.default_rng(seed)
    X = np.round(rng.random((n, f)), 4)
    y = (rng.random(n) > 0.5).astype(np.float64)
    return X, y


def test_device_trainer_world1_bit_exact():
    from paper_2103_16898_b200.workload import LogisticTrainer

    X, y = _data(700, 513, 3)
    w0, b0 = ref.logistic_train(X, y, 0.25, 4)
    tr = LogisticTrainer(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), exact=True)
    w1, b1 = tr.train(0.25, 4)
    assert np.array_equal(w0.view(np.uint64), w1.view(np.uint64)) and b0 == b1


@pytest.mark.parametrize("f", [7, 3072, 5000])
def test_device_trainer_fast_within_tolerance(f):
    from paper_2103_16898_b200.workload import LogisticTrainer

    X, y = _data(2500, f, f)
    w0, b0 = ref.logistic_train(X, y, 0.1, 3)
    tr = LogisticTrainer(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), exact=False)
    w1, b1 = tr.train(0.1, 3)
    scale = max(1.0, float(np.max(np.abs(w0))))
    assert np.max(np.abs(w1 - w0)) <= 1e-9 * scale
    assert abs(b1 - b0) <= 1e-9 * max(1.0, abs(b0))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, X, y, exact, q):
    import torch.distributed as dist

    from paper_2103_16898_b200.workload import LogisticTrainer, shard_rows

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_rows(X.shape[0], world, rank)
    tr = LogisticTrainer(torch.from_numpy(X[lo:hi]).cuda(), torch.from_numpy(y[lo:hi]).cuda(), exact=exact,
                         group=dist.group.WORLD, n_total=X.shape[0])
    w, b = tr.train(0.2, 3)
    q.put((rank, w, b))
    dist.destroy_process_group()


@pytest.mark.parametrize("exact", [True, False])
def test_two_rank_gloo_matches_single_rank(exact):
    X, y = _data(2001, 3072, 5)
    w0, b0 = ref.logistic_train(X, y, 0.2, 3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, X, y, exact, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, wa, ba), (_, wb_, bb) = sorted(out, key=lambda t: t[0])
    assert np.array_equal(wa, wb_) and ba == bb               # identical update on every rank
    scale = max(1.0, float(np.max(np.abs(w0))))
    assert np.max(np.abs(wa - w0)) <= 1e-9 * scale
    assert abs(ba - b0) <= 1e-9 * max(1.0, abs(b0))
