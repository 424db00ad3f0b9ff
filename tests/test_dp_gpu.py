"""Data-parallel step machinery on one B200: NCCL process group of world size 1 (the
all-reduce is then the identity), so the overlapped-bucket path -- grad-ready hooks, side-stream
NCCL launches, CUDA-graph segments split at bucket boundaries -- must reproduce the plain
single-GPU step bit for bit."""
import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_group():
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("model,graph_collectives", [("small_cnn", False), ("resnet18", False),
                                                      ("small_cnn", True), ("resnet18", True)])
def test_overlapped_allreduce_step_matches_single_gpu(nccl_group, model, graph_collectives):
    from bench import make_shards
    from paper_2103_16898_b200.loader import CIFAR
    from paper_2103_16898_b200.trainer import EncryptedTrainer

    key, B = bytes(range(32)), 32
    shards = make_shards(3, B, 5, key, CIFAR)
    cts = [torch.frombuffer(bytearray(s[3]), dtype=torch.uint8).cuda() for s in shards]
    aads = [torch.frombuffer(bytearray(s[2]), dtype=torch.uint8).cuda() for s in shards]
    runs = {}
    for dp in (False, True):
        tr = EncryptedTrainer(model, key, batch=B, spec=CIFAR, seed=3, force_allreduce=dp,
                              graph_collectives=graph_collectives)
        if dp:
            assert len(tr.allreduce.buckets) >= 1
            tr.allreduce.__init__(tr.net.ps, bucket_mb=0.25)     # several buckets -> several segments
        losses = []
        tr.step_resident(cts[0], shards[0][1], aads[0], B)       # eager step
        losses.append(float(tr.net.loss.item()))
        tr.capture()
        if dp and not graph_collectives:
            assert len(tr.segments) >= 2, "backward was not split at bucket boundaries"
        if dp and graph_collectives:   # one graph: NCCL captured, wgrad side stream kept on
            assert tr.segments == [] and tr.net.ps.overlap_with_hook
        for i in (1, 2):
            tr.step_resident(cts[i], shards[i][1], aads[i], B)
            losses.append(float(tr.net.loss.item()))
        torch.cuda.synchronize()
        runs[dp] = (losses, tr.net.ps.p32.clone())
    assert runs[False][0] == runs[True][0]
    assert torch.equal(runs[False][1], runs[True][1])


def test_double_buffered_host_steps_match_plain_host_steps():
    """step_host with the next shard prefetched on a copy stream == step_host staging each
    shard on the compute stream (same losses, same weights, bit for bit)."""
    from bench import make_shards
    from paper_2103_16898_b200.loader import CIFAR
    from paper_2103_16898_b200.trainer import EncryptedTrainer

    key, B = bytes(range(32)), 64
    shards = make_shards(4, B, 9, key, CIFAR)
    host = [torch.frombuffer(bytearray(s[3]), dtype=torch.uint8).pin_memory() for s in shards]
    runs = []
    for pipelined in (False, True):
        tr = EncryptedTrainer("small_cnn", key, batch=B, spec=CIFAR, seed=2)
        tr.capture()
        losses = []
        for i in range(6):
            j, k = i % 4, (i + 1) % 4
            if pipelined:
                tr.step_host(host[j], shards[j][1], shards[j][2], B, next_blob=host[k], next_aad=shards[k][2])
            else:
                tr.step_host(host[j], shards[j][1], shards[j][2], B)
            tr.check_status()
            losses.append(float(tr.loss_host[0]))
        runs.append((losses, tr.net.ps.p32.clone()))
    assert runs[0][0] == runs[1][0]
    assert torch.equal(runs[0][1], runs[1][1])


def _dp_worker(rank, world, port, q):
    import torch.distributed as dist

    from bench import make_shards
    from paper_2103_16898_b200.loader import CIFAR
    from paper_2103_16898_b200.trainer import EncryptedTrainer

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)   # both ranks share cuda:0
    key, B = bytes(range(32)), 32
    shards = make_shards(3, B, 40 + rank, key, CIFAR)                 # different data per rank
    cts = [torch.frombuffer(bytearray(s[3]), dtype=torch.uint8).cuda() for s in shards]
    aads = [torch.frombuffer(bytearray(s[2]), dtype=torch.uint8).cuda() for s in shards]
    tr = EncryptedTrainer("resnet18", key, batch=B, spec=CIFAR, seed=3, world=world, rank=rank)
    tr.allreduce.__init__(tr.net.ps, bucket_mb=4.0)
    tr.step_resident(cts[0], shards[0][1], aads[0], B)           # eager, overlapped buckets
    tr.capture()                                                  # graph segments between buckets
    for i in (1, 2):
        tr.step_resident(cts[i], shards[i][1], aads[i], B)
    torch.cuda.synchronize()
    p = tr.net.ps.p32.detach().cpu()
    ref = p.clone()
    dist.broadcast(ref, src=0)
    q.put((rank, len(tr.segments), float((p - ref).abs().max()), float(p.abs().sum())))
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_rank_data_parallel_weights_stay_identical():
    """Two ranks (gloo, sharing the one GPU), different shards, overlapped bucket all-reduce
    with the backward split into CUDA-graph segments: after 3 steps every rank holds the
    same weights bit for bit."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=500) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, nseg, diff, norm in out:
        assert nseg >= 2 and diff == 0.0 and norm > 0
