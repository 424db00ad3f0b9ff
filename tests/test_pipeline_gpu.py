"""Step pipelining of the encrypted trainer: the next shard's decrypt issued beside the
optimiser (step_resident(next_shard=...), step_host(next_nonce=...)) must give bit-identical
losses and weights to the unpipelined steps, and keep per-shard tag verdicts exact."""
import pytest
import torch

from paper_2103_16898_b200.crypto import AuthenticationFailure
from paper_2103_16898_b200.loader import CIFAR
from paper_2103_16898_b200.trainer import EncryptedTrainer

pytestmark = pytest.mark.gpu


def _shards(n, B, seed, key):
    from bench import make_shards
    return make_shards(n, B, seed, key, CIFAR)


def test_resident_decrypt_prefetch_bit_exact():
    key, B = bytes(range(32)), 64
    shards = _shards(3, B, 4, key)
    cts = [torch.frombuffer(bytearray(s[3]), dtype=torch.uint8).cuda() for s in shards]
    aads = [torch.frombuffer(bytearray(s[2]), dtype=torch.uint8).cuda() for s in shards]
    runs = []
    for pipelined in (False, True):
        tr = EncryptedTrainer("small_cnn", key, batch=B, spec=CIFAR, seed=3)
        tr.capture()
        losses = []
        for i in range(7):
            j, k = i % 3, (i + 1) % 3
            nxt = (cts[k], shards[k][1], aads[k]) if pipelined and i < 6 else None
            losses.append(float(tr.step_resident(cts[j], shards[j][1], aads[j], B, next_shard=nxt).item()))
        runs.append((losses, tr.net.ps.p32.clone()))
    assert runs[0][0] == runs[1][0]
    assert torch.equal(runs[0][1], runs[1][1])


def test_host_decrypt_prefetch_bit_exact_and_verdicts():
    key, B = bytes(range(32)), 64
    shards = _shards(4, B, 6, key)
    host = [torch.frombuffer(bytearray(s[3]), dtype=torch.uint8).pin_memory() for s in shards]
    runs = []
    for pipelined in (False, True):
        tr = EncryptedTrainer("small_cnn", key, batch=B, spec=CIFAR, seed=2)
        tr.capture()
        losses = []
        for i in range(6):
            j, k = i % 4, (i + 1) % 4
            if pipelined and i < 5:
                tr.step_host(host[j], shards[j][1], shards[j][2], B, next_blob=host[k], next_aad=shards[k][2],
                             next_nonce=shards[k][1])
            else:
                tr.step_host(host[j], shards[j][1], shards[j][2], B)
            tr.check_status()
            losses.append(float(tr.loss_host[0]))
        runs.append((losses, tr.net.ps.p32.clone()))
    assert runs[0][0] == runs[1][0]
    assert torch.equal(runs[0][1], runs[1][1])
    # a tampered shard decrypted ahead (beside the previous step's optimiser): the step that
    # trains on it reports the failure, the step before it does not
    bad = host[1].clone().pin_memory()
    bad[100] ^= 1
    tr = EncryptedTrainer("small_cnn", key, batch=B, spec=CIFAR, seed=2)
    tr.capture()
    tr.step_host(host[0], shards[0][1], shards[0][2], B, next_blob=bad, next_aad=shards[1][2],
                 next_nonce=shards[1][1])
    tr.check_status()                      # shard 0 is fine
    with pytest.raises(AuthenticationFailure):
        tr.check_status(include_pending=True)   # ... but the shard decrypted ahead is not
    w_before = tr.net.ps.p32.clone()
    m_before, step_before = tr.net.ps.m.clone(), int(tr.net.ps.step_dev.item())
    tr.step_host(bad, shards[1][1], shards[1][2], B)
    with pytest.raises(AuthenticationFailure):
        tr.check_status()
    assert torch.count_nonzero(tr.loader.x) == 0   # nothing unverified reached the step
    # the optimiser was gated on the device verdict: weights, moments and step counter unchanged
    assert torch.equal(tr.net.ps.p32, w_before)
    assert torch.equal(tr.net.ps.m, m_before)
    assert int(tr.net.ps.step_dev.item()) == step_before
    # ... and stays gated (sticky) for later good shards until the run is abandoned
    tr.step_host(host[2], shards[2][1], shards[2][2], B)
    torch.cuda.synchronize()
    assert torch.equal(tr.net.ps.p32, w_before)


def test_sticky_verdict_in_timed_loop_resident():
    """A tampered shard in the middle of a pipelined resident run (step k < K) is caught by
    the sticky run verdict after the loop, and no step from k on moved the weights."""
    key, B = bytes(range(32)), 64
    shards = _shards(4, B, 8, key)
    cts = [torch.frombuffer(bytearray(s[3]), dtype=torch.uint8).cuda() for s in shards]
    aads = [torch.frombuffer(bytearray(s[2]), dtype=torch.uint8).cuda() for s in shards]
    bad = cts[2].clone()
    bad[1000] ^= 0x10
    seq = [cts[0], cts[1], bad, cts[3], cts[0]]
    idx = [0, 1, 2, 3, 0]
    tr = EncryptedTrainer("small_cnn", key, batch=B, spec=CIFAR, seed=5)
    tr.capture()
    snaps = []
    for i in range(5):
        nxt = (seq[i + 1], shards[idx[i + 1]][1], aads[idx[i + 1]]) if i + 1 < 5 else None
        tr.step_resident(seq[i], shards[idx[i]][1], aads[idx[i]], B, next_shard=nxt)
        torch.cuda.synchronize()
        snaps.append(tr.net.ps.p32.clone())
    with pytest.raises(AuthenticationFailure):
        tr.check_status()
    assert not torch.equal(snaps[0], snaps[1])      # good steps trained
    assert torch.equal(snaps[1], snaps[2]) and torch.equal(snaps[2], snaps[4])
