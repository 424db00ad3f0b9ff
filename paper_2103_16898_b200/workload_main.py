"""The B200 training workload, run inside the (simulated) enclave.

Same contract as the reference artifact /root/reference/pkg/scenarios/assets/trainer_workload/
train.py:23-53: one canonical JSON key document on stdin (runtime.py:15-20, :132-137);
roles ``training-data`` / ``trainer-code`` / ``model-output``; exit 3 before any read if a
role key is missing, exit 4 on any failure (including an authentication failure of any
shard), exit 0 after sealing ``model.bin`` into the output volume.

``params.json`` (trainer-code volume) selects the path:
  * no ``model`` key  -> the reference logistic trainer on ``dataset.csv`` (GPU, bit-exact),
  * ``model`` in {small_cnn, resnet18, densenet121} -> CNN training over the sealed record
    shards ``shard-*.bin`` of the training volume (GPU decrypt + train), weights sealed in
    the CVC1 format.  Keys used: model, epochs (1), learning_rate (1e-3), batch_size
    (records per shard), seed (0), world_size (ranks; default every visible GPU), backend
    ("nccl" when every rank has its own GPU, else "gloo").
"""
from __future__ import annotations

import json
import os
import sys

ROLE_TRAINING = "training-data"
ROLE_CODE = "trainer-code"
ROLE_OUTPUT = "model-output"


def _read_doc() -> dict:
    line = sys.stdin.readline()
    if not line.strip():
        raise RuntimeError("no key document on stdin")
    return json.loads(line)


def _rank_train(rank: int, world: int, backend: str, rdzv: str, params: dict, vol_root: str, key_bytes: bytes,
                shards: list, conn=None):
    """One rank's training loop: its shards (round-robin by index), one shard per step, the
    whole step captured as CUDA graphs, the next shard's H2D copy and decrypt overlapping the
    current step.  Every shard's tag verdict is gated on the device (a failed shard never
    moves the weights, trainer.py) and summed over ranks with the gradients, so every rank
    raises AuthenticationFailure at the same step -> exit 4 everywhere.  Rank 0 returns (or
    sends through ``conn``) the serialized model."""
    import torch

    from .loader import CIFAR, MEDICAL, ShardSet
    from .trainer import EncryptedTrainer, serialize_cnn_model
    from .volume import Volume

    ndev = max(1, torch.cuda.device_count())
    torch.cuda.set_device(rank % ndev)
    group = None
    if world > 1:
        import torch.distributed as dist

        opts = {"device_id": torch.device("cuda", rank % ndev)} if backend == "nccl" else {}
        dist.init_process_group(backend, init_method=rdzv, rank=rank, world_size=world, **opts)
        group = dist.group.WORLD
    try:
        model = params["model"]
        spec = MEDICAL if model == "densenet121" else CIFAR
        mine = shards[rank::world]
        ss = ShardSet(Volume.open(vol_root), mine, spec)
        batch = int(params.get("batch_size", ss.nrec[0]))
        if any(n != batch for n in ss.nrec):
            raise ValueError("every shard must hold batch_size records")
        tr = EncryptedTrainer(model, key_bytes, batch=batch, spec=spec, seed=int(params.get("seed", 0)), world=world,
                              rank=rank, lr=float(params.get("learning_rate", 1e-3)))
        if group is not None and tr.allreduce is not None:
            tr.allreduce.group = group
        tr.capture()
        n = len(mine)
        for _ in range(max(0, int(params.get("epochs", 1)))):
            for i in range(n):
                if i + 1 < n:
                    tr.step_host(ss.blobs[i], ss.nonces[i], ss.aads[i], batch, next_blob=ss.blobs[i + 1],
                                 next_aad=ss.aads[i + 1], next_nonce=ss.nonces[i + 1])
                else:
                    tr.step_host(ss.blobs[i], ss.nonces[i], ss.aads[i], batch)
            tr.check_status()               # once per epoch: any failed shard on any rank
        tr.check_status(include_pending=True)
        torch.cuda.synchronize()
        out = serialize_cnn_model(tr.net) if rank == 0 else None
        if conn is not None and rank == 0:
            conn.send_bytes(out)
        return out
    finally:
        if group is not None:
            import torch.distributed as dist

            dist.destroy_process_group()


def _rank_entry(rank, world, backend, rdzv, params, vol_root, key_bytes, shards, conn):
    try:
        _rank_train(rank, world, backend, rdzv, params, vol_root, key_bytes, shards, conn)
    except BaseException as e:  # noqa: BLE001 -- reported to the parent through the exit code
        print(f"rank {rank}: training failed: {e}", file=sys.stderr)
        sys.stderr.flush()
        os._exit(4)


def _train_cnn(params: dict, data_vol, key) -> bytes:
    """CNN training over the sealed record shards, on ``world_size`` ranks (default: every
    visible GPU, at most one rank per shard).  Ranks > 1 are spawned processes -- one per GPU,
    or several sharing GPUs with backend "gloo" -- that receive the data key through the
    spawn pipe (never the environment or a file, tee.py:199-201) and rendezvous through a file
    in the enclave's private working directory.  The parent waits for all of them; any rank
    that fails makes the others stop and the run fail (exit 4)."""
    import multiprocessing as mp
    import tempfile

    import torch

    shards = [p for p in data_vol.paths() if p.startswith("shard-")]
    if not shards:
        raise ValueError("no shard-*.bin in the training volume")
    world = int(params.get("world_size", torch.cuda.device_count() or 1))
    world = max(1, min(world, len(shards)))
    if len(shards) % world:
        raise ValueError(f"{len(shards)} shards do not split evenly over {world} ranks")
    key_bytes = key.reveal_bytes()
    if world == 1:
        return _rank_train(0, 1, "", "", params, str(data_vol.root), key_bytes, shards)
    backend = params.get("backend") or ("nccl" if torch.cuda.device_count() >= world else "gloo")
    rdzv_dir = tempfile.mkdtemp(prefix=".rdzv-", dir=os.getcwd())
    rdzv = "file://" + os.path.join(rdzv_dir, "store")
    ctx = mp.get_context("spawn")
    recv, send = ctx.Pipe(duplex=False)
    procs = [ctx.Process(target=_rank_entry, args=(r, world, backend, rdzv, params, str(data_vol.root), key_bytes,
                                                   shards, send if r == 0 else None)) for r in range(world)]
    for p in procs:
        p.start()
    send.close()
    model = None
    try:
        while True:
            if model is None and recv.poll(0.05):
                try:
                    model = recv.recv_bytes()
                except EOFError:
                    pass
            codes = [p.exitcode for p in procs]
            if any(c not in (None, 0) for c in codes):
                raise RuntimeError(f"rank exit codes {codes}")
            if all(c == 0 for c in codes):
                break
    finally:
        for p in procs:
            if p.exitcode is None:
                p.terminate()
            p.join(timeout=30)
        import shutil

        shutil.rmtree(rdzv_dir, ignore_errors=True)
    if model is None:
        raise RuntimeError("rank 0 returned no model")
    return model


def main() -> int:
    doc = _read_doc()
    roles = doc.get("roles", {})
    refs = {}
    for role in (ROLE_TRAINING, ROLE_CODE, ROLE_OUTPUT):
        ref = roles.get(role)
        if ref is None or ref not in doc.get("keys", {}):
            print(f"missing key for role {role}; aborting before any read", file=sys.stderr)
            return 3
        refs[role] = ref
    from .crypto import SymmetricKey
    from .volume import Volume

    keys = {ref: SymmetricKey.from_hex(doc["keys"][ref]) for ref in refs.values()}
    paths = doc["volumes"]
    try:
        code_volume = Volume.open(paths[refs[ROLE_CODE]])
        params = json.loads(code_volume.get(keys[refs[ROLE_CODE]], "params.json"))
        data_volume = Volume.open(paths[refs[ROLE_TRAINING]])
        if "model" in params:
            model = _train_cnn(params, data_volume, keys[refs[ROLE_TRAINING]])
        else:
            from .workload import run_training

            csv_text = data_volume.get(keys[refs[ROLE_TRAINING]], "dataset.csv").decode("utf-8")
            model = run_training(params, csv_text)
    except Exception as e:  # noqa: BLE001 -- the contract maps every failure to exit 4
        print(f"training failed: {e}", file=sys.stderr)
        return 4
    out_ref = refs[ROLE_OUTPUT]
    out_name = out_ref.rpartition("/")[2]
    out_volume = Volume.create(paths[out_ref], out_name, keys[out_ref])
    out_volume.put(keys[out_ref], "model.bin", model)
    print("model sealed")
    return 0


_TRAIN_PY = '''"""B200 training workload artifact (same stdin / roles / exit-code contract as the
reference trainer_workload/train.py); generated by paper_2103_16898_b200.artifact."""
import sys

sys.path.insert(0, {repo!r})
from paper_2103_16898_b200.workload_main import main

if __name__ == "__main__":
    sys.exit(main())
'''


def make_artifact(dest) -> "Path":
    """Write the workload artifact directory (measured by the TEE as a whole)."""
    from pathlib import Path

    dest = Path(dest)
    dest.mkdir(parents=True, exist_ok=True)
    repo = str(Path(__file__).resolve().parent.parent)
    (dest / "train.py").write_text(_TRAIN_PY.format(repo=repo))
    return dest
