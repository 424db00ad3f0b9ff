"""Benchmark of the encrypted-training hot path (BASELINE.json metric: training images/s).

Workload (N=1): BASELINE.json configs[1] -- the paper-shaped small CNN on synthetic
CIFAR-10-shaped records, batch 512 per GPU, bf16 operands / fp32 accumulation.  One step =
AES-256-GCM open of one sealed 512-record shard (tag verified on device) + record decode +
forward + softmax-CE + backward + Adam.  Per-rank inputs: 96 sealed shards (151 MB of
ciphertext, larger than the 126 MB L2) resident in HBM, cycled.  Weak scaling under
torchrun: every rank has its own shards and batch, gradients all-reduced over NCCL.

Prints ONE JSON line on rank 0 (see the driver contract in the task statement):
  value     images/s over all ranks, device-resident ciphertext, CUDA-event timed
  e2e       same metric through the public host API: pinned host ciphertext -> H2D ->
            decrypt -> train -> D2H of loss + tag status inside the timed region
  roofline  dominant kernel of an instrumented replay of the step (CUDA events per launch)
  cpu_baseline  reference CPU arm on the host cores (rank 0, N=1 only; bounded sample)
``--impl reference`` runs only the CPU reference arm (oracle port of the CNN + the
reference's own AES-GCM open) and prints its line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
_REF = ROOT / "baseline" / "_ref"
if _REF.exists():
    sys.path.insert(1, str(_REF))

import numpy as np  # noqa: E402
import torch  # noqa: E402

METRIC = "training images/sec at 1/2/4/8 B200 vs reference CPU trainer on host cores"
UNIT = "images/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="resnet18", choices=["resnet18", "small_cnn", "densenet121", "logistic"])
    ap.add_argument("--rows", type=int, default=20000, help="logistic: CSV rows (x 3,072 features)")
    ap.add_argument("--batch", type=int, default=None, help="per-GPU batch (default: 512, DenseNet 128)")
    ap.add_argument("--shards", type=int, default=None, help="resident shards per rank (default: > 150 MB)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    a = ap.parse_args()
    if a.batch is None:
        a.batch = 128 if a.model == "densenet121" else 512
    return a


# BASELINE.json configs each model is the bench line of
WORKLOADS = {
    "small_cnn": ("configs[1]", "paper-shaped small CNN (4 conv+BN, 2 FC, Adam)", "CIFAR-10-shaped 32x32x3, 10 classes"),
    "resnet18": ("configs[2]", "ResNet-18 (CIFAR variant)", "CIFAR-10-shaped 32x32x3, 10 classes"),
    "densenet121": ("configs[3]", "DenseNet-121-style CNN (1-channel stem)", "medical-imaging-shaped 224x224x1, binary"),
}


def spec_for(model):
    from paper_2103_16898_b200.loader import CIFAR, MEDICAL

    return MEDICAL if model == "densenet121" else CIFAR


def rec_bytes(spec):
    return 1 + spec["c"] * spec["h"] * spec["w"]


# ---------------------------------------------------------------------------------------
# synthetic sealed dataset (reference volume format: one AES-256-GCM message per shard file,
# AAD = volume_name || 0 || path, volume.py:53-54)
# ---------------------------------------------------------------------------------------
def make_shards(n_shards, batch, seed, key, spec):
    from cryptography.hazmat.primitives.ciphers.aead import AESGCM

    c, h, w = spec["c"], spec["h"], spec["w"]
    rng = np.random.default_rng(seed)
    classes = 2 if c == 1 else 10     # medical: binary diagnosis; CIFAR: 10 classes
    templ = np.random.default_rng(0).normal(size=(classes, c * h * w)).astype(np.float32)
    aes = AESGCM(key)
    shards = []
    for i in range(n_shards):
        labels = rng.integers(0, classes, size=batch).astype(np.uint8)
        noise = rng.integers(-52, 53, size=(batch, c * h * w), dtype=np.int16)
        px = np.clip(128 + 40 * templ[labels] + noise, 0, 255).astype(np.uint8)
        pt = np.concatenate([labels[:, None], px], axis=1).tobytes()
        path = f"shard-{seed:03d}-{i:05d}.bin"
        aad = b"training-data\x00" + path.encode()
        nonce = rng.bytes(12)
        shards.append((path, nonce, aad, aes.encrypt(nonce, pt, aad), pt if i == 0 else None))
    return shards


class ClockSampler:
    """NVML clock + throttle-reason sampling every ~5 ms while the timed region runs, in a
    separate process (a thread would compete for the GIL with the launch loop and starve)."""

    CODE = r"""
import sys, time, pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
print("max", pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM), flush=True)
while True:
    try:
        print(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
              pynvml.nvmlDeviceGetCurrentClocksEventReasons(h), flush=True)
    except Exception:
        pass
    time.sleep(0.005)
"""
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, dev_index):
        self.proc = None
        try:
            self.proc = subprocess.Popen([sys.executable, "-c", self.CODE, str(dev_index)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.proc.stdout.readline()   # started (max clock line)
        except Exception:
            self.proc = None

    def summary(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            return None
        sm, reasons, mx = [], set(), 0.0
        for line in out.strip().splitlines():
            f = line.split()
            if len(f) != 2 or f[0] == "max":
                continue
            sm.append(float(f[0]))
            for nm, bit in self.REASONS.items():
                if int(f[1]) & bit:
                    reasons.add(nm)
        try:
            import pynvml

            pynvml.nvmlInit()
            mx = float(pynvml.nvmlDeviceGetMaxClockInfo(pynvml.nvmlDeviceGetHandleByIndex(0), pynvml.NVML_CLOCK_SM))
        except Exception:
            pass
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml (separate process, 5 ms period) during the timed region"}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), "measured"
    return 6650.0, 1590.0, "fallback"


# ---------------------------------------------------------------------------------------
# CPU reference arm
# ---------------------------------------------------------------------------------------
def cpu_reference(model, batch, key, spec, seconds, steps=None, warmup=0):
    """Reference CPU trainer on the host cores: the reference's own AES-GCM open
    (covault.crypto.aead_open -> OpenSSL) of the shard, then the CPU restatement of the CNN
    step (oracle/cnn_ref.py, fp32, all threads).  Returns (img/s, cores, sample, kind)."""
    from oracle.cnn_ref import RefTrainer, normalise_records
    from paper_2103_16898_b200 import nets

    cores = len(os.sched_getaffinity(0))
    torch.set_num_threads(cores)
    try:
        from covault.crypto import SymmetricKey, aead_open  # the reference package (baseline/_ref)

        rkey = SymmetricKey(key)
        opener = lambda n, a, b: aead_open(rkey, n, a, b)  # noqa: E731
        dec = "covault.crypto.aead_open (reference, OpenSSL)"
    except Exception:
        from cryptography.hazmat.primitives.ciphers.aead import AESGCM

        opener = lambda n, a, b: AESGCM(key).decrypt(n, b, a)  # noqa: E731
        dec = "cryptography AESGCM (reference's dependency)"
    m = nets.make_model(model, seed=0)
    ref = RefTrainer(model, {n: t.clone() for n, _, t in m.ps.specs}, emulate_bf16=False)
    shards = make_shards(2, batch, 7, key, spec)
    t_total, n_img, it = 0.0, 0, 0
    deadline = time.perf_counter() + seconds
    while True:
        path, nonce, aad, blob, _ = shards[it % 2]
        t0 = time.perf_counter()
        pt = opener(nonce, aad, blob)
        rec = torch.frombuffer(bytearray(pt), dtype=torch.uint8).view(batch, -1)
        x, lab = normalise_records(rec, spec["c"], spec["h"], spec["w"], spec["mean"], spec["std"], False)
        ref.step(x, lab)
        dt = time.perf_counter() - t0
        if it >= warmup:
            t_total += dt
            n_img += batch
        it += 1
        if steps is not None:
            if it >= steps + warmup:
                break
        elif time.perf_counter() > deadline and it > warmup:
            break
    sample = (f"{it - warmup} timed steps of batch {batch} ({n_img} images): {dec} of one sealed shard + "
              f"{model} fp32 train step (oracle/cnn_ref.py, torch CPU, {cores} threads)")
    return n_img / t_total, cores, sample, t_total


def run_reference(args, rank, world):
    if rank != 0:
        return
    key = bytes(range(32))
    cfg, mname, dname = WORKLOADS[args.model]
    v, cores, sample, t = cpu_reference(args.model, args.batch, key, spec_for(args.model), 0, steps=args.steps,
                                        warmup=args.warmup)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / max(1, args.steps),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
            "config": {"workload": f"{cfg}: {mname}, {dname} sealed shards, batch {args.batch} (CPU reference)",
                       "model": args.model, "global_batch": args.batch, "seq_len": None, "parallelism": "cpu"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import torch.distributed as dist

    from paper_2103_16898_b200 import kernels as K
    from paper_2103_16898_b200.trainer import EncryptedTrainer

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    spec = spec_for(args.model)
    key = bytes(range(32))
    B = args.batch
    rb = rec_bytes(spec)
    if args.shards is None:   # enough resident ciphertext to exceed the 126 MB L2
        args.shards = max(4, -(-160_000_000 // (B * rb + 16)))
    cfg, mname, dname = WORKLOADS[args.model]
    tr = EncryptedTrainer(args.model, key, batch=B, spec=spec, seed=0, world=world, rank=rank,
                          force_allreduce=bool(os.environ.get("CVB_FORCE_DIST")))
    shards = make_shards(args.shards, B, 1000 + rank, key, spec)
    # resident ciphertext + AADs in HBM (inputs larger than L2)
    cts = [torch.frombuffer(bytearray(s[3]), dtype=torch.uint8).to(dev) for s in shards]
    aads = [torch.frombuffer(bytearray(s[2]), dtype=torch.uint8).to(dev) for s in shards]
    host = [torch.frombuffer(bytearray(s[3]), dtype=torch.uint8).pin_memory() for s in shards]
    # parity gate before timing: shard 0 decrypts bit-exactly on the device, and the fused
    # decrypt-and-normalise step sees the same labels
    tr.ctx.open_device(shards[0][1], aads[0], cts[0], tr.loader.pt, tr.loader.work)
    torch.cuda.synchronize()
    assert int(tr.loader.work[4].item()) == 0, "tag check failed"
    assert bytes(tr.loader.pt[:len(shards[0][4])].cpu().numpy()) == shards[0][4], "decrypt mismatch"
    tr.step_resident(cts[0], shards[0][1], aads[0], B)
    torch.cuda.synchronize()
    want_labels = np.frombuffer(shards[0][4], dtype=np.uint8).reshape(B, rb)[:, 0]
    assert np.array_equal(tr.loader.labels[:B].cpu().numpy(), want_labels), "fused loader labels mismatch"
    tr.capture()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(steps):
            fn(i)
        e1.record()
        barrier()
        ms = torch.tensor([e0.elapsed_time(e1)], device=dev)
        if world > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return float(ms.item())

    nsh = len(cts)

    def resident_loop(count):
        """Step i of a run of `count` steps on resident ciphertext; shard i+1's decrypt is issued
        beside step i's optimiser (never past the run, so every timed step decrypts its own
        shard inside the timed region)."""
        def fn(i):
            j, k = i % nsh, (i + 1) % nsh
            nxt = (cts[k], shards[k][1], aads[k]) if i + 1 < count else None
            return tr.step_resident(cts[j], shards[j][1], aads[j], B, next_shard=nxt)
        return fn

    def e2e_loop(count):
        """e2e: each step's shard is copied from pinned host memory inside the timed region;
        shard i+1's H2D copy and decrypt overlap step i (trainer.step_host)."""
        def fn(i):
            j, k = i % nsh, (i + 1) % nsh
            if i + 1 < count:
                return tr.step_host(host[j], shards[j][1], shards[j][2], B, next_blob=host[k],
                                    next_aad=shards[k][2], next_nonce=shards[k][1])
            return tr.step_host(host[j], shards[j][1], shards[j][2], B)
        return fn

    resident = resident_loop(1)   # single unpipelined step (the instrumented pass below)
    warm = resident_loop(args.warmup)
    for i in range(args.warmup):
        warm(i)
    launches0 = K.REC.launches
    clk = ClockSampler(local_rank) if rank == 0 else None
    ms = timed(resident_loop(args.steps), args.steps)
    clocks = clk.summary() if rank == 0 else None
    tr.check_status(include_pending=True)   # sticky run verdict: every timed shard authenticated
    # graph replays do not pass through the Python wrappers: count one eager step's launches
    per_step_eager = None
    warm = e2e_loop(args.warmup)
    for i in range(args.warmup):
        warm(i)
    ms_e2e = timed(e2e_loop(args.steps), args.steps)
    tr.check_status(include_pending=True)

    # ---- roofline ---------------------------------------------------------------------
    # (1) one eager step through the kernel wrappers: launch count and, per kernel class, the
    #     algorithmic FLOPs (2*M*N*K, real channel counts) and bytes of the step's launches.
    K.REC.timing, K.REC.records = True, []
    l0 = K.REC.launches
    tr.graph = None
    resident(0)
    torch.cuda.synchronize()
    per_step_eager = K.REC.launches - l0
    K.REC.timing = False
    summ = K.REC.summary()            # {kind: [calls, ms (eager, not used), flops, bytes]}
    tr.graph = True
    # (2) per class, the in-graph time: a CUDA graph of the step captured with every other
    #     class's launches filtered out (kernels.ONLY_CLASSES) replays exactly that class's
    #     kernels back to back -- their time inside a graph, without launch gaps of an eager
    #     replay and without the rest of the step in between.  The decrypt (outside the step
    #     graphs) is timed the same way on its own stream.
    def graph_ms(body, reps=20):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                body()
        torch.cuda.current_stream().wait_stream(s)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    ar = tr.allreduce
    if ar is not None:
        ar.segment = lambda idx: None     # no collectives inside the measurement graphs
    class_ms = {}
    import warnings
    with warnings.catch_warnings():
        warnings.filterwarnings("ignore", message="The CUDA Graph is empty")
        for kind in summ:
            K.ONLY_CLASSES = {kind}
            try:
                class_ms[kind] = graph_ms(lambda: (tr._train_body(), tr._opt_body()))
            finally:
                K.ONLY_CLASSES = None
        class_ms["decrypt"] = graph_ms(lambda: tr.ctx.open_records_device(shards[1][1], aads[1], cts[1], tr.loader.x,
                                                                           tr.loader.labels, tr._works[0], spec))
    if ar is not None:
        ar.segment = None
    tr.check_status(include_pending=True)
    dec_bytes = len(shards[0][3]) + B * spec["h"] * spec["w"] * spec["c"] * 2 + B * 4   # C||T in, tile + labels out
    summ["decrypt"] = [1, 0.0, 0, dec_bytes]
    step_ms = ms / args.steps
    kind = max(class_ms, key=class_ms.get)
    calls, _, dfl, dby = summ[kind]
    dms = class_ms[kind]
    hbm, tflops, src = peaks()
    if dfl > 0:
        ach = dfl / (dms * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": ach, "peak": tflops, "unit": "TFLOP/s", "frac": ach / tflops}
    else:
        ach = dby / (dms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm}
    traffic = None
    try:   # ncu-measured DRAM bytes of this kernel class in one step (profiles/, scripts/traffic_json.py)
        tj = json.loads((ROOT / "profiles" / "traffic.json").read_text())[args.model]
        kd = tj["kinds"][kind]
        traffic = {"dram_bytes_per_launch": kd["dram_bytes"] / kd["launches"],
                   "dram_bytes_per_step": kd["dram_bytes"], "algorithmic_bytes_per_step": dby,
                   "source": tj["source"]}
    except Exception:
        pass
    roof.update({"traffic": traffic, "kernel": kind, "launches_per_step": calls,
                 "algorithmic_per_step": dfl if dfl > 0 else dby,
                 "class_ms_in_graph": round(dms, 5), "share_of_step": dms / step_ms, "peak_source": src,
                 "per_class_ms_in_graph": {k: round(v, 5) for k, v in sorted(class_ms.items(), key=lambda kv: -kv[1])},
                 "method": "per-class CUDA graph of the step (other classes filtered out), 20 replays, CUDA events",
                 "algorithmic": "sum over the step's launches of 2*M*N*K (real channel counts)"
                 if dfl > 0 else "sum over the step's launches of each input read once + each output written once"})
    if dfl > 0:   # the same class against HBM: its algorithmic bytes over the same time
        roof["hbm_gbs_at_algorithmic_bytes"] = dby / (dms * 1e-3) / 1e9
    prof = ROOT / "profiles" / "roofline_live.json"
    if rank == 0:
        try:
            prof.write_text(json.dumps({"model": args.model, "ms_per_step": step_ms,
                                        "summary": {k: v for k, v in summ.items()}, "class_ms": class_ms,
                                        "roofline": roof}, indent=1))
        except Exception:
            pass

    images = B * args.steps * world
    value = images / (ms * 1e-3)
    e2e = images / (ms_e2e * 1e-3)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, sample, _ = cpu_reference(args.model, B, key, spec, args.cpu_seconds, warmup=1)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample}
    if rank == 0:
        decrypt_launches = 1   # fused gcm_kernel<decode>: open + tag finalisation (last CTA) + NHWC-8 decode
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16 operands, fp32 accumulate", "data": "synthetic",
            "config": {"workload": f"{cfg}: {mname}, {dname} sealed shards, batch {B}/GPU, "
                                   f"decrypt+decode+fwd+bwd+Adam per step",
                       "model": args.model, "global_batch": B * world, "seq_len": None,
                       "parallelism": f"dp{world}",
                       "l2": f"{args.shards} resident shards/rank = "
                             f"{args.shards * (B * rb + 16) / 1e6:.0f} MB ciphertext (> 126 MB L2), cycled"},
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": B * rb + 16 + 64,
                    "d2h_bytes_per_step": 8},
            "gpu_launches": args.steps * (per_step_eager + decrypt_launches) if per_step_eager else None,
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "loss": float(tr.net.loss.item()),
        }
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if os.environ.get("CVB_ONE_GPU"):   # test aid: run every rank on cuda:0 (use with CVB_DIST_BACKEND=gloo)
        local_rank = 0
    if args.model == "logistic":   # the reference's own trainer (bench_logistic.py), one GPU
        import bench_logistic as BL

        if rank != 0:
            return
        if args.impl == "reference":
            BL.run_reference(args, METRIC, UNIT)
        else:
            BL.run(args, METRIC, UNIT, peaks, ClockSampler)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    force = bool(os.environ.get("CVB_FORCE_DIST"))   # exercise the NCCL path even at world 1
    if force and "RANK" not in os.environ:
        import socket

        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                          MASTER_PORT=str(sk.getsockname()[1]))
        sk.close()
    if world > 1 or force:
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        backend = os.environ.get("CVB_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    run_ours(args, rank, world, local_rank)
    if world > 1 or force:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
