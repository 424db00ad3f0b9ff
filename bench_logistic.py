"""Bench line for the reference's own trainer: covault.workload.run_training
(/root/reference/pkg/src/covault/workload.py:48-71) on the CSV rendering of CIFAR-shaped records.

Workload: N rows x 3,072 features, each feature the "%.4f" rendering of pixel/255 and the
label the class mod 2 (SURVEY 8(d) synthetic inputs), one "step" = one epoch of the reference
schedule (one full-batch gradient step over every row).  Our arm:
  value  epochs on the device-resident parsed dataset, bit-exact mode (the reference's order:
         reproduces its model bytes), CUDA events
  e2e    through the public API per step: pinned host CSV bytes -> H2D -> device CSV parse
         (bit-exact float()) -> one exact epoch -> D2H of the F+1 model values
  roofline  the exact epoch's kernels against HBM: algorithmic bytes = X read by the logit pass
         (feature-major copy) and by the gradient pass = 16 B per element
  cpu_baseline  the reference's run_training itself (baseline/_ref, pure Python, single-threaded,
         pinned to one core) on a bounded sample of the same CSV, parse + 1 epoch
``--impl reference`` prints the reference arm's line (same sample, same metric).
"""
from __future__ import annotations

import json
import os
import time

import numpy as np
import torch

F = 3072


def render_csv(n, seed=0) -> bytes:
    """CIFAR-shaped records as CSV text: 3,072 '%.4f' pixel/255 values + label (class mod 2)."""
    rng = np.random.default_rng(seed)
    templ = np.random.default_rng(0).normal(size=(10, F))
    labels = rng.integers(0, 10, size=n)
    px = np.clip(np.round(128 + 40 * templ[labels] + 30 * rng.normal(size=(n, F))), 0, 255).astype(np.int64)
    table = np.frombuffer(b"".join(f"{v / 255:.4f}".encode() for v in range(256)), dtype=np.uint8).reshape(256, 6)
    body = np.empty((n, F, 7), dtype=np.uint8)
    body[:, :, :6] = table[px]
    body[:, :, 6] = ord(",")
    tail = np.frombuffer(b"".join(f"{int(l) % 2}\n".encode() for l in labels), dtype=np.uint8).reshape(n, 2)
    return np.concatenate([body.reshape(n, -1), tail], axis=1).tobytes()


def reference_cpu(csv: bytes, epochs=1):
    """covault.workload.run_training on one pinned core: (seconds, rows, cores=1)."""
    from covault.workload import run_training

    prev = os.sched_getaffinity(0)
    os.sched_setaffinity(0, {min(prev)})
    try:
        text = csv.decode()
        t0 = time.perf_counter()
        run_training({"learning_rate": 0.1, "epochs": epochs}, text)
        dt = time.perf_counter() - t0
    finally:
        os.sched_setaffinity(0, prev)
    return dt, text.count("\n")


def run(args, metric, unit, peaks, clock_sampler):
    from paper_2103_16898_b200 import workload

    n = args.rows
    csv = render_csv(n)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    text = csv.decode()
    # parity gate before timing: device parse == the reference's float() bit for bit on a slice,
    # and one exact epoch reproduces the host oracle on it
    head = "".join(text.splitlines(keepends=True)[:64])
    Xd, yd = workload.parse_dataset_device(head)
    rows = workload.parse_dataset(head)
    assert np.array_equal(Xd.cpu().numpy().view(np.uint64),
                          np.array([f for f, _ in rows], dtype=np.float64).view(np.uint64)), "CSV parse mismatch"
    X, y = workload.parse_dataset_device(text)
    tr = workload.LogisticTrainer(X, y, exact=True)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    for _ in range(args.warmup):
        tr.epoch(0.1)
    torch.cuda.synchronize()
    clk = clock_sampler(0)
    e0, e1 = ev(), ev()
    e0.record()
    for _ in range(args.steps):
        tr.epoch(0.1)
    e1.record()
    torch.cuda.synchronize()
    clocks = clk.summary()
    ms = e0.elapsed_time(e1) / args.steps
    # e2e through the public API: host CSV -> device parse -> exact epoch -> model to host
    host = torch.frombuffer(bytearray(csv), dtype=torch.uint8).pin_memory()

    def e2e_step():
        Xs, ys = workload.parse_dataset_device(text)          # H2D of the text inside
        w, b = workload.LogisticTrainer(Xs, ys, exact=True).train(0.1, 1)
        return w, b

    for _ in range(max(1, args.warmup // 2)):
        e2e_step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    k_e2e = max(3, args.steps // 4)
    for _ in range(k_e2e):
        e2e_step()
    torch.cuda.synchronize()
    ms_e2e = (time.perf_counter() - t0) * 1e3 / k_e2e
    del host
    # parse alone (GB/s of CSV text), for the record
    t0 = time.perf_counter()
    for _ in range(3):
        workload.parse_dataset_device(text)
    torch.cuda.synchronize()
    parse_ms = (time.perf_counter() - t0) * 1e3 / 3
    hbm, _, src = peaks()
    algo = 16.0 * n * F   # X read by the logit pass (Xt) and the gradient pass (X), 8 B each
    roof = {"bound": "hbm", "achieved": algo / (ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": algo / (ms * 1e-3) / 1e9 / hbm, "traffic": None, "kernel": "lr_logits_exact + lr_grad_exact",
            "algorithmic_per_step": algo, "peak_source": src,
            "note": "exact mode: per-feature dependent add chains over rows in file order (the reference's "
                    "rounding order) bound it, not HBM"}
    cpu = None
    if not args.no_cpu_baseline:
        sample = max(200, int(args.cpu_seconds * 700))
        sub = b"".join(csv.splitlines(keepends=True)[:sample])
        dt, rr = reference_cpu(sub)
        cpu = {"value": rr / dt, "unit": unit, "cores": 1, "kind": "reference",
               "sample": f"covault.workload.run_training (baseline/_ref, pure Python) on {rr} CSV rows x {F} "
                         f"features: parse + 1 epoch, pinned to 1 core"}
    line = {"metric": metric, "value": n / (ms * 1e-3), "unit": unit, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"reference trainer (workload.py:48-71), CSV rendering of {n} CIFAR-shaped "
                                   f"records x {F} features, 1 step = 1 epoch, bit-exact mode",
                       "model": "logistic", "global_batch": n, "seq_len": None, "parallelism": "dp1",
                       "l2": f"X = {n * F * 8 / 1e9:.2f} GB (> 126 MB L2)"},
            "e2e": {"value": n / (ms_e2e * 1e-3), "unit": unit, "h2d_bytes_per_step": len(csv),
                    "d2h_bytes_per_step": 8 * (F + 1)},
            "csv_parse_gbs": len(csv) / (parse_ms * 1e-3) / 1e9,
            "gpu_launches": None, "roofline": roof, "cpu_baseline": cpu, "clocks": clocks}
    print(json.dumps(line), flush=True)


def run_reference(args, metric, unit):
    sample = max(200, int(args.cpu_seconds * 700))
    csv = render_csv(sample)
    times = []
    for i in range(args.warmup + args.steps):
        dt, rr = reference_cpu(csv)
        if i >= args.warmup:
            times.append(dt)
    v = rr * len(times) / sum(times)
    line = {"impl": "reference", "metric": metric, "value": v, "unit": unit, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"reference trainer, CSV rendering of {rr} CIFAR-shaped records x {F} features, "
                                   f"1 step = parse + 1 epoch", "model": "logistic", "global_batch": rr,
                       "seq_len": None, "parallelism": "cpu"},
            "cpu_baseline": {"value": v, "unit": unit, "cores": 1, "kind": "reference",
                             "sample": f"covault.workload.run_training on {rr} rows, 1 pinned core"},
            "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
