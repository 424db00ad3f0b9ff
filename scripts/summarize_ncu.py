"""Summaries of ncu outputs for profiles/ (run locally on the files gpurun brought back).

usage: summarize_ncu.py launches <csv> | report <ncu-rep>
"""
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (int(d["ID"]), d["Kernel Name"])
        data.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", "") or 0)
    agg, tot = {}, 0.0
    for (i, name), m in data.items():
        k = name.split("(")[0].replace("<unnamed>::", "").replace("void ", "")
        t = m.get("gpu__time_duration.sum", 0) / 1000
        a = agg.setdefault(k, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += t
        a[2] += (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e6
        tot += t
    out = [f"launches: {len(data)}, total {tot:.1f} us (ncu: cold cache, serialised -> compare shares)", "",
           "| kernel | launches | us | share | DRAM MB |", "|---|---:|---:|---:|---:|"]
    for k, (c, t, mb) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| {k} | {c} | {t:.1f} | {t / tot * 100:.1f}% | {mb:.1f} |")
    return "\n".join(out)


KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__cycles_active.avg",
]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = r[0], r[1], r[2] if len(r) > 2 else r[1]
    d = dict(zip(hdr, vals))
    un = dict(zip(hdr, units))
    out = [f"kernel: {d.get('Kernel Name', '?')[:90]}", "", "| metric | value | unit |", "|---|---|---|"]
    for k in KEYS:
        for hk, v in d.items():
            if hk == k or hk.endswith("." + k):
                out.append(f"| {k} | {v} | {un.get(hk, '')} |")
                break
    return "\n".join(out)


if __name__ == "__main__":
    print(launches(sys.argv[2]) if sys.argv[1] == "launches" else report(sys.argv[2]))
