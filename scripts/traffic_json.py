"""profiles/traffic.json: ncu-measured DRAM bytes per launch class of one training step
(from the committed launch lists), read by bench.py for roofline.traffic."""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
KIND = {"umma_gemm_kernel": "umma_gemm", "bn_bwd_fused": "bn", "bn_fwd_fused": "bn", "bn_apply": "bn",
        "chan_stats_partial": "bn", "bn_finalize": "bn", "bn_gather_dx": "bn", "head_train_kernel": "head",
        "softmax_xent_mean": "head", "transpose_batched": "layout", "adam_step_dev": "optimizer",
        "reduce_splits": "reduce", "reduce_splits_flat": "reduce", "reduce_splits_flat4": "reduce"}


def summarize(path):
    data = {}
    hdr = None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = (int(d["ID"]), d["Kernel Name"].split("(")[0].replace("<unnamed>::", "").replace("void ", ""))
        data.setdefault(k, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", "") or 0)
    out = {}
    for (_, name), m in data.items():
        kind = KIND.get(name.split("<")[0], name.split("<")[0])
        o = out.setdefault(kind, {"launches": 0, "dram_bytes": 0.0, "ncu_us": 0.0})
        o["launches"] += 1
        o["dram_bytes"] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        o["ncu_us"] += m.get("gpu__time_duration.sum", 0) / 1000
    return out


if __name__ == "__main__":
    tags = sys.argv[1:] or ["r01b"]      # first tag that has a model's launch list wins
    res = {}
    for model in ("small_cnn", "resnet18", "densenet121"):
        cands = [ROOT / "profiles" / f"{t}_launches_{model}.csv" for t in tags]
        p = next((c for c in cands if c.exists()), None)
        if p is not None:
            res[model] = {"source": str(p.relative_to(ROOT)) + " (ncu launch list of one eager step, cold cache)",
                          "kinds": summarize(p)}
    (ROOT / "profiles" / "traffic.json").write_text(json.dumps(res, indent=1))
    print(json.dumps({m: {k: round(v["dram_bytes"] / 1e6, 1) for k, v in r["kinds"].items() if k in ("umma_gemm", "bn")}
                      for m, r in res.items()}))
