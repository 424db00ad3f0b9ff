"""Top stall-sampled SASS lines of an ncu report (source page), with the CUDA source line when
the report was captured with --import-source.  usage: ncu_hot_sass.py REPORT [N]"""
import csv
import io
import subprocess
import sys

rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
tot = sum(float(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
data.sort(key=lambda d: -float(d["Warp Stall Sampling (All Samples)"] or 0))
print(f"total samples {tot:.0f}")
for d in data[:n]:
    s = float(d["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{100 * s / tot:5.1f}%  {d['Address'][-5:]}  {d['Source'].strip()[:90]}")
