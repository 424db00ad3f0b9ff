#!/bin/bash
# build, bench one model (BENCH_MODEL, default resnet18) and take the ncu launch list of one eager step
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
M=${BENCH_MODEL:-resnet18}
timeout 600 python bench.py --model $M --steps ${STEPS:-100} > gpurun_out/bench_$M.log 2>&1
tail -n 1 gpurun_out/bench_$M.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], d['e2e']['value'], r['frac'], r['per_class_ms_in_graph'])"
if [ -z "$NOLIST" ]; then
NOFULL=1 LISTS="$M ${BATCH:-512}" bash scripts/profile_r02.sh > /dev/null 2>&1
python scripts/summarize_ncu.py launches gpurun_out/prof2/launches_$M.csv 2>&1 | head -30
fi
