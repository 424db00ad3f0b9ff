#!/bin/bash
# A/B of env settings on the same box: AB_ENVS="A=1 B=2;A=0" (";"-separated), model BENCH_MODEL
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
M=${BENCH_MODEL:-resnet18}
IFS=';' read -ra SETS <<< "$AB_ENVS"
for rep in 1 2; do
  for e in "${SETS[@]}"; do
    env $e timeout 600 python bench.py --model $M --steps ${STEPS:-100} 2>/dev/null | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$e', round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['value']), round(r['frac'],4), {k: round(v,3) for k,v in r['per_class_ms_in_graph'].items()})"
  done
done
