#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
{
for d in 4 1028 6 1030; do for w in conv128 gemm conv64; do echo "== DBG=$d $w"; CVB_GEMM_DBG=$d timeout 120 python scripts/trace_gemm.py $w | grep -E "median|stages" | head -3; done; done
for d in 0 1024; do echo "== DBG=$d knobs"; CVB_GEMM_DBG=$d timeout 300 python scripts/conv_knobs.py; done
} > gpurun_out/trace6.log 2>&1
cat gpurun_out/trace6.log
