#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
{
for d in 4 516 6 518; do for w in conv128 conv256 gemm; do echo "== DBG=$d $w"; CVB_GEMM_DBG=$d timeout 120 python scripts/trace_gemm.py $w | grep -E "median|stages" | head -3; done; done
} > gpurun_out/trace5.log 2>&1
cat gpurun_out/trace5.log
