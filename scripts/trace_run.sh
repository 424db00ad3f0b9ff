#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
{
for d in 4 6 5; do for w in conv128 conv256 conv64; do echo "== DBG=$d $w"; CVB_GEMM_DBG=$d timeout 120 python scripts/trace_gemm.py $w; done; done
} > gpurun_out/trace.log 2>&1
cat gpurun_out/trace.log | grep -v "^[0-9]* prod" | head -150
