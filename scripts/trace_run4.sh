#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
{
for w in conv128 conv256; do echo "== DBG=4 $w"; CVB_GEMM_DBG=4 timeout 120 python scripts/trace_gemm.py $w | grep -E "median|stages"; done
echo "== knobs"; timeout 300 python scripts/conv_knobs.py
} > gpurun_out/trace4.log 2>&1
cat gpurun_out/trace4.log
