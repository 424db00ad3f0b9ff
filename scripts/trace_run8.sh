#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
{
timeout 300 python scripts/bn_trace.py
for w in conv128 conv256; do echo "== DBG=6 $w"; CVB_GEMM_DBG=6 timeout 120 python scripts/trace_gemm.py $w | grep -E "median|stages|total" | head -3; done
echo "== DBG=2 knobs"; CVB_GEMM_DBG=2 timeout 300 python scripts/conv_knobs.py
} > gpurun_out/trace8.log 2>&1
cat gpurun_out/trace8.log
