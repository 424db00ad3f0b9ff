#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
{
for d in 4 132 388 260; do for w in conv128 conv256; do echo "== DBG=$d $w"; CVB_GEMM_DBG=$d timeout 120 python scripts/trace_gemm.py $w | grep -E "median|stages"; done; done
for d in 0 128 384; do echo "== DBG=$d knobs"; CVB_GEMM_DBG=$d timeout 300 python scripts/conv_knobs.py; done
echo "== mma_rate"; timeout 120 python scripts/mma_rate.py | grep -E "N=128 1 issuer\(s\) A=swizzle|N=256 1 issuer\(s\) A=swizzle|N=64 1 issuer\(s\) A=swizzle"
echo "== BN"; timeout 300 python scripts/bn_probe.py
} > gpurun_out/trace2.log 2>&1
cat gpurun_out/trace2.log
