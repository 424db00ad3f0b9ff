#!/bin/bash
# What bounds the ResNet-18 convs and the BN layers: engine debug knobs (1 = skip MMA, 2 = skip
# TMA, 8 = skip epilogue), pipeline depth, and the BN kernels' per-launch fixed cost.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
{
for d in 0 1 2 8; do echo "== CVB_GEMM_DBG=$d"; CVB_GEMM_DBG=$d timeout 300 python scripts/conv_knobs.py; done
for s in 2 3 4; do echo "== CVB_STAGES=$s"; CVB_STAGES=$s timeout 300 python scripts/conv_knobs.py; done
echo "== BN"; timeout 300 python scripts/bn_probe.py
echo "== BN min elems 1M"; CVB_BN_MIN_ELEMS=1000000 timeout 300 python scripts/bn_probe.py
} > gpurun_out/gemm_bound.log 2>&1
cat gpurun_out/gemm_bound.log
