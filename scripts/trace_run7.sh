#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
{
for w in conv128 conv256 gemm; do echo "== DBG=4 $w"; CVB_GEMM_DBG=4 timeout 120 python scripts/trace_gemm.py $w | grep -E "median|stages" | head -3; done
echo "== knobs pair"; timeout 300 python scripts/conv_knobs.py
echo "== knobs nopair"; CVB_NO_KB_PAIR=1 timeout 300 python scripts/conv_knobs.py
timeout 600 python -m pytest -q -x tests/test_umma_gpu.py tests/test_blocks_gpu.py tests/test_head_gpu.py 2>&1 | tail -3
} > gpurun_out/trace7.log 2>&1
cat gpurun_out/trace7.log
