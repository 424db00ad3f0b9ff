#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
{
timeout 300 python scripts/bn_trace.py
timeout 300 python scripts/bn_probe.py
timeout 600 python -m pytest -q -x tests/test_nn_kernels_gpu.py tests/test_blocks_gpu.py tests/test_head_gpu.py tests/test_dp_gpu.py 2>&1 | tail -3
} > gpurun_out/trace9.log 2>&1
cat gpurun_out/trace9.log
