#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
{
timeout 300 python scripts/wgrad_debug.py 2>&1 | grep -E "kh1|used"
timeout 600 python -m pytest -q -x tests/test_umma_gpu.py -k wgrad 2>&1 | tail -2
echo "== pair 2box"; timeout 300 python scripts/wgrad_time.py
} > gpurun_out/trace11.log 2>&1
cat gpurun_out/trace11.log
