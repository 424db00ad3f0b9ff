#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
{
timeout 600 python -m pytest -q -x tests/test_umma_gpu.py tests/test_blocks_gpu.py tests/test_cnn_gpu.py -k "wgrad or block or mask_matched or configs1" 2>&1 | tail -3
echo "== pair"; timeout 300 python scripts/wgrad_time.py
echo "== nopair"; CVB_NO_WGRAD_PAIR=1 timeout 300 python scripts/wgrad_time.py
} > gpurun_out/trace10.log 2>&1
cat gpurun_out/trace10.log
