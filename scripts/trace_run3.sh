#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python scripts/mma_rate2.py > gpurun_out/mma_rate2.log 2>&1
cat gpurun_out/mma_rate2.log
