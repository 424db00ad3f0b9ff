#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest -q tests/test_cnn_gpu.py tests/test_csv_gpu.py > gpurun_out/t_b.log 2>&1
echo "tests rc=$?" >> gpurun_out/t_b.log
tail -n 12 gpurun_out/t_b.log
bash scripts/profile_r02.sh
