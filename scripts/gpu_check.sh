#!/bin/bash
# One GPU-box pass: gpu tests, smoke, bench (both arms).  Outputs under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
for m in ${EXTRA_MODELS}; do timeout 900 python bench.py --model $m --no-cpu-baseline --steps 20 > gpurun_out/bench_$m.log 2>&1; done
tail -3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench*.log
