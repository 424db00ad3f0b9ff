#!/bin/bash
# full GPU pass: build, every -m gpu test, smoke, and the bench lines of every workload
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -q -m gpu ${PYTEST_ARGS} > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -n 8 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > gpurun_out/smoke.log 2>&1
tail -n 2 gpurun_out/smoke.log
for m in ${BENCH:-resnet18 small_cnn}; do
  timeout 900 python bench.py --model $m ${BENCH_ARGS} > gpurun_out/bench_$m.log 2>&1
  tail -n 1 gpurun_out/bench_$m.log | cut -c1-600
done
