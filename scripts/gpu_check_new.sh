#!/bin/bash
# development GPU pass: build, the new/changed GPU tests, the CNN parity probe, the bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -q ${TESTS:-tests/test_csv_gpu.py tests/test_reference_suites_gpu.py tests/test_gate_gpu.py tests/test_sha256_gpu.py tests/test_dp_gpu.py tests/test_logistic_dp_gpu.py tests/test_pipeline_gpu.py tests/test_artifact_gpu.py} > gpurun_out/t_new.log 2>&1
echo "tests rc=$?" >> gpurun_out/t_new.log
tail -n 15 gpurun_out/t_new.log
if [ -n "$PROBE" ]; then
  timeout 1200 python scripts/parity_probe.py $PROBE > gpurun_out/parity_probe.log 2>&1
  tail -n 30 gpurun_out/parity_probe.log
fi
if [ -n "$BENCH" ]; then
  for m in $BENCH; do
    timeout 600 python bench.py --model $m --steps 30 --warmup 5 > gpurun_out/bench_$m.log 2>&1
    tail -n 2 gpurun_out/bench_$m.log
  done
fi
