#!/bin/bash
# Round-end measurements on one B200: bench lines of every workload (resnet18 default, small CNN,
# DenseNet, reference trainer, reference arm), and the configs[4] decrypt sweep.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final/build.log 2>&1 || { tail -20 gpurun_out/final/build.log; exit 1; }
for m in resnet18 small_cnn densenet121 logistic; do
  timeout 900 python bench.py --model $m > gpurun_out/final/bench_$m.log 2>&1
  tail -n 1 gpurun_out/final/bench_$m.log | cut -c1-300
done
timeout 900 python bench.py --impl reference > gpurun_out/final/bench_reference.log 2>&1
tail -n 1 gpurun_out/final/bench_reference.log | cut -c1-300
timeout 1500 python scripts/decrypt_sweep.py > gpurun_out/final/decrypt_sweep.log 2>&1
tail -n 3 gpurun_out/final/decrypt_sweep.log | cut -c1-600
