#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over small workloads of every kernel family;
# logs in gpurun_out/sanitize/ (summaries copied to profiles/ by hand)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for w in "crypto" "cnn small_cnn 32" "cnn resnet18 16"; do
    tag=$(echo $w | tr ' ' '_')
    timeout 1200 $CS --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize_step.py $w \
      > gpurun_out/sanitize/${tool}_${tag}.log 2>&1
    echo "$tool $tag rc=$?" | tee -a gpurun_out/sanitize/summary.txt
  done
done
