#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over small workloads of every kernel family;
# logs in gpurun_out/sanitize/ (summaries copied to profiles/)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool tag args...
  local tool=$1 tag=$2; shift 2
  timeout ${SAN_TIMEOUT:-900} $CS --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize_step.py "$@" \
    > gpurun_out/sanitize/${tool}_${tag}.log 2>&1
  echo "$tool $tag rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Error' gpurun_out/sanitize/${tool}_${tag}.log | tail -1)" \
    | tee -a gpurun_out/sanitize/summary.txt
}
rm -f gpurun_out/sanitize/summary.txt
run memcheck crypto crypto
run memcheck small_cnn cnn small_cnn 32
run memcheck resnet18 cnn resnet18 16
run racecheck crypto crypto
run racecheck small_cnn cnn small_cnn 32
run synccheck crypto crypto
run synccheck small_cnn cnn small_cnn 32
