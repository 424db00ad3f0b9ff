#!/bin/bash
# Round profiling on the GPU box: launch list of the bench command + full ncu captures of the
# dominant kernels.  Outputs land in gpurun_out/ (summaries are copied to profiles/ locally).
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
# 1) every launch of a short bench run (cold-cache, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 400 --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --shards 8 > gpurun_out/launches_bench.log 2>&1
# 2) full capture of the top GEMM launches of one eager step (conv2 fwd = 2nd umma launch)
timeout 900 ncu --profile-from-start off -k regex:umma_gemm -s 1 -c 1 --set full --import-source on \
  --clock-control none -o gpurun_out/r01_umma_conv2_fwd python scripts/profile_step.py small_cnn 512 \
  > gpurun_out/r01_umma.log 2>&1
# 3) full capture of the AES-GCM open kernel at 256 MiB
timeout 900 ncu -k regex:gcm_kernel -s 3 -c 1 --set full --import-source on --clock-control none \
  -o gpurun_out/r01_gcm python scripts/gcm_bench.py > gpurun_out/r01_gcm.log 2>&1
ls -la gpurun_out
