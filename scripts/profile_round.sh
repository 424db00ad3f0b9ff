#!/bin/bash
# Round profiling on the GPU box (1 GPU).  Outputs land in gpurun_out/prof/ and are summarised
# into profiles/ locally (scripts/summarize_ncu.py).
#  1) per-model launch list of one eager training step (duration + DRAM bytes per launch)
#  2) ncu --set full of the top kernels: small-CNN conv2 forward (umma_gemm), the fused BN
#     backward, and the AES-GCM open kernel at 256 MiB
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/prof
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none"
for cfg in "small_cnn 512" "resnet18 512" "densenet121 128"; do
  set -- $cfg
  timeout 900 ncu --profile-from-start off $M --csv --log-file gpurun_out/prof/launches_$1.csv \
    python scripts/profile_step.py $1 $2 > gpurun_out/prof/launches_$1.log 2>&1
done
timeout 900 ncu --profile-from-start off -k regex:umma_gemm -s 1 -c 1 --set full --import-source on \
  --clock-control none -o gpurun_out/prof/umma_small_conv2_fwd python scripts/profile_step.py small_cnn 512 \
  > gpurun_out/prof/umma.log 2>&1
timeout 900 ncu --profile-from-start off -k regex:bn_bwd_fused -s 2 -c 1 --set full --import-source on \
  --clock-control none -o gpurun_out/prof/bn_bwd_small python scripts/profile_step.py small_cnn 512 \
  > gpurun_out/prof/bn.log 2>&1
timeout 900 ncu --profile-from-start off -k regex:umma_gemm -s 8 -c 1 --set full --import-source on \
  --clock-control none -o gpurun_out/prof/umma_r18_stage3 python scripts/profile_step.py resnet18 512 \
  > gpurun_out/prof/umma_r18.log 2>&1
timeout 900 ncu -k regex:gcm_kernel -s 1 -c 1 --set full --import-source on --clock-control none \
  -o gpurun_out/prof/gcm_open_256m python scripts/gcm_one.py 256 > gpurun_out/prof/gcm.log 2>&1
timeout 900 ncu -k regex:gcm_kernel -s 3 -c 1 --set full --import-source on --clock-control none \
  -o gpurun_out/prof/gcm_shard_512 python scripts/gcm_shard.py > gpurun_out/prof/gcm_shard.log 2>&1
timeout 900 ncu --profile-from-start off -k regex:head_train -c 1 --set full --import-source on \
  --clock-control none -o gpurun_out/prof/head_small python scripts/profile_step.py small_cnn 512 \
  > gpurun_out/prof/head.log 2>&1
ls -la gpurun_out/prof
