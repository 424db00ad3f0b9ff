#!/bin/bash
# Round-2 profiling (1 GPU): launch list of one eager ResNet-18 / small-CNN step (duration + DRAM
# bytes per launch; scripts/traffic_json.py turns it into profiles/traffic.json) and ncu --set full
# captures of the kernels the round-2 work targets.  Outputs in gpurun_out/prof2/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/prof2
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none"
for cfg in ${LISTS:-"resnet18 512" "small_cnn 512"}; do
  set -- $cfg
  timeout 900 ncu --profile-from-start off $M --csv --log-file gpurun_out/prof2/launches_$1.csv \
    python scripts/profile_step.py $1 $2 > gpurun_out/prof2/launches_$1.log 2>&1
done
full() {  # name kernel-regex skip model batch
  timeout 900 ncu --profile-from-start off -k regex:$2 -s $3 -c 1 --set full --import-source on \
    --clock-control none -o gpurun_out/prof2/$1 python scripts/profile_step.py $4 $5 > gpurun_out/prof2/$1.log 2>&1
}
if [ -z "$NOFULL" ]; then
  full r18_bn_fwd_stage4 bn_fwd_fused 16 resnet18 512
  full r18_bn_bwd_stage1 bn_bwd_fused 15 resnet18 512
  full r18_wgrad_stage1 umma_gemm 59 resnet18 512
  full r18_fwd_stage2 umma_gemm 7 resnet18 512
fi
ls -la gpurun_out/prof2
