#!/bin/bash
# Round-2 final profiling (r02c) (1 GPU): launch lists of one eager step per model (duration + DRAM bytes
# per launch) and ncu --set full captures of the CTA-pair GEMMs (stage-2/3 forward, stage-3
# weight gradient), the stage-1 halo conv and the stage-1 BN backward.  Outputs: gpurun_out/prof5/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD_FAIL; exit 1; }
mkdir -p gpurun_out/prof5
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none"
for cfg in "resnet18 512" "small_cnn 512" "densenet121 128"; do
  set -- $cfg
  timeout 900 ncu --profile-from-start off $M --csv --log-file gpurun_out/prof5/launches_$1.csv \
    python scripts/profile_step.py $1 $2 > gpurun_out/prof5/launches_$1.log 2>&1
done
full() {  # name kernel-regex skip model batch
  timeout 900 ncu --profile-from-start off -k regex:$2 -s $3 -c 1 --set full --import-source on \
    --clock-control none -o gpurun_out/prof5/$1 python scripts/profile_step.py $4 $5 > gpurun_out/prof5/$1.log 2>&1
}
full r18_fwd_stage3_pair umma_gemm 12 resnet18 512
full r18_fwd_stage2_pair umma_gemm 7 resnet18 512
full r18_wgrad_stage3_pair umma_gemm 33 resnet18 512
full r18_fwd_stage1_halo umma_gemm 1 resnet18 512
full small_wgrad_conv2_quad umma_gemm 11 small_cnn 512
full dense_wgrad_conv2_quad umma_gemm 334 densenet121 128
full r18_bn_bwd_stage1 bn_bwd_fused 15 resnet18 512
ls -la gpurun_out/prof5
