#!/bin/bash
# Round-2 closing profiles (r02d) (1 GPU): launch lists of one eager step per model (duration +
# DRAM bytes per launch) and ncu --set full captures of the kernels the round-2 changes touched:
# the stage-1 halo conv, the stage-2 halo conv with streamed weights, the stage-3 pair conv, the
# stage-2 row-parity stride-2 dgrad (4-tap conv), the stage-1 BN backward, DenseNet's 1x1 row
# GEMM and its block-1 input-gradient gather.  Outputs: gpurun_out/prof9/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD_FAIL; exit 1; }
mkdir -p gpurun_out/prof9
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none"
for cfg in "resnet18 512" "small_cnn 512" "densenet121 128"; do
  set -- $cfg
  timeout 900 ncu --profile-from-start off $M --csv --log-file gpurun_out/prof9/launches_$1.csv \
    python scripts/profile_step.py $1 $2 > gpurun_out/prof9/launches_$1.log 2>&1
done
full() {  # name kernel-regex skip model batch
  timeout 900 ncu --profile-from-start off -k regex:$2 -s $3 -c 1 --set full --import-source on \
    --clock-control none -o gpurun_out/prof9/$1 python scripts/profile_step.py $4 $5 > gpurun_out/prof9/$1.log 2>&1
}
full r18_fwd_stage1_halo umma_gemm 1 resnet18 512
full r18_fwd_stage2_hs umma_gemm 7 resnet18 512
full r18_fwd_stage3_pair umma_gemm 12 resnet18 512
full r18_dgrad_s2_rows_stage2 umma_gemm 50 resnet18 512
full r18_bn_bwd_stage1 bn_bwd_fused 16 resnet18 512
full dense_conv1x1_rows umma_gemm 1 densenet121 128
full dense_gather_block1 bn_gather_dx 61 densenet121 128
ls -la gpurun_out/prof9
