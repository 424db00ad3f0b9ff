#!/bin/bash
# ncu --set full of DenseNet's block-1 dense-layer convs (1x1 64->128 and 3x3 128->32 at 56x56)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD_FAIL; exit 1; }
mkdir -p gpurun_out/prof7
for s in ${SKIPS:-1 2}; do
  timeout 900 ncu --profile-from-start off -k regex:umma_gemm -s $s -c 1 --set full --import-source on \
    --clock-control none -o gpurun_out/prof7/dense_conv_$s python scripts/profile_step.py densenet121 128 \
    > gpurun_out/prof7/dense_conv_$s.log 2>&1
done
ls -la gpurun_out/prof7
