#!/bin/bash
# ncu --set full of DenseNet's bn_gather_dx launches (block-1 input gather, a block-2 slice gather)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD_FAIL; exit 1; }
mkdir -p gpurun_out/prof6
for s in ${SKIPS:-61 30}; do
  timeout 900 ncu --profile-from-start off -k regex:bn_gather_dx -s $s -c 1 --set full --import-source on \
    --clock-control none -o gpurun_out/prof6/gather_$s python scripts/profile_step.py densenet121 128 \
    > gpurun_out/prof6/gather_$s.log 2>&1
done
ls -la gpurun_out/prof6
