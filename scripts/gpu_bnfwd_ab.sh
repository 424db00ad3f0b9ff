#!/bin/bash
# A/B: BN forward kernel at 2 CTAs/SM (launch bounds 512, 2 -> <= 64 registers) vs current
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD_FAIL
rm -rf /tmp/lb && mkdir -p /tmp/lb && cp -r paper_2103_16898_b200/csrc /tmp/lb/csrc && rm -rf /tmp/lb/csrc/_build
sed -i 's/__global__ void __launch_bounds__(THREADS) bn_fwd_fused(const FwdArgs a)/__global__ void __launch_bounds__(THREADS, 2) bn_fwd_fused(const FwdArgs a)/' /tmp/lb/csrc/bn_fused.cu
grep -c "__launch_bounds__(THREADS, 2) bn_fwd_fused" /tmp/lb/csrc/bn_fused.cu
make -s -j 16 -C /tmp/lb/csrc > /tmp/lb/build.log 2>&1 || tail /tmp/lb/build.log
grep -A3 "bn_fwd_fused" /tmp/lb/csrc/_build/bn_fused.ptxas.log | grep "registers\|spill"
AB_ENVS="CVB_LIB=/tmp/lb/libcovault_b200.so;X=1" bash scripts/gpu_ab.sh
AB_ENVS="CVB_LIB=/tmp/lb/libcovault_b200.so;X=1" BENCH_MODEL=small_cnn bash scripts/gpu_ab.sh
