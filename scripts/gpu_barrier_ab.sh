#!/bin/bash
# A/B of the grid-barrier implementation (current acq_rel form vs the round-1 threadfence form)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD_FAIL
rm -rf /tmp/lb && mkdir -p /tmp/lb && cp -r paper_2103_16898_b200/csrc /tmp/lb/csrc && rm -rf /tmp/lb/csrc/_build
python - <<'PY'
p='/tmp/lb/csrc/cvb_common.cuh'
s=open(p).read()
a=s.index('__device__ __forceinline__ void cvb_grid_barrier(unsigned* bar) {')
b=s.index('#endif', a)
s=s[:a]+'''__device__ __forceinline__ void cvb_grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = bar + 1;
    const unsigned g = *vgen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*vgen == g) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}
'''+s[b:]
open(p,'w').write(s)
PY
make -s -j 16 -C /tmp/lb/csrc > /tmp/lb/build.log 2>&1 || tail /tmp/lb/build.log
ls -la /tmp/lb/libcovault_b200.so
AB_ENVS="CVB_LIB=/tmp/lb/libcovault_b200.so;X=1" bash scripts/gpu_ab.sh
