#!/bin/bash
# A/B: BN backward with explicit rounding steps (current) vs compiler-contracted expressions
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD_FAIL
rm -rf /tmp/lb && mkdir -p /tmp/lb && cp -r paper_2103_16898_b200/csrc /tmp/lb/csrc && rm -rf /tmp/lb/csrc/_build
python - <<'PY'
p='/tmp/lb/csrc/bn_fused.cu'
s=open(p).read()
s=s.replace("__fmul_rn(__fsub_rn(xv[k], mu[k]), rs[k])","(xv[k] - mu[k]) * rs[k]")
s=s.replace("__fmaf_rn(xh[k], ga[k], be[k])","xh[k] * ga[k] + be[k]")
s=s.replace("__fmul_rn(kk[k], __fmaf_rn(-xh[k], kg[k], __fsub_rn(d[k], kb[k])))","kk[k] * (d[k] - kb[k] - xh[k] * kg[k])")
s=s.replace("o[0] = __fadd_rn(u.x, o[0]); o[1] = __fadd_rn(u.y, o[1]); o[2] = __fadd_rn(u.z, o[2]);","o[0] += u.x; o[1] += u.y; o[2] += u.z;")
s=s.replace("o[3] = __fadd_rn(u.w, o[3]); o[4] = __fadd_rn(w.x, o[4]); o[5] = __fadd_rn(w.y, o[5]);","o[3] += u.w; o[4] += w.x; o[5] += w.y;")
s=s.replace("o[6] = __fadd_rn(w.z, o[6]); o[7] = __fadd_rn(w.w, o[7]);","o[6] += w.z; o[7] += w.w;")
open(p,'w').write(s)
PY
make -s -j 16 -C /tmp/lb/csrc > /tmp/lb/build.log 2>&1 || tail /tmp/lb/build.log
grep -A3 "bn_bwd_fused" /tmp/lb/csrc/_build/bn_fused.ptxas.log | grep "registers\|spill"
AB_ENVS="CVB_LIB=/tmp/lb/libcovault_b200.so;X=1" bash scripts/gpu_ab.sh
AB_ENVS="CVB_LIB=/tmp/lb/libcovault_b200.so;X=1" BENCH_MODEL=small_cnn bash scripts/gpu_ab.sh
