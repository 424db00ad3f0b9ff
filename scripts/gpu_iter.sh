#!/bin/bash
# iteration loop on the GPU box: build, the named test files (TESTS), then bench + launch list
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest $TESTS -x -q -m gpu > gpurun_out/iter_tests.log 2>&1
  echo "tests rc=$?"; tail -n 15 gpurun_out/iter_tests.log
fi
[ -n "$NOBENCH" ] || bash scripts/gpu_step_check.sh
