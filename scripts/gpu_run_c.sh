#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash scripts/profile_r02.sh > /dev/null 2>&1
ls gpurun_out/prof2
bash scripts/sanitize.sh
