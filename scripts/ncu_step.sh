#!/bin/bash
# ncu launch list (per-kernel duration + DRAM bytes) of one eager training step of MODEL.
# usage: scripts/ncu_step.sh MODEL BATCH OUT_CSV
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file "$3" python scripts/profile_step.py "$1" "$2" > /dev/null 2>&1
