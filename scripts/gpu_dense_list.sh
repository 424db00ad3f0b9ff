cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/prof4
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/prof4/launches_densenet121.csv python scripts/profile_step.py densenet121 128 > /dev/null 2>&1
python scripts/summarize_ncu.py launches gpurun_out/prof4/launches_densenet121.csv | head -20
