cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD_FAIL
timeout 300 python -m pytest tests/test_umma_gpu.py -x -q 2>&1 | tail -4
CVB_GEMM_PAIR_HALO=1 timeout 120 python scripts/pair_probe.py 2>&1 | head -6
timeout 120 python scripts/pair_probe.py 2>&1 | head -6
NOLIST=1 bash scripts/gpu_step_check.sh
BENCH_MODEL=small_cnn NOLIST=1 bash scripts/gpu_step_check.sh
