cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD_FAIL
timeout 300 python -m pytest tests/test_umma_gpu.py -x -q 2>&1 | tail -5
CVB_NO_WGRAD_ROWPAD=1 timeout 120 python scripts/wgrad_pair_probe.py 2>&1 | tail -5
timeout 120 python scripts/wgrad_pair_probe.py 2>&1 | tail -5
AB_ENVS="CVB_NO_WGRAD_ROWPAD=1;X=1" BENCH_MODEL=small_cnn bash scripts/gpu_ab.sh; AB_ENVS="CVB_NO_WGRAD_ROWPAD=1;X=1" bash scripts/gpu_ab.sh
