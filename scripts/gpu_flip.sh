cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD_FAIL
timeout 300 python -m pytest tests/test_nn_kernels_gpu.py tests/test_umma_gpu.py -x -q 2>&1 | tail -3
CVB_EPI8_SHORTK=0 timeout 120 python scripts/pair_probe.py 2>&1 | head -3
CVB_EPI8_SHORTK=1 timeout 120 python scripts/pair_probe.py 2>&1 | head -3
AB_ENVS="CVB_EPI8_SHORTK=0;CVB_EPI8_SHORTK=1" bash scripts/gpu_ab.sh
