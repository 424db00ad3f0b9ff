cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD_FAIL
timeout 300 python -m pytest tests/test_umma_gpu.py -x -q 2>&1 | tail -15
CVB_NO_HALO_STREAM=1 timeout 120 python scripts/pair_probe.py 2>&1 | grep "128->128\|256->256"
timeout 120 python scripts/pair_probe.py 2>&1 | grep "128->128\|256->256"
