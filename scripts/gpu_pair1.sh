cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD_FAIL
timeout 300 python -m pytest tests/test_umma_gpu.py -x -q 2>&1 | tail -15
for pr in 0 1; do CVB_GEMM_PAIR=$pr timeout 120 python scripts/pair_probe.py 2>&1 | tail -8; done
CVB_GEMM_PAIR=1 CVB_KB_PAIR=0 timeout 120 python scripts/pair_probe.py 2>&1 | tail -8
