cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD_FAIL
for e in "X=1" "CVB_NO_HALO_ROWS=1" "CVB_NO_KWBOX=1" "CVB_STAGES=2"; do
  env $e timeout 120 python scripts/pair_probe.py 2>&1 | sed -n 4,9p | sed "s/^/$e /"
done
