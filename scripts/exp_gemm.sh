cd $GRAFT_REPO_ROOT
cat > /tmp/m.py <<'PY'
import sys; sys.path.insert(0,'.')
from scripts.gemm_micro import dense, conv
dense(8192, 256, 8192); dense(4096, 4096, 4096); conv(512, 32, 32, 32, 3, 1, 1)
PY
for cfg in "0 0" "1 0" "2 0" "0 2" "0 4"; do set -- $cfg; echo "== dbg=$1 stages=$2"; CVB_GEMM_DBG=$1 CVB_STAGES=$2 timeout 120 python /tmp/m.py 2>&1 | grep -v wgrad; done
