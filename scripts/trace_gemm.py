"""Timeline of CTA 0 of one tcgen05 GEMM launch (needs CVB_GEMM_DBG=4)."""
import ctypes, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2103_16898_b200 import kernels as K, _lib
which = sys.argv[1] if len(sys.argv) > 1 else "conv"
if which == "stem":
    x = torch.randn(512, 32, 32, 8, device="cuda").bfloat16(); w = torch.randn(32, 3, 3, 8, device="cuda").bfloat16()
    y = torch.empty(512, 32, 32, 32, device="cuda", dtype=torch.bfloat16)
    f = lambda: K.conv2d_fwd(x, w, 1, 1, out=y)
elif which == "stemwg":
    x = torch.randn(512, 32, 32, 8, device="cuda").bfloat16(); dy = torch.randn(512, 32, 32, 32, device="cuda").bfloat16()
    f = lambda: K.conv2d_wgrad_partials(dy, x, 3, 3, 1, 1)
elif which == "wg32":
    x = torch.randn(512, 32, 32, 32, device="cuda").bfloat16(); dy = torch.randn(512, 32, 32, 32, device="cuda").bfloat16()
    f = lambda: K.conv2d_wgrad_partials(dy, x, 3, 3, 1, 1)
elif which == "conv64":
    x = torch.randn(512, 32, 32, 64, device="cuda").bfloat16(); w = torch.randn(64, 3, 3, 64, device="cuda").bfloat16()
    y = torch.empty(512, 32, 32, 64, device="cuda", dtype=torch.bfloat16)
    f = lambda: K.conv2d_fwd(x, w, 1, 1, out=y)
elif which in ("conv128", "conv256"):
    c, hw = (128, 16) if which == "conv128" else (256, 8)
    x = torch.randn(512, hw, hw, c, device="cuda").bfloat16(); w = torch.randn(c, 3, 3, c, device="cuda").bfloat16()
    y = torch.empty(512, hw, hw, c, device="cuda", dtype=torch.bfloat16)
    f = lambda: K.conv2d_fwd(x, w, 1, 1, out=y)
elif which == "c1x1":   # DenseNet conv1 dgrad shape: 1x1 conv 128 -> 256 at 56x56, batch 128
    x = torch.randn(128, 56, 56, 128, device="cuda").bfloat16(); w = torch.randn(256, 1, 1, 128, device="cuda").bfloat16()
    y = torch.empty(128, 56, 56, 256, device="cuda", dtype=torch.bfloat16)
    f = lambda: K.conv2d_fwd(x, w, 1, 0, out=y)
elif which == "dwg":   # DenseNet conv2 weight gradient (128 -> 32, 56x56, batch 128)
    x = torch.randn(128, 56, 56, 128, device="cuda").bfloat16(); dy = torch.randn(128, 56, 56, 32, device="cuda").bfloat16()
    f = lambda: K.conv2d_wgrad_partials(dy, x, 3, 3, 1, 1)
elif which in ("ds64", "ds256"):   # 1x1 stride-2 downsample convs of ResNet-18
    c, hw = (64, 32) if which == "ds64" else (256, 8)
    x = torch.randn(512, hw, hw, c, device="cuda").bfloat16(); w = torch.randn(2 * c, 1, 1, c, device="cuda").bfloat16()
    y = torch.empty(512, hw // 2, hw // 2, 2 * c, device="cuda", dtype=torch.bfloat16)
    f = lambda: K.conv2d_fwd(x, w, 2, 0, out=y)
elif which == "conv":
    x = torch.randn(512, 32, 32, 32, device="cuda").bfloat16(); w = torch.randn(32, 3, 3, 32, device="cuda").bfloat16()
    y = torch.empty(512, 32, 32, 32, device="cuda", dtype=torch.bfloat16)
    f = lambda: K.conv2d_fwd(x, w, 1, 1, out=y)
else:
    a = torch.randn(4096, 4096, device="cuda").bfloat16(); b = torch.randn(4096, 4096, device="cuda").bfloat16()
    o = torch.empty(4096, 4096, device="cuda", dtype=torch.bfloat16)
    f = lambda: K.gemm(a, b, 4096, 4096, 4096, out=o)
for _ in range(3): f()
torch.cuda.synchronize()
L = _lib.load(); L.cvb_debug_trace.argtypes = [ctypes.c_void_p]
buf = np.zeros(8 * 4096, dtype=np.int64)
L.cvb_debug_trace(buf.ctypes.data)
t = buf.reshape(8, 4096)
base = t[0][0]
names = ["prod_empty_ok", "mma_full_ok", "mma_committed", "epi_tfull_ok", "epi_done"]
n_it = int((t[1] > 0).sum()); n_t = int((t[3] > 0).sum())
print("stages", n_it, "tiles", n_t, "total cycles", t[4][n_t - 1] - base)
for i in list(range(min(n_it, 24))):
    print(i, " ".join(f"{names[k]}={t[k][i] - base:8d}" for k in range(3)))
for i in range(min(n_t, 12)):
    print("tile", i, f"tfull_ok={t[3][i]-base} epi_done={t[4][i]-base}")
d = np.diff(t[1][:n_it])
print("median cycles between MMA stage starts", np.median(d), "mean", d.mean())
print("median full-wait->commit", np.median(t[2][:n_it] - t[1][:n_it]))
print("median producer empty_ok - prev mma commit of slot", )
e = t[4][:n_t] - t[3][:n_t]
print("median epilogue cycles (tfull_ok -> done)", np.median(e), "tile period", np.median(np.diff(t[3][:n_t])))
if (t[5] > 0).sum():
    print("epilogue phases (median cycles from tfull_ok): tmem loaded", np.median(t[5][:n_t] - t[3][:n_t]),
          "buffer free", np.median(t[6][:n_t] - t[3][:n_t]), "store issued", np.median(t[7][:n_t] - t[3][:n_t]))
print("per-tile timeline (cycles rel. to CTA start): prod_empty_ok mma_full_ok mma_commit | epi: tfull tmem_ld buf_free store_issued done")
for i in range(10, 16):
    print(i, [int(t[k][i] - base) for k in (0, 1, 2)], "|", [int(t[k][i] - base) for k in (3, 5, 6, 7, 4)])
