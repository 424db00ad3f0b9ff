"""Print the CNN parity numbers the tolerances in tests/cnn_parity.py are set from."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from tests import cnn_parity as P  # noqa: E402

torch.set_num_threads(max(1, torch.get_num_threads()))
what = sys.argv[1:] or ["forced_small", "forced_r18", "free20", "r18_512", "dn128"]
if "forced_small" in what:
    for b in (64, 512):
        t = time.time()
        out = P.run_forced("small_cnn", batch=b, steps=3)
        for s, (lg, lr_, g, w) in enumerate(out):
            print(f"small b{b} s{s}: dloss {abs(lg-lr_)/max(1,abs(lr_)):.2e} gmax {max(g.values()):.2e} "
                  f"({max(g, key=g.get)}) wmax {max(w.values()):.2e} ({max(w, key=w.get)})", flush=True)
        print("  t", time.time() - t)
if "forced_r18" in what:
    for b in (32,):
        out = P.run_forced("resnet18", batch=b, steps=2)
        for s, (lg, lr_, g, w) in enumerate(out):
            print(f"r18 b{b} s{s}: dloss {abs(lg-lr_)/max(1,abs(lr_)):.2e} gmax {max(g.values()):.2e} "
                  f"({max(g, key=g.get)}) wmax {max(w.values()):.2e} ({max(w, key=w.get)})", flush=True)
if "free20" in what:
    rep, wrel = P.run_parity("small_cnn", batch=64, steps=20, lr=1e-3)
    print("free20 losses gpu", [round(r["loss_gpu"], 4) for r in rep])
    print("free20 losses ref", [round(r["loss_ref"], 4) for r in rep])
    print("free20 max rel dloss", max(abs(r["loss_gpu"] - r["loss_ref"]) / max(1, abs(r["loss_ref"])) for r in rep),
          "wrel", wrel, flush=True)
if "r18_512" in what:
    t = time.time()
    out = P.run_forced("resnet18", batch=512, steps=1)
    lg, lr_, g, w = out[0]
    print(f"r18 b512: dloss {abs(lg-lr_)/max(1,abs(lr_)):.2e} gmax {max(g.values()):.2e} ({max(g, key=g.get)}) "
          f"wmax {max(w.values()):.2e} t {time.time()-t:.1f}s", flush=True)
if "dn128" in what:
    t = time.time()
    rep, wrel = P.run_parity("densenet121", batch=128, steps=1)
    r = rep[0]
    print(f"dn128: loss {r['loss_gpu']:.5f} vs {r['loss_ref']:.5f} cos {r['cos']:.4f} "
          f"gmax {max(r['grads'].values()):.3f} t {time.time()-t:.1f}s", flush=True)
