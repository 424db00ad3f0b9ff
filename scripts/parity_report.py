import sys; sys.path.insert(0, '.')
from tests import cnn_parity as P
for model, b in [(m, int(b)) for m, b in (a.split(":") for a in sys.argv[1:])]:
    rep, wrel = P.run_parity(model, batch=b, steps=3)
    for r in rep:
        worst = sorted(r["grads"].items(), key=lambda kv: -kv[1])[:3]
        print(model, b, "step", r["step"], "loss", r["loss_gpu"], r["loss_ref"], "worst grads", [(k, round(v, 4)) for k, v in worst])
    print(model, b, "cos", [round(r["cos"], 5) for r in rep], "w rel", wrel)
