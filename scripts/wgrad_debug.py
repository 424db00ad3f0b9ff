import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import torch.nn.functional as F
from paper_2103_16898_b200 import kernels as K
for (n, h, w) in [(3, 16, 16), (4, 32, 32), (1, 16, 16)]:
    cin = cout = 64; k = 3
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(n, h, w, cin, device="cuda", generator=g).to(torch.bfloat16)
    dy = torch.randn(n, h, w, cout, device="cuda", generator=g).to(torch.bfloat16)
    part, used = K.conv2d_wgrad_partials(dy, x, k, k, 1, 1)
    dw = part[:used].sum(0).view(cout, k, k, cin)
    xr = x.permute(0, 3, 1, 2).float().requires_grad_(True)
    wr = torch.zeros(cout, cin, k, k, device="cuda", requires_grad=True)
    F.conv2d(xr, wr, stride=1, padding=1).backward(dy.permute(0, 3, 1, 2).float())
    ref = wr.grad.permute(0, 2, 3, 1)
    print(n, h, w, "used", used)
    for kh in range(3):
        for kw in range(3):
            d = (dw[:, kh, kw] - ref[:, kh, kw]).abs().max().item()
            # which reference tap does it match?
            best = min(((dw[:, kh, kw] - ref[:, a, b]).abs().max().item(), (a, b)) for a in range(3) for b in range(3))
            print(f"  kh{kh} kw{kw}: err {d:.3g} best match {best[1]} err {best[0]:.3g} rows0-31 {(dw[:32, kh, kw]-ref[:32, kh, kw]).abs().max().item():.3g} rows32-63 {(dw[32:, kh, kw]-ref[32:, kh, kw]).abs().max().item():.3g}")
