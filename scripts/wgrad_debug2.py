import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import torch.nn.functional as F
from paper_2103_16898_b200 import kernels as K
n, h, w = 1, 16, 16
cin = cout = 64
g = torch.Generator(device="cuda").manual_seed(7)
x = torch.randn(n, h, w, cin, device="cuda", generator=g).to(torch.bfloat16)
dy = torch.randn(n, h, w, cout, device="cuda", generator=g).to(torch.bfloat16)
part, used = K.conv2d_wgrad_partials(dy, x, 3, 3, 1, 1)
dw = part[:used].sum(0).view(cout, 3, 3, cin).float()
X = F.pad(x.float().permute(0, 3, 1, 2), (4, 4, 4, 4))[0]    # [ci][H+8][W+8]
D = dy.float().permute(0, 3, 1, 2)[0]                          # [co][H][W]
def C(dr, dc_kw):   # sum_y,x D[co][y][x] * X[ci][y+dr][x+dc]
    Xs = X[:, 4 + dr:4 + dr + h, 4 + dc_kw:4 + dc_kw + w]
    return torch.einsum("oyx,iyx->oi", D, Xs)
for kw in range(3):
    got = dw[:, 1, kw]
    res = []
    for dr in range(-3, 4):
        for dc in range(-3, 4):
            res.append(((got - C(dr, dc)).abs().max().item(), dr, dc))
    res.sort()
    print("kh1 kw", kw, "best (err, drow, dcol):", [tuple(round(v, 3) if isinstance(v, float) else v for v in r) for r in res[:3]])
    # also partial: rows 0-31 vs 32-63
