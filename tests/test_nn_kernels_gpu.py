"""Every memory-bound training-step kernel vs a torch fp32 reference of the same op, on
identical (bf16) inputs.  Tolerances are per-op and stated inline."""
import pytest
import torch
import torch.nn.functional as F

from paper_2103_16898_b200 import kernels as K

pytestmark = pytest.mark.gpu
dev = "cuda"


def rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-12)).item()


def nchw(t):
    return t.float().permute(0, 3, 1, 2)


@pytest.mark.parametrize("rows,C", [(512 * 32 * 32, 32), (4096, 64), (1000, 512), (98 * 7, 1024)])
def test_bn_forward_backward(rows, C):
    g = torch.Generator(device=dev).manual_seed(rows + C)
    z = (torch.randn(rows, C, device=dev, generator=g) * 2 + 0.5).bfloat16()
    gamma = torch.rand(C, device=dev, generator=g) + 0.5
    beta = torch.randn(C, device=dev, generator=g) * 0.1
    mean, rstd = torch.empty(C, device=dev), torch.empty(C, device=dev)
    rm, rv = torch.zeros(C, device=dev), torch.ones(C, device=dev)
    ws = K.bn_workspace(rows, C)
    K.bn_stats(z, rows, C, C, ws, mean, rstd, run_mean=rm, run_var=rv)
    zf = z.float()
    assert rel(mean, zf.mean(0)) < 1e-5
    assert rel(rstd, 1 / torch.sqrt(zf.var(0, unbiased=False) + 1e-5)) < 1e-5
    assert rel(rv, 0.9 + 0.1 * zf.var(0, unbiased=True)) < 1e-5
    y = torch.empty(rows, C, device=dev, dtype=torch.bfloat16)
    K.bn_apply(z, rows, C, C, mean, rstd, gamma, beta, y, C, relu=True)
    zr = zf.clone().requires_grad_(True)
    gr, br = gamma.clone().requires_grad_(True), beta.clone().requires_grad_(True)
    yr = F.relu(F.batch_norm(zr, None, None, gr, br, training=True, eps=1e-5))
    assert rel(y, yr) < 4e-3          # bf16 output rounding
    dy = torch.randn(rows, C, device=dev, generator=g).bfloat16()
    yr.backward(dy.float())
    dg, db = torch.empty(C, device=dev), torch.empty(C, device=dev)
    dx = torch.empty(rows, C, device=dev, dtype=torch.bfloat16)
    K.bn_backward(dy, C, z, C, rows, C, mean, rstd, gamma, beta, ws, dg, db, relu=True, dx=dx, dxcs=C)
    assert rel(db, br.grad) < 1e-4
    assert rel(dg, gr.grad) < 1e-4
    assert rel(dx, zr.grad) < 5e-3    # bf16 output rounding


def test_bn_residual_and_dz_out():
    rows, C = 2048, 64
    z = torch.randn(rows, C, device=dev).bfloat16()
    res = torch.randn(rows, C, device=dev).bfloat16()
    gamma, beta = torch.rand(C, device=dev) + 0.5, torch.randn(C, device=dev) * 0.1
    mean, rstd, ws = torch.empty(C, device=dev), torch.empty(C, device=dev), K.bn_workspace(rows, C)
    K.bn_stats(z, rows, C, C, ws, mean, rstd)
    y = torch.empty(rows, C, device=dev, dtype=torch.bfloat16)
    K.bn_apply(z, rows, C, C, mean, rstd, gamma, beta, y, C, relu=True, res=res, rcs=C)
    zr = z.float().requires_grad_(True)
    rr = res.float().requires_grad_(True)
    yr = F.relu(F.batch_norm(zr, None, None, gamma, beta, training=True, eps=1e-5) + rr)
    assert rel(y, yr) < 4e-3
    dy = torch.randn(rows, C, device=dev).bfloat16()
    yr.backward(dy.float())
    dg, db = torch.empty(C, device=dev), torch.empty(C, device=dev)
    dx = torch.empty_like(z)
    dres = torch.empty_like(z)
    K.bn_backward(dy, C, z, C, rows, C, mean, rstd, gamma, beta, ws, dg, db, relu=True, y=y, ycs=C, dx=dx, dxcs=C,
                  dz_out=dres)
    assert rel(dres, rr.grad) < 1e-6  # exact masking of bf16 values
    assert rel(dx, zr.grad) < 5e-3


@pytest.mark.parametrize("rows,C,xcs,res", [(512 * 32 * 32, 64, 64, True), (3000, 96, 160, False),
                                              (98 * 49, 1024, 1024, False), (77, 32, 32, True)])
def test_bn_single_launch_forward_backward(rows, C, xcs, res):
    """cvb_bn_forward / cvb_bn_backward_fused (one cooperative launch each) vs torch fp32:
    strided input (DenseNet concat prefix), output at a channel offset, residual add, fp32
    accumulated dx.  Same tolerances as the three-kernel path."""
    g = torch.Generator(device=dev).manual_seed(rows + C + xcs)
    zfull = (torch.randn(rows, xcs, device=dev, generator=g) * 1.5 + 0.3).bfloat16()
    z = zfull[:, :C]
    gamma = torch.rand(C, device=dev, generator=g) + 0.5
    beta = torch.randn(C, device=dev, generator=g) * 0.1
    r = torch.randn(rows, C, device=dev, generator=g).bfloat16() if res else None
    mean, rstd = torch.empty(C, device=dev), torch.empty(C, device=dev)
    rm, rv = torch.zeros(C, device=dev), torch.ones(C, device=dev)
    ws = K.bn_workspace(rows, C)
    yfull = torch.zeros(rows, C + 16, device=dev, dtype=torch.bfloat16)
    K.bn_forward(zfull, rows, C, xcs, ws, mean, rstd, gamma, beta, yfull, C + 16, ycoff=8, relu=True, res=r,
                 rcs=C, run_mean=rm, run_var=rv)
    zf = z.float()
    assert rel(mean, zf.mean(0)) < 1e-5
    assert rel(rstd, 1 / torch.sqrt(zf.var(0, unbiased=False) + 1e-5)) < 1e-5
    assert rel(rv, 0.9 + 0.1 * zf.var(0, unbiased=True)) < 1e-5
    zr = zf.clone().requires_grad_(True)
    gr, br = gamma.clone().requires_grad_(True), beta.clone().requires_grad_(True)
    pre = F.batch_norm(zr, None, None, gr, br, training=True, eps=1e-5)
    yr = F.relu(pre + r.float() if res else pre)
    assert rel(yfull[:, 8:8 + C], yr) < 4e-3
    assert yfull[:, :8].abs().max().item() == 0 and yfull[:, 8 + C:].abs().max().item() == 0
    dy = torch.randn(rows, C, device=dev, generator=g).bfloat16()
    dg, db = torch.empty(C, device=dev), torch.empty(C, device=dev)
    base = torch.randn(rows, xcs, device=dev, generator=g)
    dx32 = base.clone()
    y = yfull[:, 8:8 + C].contiguous()
    K.bn_backward(dy, C, zfull, xcs, rows, C, mean, rstd, gamma, beta, ws, dg, db, relu=True, y=y, ycs=C,
                  dx32=dx32, dxcs=xcs, accum32=True)
    # fp64 reference with the kernel's own ReLU mask (y > 0): near-zero pre-activations may
    # round to the other side of zero between fp32 and torch's order of operations
    d = dy.double() * (y.double() > 0)
    xh = (zf.double() - zf.double().mean(0)) / torch.sqrt(zf.double().var(0, unbiased=False) + 1e-5)
    rdb, rdg = d.sum(0), (d * xh).sum(0)
    rdx = gamma.double() / torch.sqrt(zf.double().var(0, unbiased=False) + 1e-5) * (d - rdb / rows - xh * rdg / rows)
    assert rel(db, rdb) < 1e-4
    assert rel(dg, rdg) < 1e-4
    assert rel(dx32[:, :C] - base[:, :C], rdx) < 1e-4
    assert torch.equal(dx32[:, C:], base[:, C:])


@pytest.mark.parametrize("k,s,p,h", [(2, 2, 0, 32), (3, 2, 1, 112), (2, 2, 0, 8), (3, 2, 1, 9), (3, 2, 1, 8)])
def test_maxpool_exact(k, s, p, h):
    x = torch.randn(4, h, h, 64, device=dev).bfloat16()
    x[0, :4, :4] = 1.0   # ties: first max wins, like torch
    oh = (h + 2 * p - k) // s + 1
    y = torch.empty(4, oh, oh, 64, device=dev, dtype=torch.bfloat16)
    K.maxpool_fwd(x, k, s, p, y)
    xr = nchw(x).cpu().requires_grad_(True)
    yr = F.max_pool2d(xr, k, s, p)
    assert torch.equal(nchw(y).cpu(), yr.detach())
    dy = torch.randn(4, oh, oh, 64, device=dev).bfloat16()
    dx = torch.empty_like(x)
    K.maxpool_bwd(x, dy, k, s, p, dx)
    yr.backward(nchw(dy).cpu())
    assert rel(nchw(dx).cpu(), xr.grad) < 4e-3   # overlapping windows sum in fp32 -> bf16
    # arg-max variant: identical forward, identical backward (same first-max rule, same order)
    y2 = torch.empty_like(y)
    idx = torch.empty(4, oh, oh, 64, device=dev, dtype=torch.uint8)
    K.maxpool_fwd(x, k, s, p, y2, idx=idx)
    assert torch.equal(y2, y)
    dx2 = torch.empty_like(x)
    K.maxpool_bwd(x, dy, k, s, p, dx2, idx=idx)
    assert torch.equal(dx2, dx)


def test_avgpool_and_gap():
    x = torch.randn(4, 14, 14, 128, device=dev).bfloat16()
    y = torch.empty(4, 7, 7, 128, device=dev, dtype=torch.bfloat16)
    K.avgpool_fwd(x, 4, 14, 14, 128, 128, 2, y)
    assert rel(nchw(y), F.avg_pool2d(nchw(x), 2)) < 4e-3
    xf = x.float()   # the kernel's exact arithmetic: fp32 sum in window order, * 0.25, bf16 round
    ref2 = ((((xf[:, 0::2, 0::2] + xf[:, 0::2, 1::2]) + xf[:, 1::2, 0::2]) + xf[:, 1::2, 1::2]) * 0.25).bfloat16()
    assert torch.equal(y, ref2)
    dy = torch.randn(4, 7, 7, 128, device=dev).bfloat16()
    dx = torch.empty_like(x)
    K.avgpool_bwd(dy, 4, 14, 14, 128, 2, dx, 128)
    xr = nchw(x).requires_grad_(True)
    F.avg_pool2d(xr, 2).backward(nchw(dy))
    assert rel(nchw(dx), xr.grad) < 1e-6
    g = torch.empty(4, 128, device=dev, dtype=torch.bfloat16)
    K.gap_fwd(x, 4, 196, 128, 128, g)
    assert rel(g, x.float().mean(dim=(1, 2))) < 4e-3
    dg = torch.randn(4, 128, device=dev).bfloat16()
    dxx = torch.empty_like(x)
    K.gap_bwd(dg, 4, 196, 128, dxx)
    assert rel(dxx, (dg.float() / 196)[:, None, None, :].expand_as(dxx)) < 4e-3


def test_softmax_xent():
    B, C, ld = 512, 10, 16
    logits = torch.randn(B, ld, device=dev) * 3
    labels = torch.randint(0, C, (B,), device=dev, dtype=torch.int32)
    rows, loss = torch.empty(B, device=dev), torch.empty(1, device=dev)
    dl = torch.zeros(B, ld, device=dev, dtype=torch.bfloat16)
    K.softmax_xent(logits, B, C, labels, 1.0 / B, rows, loss, dl)
    lr = logits[:, :C].clone().requires_grad_(True)
    ref = F.cross_entropy(lr, labels.long())
    ref.backward()
    assert abs(loss.item() - ref.item()) < 1e-5 * max(1, ref.item())
    assert rel(dl[:, :C], lr.grad) < 4e-3 and dl[:, C:].abs().max().item() == 0


def test_adam_matches_torch():
    n = 10_000
    p0 = torch.randn(n, device=dev)
    p, g = p0.clone(), torch.randn(n, device=dev)
    m, v = torch.zeros(n, device=dev), torch.zeros(n, device=dev)
    pb = torch.empty(n, device=dev, dtype=torch.bfloat16)
    step_dev, sched = torch.zeros(1, dtype=torch.int32, device=dev), torch.zeros(4, device=dev)
    pr = p0.clone().requires_grad_(True)
    opt = torch.optim.Adam([pr], lr=1e-3, foreach=False)
    for _ in range(3):
        K.adam_step(p, g, m, v, pb, 1e-3, 0.9, 0.999, 1e-8, step_dev=step_dev, sched_dev=sched)
        pr.grad = g.clone()
        opt.step()
    assert rel(p, pr.detach()) < 1e-6
    assert torch.equal(pb, p.bfloat16())
    assert int(step_dev.item()) == 3 and sched[2].view(torch.int32).item() == 0   # counter advanced, CTA count reset
    assert int(step_dev.item()) == 3


def test_sgd_matches_torch():
    n = 1000
    p0, g = torch.randn(n, device=dev), torch.randn(n, device=dev)
    p, buf = p0.clone(), torch.zeros(n, device=dev)
    pr = p0.clone().requires_grad_(True)
    opt = torch.optim.SGD([pr], lr=0.1, momentum=0.9, weight_decay=5e-4)
    for i in range(3):
        K.sgd_step(p, g, buf, None, 0.1, 0.9, 5e-4, first=(i == 0))
        pr.grad = g.clone()
        opt.step()
    assert rel(p, pr.detach()) < 1e-6


def test_layout_helpers():
    w = torch.randn(64, 3, 3, 32, device=dev).bfloat16()
    wt = torch.empty(32, 3, 3, 64, device=dev, dtype=torch.bfloat16)
    K.weight_flip(w, wt)
    assert torch.equal(wt, w.flip(1, 2).permute(3, 1, 2, 0).contiguous())
    dy = torch.randn(2, 4, 5, 16, device=dev).bfloat16()
    up = torch.empty(2, 7, 9, 16, device=dev, dtype=torch.bfloat16)
    K.zero_upsample(dy, up)
    want = torch.zeros_like(up)
    want[:, ::2, ::2] = dy
    assert torch.equal(up, want)
    x = torch.randn(300, 48, device=dev)
    out = torch.empty(48, device=dev)
    K.col_sum(x, 300, 48, 48, out)
    assert rel(out, x.sum(0)) < 1e-6
    part = torch.randn(5, 1000, device=dev)
    red = torch.zeros(1000, device=dev)
    K.reduce_splits(part, 5, 1000, red)
    assert rel(red, part.sum(0)) < 1e-6


def test_weight_flip_batched_matches_torch():
    """Batched dgrad weight flip ([cout][kh][kw][cin] -> [cin][kh'][kw'][cout], both spatial
    axes reversed) for several layers in one launch, incl. channel counts off the 32-tile."""
    shapes = [(64, 3, 3, 64), (128, 3, 3, 72), (40, 1, 1, 24), (512, 3, 3, 512)]
    ws = [torch.randn(s, device=dev).bfloat16() for s in shapes]
    pb = torch.cat([w.reshape(-1) for w in ws])
    fb = torch.zeros_like(pb)
    desc, off = [], 0
    for s in shapes:
        n = s[0] * s[1] * s[2] * s[3]
        desc += [off, off, s[0], s[1], s[2], s[3]]
        off += n
    desc_dev = torch.tensor(desc, dtype=torch.int64, device=dev)
    K.weight_flip_batched(pb, fb, desc_dev, len(shapes), max(s[0] * s[1] * s[2] * s[3] for s in shapes), 0)
    off = 0
    for w in ws:
        n = w.numel()
        want = w.flip(1, 2).permute(3, 1, 2, 0).contiguous().reshape(-1)
        assert torch.equal(fb[off:off + n], want)
        off += n


@pytest.mark.gpu
def test_transpose_batched_matches_torch():
    """Batched transposes in one launch (the per-step flipped / class dgrad weights): vector jobs
    (everything a multiple of 8) and element jobs (odd extents / offsets / strides), tiles
    partially outside the matrix, and more jobs than one launch's shared-memory prefix holds."""
    g = torch.Generator().manual_seed(7)
    shapes = [(64, 64), (512, 512), (32, 128), (8, 24), (72, 40), (13, 7), (130, 66), (1, 1), (200, 8)]
    shapes += [(8 * int(torch.randint(1, 9, (1,), generator=g)), 8 * int(torch.randint(1, 9, (1,), generator=g)))
               for _ in range(60)]
    src = torch.randn(sum(r * c + 16 for r, c in shapes) + 8, device=dev).bfloat16()
    dst = torch.zeros(sum(r * c + 16 for r, c in shapes) + 8, dtype=torch.bfloat16, device=dev)
    up8 = lambda v: (v + 7) // 8 * 8
    desc, so, do = [], 8, 0
    for i, (r, c) in enumerate(shapes):
        odd = i == 4   # an element job with an unaligned source offset
        s0 = so + (1 if odd else 0)
        desc += [s0, do, r, c, c, r]
        so += up8(r * c + 5)
        do += up8(r * c + 3)
    desc_dev = torch.tensor(desc, dtype=torch.int64, device=dev)
    max_elems = max(r * c for r, c in shapes)
    K.transpose_batched(src, dst, desc_dev, len(shapes), max_elems, 0)
    for j in range(len(shapes)):
        s0, d0, r, c = desc[6 * j:6 * j + 4]
        want = src[s0:s0 + r * c].view(r, c).t().contiguous().reshape(-1)
        assert torch.equal(dst[d0:d0 + r * c], want), (j, r, c)
    # > 8192 jobs: several launches
    n = 9000
    src2 = torch.randn(n * 64, device=dev).bfloat16()
    dst2 = torch.zeros_like(src2)
    desc2 = torch.tensor([[64 * j, 64 * j, 8, 8, 8, 8] for j in range(n)], dtype=torch.int64, device=dev).reshape(-1)
    K.transpose_batched(src2, dst2, desc2, n, 64, 0)
    assert torch.equal(dst2.view(n, 8, 8), src2.view(n, 8, 8).transpose(1, 2))


@pytest.mark.parametrize("rows,C", [(512 * 32 * 32, 64), (3000, 128), (77, 512)])
def test_bn_relu_mask_replaces_y(rows, C):
    """Residual BN: the forward's ReLU mask bits equal (y > 0) of the stored bf16 y, and the
    backward reading the mask is bit-identical to the backward reading y."""
    g = torch.Generator(device=dev).manual_seed(rows * 3 + C)
    z = (torch.randn(rows, C, device=dev, generator=g) * 1.5).bfloat16()
    res = torch.randn(rows, C, device=dev, generator=g).bfloat16()
    res[0, :8] = 0   # exact zeros around the ReLU edge
    gamma = torch.rand(C, device=dev, generator=g) + 0.5
    beta = torch.randn(C, device=dev, generator=g) * 0.1
    mean, rstd, ws = torch.empty(C, device=dev), torch.empty(C, device=dev), K.bn_workspace(rows, C)
    y = torch.empty(rows, C, device=dev, dtype=torch.bfloat16)
    mask = torch.full((rows, C // 8), 0xA5, dtype=torch.uint8, device=dev)
    K.bn_forward(z, rows, C, C, ws, mean, rstd, gamma, beta, y, C, relu=True, res=res, rcs=C, mask=mask)
    y2 = torch.empty_like(y)
    K.bn_forward(z, rows, C, C, ws, mean, rstd, gamma, beta, y2, C, relu=True, res=res, rcs=C)
    assert torch.equal(y, y2)
    bits = (y.view(rows, C // 8, 8) > 0).to(torch.int32) << torch.arange(8, device=dev, dtype=torch.int32)
    assert torch.equal(bits.sum(-1).to(torch.uint8), mask)
    dy = torch.randn(rows, C, device=dev, generator=g).bfloat16()
    outs = []
    for use_mask in (False, True):
        dg, db = torch.empty(C, device=dev), torch.empty(C, device=dev)
        dx, dres = torch.empty_like(z), torch.empty_like(z)
        K.bn_backward(dy, C, z, C, rows, C, mean, rstd, gamma, beta, ws, dg, db, relu=True,
                      y=None if use_mask else y, ycs=C, dx=dx, dxcs=C, dz_out=dres, mask=mask if use_mask else None)
        outs.append((dg, db, dx, dres))
    for a, b in zip(*outs):
        assert torch.equal(a, b)
