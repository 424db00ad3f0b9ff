"""Layer-composition parity with identical inputs (no upstream trajectory divergence):
one ConvBN layer, one residual BasicBlock (identity and downsample) and one Linear layer,
forward and backward, GPU kernels vs the bf16-emulating CPU restatement."""
import pytest
import torch

from oracle.cnn_ref import RefModel
from paper_2103_16898_b200 import nets

pytestmark = pytest.mark.gpu


def rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-12)).item()


def nchw(t):
    return t.float().cpu().permute(0, 3, 1, 2)


def nhwc(t):
    return t.permute(0, 2, 3, 1)


@pytest.mark.parametrize("cin,cout,stride,n,h", [(64, 64, 1, 32, 16), (64, 128, 2, 32, 16), (128, 128, 1, 16, 8)])
def test_basic_block(cin, cout, stride, n, h):
    g = torch.Generator().manual_seed(cin + cout + stride)
    ps, S = nets.ParamStore(), nets.Scratch()
    blk = nets.BasicBlock(ps, "b", cin, cout, stride, g)
    oh, ow = blk.build(n, h, h, S, "cuda")
    S.finalize("cuda")
    ps.finalize("cuda")
    x = torch.randn(n, h, h, cin, generator=g).bfloat16()
    dout = torch.randn(n, oh, ow, cout, generator=g).bfloat16()
    xd, out = x.cuda(), torch.empty(n, oh, ow, cout, dtype=torch.bfloat16, device="cuda")
    dx = torch.empty_like(xd)
    blk.forward(ps, xd, out)
    blk.backward(ps, dout.cuda(), xd, out, dx)
    torch.cuda.synchronize()

    ref = RefModel(ps.state_cpu())
    xr = nchw(x).requires_grad_(True)
    o1 = ref.conv_bn(xr, "b.conv1", stride, 1)
    sc = xr
    if blk.down is not None:
        sc = ref.conv_bn(xr, "b.down", stride, 0, relu=False)
    y = ref.conv_bn(o1, "b.conv2", 1, 1, res=sc)
    y.backward(nchw(dout))
    assert rel(nchw(out), y.detach()) < 1e-2
    assert rel(nchw(dx), xr.grad) < 3e-2
    for k, p in ref.params.items():
        name = k.replace("__", ".")
        assert rel(ps.g[name].cpu(), p.grad) < 5e-2, (name, rel(ps.g[name].cpu(), p.grad))


def test_dense_block_and_transition():
    """3 DenseNet layers on a 64-channel block input + a transition, identical inputs."""
    g = torch.Generator().manual_seed(5)
    n, h, w, c0, gr = 8, 8, 8, 64, 32
    ps, S = nets.ParamStore(), nets.Scratch()
    layers = [nets.DenseLayer(ps, f"b.l{i}", c0 + i * gr, gr, 4, g) for i in range(3)]
    c1 = c0 + 3 * gr
    tbn = nets.BNAct(ps, "t.norm", c1)
    tconv = nets.Conv(ps, "t.conv", c1, c1 // 2, 1, 1, 0, g)
    for L in layers:
        L.build(n, h, w, S, "cuda")
    tbn.build(n * h * w, S, "cuda")
    tconv.build(n, h, w, S)
    S.finalize("cuda")
    ps.finalize("cuda")
    e = lambda *s: torch.empty(*s, dtype=torch.bfloat16, device="cuda")  # noqa: E731
    x0 = torch.randn(n, h, w, c0, generator=g).bfloat16()
    blk = torch.zeros(n, h, w, c1, dtype=torch.bfloat16, device="cuda")
    blk[..., :c0] = x0.cuda()
    from paper_2103_16898_b200 import kernels as K

    bm, br = torch.zeros(c1, device="cuda"), torch.zeros(c1, device="cuda")
    for L in layers:
        L.bn1.use_stats(bm[:L.cin], br[:L.cin])
        L.slice_stats = (bm[L.cin:L.cin + gr], br[L.cin:L.cin + gr])
    tbn.use_stats(bm, br)
    K.bn_stats(blk, n * h * w, c0, c1, S.bnws, bm[:c0], br[:c0])
    y1, y2 = e(n * h * w * c1), e(n * h * w * 128)
    for L in layers:
        L.forward(ps, blk, y1[:n * h * w * L.cin].view(n, h, w, L.cin), y2.view(n, h, w, 128))
    y = e(n, h, w, c1)
    tbn.forward(ps, blk, c1, y, c1)
    t = e(n, h, w, c1 // 2)
    tconv.forward(ps, y, t)
    dt = torch.randn(n, h, w, c1 // 2, generator=g).bfloat16()
    dblk = torch.empty(n, h, w, c1, dtype=torch.float32, device="cuda")
    dy = e(n, h, w, c1)
    tconv.backward(ps, dt.cuda(), y, dx=dy)
    tbn.backward(ps, dy, c1, blk, c1, dblk, c1, accumulate=False)
    dz2, dy2, dz1, dy1 = e(n * h * w * gr), e(n * h * w * 128), e(n * h * w * 128), e(n * h * w * c1)
    for L in reversed(layers):
        L.backward(ps, blk, dblk, y1[:n * h * w * L.cin].view(n, h, w, L.cin), y2.view(n, h, w, 128),
                   dz2.view(n, h, w, gr), dy2.view(n, h, w, 128), dz1.view(n, h, w, 128),
                   dy1[:n * h * w * L.cin].view(n, h, w, L.cin))
    torch.cuda.synchronize()

    from oracle.cnn_ref import DenseNet121Ref
    ref = DenseNet121Ref(ps.state_cpu())
    xr = nchw(x0).requires_grad_(True)
    feats = [xr]
    for i, L in enumerate(layers):
        cat = torch.cat(feats, 1)
        yy1 = ref.bn_relu(cat, f"b.l{i}.norm1")
        z1 = ref.conv(yy1, f"b.l{i}.conv1", 1, 0)
        yy2 = ref.bn_relu(z1, f"b.l{i}.norm2")
        feats.append(ref.conv(yy2, f"b.l{i}.conv2", 1, 1))
    cat = torch.cat(feats, 1)
    tt = ref.conv(ref.bn_relu(cat, "t.norm"), "t.conv", 1, 0)
    assert rel(nchw(blk), cat.detach()) < 1e-2
    assert rel(nchw(t), tt.detach()) < 1e-2
    tt.backward(nchw(dt))
    assert rel(nchw(dblk[..., :c0]), xr.grad) < 3e-2, rel(nchw(dblk[..., :c0]), xr.grad)
    for k, p in ref.params.items():
        name = k.replace("__", ".")
        assert rel(ps.g[name].cpu(), p.grad) < 5e-2, (name, rel(ps.g[name].cpu(), p.grad))


def test_linear_layer():
    g = torch.Generator().manual_seed(3)
    ps, S = nets.ParamStore(), nets.Scratch()
    lin = nets.Linear(ps, "fc", 512, 10, g)
    lin.build(64, S)
    S.finalize("cuda")
    ps.finalize("cuda")
    x = torch.randn(64, 512, generator=g).bfloat16().cuda()
    y = torch.empty(64, 16, device="cuda")
    lin.forward(ps, x, y, out_f32=True)
    dy = torch.randn(64, 16, generator=g).bfloat16()
    dy[:, 10:] = 0
    dx = torch.empty_like(x)
    lin.backward(ps, dy.cuda(), x, dx)
    W, b = ps.p["fc.w"], ps.p["fc.b"]
    Wb = W.bfloat16().float()
    assert rel(y, x.float() @ Wb.t() + b) < 1e-5
    assert rel(ps.g["fc.w"], dy.cuda().float().t() @ x.float()) < 1e-5
    assert rel(ps.g["fc.b"], dy.cuda().float().sum(0)) < 1e-5
    assert rel(dx, dy.cuda().float() @ Wb) < 4e-3
