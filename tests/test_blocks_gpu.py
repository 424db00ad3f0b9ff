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
