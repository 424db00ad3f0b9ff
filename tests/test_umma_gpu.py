"""tcgen05 implicit-GEMM engine vs a torch fp32 reference of the same op (bf16-rounded
operands, fp32 accumulation on both sides; tolerance 2e-3 relative to the output scale)."""
import pytest
import torch
import torch.nn.functional as F

from paper_2103_16898_b200 import kernels as K

pytestmark = pytest.mark.gpu
TOL = 2e-3


def _close(got, want, tol=TOL):
    got, want = got.float(), want.float()
    scale = want.abs().max().item() + 1e-6
    err = (got - want).abs().max().item()
    assert err <= tol * scale, f"max err {err:.3e} vs scale {scale:.3e}"


def _ref_conv(x, w, stride, pad):
    # x NHWC bf16, w [co,kh,kw,ci] -> NHWC fp32
    y = F.conv2d(x.permute(0, 3, 1, 2).float(), w.permute(0, 3, 1, 2).float(), stride=stride, padding=pad)
    return y.permute(0, 2, 3, 1)


CONV_CASES = [
    # n, h, w, cin, cout, k, stride, pad
    (2, 32, 32, 8, 32, 3, 1, 1),
    (2, 32, 32, 32, 32, 3, 1, 1),
    (2, 16, 16, 32, 64, 3, 1, 1),
    (3, 16, 16, 64, 64, 3, 1, 1),
    (4, 8, 8, 64, 128, 3, 2, 1),
    (4, 8, 8, 64, 128, 1, 2, 0),
    (2, 14, 14, 96, 128, 1, 1, 0),
    (3, 7, 7, 128, 32, 3, 1, 1),
    (2, 28, 28, 16, 48, 3, 1, 1),
    (1, 56, 56, 8, 64, 7, 2, 3),
    (8, 4, 4, 256, 512, 3, 1, 1),
    (2, 32, 32, 64, 256, 3, 1, 1),
    (4, 32, 32, 64, 64, 3, 1, 1),      # kh-paired wgrad (Cout 64): ResNet-18 stage-1 geometry
    (2, 24, 48, 64, 64, 3, 1, 1),
    # CTA-pair (cta_group::2) gathered convs: ResNet-18 stage 2-4 geometries, the stride-2
    # downsample, and an odd number of M tiles (single-CTA fallback)
    (4, 16, 16, 128, 128, 3, 1, 1),
    (4, 8, 8, 256, 256, 3, 1, 1),
    (16, 4, 4, 512, 512, 3, 1, 1),
    (8, 16, 16, 64, 128, 3, 2, 1),
    (5, 8, 8, 128, 128, 3, 1, 1),
    # halo weight gradients over several 64-channel groups (N tile = (kh, group)): DenseNet's
    # 128 -> 32 conv2, a 192-channel input with Cout 64 (no kh pairing)
    (2, 28, 28, 128, 32, 3, 1, 1),
    (2, 16, 16, 192, 64, 3, 1, 1),
    (3, 32, 32, 64, 32, 3, 1, 1),      # kh-quad packing with one input group
    (2, 16, 16, 16, 32, 3, 1, 1),      # 16-channel input as zero-padded 64-channel rows
    (3, 16, 16, 8, 32, 3, 1, 1),       # ... and an 8-channel (padded RGB) input, kh-quad
    # halo conv with streamed weights (wide stride-1 3x3): CTA pair, single-CTA (odd tile
    # count), 256 output channels, 192-channel input
    (3, 16, 8, 128, 128, 3, 1, 1),
    (2, 32, 16, 128, 256, 3, 1, 1),
    (2, 16, 16, 192, 64, 3, 1, 1),
    # 1x1 stride-1 convs as plain row GEMMs: DenseNet widths, a partial last row tile, 32 channels
    (2, 56, 56, 64, 128, 1, 1, 0),
    (3, 7, 7, 512, 128, 1, 1, 0),
    (1, 10, 10, 32, 96, 1, 1, 0),
]


@pytest.mark.parametrize("n,h,w,cin,cout,k,s,p", CONV_CASES)
def test_conv_fwd(n, h, w, cin, cout, k, s, p):
    g = torch.Generator(device="cuda").manual_seed(n * 1000 + h + cin + cout)
    x = torch.randn(n, h, w, cin, device="cuda", generator=g).to(torch.bfloat16)
    wt = (torch.randn(cout, k, k, cin, device="cuda", generator=g) / (k * k * cin) ** 0.5).to(torch.bfloat16)
    bias = torch.randn(cout, device="cuda", generator=g)
    y = K.conv2d_fwd(x, wt, s, p, bias=bias, out_f32=True)
    _close(y, _ref_conv(x, wt, s, p) + bias)
    yb = K.conv2d_fwd(x, wt, s, p)   # bf16 output path
    _close(yb, _ref_conv(x, wt, s, p), tol=1e-2)


def test_conv_fwd_channel_slices():
    # DenseNet-style: read channels [0,cin) of a wider buffer, write at an offset of another
    x_full = torch.randn(2, 8, 8, 160, device="cuda").to(torch.bfloat16)
    wt = (torch.randn(32, 3, 3, 96, device="cuda") * 0.1).to(torch.bfloat16)
    out = torch.zeros(2, 8, 8, 256, device="cuda", dtype=torch.bfloat16)
    K.conv2d_fwd(x_full, wt, 1, 1, out=out, cin=96, out_coff=64)
    _close(out[..., 64:96], _ref_conv(x_full[..., :96].contiguous(), wt, 1, 1), tol=1e-2)
    assert out[..., :64].abs().max().item() == 0 and out[..., 96:].abs().max().item() == 0


@pytest.mark.parametrize("acc", [False, True])
def test_conv1x1_row_gemm_slices(acc):
    # 1x1 conv (row-GEMM plan) reading channels [0, cin) of a wider buffer and writing / adding
    # at a channel offset of another
    g = torch.Generator(device="cuda").manual_seed(5 + acc)
    x_full = torch.randn(2, 28, 28, 192, device="cuda", generator=g).to(torch.bfloat16)
    wt = (torch.randn(128, 1, 1, 160, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    base = torch.randn(2, 28, 28, 256, device="cuda", generator=g)
    out = base.clone() if acc else torch.zeros_like(base)
    K.conv2d_fwd(x_full, wt, 1, 0, out=out, out_f32=True, cin=160, out_coff=64, accumulate=acc)
    ref = _ref_conv(x_full[..., :160].contiguous(), wt, 1, 0)
    _close(out[..., 64:192] - (base[..., 64:192] if acc else 0), ref)
    want_rest = base if acc else torch.zeros_like(base)
    assert torch.equal(out[..., :64], want_rest[..., :64]) and torch.equal(out[..., 192:], want_rest[..., 192:])


@pytest.mark.parametrize("k,p", [(3, 1), (4, 2)])
def test_conv_fwd_cin32_of_wider_buffer(k, p):
    # 32 input channels read as zero-padded 128-byte rows (h_rowpad): the pad half must be TMA
    # zero fill even when the buffer holds more channels past cin
    g = torch.Generator(device="cuda").manual_seed(31 + k)
    x_full = torch.randn(2, 16, 16, 64, device="cuda", generator=g).to(torch.bfloat16)
    wt = (torch.randn(48, k, k, 32, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    y = K.conv2d_fwd(x_full, wt, 1, p, out_f32=True, cin=32)
    _close(y, _ref_conv(x_full[..., :32].contiguous(), wt, 1, p))


@pytest.mark.parametrize("n,h,w,cin,cout,k,s,p", CONV_CASES)
def test_conv_wgrad(n, h, w, cin, cout, k, s, p):
    g = torch.Generator(device="cuda").manual_seed(7 + n + h + cin + cout)
    x = torch.randn(n, h, w, cin, device="cuda", generator=g).to(torch.bfloat16)
    oh, ow = K.conv_out_hw(h, w, k, s, p)
    dy = torch.randn(n, oh, ow, cout, device="cuda", generator=g).to(torch.bfloat16)
    part, used = K.conv2d_wgrad_partials(dy, x, k, k, s, p)
    dw = part[:used].sum(0).view(cout, k, k, cin)
    xr = x.permute(0, 3, 1, 2).float().requires_grad_(True)
    wr = torch.zeros(cout, cin, k, k, device="cuda", requires_grad=True)
    yr = F.conv2d(xr, wr, stride=s, padding=p)
    yr.backward(dy.permute(0, 3, 1, 2).float())
    _close(dw, wr.grad.permute(0, 2, 3, 1))


@pytest.mark.parametrize("n,h,w,cin,cout,k,s,p", CONV_CASES)
def test_conv_dgrad_via_flipped_conv(n, h, w, cin, cout, k, s, p):
    """dgrad = stride-1 conv of dY (zero-upsampled for stride 2) with flipped weights."""
    g = torch.Generator(device="cuda").manual_seed(11 + n + h + cin + cout)
    wt = (torch.randn(cout, k, k, cin, device="cuda", generator=g) / (k * k * cin) ** 0.5).to(torch.bfloat16)
    oh, ow = K.conv_out_hw(h, w, k, s, p)
    dy = torch.randn(n, oh, ow, cout, device="cuda", generator=g).to(torch.bfloat16)
    flip = torch.empty(cin, k, k, cout, device="cuda", dtype=torch.bfloat16)
    K.weight_flip(wt, flip)
    src = dy
    if s == 2:
        src = torch.empty(n, 2 * oh - 1, 2 * ow - 1, cout, device="cuda", dtype=torch.bfloat16)
        K.zero_upsample(dy, src)
    dx = torch.zeros(n, h, w, cin, device="cuda", dtype=torch.float32)
    K.conv2d_fwd(src, flip, 1, k - 1 - p, out=dx, out_f32=True, out_hw=(h, w))
    xr = torch.zeros(n, cin, h, w, device="cuda", requires_grad=True)
    F.conv2d(xr, wt.permute(0, 3, 1, 2).float(), stride=s, padding=p).backward(dy.permute(0, 3, 1, 2).float())
    _close(dx, xr.grad.permute(0, 2, 3, 1))
    # accumulate mode adds onto the existing output
    base = torch.randn(n, h, w, cin, device="cuda", generator=g)
    acc = base.clone()
    K.conv2d_fwd(src, flip, 1, k - 1 - p, out=acc, out_f32=True, out_hw=(h, w), accumulate=True)
    _close(acc, base + xr.grad.permute(0, 2, 3, 1))


@pytest.mark.parametrize("M,N,Kd,am,bm,splits", [
    (512, 256, 4096, 0, 0, 1), (512, 10, 256, 0, 0, 1), (512, 4096, 256, 0, 1, 1),
    (256, 4096, 512, 1, 1, 4), (10, 256, 512, 1, 1, 2), (300, 200, 136, 0, 0, 1),
])
def test_dense(M, N, Kd, am, bm, splits):
    g = torch.Generator(device="cuda").manual_seed(M + N + Kd)
    A = torch.randn(M, Kd, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(N, Kd, device="cuda", generator=g).to(torch.bfloat16)
    a = A if am == 0 else A.t().contiguous()
    if bm == 1 and N % 8:
        pytest.skip("MN-major operand needs N % 8 == 0")
    b = B if bm == 0 else B.t().contiguous()
    if am == 1 and M % 8:
        pytest.skip("MN-major operand needs M % 8 == 0")
    bias = torch.randn(N, device="cuda", generator=g)
    out = K.gemm(a, b, M, N, Kd, am, bm, out_f32=True, bias=None if splits > 1 else bias, splits=splits)
    want = A.float() @ B.float().t()
    if out.dim() == 3:
        out = out.sum(0)
    else:
        want = want + bias
    _close(out, want)


@pytest.mark.parametrize("n,h,w,cin,cout,k,s,p", [(4, 32, 32, 64, 64, 3, 1, 1), (2, 16, 16, 32, 48, 3, 1, 1),
                                                   (3, 7, 7, 64, 32, 1, 1, 0), (4, 8, 8, 32, 64, 3, 2, 1)])
def test_conv_accumulate_bf16_slice(n, h, w, cin, cout, k, s, p):
    """bf16 accumulate into a channel slice of a wider buffer (the residual / concat
    gradient case): neighbouring channels untouched, slice = old + conv (bf16 rounding)."""
    g = torch.Generator(device="cuda").manual_seed(5 + n + h + cin + cout)
    x = torch.randn(n, h, w, cin, device="cuda", generator=g).to(torch.bfloat16)
    wt = (torch.randn(cout, k, k, cin, device="cuda", generator=g) / (k * k * cin) ** 0.5).to(torch.bfloat16)
    oh, ow = K.conv_out_hw(h, w, k, s, p)
    wide = torch.randn(n, oh, ow, cout + 32, device="cuda", generator=g).to(torch.bfloat16)
    before = wide.clone()
    K.conv2d_fwd(x, wt, s, p, out=wide, out_coff=16, accumulate=True)
    want = before[..., 16:16 + cout].float() + _ref_conv(x, wt, s, p)
    _close(wide[..., 16:16 + cout], want, tol=1e-2)
    assert torch.equal(wide[..., :16], before[..., :16]) and torch.equal(wide[..., 16 + cout:], before[..., 16 + cout:])


@pytest.mark.parametrize("n,h,w,cin,cout,k,p,acc", [(4, 8, 8, 64, 128, 3, 1, False), (4, 8, 8, 64, 128, 1, 0, True),
                                                    (2, 32, 32, 64, 128, 3, 1, True), (8, 16, 16, 128, 256, 3, 1, False),
                                                    (3, 16, 16, 32, 64, 1, 0, True)])
def test_conv_dgrad_stride2_parity_classes(n, h, w, cin, cout, k, p, acc):
    """Stride-2 dgrad as 4 output-parity gather convs of dY (no zero-upsampled copy) vs torch."""
    g = torch.Generator(device="cuda").manual_seed(13 + n + h + cin + cout + k)
    wt = (torch.randn(cout, k, k, cin, device="cuda", generator=g) / (k * k * cin) ** 0.5).to(torch.bfloat16)
    oh, ow = K.conv_out_hw(h, w, k, 2, p)
    dy = torch.randn(n, oh, ow, cout, device="cuda", generator=g).to(torch.bfloat16)
    base = torch.randn(n, h, w, cin, device="cuda", generator=g).to(torch.bfloat16) if acc else \
        torch.full((n, h, w, cin), 7.0, device="cuda", dtype=torch.bfloat16)
    dx = base.clone()
    assert K.conv2d_dgrad_s2(dy, wt, p, dx, accumulate=acc)
    xr = torch.zeros(n, cin, h, w, device="cuda", requires_grad=True)
    F.conv2d(xr, wt.permute(0, 3, 1, 2).float(), stride=2, padding=p).backward(dy.permute(0, 3, 1, 2).float())
    want = xr.grad.permute(0, 2, 3, 1) + (base.float() if acc else 0)
    _close(dx, want, tol=1e-2)


def test_conv_dgrad_stride2_rejects_without_launch():
    # 1x1 stride 2 without accumulate: odd positions have no taps -> refused, dx untouched
    wt = torch.randn(64, 1, 1, 32, device="cuda").to(torch.bfloat16)
    dy = torch.randn(2, 4, 4, 64, device="cuda").to(torch.bfloat16)
    dx = torch.full((2, 8, 8, 32), 3.0, device="cuda", dtype=torch.bfloat16)
    assert not K.conv2d_dgrad_s2(dy, wt, 0, dx, accumulate=False)
    assert (dx == 3.0).all()


def test_dense_narrow_n_tiles_split_k():
    """cvb_gemm_ex with 64-column N tiles + split-K (the FC forward configuration)."""
    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randn(512, 4096, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(256, 4096, device="cuda", generator=g).to(torch.bfloat16)
    out = K.gemm(A, B, 512, 256, 4096, 0, 0, splits=9, max_bn=64)
    _close(out.sum(0), A.float() @ B.float().t())


@pytest.mark.parametrize("cin,cout,k,p", [(64, 128, 3, 1), (128, 256, 1, 0)])
def test_dgrad_s2_with_batched_class_weights(cin, cout, k, p):
    """Stride-2 dgrad with the parity-class weight matrices produced by the batched transpose
    jobs (ParamStore.flip_all's layout) == the dgrad that permutes them itself, bit for bit."""
    g = torch.Generator(device="cuda").manual_seed(cin + cout + k)
    n, h, w = 4, 16, 16
    wt = (torch.randn(cout, k, k, cin, device="cuda", generator=g) / (k * k * cin) ** 0.5).to(torch.bfloat16)
    oh, ow = K.conv_out_hw(h, w, k, 2, p)
    dy = torch.randn(n, oh, ow, cout, device="cuda", generator=g).to(torch.bfloat16)
    acc = k == 1
    dx_ref = torch.zeros(n, h, w, cin, device="cuda", dtype=torch.bfloat16)
    assert K.conv2d_dgrad_s2(dy, wt, p, dx_ref, accumulate=acc)
    desc, coff, taps = [], 0, k * k
    for _, taplist in K.dgrad_s2_classes(k, k, p):
        for t, (y, x) in enumerate(taplist):
            desc += [(y * k + x) * cin, coff + t * cout, cout, cin, taps * cin, len(taplist) * cout]
        coff += cin * len(taplist) * cout
    cw = torch.zeros(wt.numel(), device="cuda", dtype=torch.bfloat16)
    K.transpose_batched(wt.reshape(-1), cw, torch.tensor(desc, dtype=torch.int64, device="cuda"), len(desc) // 6,
                        cout * cin, 0)
    dx = torch.zeros_like(dx_ref)
    assert K.conv2d_dgrad_s2(dy, wt, p, dx, accumulate=acc, wscratch=cw, class_weights_ready=True)
    assert torch.equal(dx, dx_ref)


@pytest.mark.parametrize("n,h,cin,cout", [(8, 32, 64, 128), (8, 16, 128, 256), (16, 8, 256, 512), (4, 32, 32, 64)])
@pytest.mark.parametrize("acc", [False, True])
def test_dgrad_s2_rows_matches_torch(n, h, cin, cout, acc):
    """3x3 pad-1 stride-2 dgrad as two row-parity convs (cvb_conv2d_dgrad_s2_rows, weights from
    the batched transpose jobs) vs the fp32 transposed convolution; accumulate adds into dx."""
    g = torch.Generator(device="cuda").manual_seed(n + h + cin + cout)
    wt = (torch.randn(cout, 3, 3, cin, device="cuda", generator=g) / (9 * cin) ** 0.5).to(torch.bfloat16)
    oh = h // 2
    dy = torch.randn(n, oh, oh, cout, device="cuda", generator=g).to(torch.bfloat16)
    wrows = torch.zeros(12 * cin * cout, device="cuda", dtype=torch.bfloat16)
    desc = K.dgrad_s2_row_jobs(0, 3, 3, cin, cout, 1, 0)
    K.transpose_batched(wt.reshape(-1), wrows, torch.tensor(desc, dtype=torch.int64, device="cuda"), len(desc) // 6,
                        cout * cin, 0)
    base = torch.randn(n, h, h, cin, device="cuda", generator=g).to(torch.bfloat16)
    dx = base.clone() if acc else torch.zeros_like(base)
    assert K.conv2d_dgrad_s2_rows(dy, wrows, cin, dx, accumulate=acc)
    ref = torch.nn.functional.conv_transpose2d(dy.permute(0, 3, 1, 2).float(), wt.permute(0, 3, 1, 2).float(),
                                               stride=2, padding=1, output_padding=1).permute(0, 2, 3, 1)
    if acc:
        ref = ref + base.float()
    err = (dx.float() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 8e-3, err
    # against the four-class form on the same inputs (same products, other summation order)
    dxc = base.clone() if acc else torch.zeros_like(base)
    assert K.conv2d_dgrad_s2(dy, wt, 1, dxc, accumulate=acc)
    assert (dx.float() - dxc.float()).abs().max().item() / ref.abs().max().item() < 8e-3
