"""Torch-tensor front end of the sm_100a kernels (no compute here, only argument plumbing).

Every function launches one or more of the library's CUDA kernels on the current torch
stream.  Activations are NHWC bf16; weights are bf16 [Cout][KH][KW][Cin] (K-major);
gradients and optimiser state are fp32.  There is no fallback: a missing library raises.
"""
from __future__ import annotations

import ctypes
import os
import sys

import torch

from . import _lib

BF16 = torch.bfloat16
F32 = torch.float32


class Recorder:
    """Launch accounting: counts every kernel this module launches and, when `timing` is on,
    brackets each call with CUDA events on the launching stream and records its algorithmic
    FLOPs / bytes (bench.py uses it for the roofline of the dominant kernel)."""

    def __init__(self):
        self.launches = 0
        self.timing = False
        self.records = []   # (kind, flops, bytes, ev_start, ev_end)

    def begin(self, n_kernels, kind, flops=0, nbytes=0):
        self.launches += n_kernels
        if not self.timing:
            return None
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()
        f1, f2 = sys._getframe(1), sys._getframe(2)   # kernel wrapper, and the layer that called it
        site = f"{f1.f_code.co_name}<-{f2.f_code.co_name}:{f2.f_lineno}"
        return (kind, flops, nbytes, e0, site)

    def end(self, tok):
        if tok is None:
            return
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        self.records.append((*tok[:4], e1, tok[4]))

    def summary(self):
        """{kind: [calls, ms, flops, bytes]} (call after a synchronize)."""
        out = {}
        for kind, fl, nb, e0, e1, _ in self.records:
            c = out.setdefault(kind, [0, 0.0, 0, 0])
            c[0] += 1
            c[1] += e0.elapsed_time(e1)
            c[2] += fl
            c[3] += nb
        return out

    def per_launch(self):
        """[(site, kind, ms, flops, bytes)] in launch order (call after a synchronize)."""
        return [(site, kind, e0.elapsed_time(e1), fl, nb) for kind, fl, nb, e0, e1, site in self.records]


REC = Recorder()
_UNFUSED_BN = bool(os.environ.get("CVB_BN_UNFUSED"))   # A/B switch: three-kernel BN


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


# launch entry point -> kernel class (the roofline / per-class timing vocabulary of bench.py)
LAUNCH_CLASS = {
    **{n: "umma_gemm" for n in ("cvb_conv2d_dgrad_s2_rows", "cvb_conv2d_fwd", "cvb_conv2d_wgrad", "cvb_gemm", "cvb_gemm_ex",
                                "cvb_conv2d_dgrad_s2")},
    **{n: "bn" for n in ("cvb_bn_stats", "cvb_bn_forward", "cvb_bn_forward_range", "cvb_bn_apply", "cvb_bn_backward",
                         "cvb_bn_backward_fused", "cvb_bn_gather_dx", "cvb_bn_forward_mask",
                         "cvb_bn_backward_fused_mask")},
    **{n: "pool" for n in ("cvb_maxpool_fwd", "cvb_maxpool_fwd_idx", "cvb_maxpool_bwd", "cvb_maxpool_bwd_idx",
                           "cvb_avgpool_fwd", "cvb_avgpool_bwd", "cvb_gap_fwd", "cvb_gap_bwd")},
    **{n: "head" for n in ("cvb_softmax_xent", "cvb_head_train")},
    **{n: "reduce" for n in ("cvb_reduce_splits", "cvb_reduce_splits_act", "cvb_col_sum")},
    **{n: "layout" for n in ("cvb_weight_flip", "cvb_weight_flip_batched", "cvb_transpose_batched",
                             "cvb_space_to_depth2", "cvb_s2d_weights",
                             "cvb_s2d_weights_grad", "cvb_zero_upsample", "cvb_cast_rows", "cvb_cast_f32_bf16")},
    **{n: "eltwise" for n in ("cvb_relu_fwd", "cvb_relu_bwd")},
    **{n: "optimizer" for n in ("cvb_adam_step", "cvb_sgd_step")},
    "cvb_verdict_snapshot": "verdict",
}
# Measurement only (bench.py): when set to a set of class names, launches of every other class
# become no-ops, so a CUDA graph captured under the filter replays exactly that class's
# kernels of a step -- their in-graph time without the rest of the step in between.
ONLY_CLASSES = None
# Measurement only (scripts/graph_layer_times.py): with ONLY_CLASSES set, keep just the
# ONLY_INDEX-th launch call of the kept classes (ONLY_SEEN counts and names the calls).
ONLY_INDEX = None
ONLY_SEEN = []


class _ClassFilter:
    def __init__(self, lib, keep):
        self._lib, self._keep = lib, keep

    def __getattr__(self, name):
        cls = LAUNCH_CLASS.get(name)
        if cls is None:
            return getattr(self._lib, name)
        if cls in self._keep:
            if ONLY_INDEX is None:
                return getattr(self._lib, name)
            ONLY_SEEN.append(name)
            if len(ONLY_SEEN) - 1 == ONLY_INDEX:
                return getattr(self._lib, name)
        return lambda *args: 0


def _lib_bound():
    _lib.bind_device()
    if ONLY_CLASSES is not None:
        return _ClassFilter(_lib.load(), ONLY_CLASSES)
    return _lib.load()


def conv_out_hw(h, w, k, stride, pad):
    return (h + 2 * pad - k) // stride + 1, (w + 2 * pad - k) // stride + 1


def conv2d_fwd(x, w, stride=1, pad=0, bias=None, out=None, out_f32=False, cin=None, out_coff=0, out_hw=None,
               accumulate=False, acct_flops=None, kind="umma_gemm"):
    """x: [N,H,W,Cs] bf16 (channels [0,cin) used, stride Cs); w: [Cout,KH,KW,cin] bf16.

    Returns y [N,OH,OW,Cout] (or writes into `out` at channel offset out_coff; adds into it
    when accumulate).  out_hw overrides the output extent (transposed-conv dgrad)."""
    lib = _lib_bound()
    n, h, wd, cs = x.shape
    cin = cs if cin is None else cin
    cout, kh, kw, wc = w.shape
    assert wc == cin and x.stride(-1) == 1 and w.is_contiguous()
    oh, ow = conv_out_hw(h, wd, kh, stride, pad) if out_hw is None else out_hw
    if out is None:
        out = torch.empty((n, oh, ow, cout), dtype=F32 if out_f32 else BF16, device=x.device)
    ycs = out.shape[-1]
    assert out.shape[:3] == (n, oh, ow) and (out.dtype == F32) == bool(out_f32)
    flops = acct_flops if acct_flops is not None else 2 * n * oh * ow * cout * kh * kw * cin
    # algorithmic bytes: input and weights read once, output written once (+ read when accumulating)
    nbytes = 2 * (n * h * wd * cin + w.numel()) + n * oh * ow * cout * out.element_size() * (2 if accumulate else 1)
    tok = REC.begin(1, kind, flops, nbytes)
    rc = lib.cvb_conv2d_fwd(x.data_ptr(), n, h, wd, cin, x.stride(2), w.data_ptr(), cout, kh, kw, stride, pad,
                            out.data_ptr(), oh, ow, ycs, out_coff, _ptr(bias), int(out_f32), int(accumulate),
                            _stream())
    REC.end(tok)
    _lib.check(rc, "conv2d_fwd")
    return out


def conv2d_dgrad_s2(dy, w, pad, dx, accumulate=False, wscratch=None, acct_flops=None, class_weights_ready=False):
    """dX of a stride-2 conv by output-parity classes (csrc/umma_gemm.cu).  Returns False,
    launching nothing, when the geometry is unsupported (caller uses the upsampled form).
    class_weights_ready: wscratch already holds the parity-class weight matrices (written by
    ParamStore.flip_all's batched transposes), so no permutation launch runs here."""
    n, oh, ow, cout = dy.shape
    cout_w, kh, kw, cin = w.shape
    _, h, wd, dcs = dx.shape
    assert cout_w == cout and w.is_contiguous() and dx.dtype == BF16
    if wscratch is None:
        assert not class_weights_ready
        wscratch = torch.empty(w.numel(), dtype=BF16, device=w.device)
    w_src = None if class_weights_ready else w
    lib = _lib_bound()
    nbytes = 2 * (dy.numel() + w.numel() + n * h * wd * cin * (2 if accumulate else 1))
    tok = REC.begin(5, "umma_gemm", acct_flops if acct_flops is not None else 2 * n * oh * ow * cout * kh * kw * cin,
                    nbytes)
    rc = lib.cvb_conv2d_dgrad_s2(dy.data_ptr(), n, oh, ow, cout, dy.stride(2), _ptr(w_src), cin, kh, kw, pad,
                                 dx.data_ptr(), h, wd, dx.stride(2), int(accumulate), wscratch.data_ptr(), _stream())
    REC.end(tok)
    if rc == -1:
        return False
    _lib.check(rc, "conv2d_dgrad_s2")
    return True


# cvb_conv2d_dgrad_s2_rows: the dY taps (dh, dw) of the two row-parity convs (3x3, pad 1)
DGRAD_S2_ROW_TAPS = ([(0, 0), (0, 1)], [(0, 0), (0, 1), (1, 0), (1, 1)])


def dgrad_s2_row_jobs(w_off, kh, kw, cin, cout, pad, dst_off):
    """Transpose jobs {src, dst, rows, cols, src ld, dst ld} writing the row-parity weight
    matrices of cvb_conv2d_dgrad_s2_rows (rows (b, ci) of tap (dh, dw) = w[co][a + pad - 2dh]
    [b + pad - 2dw][ci]) from w [cout][kh][kw][cin] at w_off into a ZEROED buffer at dst_off
    (12 * cin * cout elements; taps that do not exist stay zero)."""
    jobs, off = [], dst_off
    for a, taps in enumerate(DGRAD_S2_ROW_TAPS):
        nt = len(taps)
        for t, (dh, dw) in enumerate(taps):
            for b in (0, 1):
                y, x = a + pad - 2 * dh, b + pad - 2 * dw
                if 0 <= y < kh and 0 <= x < kw:
                    jobs += [w_off + (y * kw + x) * cin, off + b * cin * nt * cout + t * cout, cout, cin,
                             kh * kw * cin, nt * cout]
        off += 2 * cin * nt * cout
    return jobs


def conv2d_dgrad_s2_rows(dy, wrows, cin, dx, accumulate=False, acct_flops=None):
    """dX of a 3x3 pad-1 stride-2 conv as two row-parity gather convs (csrc/umma_gemm.cu
    cvb_conv2d_dgrad_s2_rows) from the weights dgrad_s2_row_jobs wrote.  Returns False,
    launching nothing, when dx is not [n][2oh][2ow][cin] contiguous."""
    n, oh, ow, cout = dy.shape
    _, h, wd, dcs = dx.shape
    nbytes = 2 * (dy.numel() + 9 * cin * cout + n * h * wd * cin * (2 if accumulate else 1))
    tok = REC.begin(2, "umma_gemm", acct_flops if acct_flops is not None else 2 * n * h * wd * cout * 9 * cin // 4,
                    nbytes)
    rc = _lib_bound().cvb_conv2d_dgrad_s2_rows(dy.data_ptr(), n, oh, ow, cout, dy.stride(2), cin, dx.data_ptr(), h, wd,
                                               dx.stride(2), int(accumulate), wrows.data_ptr(), _stream())
    REC.end(tok)
    if rc == -1:
        return False
    _lib.check(rc, "conv2d_dgrad_s2_rows")
    return True


def conv2d_wgrad_partials(dy, x, kh, kw, stride, pad, cin=None, max_splits=148, part=None, acct_flops=None):
    """fp32 partial weight gradients [splits, Cout, KH*KW*cin]; returns (part, splits)."""
    lib = _lib_bound()
    n, oh, ow, cout = dy.shape
    _, h, wd, cs = x.shape
    cin = cs if cin is None else cin
    ncols = kh * kw * cin
    if part is None:
        part = torch.empty((max_splits, cout, ncols), dtype=F32, device=dy.device)
    used = ctypes.c_int(0)
    flops = acct_flops if acct_flops is not None else 2 * n * oh * ow * cout * ncols
    nbytes = 2 * (dy.numel() + n * h * wd * cin) + 4 * cout * ncols   # dY, X read once; dW (fp32) written once
    tok = REC.begin(1, "umma_gemm", flops, nbytes)
    rc = lib.cvb_conv2d_wgrad(dy.data_ptr(), n, oh, ow, cout, dy.stride(2), x.data_ptr(), h, wd, cin, x.stride(2),
                              kh, kw, stride, pad, part.data_ptr(), min(max_splits, part.shape[0]),
                              ctypes.byref(used), _stream())
    REC.end(tok)
    _lib.check(rc, "conv2d_wgrad")
    return part, used.value


def splits_used(K, splits):
    return _lib_bound().cvb_gemm_splits_used(K, splits)


def gemm(a, b, M, N, K, a_major=0, b_major=0, out=None, out_f32=False, bias=None, splits=1, accumulate=False,
         acct_flops=None, max_bn=256):
    """C[M,N] = sum_k A(m,k) B(n,k) with A [M,K] (a_major 0) or [K,M] (1), B [N,K] (0) or [K,N] (1)."""
    lib = _lib_bound()
    used = lib.cvb_gemm_splits_used(K, splits)
    if out is None:
        if used > 1:
            out = torch.empty((used, M, N), dtype=F32, device=a.device)
        else:
            out = torch.empty((M, N), dtype=F32 if out_f32 else BF16, device=a.device)
    nbytes = 2 * (M * K + N * K) + M * N * (4 if (out_f32 or used > 1) else 2)   # A, B once; C once
    tok = REC.begin(1, "umma_gemm", acct_flops if acct_flops is not None else 2 * M * N * K, nbytes)
    rc = lib.cvb_gemm_ex(a.data_ptr(), a_major, a.stride(0), b.data_ptr(), b_major, b.stride(0), M, N, K,
                         out.data_ptr(), out.stride(-2), int(out_f32 or used > 1), _ptr(bias), splits, int(accumulate),
                         max_bn, _stream())
    REC.end(tok)
    _lib.check(rc, "gemm")
    return out


# ---------------------------------------------------------------------------------------
# memory-bound kernels (csrc/nn.cu); `nbytes` = algorithmic HBM bytes (reads + writes)
# ---------------------------------------------------------------------------------------
def bn_workspace(rows, C, device="cuda"):
    n = _lib_bound().cvb_bn_workspace_floats(rows, C)
    return torch.empty(max(1, n), dtype=F32, device=device)


def bn_stats(x, rows, C, xcs, ws, mean, rstd, eps=1e-5, run_mean=None, run_var=None, momentum=0.1):
    tok = REC.begin(2 if _UNFUSED_BN else 1, "bn", 0, rows * C * 2)
    if _UNFUSED_BN:
        rc = _lib_bound().cvb_bn_stats(x.data_ptr(), rows, C, xcs, ws.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
                                       eps, _ptr(run_mean), _ptr(run_var), momentum, _stream())
    else:   # single launch, statistics only
        rc = _lib_bound().cvb_bn_forward(x.data_ptr(), rows, C, xcs, ws.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
                                         eps, _ptr(run_mean), _ptr(run_var), momentum, None, None, None, 0, 0, None,
                                         0, 0, _stream())
    REC.end(tok)
    _lib.check(rc, "bn_stats")


def bn_forward(x, rows, C, xcs, ws, mean, rstd, gamma, beta, y, ycs, ycoff=0, relu=True, res=None, rcs=0, eps=1e-5,
               run_mean=None, run_var=None, momentum=0.1, mask=None):
    """Statistics + normalisation (+residual, +ReLU) of one BN layer in a single launch.
    mask (uint8 [rows][C/8]): also write y's ReLU mask bits (for bn_backward(mask=...))."""
    if _UNFUSED_BN:
        if mask is not None:
            raise RuntimeError("bn_forward: the ReLU mask needs the fused BN kernels")
        bn_stats(x, rows, C, xcs, ws, mean, rstd, eps, run_mean, run_var, momentum)
        bn_apply(x, rows, C, xcs, mean, rstd, gamma, beta, y, ycs, ycoff, relu, res, rcs)
        return
    # algorithmic bytes: x (+res) read once, y (+mask) written once (the statistics pass's read of x is traffic)
    tok = REC.begin(1, "bn", 0, rows * C * 2 * (3 if res is not None else 2) + (rows * C // 8 if mask is not None else 0))
    lib = _lib_bound()
    if mask is not None:
        rc = lib.cvb_bn_forward_mask(x.data_ptr(), rows, C, xcs, ws.data_ptr(), mean.data_ptr(), rstd.data_ptr(), eps,
                                     _ptr(run_mean), _ptr(run_var), momentum, gamma.data_ptr(), beta.data_ptr(),
                                     _ptr(res), rcs, int(relu), y.data_ptr(), ycs, ycoff, mask.data_ptr(), _stream())
    else:
        rc = lib.cvb_bn_forward(x.data_ptr(), rows, C, xcs, ws.data_ptr(), mean.data_ptr(), rstd.data_ptr(), eps,
                                _ptr(run_mean), _ptr(run_var), momentum, gamma.data_ptr(), beta.data_ptr(),
                                _ptr(res), rcs, int(relu), y.data_ptr(), ycs, ycoff, _stream())
    REC.end(tok)
    _lib.check(rc, "bn_forward")


def bn_forward_range(x, rows, C, xcs, ws, mean, rstd, gamma, beta, y, ycs, st_off, st_C, ycoff=0, relu=True, eps=1e-5):
    """Batch norm (+ReLU) of all C channels whose statistics are computed here only for channels
    [st_off, st_off + st_C) (the others' mean/rstd are given): one launch."""
    tok = REC.begin(1, "bn", 0, rows * (C * 4 + st_C * 2))
    rc = _lib_bound().cvb_bn_forward_range(x.data_ptr(), rows, C, xcs, ws.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
                                           eps, None, None, 0.0, gamma.data_ptr(), beta.data_ptr(), None, 0, int(relu),
                                           y.data_ptr(), ycs, ycoff, st_off, st_C, _stream())
    REC.end(tok)
    _lib.check(rc, "bn_forward_range")


def bn_apply(x, rows, C, xcs, mean, rstd, gamma, beta, y, ycs, ycoff=0, relu=True, res=None, rcs=0):
    tok = REC.begin(1, "bn", 0, rows * C * 2 * (3 if res is not None else 2))
    rc = _lib_bound().cvb_bn_apply(x.data_ptr(), rows, C, xcs, mean.data_ptr(), rstd.data_ptr(), gamma.data_ptr(),
                                   beta.data_ptr(), _ptr(res), rcs, int(relu), y.data_ptr(), ycs, ycoff, _stream())
    REC.end(tok)
    _lib.check(rc, "bn_apply")


def bn_backward(dy, dycs, x, xcs, rows, C, mean, rstd, gamma, beta, ws, dgamma, dbeta, relu=True, y=None, ycs=0,
                dx=None, dxcs=0, dx32=None, accum32=False, dz_out=None, mask=None):
    # algorithmic bytes: dy, x (, y) read once, dz (bf16) and dx written once -- dx as bf16, fp32, or fp32
    # read-modify-write when accumulating. The kernel's second pass re-reads its inputs (mostly from L2);
    # those re-reads are traffic, not algorithmic bytes.
    dx_b = 8 if (dx32 is not None and accum32) else 4 if dx32 is not None else 2 if dx is not None else 0
    nb = rows * C * (2 * (3 if y is not None else 2) + (2 if dz_out is not None else 0) + dx_b)
    if mask is not None:   # the ReLU mask of y (bn_forward(mask=...)) in place of y
        if _UNFUSED_BN:
            raise RuntimeError("bn_backward: the ReLU mask needs the fused BN kernels")
        tok = REC.begin(1, "bn", 0, nb + rows * C // 8)
        rc = _lib_bound().cvb_bn_backward_fused_mask(
            dy.data_ptr(), dycs, x.data_ptr(), xcs, mask.data_ptr(), rows, C, mean.data_ptr(), rstd.data_ptr(),
            gamma.data_ptr(), beta.data_ptr(), int(relu), ws.data_ptr(), dgamma.data_ptr(), dbeta.data_ptr(),
            _ptr(dx), dxcs, _ptr(dx32), int(accum32), _ptr(dz_out), _stream())
        REC.end(tok)
        _lib.check(rc, "bn_backward_mask")
        return
    fn = _lib_bound().cvb_bn_backward if _UNFUSED_BN else _lib_bound().cvb_bn_backward_fused
    tok = REC.begin((3 if (dx is not None or dx32 is not None) else 2) if _UNFUSED_BN else 1, "bn", 0, nb)
    rc = fn(dy.data_ptr(), dycs, x.data_ptr(), xcs, _ptr(y), ycs, rows, C, mean.data_ptr(),
                                      rstd.data_ptr(), gamma.data_ptr(), beta.data_ptr(), int(relu), ws.data_ptr(),
                                      dgamma.data_ptr(), dbeta.data_ptr(), _ptr(dx), dxcs, _ptr(dx32), int(accum32),
                                      _ptr(dz_out), _stream())
    REC.end(tok)
    _lib.check(rc, "bn_backward")


def bn_gather_dx(x, xcs, rows, nc, mean, rstd, layers, out, ocs, base=None, bcs=0):
    """DenseNet deferred BN input gradient over nc channels (csrc/bn_fused.cu bn_gather_dx).

    layers: [(dy, dycs, gamma, beta, dgamma, dbeta)] in summation order, every tensor already
    sliced to the range's first channel; out bf16 or fp32 (may alias base)."""
    nl = len(layers)
    P = ctypes.c_void_p * max(1, nl)
    I = ctypes.c_int * max(1, nl)
    dy = P(*[t[0].data_ptr() for t in layers])
    dycs = I(*[t[1] for t in layers])
    ga, be, dg, db = (P(*[t[i].data_ptr() for t in layers]) for i in (2, 3, 4, 5))
    out_f32 = out.dtype == F32
    nb = rows * nc * (2 + (4 if base is not None else 0) + (4 if out_f32 else 2) + 2 * nl)
    tok = REC.begin(1, "bn", 0, nb)
    rc = _lib_bound().cvb_bn_gather_dx(x.data_ptr(), xcs, rows, nc, mean.data_ptr(), rstd.data_ptr(), _ptr(base), bcs,
                                       nl, dy, dycs, ga, be, dg, db, out.data_ptr(), ocs, int(out_f32), _stream())
    REC.end(tok)
    _lib.check(rc, "bn_gather_dx")


def maxpool_fwd(x, k, s, p, y, idx=None):
    """idx (uint8 [n][oh][ow][C], optional): keep the window arg-max for maxpool_bwd."""
    n, h, w, c = x.shape
    _, oh, ow, _ = y.shape
    tok = REC.begin(1, "pool", 0, (x.numel() + y.numel()) * 2 + (idx.numel() if idx is not None else 0))
    if idx is not None:
        rc = _lib_bound().cvb_maxpool_fwd_idx(x.data_ptr(), n, h, w, c, k, s, p, y.data_ptr(), oh, ow, y.stride(2),
                                              idx.data_ptr(), _stream())
    else:
        rc = _lib_bound().cvb_maxpool_fwd(x.data_ptr(), n, h, w, c, k, s, p, y.data_ptr(), oh, ow, y.stride(2),
                                          _stream())
    REC.end(tok)
    _lib.check(rc, "maxpool_fwd")


def maxpool_bwd(x, dy, k, s, p, dx, idx=None):
    n, h, w, c = x.shape
    _, oh, ow, _ = dy.shape
    if idx is not None:
        tok = REC.begin(1, "pool", 0, dy.numel() * 2 + idx.numel() + dx.numel() * 2)
        rc = _lib_bound().cvb_maxpool_bwd_idx(idx.data_ptr(), dy.data_ptr(), n, h, w, c, k, s, p, oh, ow,
                                              dx.data_ptr(), _stream())
    else:
        tok = REC.begin(1, "pool", 0, (2 * x.numel() + dy.numel()) * 2)
        rc = _lib_bound().cvb_maxpool_bwd(x.data_ptr(), dy.data_ptr(), n, h, w, c, k, s, p, oh, ow, dx.data_ptr(),
                                          _stream())
    REC.end(tok)
    _lib.check(rc, "maxpool_bwd")


def avgpool_fwd(x, n, h, w, c, xcs, k, y, ycs=None):
    tok = REC.begin(1, "pool", 0, n * h * w * c * 2 * 5 // 4)
    rc = _lib_bound().cvb_avgpool_fwd(x.data_ptr(), n, h, w, c, xcs, k, y.data_ptr(), c if ycs is None else ycs,
                                      _stream())
    REC.end(tok)
    _lib.check(rc, "avgpool_fwd")


def avgpool_bwd(dy, n, h, w, c, k, dx, dxcs):
    tok = REC.begin(1, "pool", 0, n * h * w * c * 2 * 5 // 4)
    rc = _lib_bound().cvb_avgpool_bwd(dy.data_ptr(), n, h, w, c, k, dx.data_ptr(), dxcs, _stream())
    REC.end(tok)
    _lib.check(rc, "avgpool_bwd")


def gap_fwd(x, n, hw, c, xcs, y):
    tok = REC.begin(1, "pool", 0, n * hw * c * 2)
    rc = _lib_bound().cvb_gap_fwd(x.data_ptr(), n, hw, c, xcs, y.data_ptr(), _stream())
    REC.end(tok)
    _lib.check(rc, "gap_fwd")


def gap_bwd(dy, n, hw, c, dx):
    tok = REC.begin(1, "pool", 0, n * hw * c * 2)
    rc = _lib_bound().cvb_gap_bwd(dy.data_ptr(), n, hw, c, dx.data_ptr(), _stream())
    REC.end(tok)
    _lib.check(rc, "gap_bwd")


def softmax_xent(logits, B, C, labels, grad_scale, row_ws, loss_out, dlogits):
    ld = logits.shape[-1]
    assert dlogits.shape[-1] == ld
    tok = REC.begin(1, "head", 0, B * ld * 6)
    rc = _lib_bound().cvb_softmax_xent(logits.data_ptr(), B, C, labels.data_ptr(), grad_scale, row_ws.data_ptr(),
                                       loss_out.data_ptr(), dlogits.data_ptr(), ld, _stream())
    REC.end(tok)
    _lib.check(rc, "softmax_xent")


def head_workspace_floats(B, fin):
    return int(_lib_bound().cvb_head_workspace_floats(B, fin))


def head_train(x, w, bias, labels, B, C, scale, logits, dlogits, row_loss, loss, dw, db, part, dx=None,
               relu_mask=False, dprev_b=None):
    """Fused classifier head (csrc/head.cu): forward + softmax-CE + backward of Linear(fin -> C <= 16)."""
    fin = w.shape[-1]
    nb = (B * x.stride(0) * 2 + w.numel() * 2 + B * 16 * 6 + dw.numel() * 4
          + (B * fin * 2 if dx is not None else 0))
    tok = REC.begin(1, "head", 0, nb)   # CUDA-core kernel: accounted by bytes
    rc = _lib_bound().cvb_head_train(x.data_ptr(), x.stride(0), w.data_ptr(), bias.data_ptr(), labels.data_ptr(), B,
                                     fin, C, scale, int(relu_mask), logits.data_ptr(), dlogits.data_ptr(),
                                     row_loss.data_ptr(), loss.data_ptr(), _ptr(dx),
                                     dx.stride(0) if dx is not None else 0, dw.data_ptr(), db.data_ptr(),
                                     _ptr(dprev_b), part.data_ptr(), _stream())
    REC.end(tok)
    _lib.check(rc, "head_train")


def reduce_splits(part, splits, count, out, accumulate=False, scale=1.0):
    tok = REC.begin(1, "reduce", 0, (splits + 1) * count * 4)
    rc = _lib_bound().cvb_reduce_splits(part.data_ptr(), splits, count, out.data_ptr(), int(accumulate), scale, _stream())
    REC.end(tok)
    _lib.check(rc, "reduce_splits")


def reduce_splits_act(part, splits, rows, cols, out, bias=None, relu=False):
    tok = REC.begin(1, "reduce", 0, (splits * 4 + out.element_size()) * rows * cols)
    rc = _lib_bound().cvb_reduce_splits_act(part.data_ptr(), splits, rows, cols, _ptr(bias), int(relu), out.data_ptr(),
                                            int(out.dtype == F32), out.stride(0), _stream())
    REC.end(tok)
    _lib.check(rc, "reduce_splits_act")


def weight_flip(w, wt):
    cout, kh, kw, cin = w.shape
    tok = REC.begin(1, "layout", 0, w.numel() * 4)
    rc = _lib_bound().cvb_weight_flip(w.data_ptr(), cout, kh, kw, cin, wt.data_ptr(), _stream())
    REC.end(tok)
    _lib.check(rc, "weight_flip")


def weight_flip_batched(pb, fb, desc_dev, nlayers, max_elems, nbytes):
    tok = REC.begin(1, "layout", 0, nbytes)
    rc = _lib_bound().cvb_weight_flip_batched(pb.data_ptr(), fb.data_ptr(), desc_dev.data_ptr(), nlayers, max_elems,
                                              _stream())
    REC.end(tok)
    _lib.check(rc, "weight_flip_batched")


def transpose_batched(src, dst, desc_dev, njobs, max_elems, nbytes):
    """Batched bf16 transposes (csrc/nn.cu transpose_batched): desc rows {src off, dst off, rows,
    cols, src ld, dst ld}."""
    tok = REC.begin(1, "layout", 0, nbytes)
    rc = _lib_bound().cvb_transpose_batched(src.data_ptr(), dst.data_ptr(), desc_dev.data_ptr(), njobs, max_elems,
                                            _stream())
    REC.end(tok)
    _lib.check(rc, "transpose_batched")


def dgrad_s2_classes(kh, kw, pad):
    """Output-parity classes of a stride-2 dgrad: [(class, [(ky, kx) taps])] in the order the
    C-ABI lays out their weight matrices (csrc/umma_gemm.cu cvb_conv2d_dgrad_s2)."""
    out = []
    for c in range(4):
        ph, pw = c >> 1, c & 1
        out.append((c, [(y, x) for y in range(kh) for x in range(kw)
                        if ((y - ph - pad) & 1) == 0 and ((x - pw - pad) & 1) == 0]))
    return out


def space_to_depth2(x, xs):
    n, h, w, c = x.shape
    tok = REC.begin(1, "layout", 0, x.numel() * 4)
    rc = _lib_bound().cvb_space_to_depth2(x.data_ptr(), n, h, w, c, xs.data_ptr(), _stream())
    REC.end(tok)
    _lib.check(rc, "space_to_depth2")


def s2d_weights(w7, ws):
    cout, _, _, c = w7.shape
    tok = REC.begin(1, "layout", 0, ws.numel() * 4)
    rc = _lib_bound().cvb_s2d_weights(w7.data_ptr(), cout, c, ws.data_ptr(), _stream())
    REC.end(tok)
    _lib.check(rc, "s2d_weights")


def s2d_weights_grad(dws, dw7):
    cout, _, _, c = dw7.shape
    tok = REC.begin(1, "layout", 0, dw7.numel() * 8)
    rc = _lib_bound().cvb_s2d_weights_grad(dws.data_ptr(), cout, c, dw7.data_ptr(), _stream())
    REC.end(tok)
    _lib.check(rc, "s2d_weights_grad")


def zero_upsample(dy, out):
    n, oh, ow, c = dy.shape
    tok = REC.begin(1, "layout", 0, (dy.numel() + out.numel()) * 2)
    rc = _lib_bound().cvb_zero_upsample(dy.data_ptr(), n, oh, ow, c, dy.stride(2), out.data_ptr(), _stream())
    REC.end(tok)
    _lib.check(rc, "zero_upsample")


def col_sum(x, rows, cols, ld, out, accumulate=False):
    tok = REC.begin(1, "reduce", 0, rows * cols * x.element_size())
    rc = _lib_bound().cvb_col_sum(x.data_ptr(), int(x.dtype == F32), rows, cols, ld, out.data_ptr(), int(accumulate),
                                  _stream())
    REC.end(tok)
    _lib.check(rc, "col_sum")


def relu_fwd(x):
    tok = REC.begin(1, "eltwise", 0, x.numel() * 4)
    rc = _lib_bound().cvb_relu_fwd(x.data_ptr(), x.numel(), _stream())
    REC.end(tok)
    _lib.check(rc, "relu_fwd")


def relu_bwd(dy, y):
    tok = REC.begin(1, "eltwise", 0, dy.numel() * 6)
    rc = _lib_bound().cvb_relu_bwd(dy.data_ptr(), y.data_ptr(), dy.numel(), _stream())
    REC.end(tok)
    _lib.check(rc, "relu_bwd")


def adam_step(p, g, m, v, pb, lr, b1, b2, eps, step=0, grad_scale=1.0, step_dev=None, sched_dev=None, skip_dev=None):
    if step <= 0 and (sched_dev is None or sched_dev.numel() < 4):
        raise ValueError("adam_step: device-counter mode needs sched_dev with 4 floats (factors + CTA counter)")
    tok = REC.begin(1, "optimizer", 0, p.numel() * (4 * 7 + 2))   # one launch in either mode
    rc = _lib_bound().cvb_adam_step(p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), _ptr(pb), p.numel(), lr, b1,
                                    b2, eps, step, grad_scale, _ptr(step_dev), _ptr(sched_dev), _ptr(skip_dev),
                                    _stream())
    REC.end(tok)
    _lib.check(rc, "adam_step")


def verdict_snapshot(word, slot):
    """slot[0] = 1.0 if the sticky decrypt verdict word is set else 0.0 (one tiny launch)."""
    rc = _lib_bound().cvb_verdict_snapshot(word.data_ptr(), slot.data_ptr(), _stream())
    _lib.check(rc, "verdict_snapshot")


def sgd_step(p, g, buf, pb, lr, momentum=0.0, wd=0.0, grad_scale=1.0, first=False):
    tok = REC.begin(1, "optimizer", 0, p.numel() * (4 * 5 + 2))
    rc = _lib_bound().cvb_sgd_step(p.data_ptr(), g.data_ptr(), buf.data_ptr(), _ptr(pb), p.numel(), lr, momentum, wd,
                                   grad_scale, int(first), _stream())
    REC.end(tok)
    _lib.check(rc, "sgd_step")


def cast_rows(x, ldx, y, ldy, rows, cols):
    tok = REC.begin(1, "layout", 0, rows * cols * 6)
    rc = _lib_bound().cvb_cast_rows(x.data_ptr(), ldx, y.data_ptr(), ldy, rows, cols, _stream())
    REC.end(tok)
    _lib.check(rc, "cast_rows")


def cast_f32_bf16(x, y):
    tok = REC.begin(1, "layout", 0, x.numel() * 6)
    rc = _lib_bound().cvb_cast_f32_bf16(x.data_ptr(), y.data_ptr(), x.numel(), _stream())
    REC.end(tok)
    _lib.check(rc, "cast_f32_bf16")
