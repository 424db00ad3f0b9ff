"""Torch-tensor front end of the sm_100a kernels (no compute here, only argument plumbing).

Every function launches one of the library's CUDA kernels on the current torch stream.
Activations are NHWC bf16; weights are bf16 [Cout][KH][KW][Cin] (K-major); gradients and
optimiser state are fp32.  There is no fallback: a missing library raises.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib

BF16 = torch.bfloat16
F32 = torch.float32


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _lib_bound():
    _lib.bind_device()
    return _lib.load()


def conv_out_hw(h, w, k, stride, pad):
    return (h + 2 * pad - k) // stride + 1, (w + 2 * pad - k) // stride + 1


def conv2d_fwd(x, w, stride=1, pad=0, bias=None, out=None, out_f32=False, cin=None, out_coff=0):
    """x: [N,H,W,Cs] bf16 (channels [0,cin) used, stride Cs); w: [Cout,KH,KW,cin] bf16.

    Returns y [N,OH,OW,Cout] (or writes into `out` at channel offset out_coff)."""
    lib = _lib_bound()
    n, h, wd, cs = x.shape
    cin = cs if cin is None else cin
    cout, kh, kw, wc = w.shape
    assert wc == cin and x.stride(-1) == 1 and w.is_contiguous()
    oh, ow = conv_out_hw(h, wd, kh, stride, pad)
    if out is None:
        out = torch.empty((n, oh, ow, cout), dtype=F32 if out_f32 else BF16, device=x.device)
    ycs = out.shape[-1]
    assert out.shape[:3] == (n, oh, ow) and (out.dtype == F32) == bool(out_f32)
    rc = lib.cvb_conv2d_fwd(x.data_ptr(), n, h, wd, cin, x.stride(2), w.data_ptr(), cout, kh, kw, stride, pad,
                            out.data_ptr(), oh, ow, ycs, out_coff, _ptr(bias), int(out_f32), _stream())
    _lib.check(rc, "conv2d_fwd")
    return out


def conv2d_wgrad_partials(dy, x, kh, kw, stride, pad, cin=None, max_splits=148, part=None):
    """fp32 partial weight gradients [splits, Cout, KH*KW*cin]; returns (part, splits)."""
    lib = _lib_bound()
    n, oh, ow, cout = dy.shape
    _, h, wd, cs = x.shape
    cin = cs if cin is None else cin
    ncols = kh * kw * cin
    if part is None:
        part = torch.empty((max_splits, cout, ncols), dtype=F32, device=dy.device)
    used = ctypes.c_int(0)
    rc = lib.cvb_conv2d_wgrad(dy.data_ptr(), n, oh, ow, cout, dy.stride(2), x.data_ptr(), h, wd, cin, x.stride(2),
                              kh, kw, stride, pad, part.data_ptr(), min(max_splits, part.shape[0]),
                              ctypes.byref(used), _stream())
    _lib.check(rc, "conv2d_wgrad")
    return part, used.value


def gemm(a, b, M, N, K, a_major=0, b_major=0, out=None, out_f32=False, bias=None, splits=1):
    """C[M,N] = sum_k A(m,k) B(n,k) with A [M,K] (a_major 0) or [K,M] (1), B [N,K] (0) or [K,N] (1)."""
    lib = _lib_bound()
    used = lib.cvb_gemm_splits_used(K, splits)
    if out is None:
        if used > 1:
            out = torch.empty((used, M, N), dtype=F32, device=a.device)
        else:
            out = torch.empty((M, N), dtype=F32 if out_f32 else BF16, device=a.device)
    rc = lib.cvb_gemm(a.data_ptr(), a_major, a.stride(0), b.data_ptr(), b_major, b.stride(0), M, N, K,
                      out.data_ptr(), out.stride(-2), int(out_f32 or used > 1), _ptr(bias), splits, _stream())
    _lib.check(rc, "gemm")
    return out
