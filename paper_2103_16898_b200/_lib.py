"""Loader for the in-tree C-ABI library ``libcovault_b200.so`` (sm_100a kernels).

There is no fallback: if the library is missing or cannot be loaded the import of any
compute entry point raises :class:`NativeLibraryMissing`.  Build it with
``python -c "import __graft_entry__ as g; g.build()"`` (or ``make -C
paper_2103_16898_b200/csrc``).
"""
from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("CVB_LIB", _HERE / "libcovault_b200.so"))

_lock = threading.Lock()
_lib = None

# status codes (include/covault_b200.h)
CVB_OK = 0
CVB_AUTH_FAIL = 1
CVB_EINVAL = -1
CVB_ECUDA = -2
CVB_ENOMEM = -3

_c = ctypes
_P = _c.c_void_p
_SZ = _c.c_size_t
_I64 = _c.c_int64
_INT = _c.c_int

# name -> (restype, argtypes); every symbol declared in include/*.h is listed here
SIGNATURES = {
    "cvb_version": (_INT, []),
    "cvb_last_error": (_c.c_char_p, []),
    "cvb_set_device": (_INT, [_INT]),
    "cvb_device_sync": (_INT, []),
    "cvb_aes256_encrypt_block_host": (_INT, [_P, _P, _P]),
    "cvb_aead_open": (_INT, [_P, _P, _P, _SZ, _P, _SZ, _P]),
    "cvb_aead_seal": (_INT, [_P, _P, _P, _SZ, _P, _SZ, _P]),
    "cvb_aead_seal_named": (_INT, [_P, _P, _P, _SZ, _P, _SZ, _P, _P]),
    "cvb_gcm_ctx_create": (_INT, [_P, _c.POINTER(_P)]),
    "cvb_gcm_ctx_destroy": (None, [_P]),
    "cvb_gcm_ctx_set_verdict": (_INT, [_P, _P]),
    "cvb_aead_cache_clear": (None, []),
    "cvb_gcm_open_dev": (_INT, [_P, _P, _P, _SZ, _P, _SZ, _P, _P, _P]),
    "cvb_gcm_seal_dev": (_INT, [_P, _P, _P, _SZ, _P, _SZ, _P, _P, _P]),
    "cvb_gcm_open_records_dev": (_INT, [_P, _P, _P, _SZ, _P, _SZ, _I64, _INT, _I64, _P, _P, _P, _P, _P, _P]),
    "cvb_records_to_nhwc": (_INT, [_P, _I64, _I64, _I64, _I64, _I64, _P, _P, _INT, _P, _P, _P]),
    "cvb_sha256_batch_dev": (_INT, [_P, _P, _I64, _P, _P]),
    "cvb_sha256_batch": (_INT, [_P, _P, _I64, _P]),
    "cvb_sha256_spans_dev": (_INT, [_P, _P, _I64, _P, _P]),
    "cvb_csv_index": (_INT, [_P, _SZ, _P, _c.POINTER(_P), _P]),
    "cvb_csv_fill": (_INT, [_P, _P, _P, _P]),
    "cvb_csv_free": (None, [_P]),
    "cvb_logistic_train": (_INT, [_P, _P, _I64, _I64, _c.c_double, _I64, _INT, _P, _P]),
    "cvb_logistic_scratch_doubles": (_I64, [_I64, _I64, _INT]),
    "cvb_logistic_transpose_dev": (_INT, [_P, _I64, _I64, _P, _P]),
    "cvb_logistic_grad_dev": (_INT, [_P, _P, _P, _I64, _I64, _P, _P, _INT, _P, _P, _P]),
    "cvb_logistic_apply_dev": (_INT, [_P, _I64, _c.c_double, _c.c_double, _P, _P, _P]),
    # tcgen05 implicit-GEMM engine (include/cvb_nn.h)
    "cvb_conv2d_fwd": (_INT, [_P, _INT, _INT, _INT, _INT, _INT, _P, _INT, _INT, _INT, _INT, _INT, _P, _INT, _INT,
                              _INT, _INT, _P, _INT, _INT, _P]),
    "cvb_bn_gather_dx": (_INT, [_P, _INT, _I64, _INT, _P, _P, _P, _INT, _INT, _P, _P, _P, _P, _P, _P, _P, _INT,
                                _INT, _P]),
    "cvb_conv2d_wgrad": (_INT, [_P, _INT, _INT, _INT, _INT, _INT, _P, _INT, _INT, _INT, _INT, _INT, _INT, _INT,
                                _INT, _P, _INT, _c.POINTER(_INT), _P]),
    "cvb_gemm": (_INT, [_P, _INT, _I64, _P, _INT, _I64, _INT, _INT, _INT, _P, _I64, _INT, _P, _INT, _INT, _P]),
    "cvb_gemm_ex": (_INT, [_P, _INT, _I64, _P, _INT, _I64, _INT, _INT, _INT, _P, _I64, _INT, _P, _INT, _INT, _INT, _P]),
    "cvb_gemm_splits_used": (_INT, [_INT, _INT]),
    "cvb_bn_workspace_floats": (_I64, [_I64, _INT]),
    "cvb_bn_stats": (_INT, [_P, _I64, _INT, _INT, _P, _P, _P, _c.c_float, _P, _P, _c.c_float, _P]),
    "cvb_bn_apply": (_INT, [_P, _I64, _INT, _INT, _P, _P, _P, _P, _P, _INT, _INT, _P, _INT, _INT, _P]),
    "cvb_bn_backward": (_INT, [_P, _INT, _P, _INT, _P, _INT, _I64, _INT, _P, _P, _P, _P, _INT, _P, _P, _P, _P, _INT,
                               _P, _INT, _P, _P]),
    "cvb_bn_fused_workspace_floats": (_I64, [_INT]),
    "cvb_conv2d_dgrad_s2": (_INT, [_P, _INT, _INT, _INT, _INT, _INT, _P, _INT, _INT, _INT, _INT, _P, _INT, _INT, _INT,
                                   _INT, _P, _P]),
    "cvb_bn_forward": (_INT, [_P, _I64, _INT, _INT, _P, _P, _P, _c.c_float, _P, _P, _c.c_float, _P, _P, _P, _INT, _INT,
                              _P, _INT, _INT, _P]),
    "cvb_bn_forward_range": (_INT, [_P, _I64, _INT, _INT, _P, _P, _P, _c.c_float, _P, _P, _c.c_float, _P, _P, _P,
                                    _INT, _INT, _P, _INT, _INT, _INT, _INT, _P]),
    "cvb_bn_backward_fused": (_INT, [_P, _INT, _P, _INT, _P, _INT, _I64, _INT, _P, _P, _P, _P, _INT, _P, _P, _P, _P,
                                     _INT, _P, _INT, _P, _P]),
    "cvb_conv2d_dgrad_s2_rows": (_INT, [_P, _INT, _INT, _INT, _INT, _INT, _INT, _P, _INT, _INT, _INT, _INT, _P, _P]),
    "cvb_bn_forward_mask": (_INT, [_P, _I64, _INT, _INT, _P, _P, _P, _c.c_float, _P, _P, _c.c_float, _P, _P, _P,
                                   _INT, _INT, _P, _INT, _INT, _P, _P]),
    "cvb_bn_backward_fused_mask": (_INT, [_P, _INT, _P, _INT, _P, _I64, _INT, _P, _P, _P, _P, _INT, _P, _P, _P, _P,
                                          _INT, _P, _INT, _P, _P]),
    "cvb_weight_flip_batched": (_INT, [_P, _P, _P, _INT, _I64, _P]),
    "cvb_transpose_batched": (_INT, [_P, _P, _P, _INT, _I64, _P]),
    "cvb_space_to_depth2": (_INT, [_P, _INT, _INT, _INT, _INT, _P, _P]),
    "cvb_s2d_weights": (_INT, [_P, _INT, _INT, _P, _P]),
    "cvb_s2d_weights_grad": (_INT, [_P, _INT, _INT, _P, _P]),
    "cvb_maxpool_fwd_idx": (_INT, [_P, _INT, _INT, _INT, _INT, _INT, _INT, _INT, _P, _INT, _INT, _INT, _P, _P]),
    "cvb_maxpool_bwd_idx": (_INT, [_P, _P, _INT, _INT, _INT, _INT, _INT, _INT, _INT, _INT, _INT, _P, _P]),
    "cvb_maxpool_fwd": (_INT, [_P, _INT, _INT, _INT, _INT, _INT, _INT, _INT, _P, _INT, _INT, _INT, _P]),
    "cvb_maxpool_bwd": (_INT, [_P, _P, _INT, _INT, _INT, _INT, _INT, _INT, _INT, _INT, _INT, _P, _P]),
    "cvb_avgpool_fwd": (_INT, [_P, _INT, _INT, _INT, _INT, _INT, _INT, _P, _INT, _P]),
    "cvb_avgpool_bwd": (_INT, [_P, _INT, _INT, _INT, _INT, _INT, _P, _INT, _P]),
    "cvb_gap_fwd": (_INT, [_P, _INT, _INT, _INT, _INT, _P, _P]),
    "cvb_gap_bwd": (_INT, [_P, _INT, _INT, _INT, _P, _P]),
    "cvb_softmax_xent": (_INT, [_P, _INT, _INT, _P, _c.c_float, _P, _P, _P, _INT, _P]),
    "cvb_head_train": (_INT, [_P, _I64, _P, _P, _P, _INT, _INT, _INT, _c.c_float, _INT, _P, _P, _P, _P, _P, _I64,
                              _P, _P, _P, _P, _P]),
    "cvb_head_workspace_floats": (_I64, [_INT, _INT]),
    "cvb_reduce_splits": (_INT, [_P, _INT, _I64, _P, _INT, _c.c_float, _P]),
    "cvb_reduce_splits_act": (_INT, [_P, _INT, _INT, _INT, _P, _INT, _P, _INT, _I64, _P]),
    "cvb_weight_flip": (_INT, [_P, _INT, _INT, _INT, _INT, _P, _P]),
    "cvb_debug_mma_cycles": (_c.c_longlong, [_INT, _INT, _INT, _INT]),
    "cvb_debug_trace": (_INT, [_P]),
    "cvb_zero_upsample": (_INT, [_P, _INT, _INT, _INT, _INT, _INT, _P, _P]),
    "cvb_col_sum": (_INT, [_P, _INT, _I64, _INT, _I64, _P, _INT, _P]),
    "cvb_relu_fwd": (_INT, [_P, _I64, _P]),
    "cvb_relu_bwd": (_INT, [_P, _P, _I64, _P]),
    "cvb_adam_step": (_INT, [_P, _P, _P, _P, _P, _I64, _c.c_float, _c.c_float, _c.c_float, _c.c_float, _I64,
                             _c.c_float, _P, _P, _P, _P]),
    "cvb_verdict_snapshot": (_INT, [_P, _P, _P]),
    "cvb_sgd_step": (_INT, [_P, _P, _P, _P, _I64, _c.c_float, _c.c_float, _c.c_float, _c.c_float, _INT, _P]),
    "cvb_cast_f32_bf16": (_INT, [_P, _P, _I64, _P]),
    "cvb_cast_rows": (_INT, [_P, _I64, _P, _I64, _I64, _INT, _P]),
}


class NativeLibraryMissing(RuntimeError):
    pass


class NativeError(RuntimeError):
    pass


def load():
    """Return the loaded ctypes library (raises NativeLibraryMissing if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise NativeLibraryMissing(
                f"{LIB_PATH} not built; run `make -C {_HERE / 'csrc'}` (no CPU fallback exists)")
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int, what: str) -> int:
    if rc < 0:
        msg = load().cvb_last_error().decode("utf-8", "replace")
        raise NativeError(f"{what} failed ({rc}): {msg}")
    return rc


_tls = threading.local()


def bind_device(dev: int | None = None) -> None:
    """Point the library's CUDA runtime at torch's current device.

    The library links cudart statically, so its current device is its own and per thread:
    re-bind whenever the calling thread's torch device differs from what this thread last
    bound (torch cuda:0 -> cuda:1 -> cuda:0 and new threads are all handled).  Without
    torch imported (the host AEAD path) the device is left at the thread's default."""
    if dev is None:
        import sys

        torch = sys.modules.get("torch")
        if torch is None or not torch.cuda.is_available() or not torch.cuda.is_initialized():
            return
        dev = torch.cuda.current_device()
    if getattr(_tls, "dev", None) != dev:
        check(load().cvb_set_device(int(dev)), "cvb_set_device")
        _tls.dev = dev


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
