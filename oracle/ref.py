"""ctypes front-end of the C oracle -- TEST INFRASTRUCTURE ONLY.

Mirrors the reference call signatures so tests read like the reference's own:
  gcm_open(key, nonce, aad, blob) -> bytes      ~ covault.crypto.aead_open  (crypto.py:265-272)
  gcm_seal(key, nonce, aad, plaintext) -> bytes ~ covault.crypto.aead_seal  (crypto.py:258-262)
  logistic_train(rows, lr, epochs) -> (w, b)    ~ covault.workload.run_training numeric core
                                                  (workload.py:48-71)
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_DIR = Path(__file__).resolve().parent
_SO = _DIR / "_build" / "liboracle.so"
_lib = None


class OracleAuthFailure(Exception):
    pass


def build() -> Path:
    srcs = [_DIR / "gcm_ref.c", _DIR / "logistic_ref.c"]
    if not _SO.exists() or any(s.stat().st_mtime > _SO.stat().st_mtime for s in srcs):
        subprocess.run(["make", "-s", "-C", str(_DIR)], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_SO))
        u8p = ctypes.c_char_p
        L.ref_gcm_seal.argtypes = [u8p, u8p, u8p, ctypes.c_size_t, u8p, ctypes.c_size_t, ctypes.c_void_p]
        L.ref_gcm_open.argtypes = [u8p, u8p, u8p, ctypes.c_size_t, u8p, ctypes.c_size_t, ctypes.c_void_p]
        L.ref_gcm_open.restype = ctypes.c_int
        L.ref_aes256_expand.argtypes = [u8p, ctypes.c_void_p]
        L.ref_aes256_encrypt_block.argtypes = [u8p, u8p, ctypes.c_void_p]
        L.ref_gf128_mul.argtypes = [u8p, u8p, ctypes.c_void_p]
        L.ref_logistic_train.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_double, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        _lib = L
    return _lib


def aes256_expand(key: bytes) -> bytes:
    out = ctypes.create_string_buffer(240)
    lib().ref_aes256_expand(key, out)
    return out.raw


def aes256_block(key: bytes, block: bytes) -> bytes:
    rk = aes256_expand(key)
    out = ctypes.create_string_buffer(16)
    lib().ref_aes256_encrypt_block(rk, block, out)
    return out.raw


def gf128_mul(x: bytes, y: bytes) -> bytes:
    out = ctypes.create_string_buffer(16)
    lib().ref_gf128_mul(x, y, out)
    return out.raw


def gcm_seal(key: bytes, nonce: bytes, aad: bytes, plaintext: bytes) -> bytes:
    assert len(key) == 32 and len(nonce) == 12
    out = ctypes.create_string_buffer(len(plaintext) + 16)
    lib().ref_gcm_seal(key, nonce, aad, len(aad), plaintext, len(plaintext), out)
    return out.raw


def gcm_open(key: bytes, nonce: bytes, aad: bytes, blob: bytes) -> bytes:
    assert len(key) == 32 and len(nonce) == 12
    if len(blob) < 16:
        raise OracleAuthFailure("blob shorter than the tag")
    out = ctypes.create_string_buffer(max(1, len(blob) - 16))
    rc = lib().ref_gcm_open(key, nonce, aad, len(aad), blob, len(blob), out)
    if rc != 0:
        raise OracleAuthFailure("AEAD authentication failed")
    return out.raw[: len(blob) - 16]


def logistic_train(X: np.ndarray, y: np.ndarray, lr: float, epochs: int):
    X = np.ascontiguousarray(X, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    n, f = X.shape
    w = np.zeros(f, dtype=np.float64)
    b = np.zeros(1, dtype=np.float64)
    lib().ref_logistic_train(X.ctypes.data, y.ctypes.data, n, f, float(lr), int(epochs),
                             w.ctypes.data, b.ctypes.data)
    return w, float(b[0])
