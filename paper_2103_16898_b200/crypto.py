"""GPU AES-256-GCM behind the reference's AEAD API.

Same signatures, argument meaning and exceptions as
  covault.crypto.aead_seal(key, nonce, aad, plaintext) -> bytes   crypto.py:258-262
  covault.crypto.aead_open(key, nonce, aad, ciphertext) -> bytes  crypto.py:265-272
  covault.crypto.SymmetricKey                                     crypto.py:213-255
When the reference package is importable its exception classes are used, so these
functions can be monkeypatched into ``covault.crypto`` and the reference's own tests keep
catching the same types.  The device-side API (``GcmContext``) keeps
ciphertext and plaintext in HBM for the training loader.
"""
from __future__ import annotations

import collections
import ctypes
import hashlib
import secrets

from . import _lib

AEAD_NONCE_SIZE = 12
SYMMETRIC_KEY_SIZE = 32
KEY_COMMITMENT_TAG = b"covault.key-commitment.v1"   # crypto.py:38

# host-API calls that ran on the GPU, by entry point (evidence that a patched reference
# test suite really exercised this path; see tests/test_reference_suites_gpu.py)
CALLS = collections.Counter()

try:  # share exception identity with the reference when it is installed
    from covault.crypto import AuthenticationFailure, CryptoError, DecodeError  # type: ignore
except Exception:  # pragma: no cover - standalone use
    class CryptoError(Exception):
        """Base class for failures in this module (crypto.py:42-43)."""

    class DecodeError(CryptoError):
        """Malformed key or nonce (crypto.py:46-47)."""

    class AuthenticationFailure(CryptoError):
        """AEAD open failed (crypto.py:50-51)."""


class SymmetricKey:
    """32 bytes of key material plus its commitment key_id = SHA-256(key || tag)."""

    __slots__ = ("_bytes", "key_id")

    def __init__(self, raw: bytes) -> None:
        if len(raw) != SYMMETRIC_KEY_SIZE:
            raise DecodeError(f"symmetric key must be {SYMMETRIC_KEY_SIZE} bytes")
        self._bytes = bytes(raw)
        self.key_id = hashlib.sha256(self._bytes + KEY_COMMITMENT_TAG).digest()

    @classmethod
    def from_hex(cls, text: str) -> "SymmetricKey":
        try:
            return cls(bytes.fromhex(text))
        except ValueError as e:
            raise DecodeError(f"bad key hex: {e}") from e

    @classmethod
    def generate(cls) -> "SymmetricKey":
        return cls(secrets.token_bytes(SYMMETRIC_KEY_SIZE))

    def reveal_bytes(self) -> bytes:
        return self._bytes

    def __repr__(self) -> str:
        return f"SymmetricKey(id={self.key_id.hex()[:12]}…)"


def _key_bytes(key) -> bytes:
    raw = key.reveal_bytes() if hasattr(key, "reveal_bytes") else bytes(key)
    if len(raw) != SYMMETRIC_KEY_SIZE:
        raise DecodeError(f"symmetric key must be {SYMMETRIC_KEY_SIZE} bytes")
    return raw


def aead_seal(key, nonce: bytes, aad: bytes, plaintext: bytes) -> bytes:
    """AES-256-GCM seal on the GPU -> C || T (crypto.py:258-262)."""
    CALLS["aead_seal"] += 1
    if len(nonce) != AEAD_NONCE_SIZE:
        raise DecodeError(f"nonce must be {AEAD_NONCE_SIZE} bytes")
    lib = _lib.load()
    _lib.bind_device()
    kb = _key_bytes(key)
    out = ctypes.create_string_buffer(len(plaintext) + 16)
    rc = lib.cvb_aead_seal(kb, bytes(nonce), bytes(aad), len(aad), bytes(plaintext), len(plaintext), out)
    _lib.check(rc, "aead_seal")
    return out.raw


def aead_seal_named(key, nonce: bytes, aad: bytes, plaintext: bytes) -> tuple[bytes, bytes]:
    """aead_seal plus SHA-256 of the sealed blob computed on the device in the same round trip:
    (blob, digest) -- Volume.put's seal + blob name (volume.py:168-171)."""
    CALLS["aead_seal"] += 1
    if len(nonce) != AEAD_NONCE_SIZE:
        raise DecodeError(f"nonce must be {AEAD_NONCE_SIZE} bytes")
    lib = _lib.load()
    _lib.bind_device()
    kb = _key_bytes(key)
    out = ctypes.create_string_buffer(len(plaintext) + 16)
    dig = ctypes.create_string_buffer(32)
    rc = lib.cvb_aead_seal_named(kb, bytes(nonce), bytes(aad), len(aad), bytes(plaintext), len(plaintext), out, dig)
    _lib.check(rc, "aead_seal_named")
    return out.raw, dig.raw


def aead_open(key, nonce: bytes, aad: bytes, ciphertext: bytes) -> bytes:
    """AES-256-GCM open on the GPU; raises AuthenticationFailure on any mismatch."""
    CALLS["aead_open"] += 1
    if len(nonce) != AEAD_NONCE_SIZE:
        raise DecodeError(f"nonce must be {AEAD_NONCE_SIZE} bytes")
    lib = _lib.load()
    _lib.bind_device()
    kb = _key_bytes(key)
    n = len(ciphertext)
    out = ctypes.create_string_buffer(max(1, n - 16))
    rc = lib.cvb_aead_open(kb, bytes(nonce), bytes(aad), len(aad), bytes(ciphertext), n, out)
    _lib.check(rc, "aead_open")
    if rc == _lib.CVB_AUTH_FAIL:
        raise AuthenticationFailure("AEAD authentication failed")
    return out.raw[: n - 16]


def sha256_many(messages) -> list[bytes]:
    """SHA-256 of each message (bytes-like) on the GPU, one launch for the whole batch --
    the batched form of covault.crypto.hash_bytes (crypto.py:91-93)."""
    msgs = [bytes(m) for m in messages]
    n = len(msgs)
    CALLS["sha256"] += n
    if n == 0:
        return []
    lib = _lib.load()
    _lib.bind_device()
    ptrs = (ctypes.c_char_p * n)(*msgs)
    lens = (ctypes.c_size_t * n)(*[len(m) for m in msgs])
    out = ctypes.create_string_buffer(32 * n)
    _lib.check(lib.cvb_sha256_batch(ctypes.cast(ptrs, ctypes.c_void_p), lens, n, out), "sha256_batch")
    raw = out.raw
    return [raw[32 * i:32 * i + 32] for i in range(n)]


def sha256_device(data_dev, offsets_dev, stream=None):
    """Digests (uint8 CUDA tensor [n, 32]) of the n messages data_dev[offsets[i]:offsets[i+1]]
    of a uint8 CUDA arena; stream-ordered, the messages never leave HBM."""
    import torch

    _lib.bind_device()
    n = offsets_dev.numel() - 1
    out = torch.empty((max(0, n), 32), dtype=torch.uint8, device=data_dev.device)
    if n > 0:
        if offsets_dev.dtype != torch.int64 or not offsets_dev.is_cuda:
            raise ValueError("offsets must be an int64 CUDA tensor")
        _lib.check(_lib.load().cvb_sha256_batch_dev(data_dev.data_ptr(), offsets_dev.data_ptr(), n, out.data_ptr(),
                                                    _lib.stream_ptr(stream)), "sha256_batch_dev")
    return out


def sha256_tensors(tensors, stream=None):
    """Digests (uint8 CUDA tensor [n, 32]) of n uint8 CUDA tensors in separate allocations, one
    launch; stream-ordered, nothing leaves HBM but the pointer/length table going in."""
    import torch

    _lib.bind_device()
    n = len(tensors)
    dev = tensors[0].device if n else torch.device("cuda")
    out = torch.empty((n, 32), dtype=torch.uint8, device=dev)
    if n:
        meta = torch.tensor([t.data_ptr() for t in tensors] + [t.numel() for t in tensors], dtype=torch.int64)
        meta = meta.pin_memory().to(dev, non_blocking=True)
        if stream is not None:
            meta.record_stream(stream)
        _lib.check(_lib.load().cvb_sha256_spans_dev(meta.data_ptr(), meta.data_ptr() + 8 * n, n, out.data_ptr(),
                                                    _lib.stream_ptr(stream)), "sha256_spans_dev")
    return out


def fresh_nonce() -> bytes:
    return secrets.token_bytes(AEAD_NONCE_SIZE)


class GcmContext:
    """Per-key device context: expanded key + GHASH power tables resident in HBM.

    ``open_device`` / ``seal_device`` are stream-ordered and never synchronise; the tag
    verdict lands in a device status word (``status_tensor``) and, on a mismatch, the
    plaintext is zeroed on-stream before any later kernel can read it.
    """

    def __init__(self, key):
        import torch

        _lib.bind_device()
        self._lib = _lib.load()
        self._ptr = ctypes.c_void_p()
        _lib.check(self._lib.cvb_gcm_ctx_create(_key_bytes(key), ctypes.byref(self._ptr)), "gcm_ctx_create")
        self._torch = torch

    def set_verdict(self, word) -> None:
        """Attach a zeroed int32 CUDA word that every later open / decode through this context
        ORs its tag verdict into (sticky over a whole run; ``None`` detaches).  The caller
        keeps ``word`` alive while launches that may write it are in flight."""
        self._verdict = word
        _lib.check(self._lib.cvb_gcm_ctx_set_verdict(self._ptr, word.data_ptr() if word is not None else None),
                   "gcm_ctx_set_verdict")

    def close(self):
        if self._ptr:
            self._lib.cvb_gcm_ctx_destroy(self._ptr)
            self._ptr = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def new_workspace(self, device=None):
        """8 zeroed uint32 words: GHASH accumulator [0:4] + status [4]."""
        return self._torch.zeros(8, dtype=self._torch.int32, device=device or "cuda")

    def open_device(self, nonce: bytes, aad_dev, blob_dev, out_dev, work, stream=None):
        """blob_dev: uint8 CUDA tensor C||T; out_dev: uint8 CUDA tensor of len(C)."""
        if len(nonce) != AEAD_NONCE_SIZE:
            raise DecodeError(f"nonce must be {AEAD_NONCE_SIZE} bytes")
        n = blob_dev.numel()
        if out_dev.numel() < n - 16:
            raise ValueError("output buffer too small")
        aad_ptr = aad_dev.data_ptr() if aad_dev is not None and aad_dev.numel() else None
        aad_len = aad_dev.numel() if aad_dev is not None else 0
        rc = self._lib.cvb_gcm_open_dev(self._ptr, bytes(nonce), aad_ptr, aad_len, blob_dev.data_ptr(), n,
                                        out_dev.data_ptr(), work.data_ptr(), _lib.stream_ptr(stream))
        _lib.check(rc, "gcm_open_dev")

    def seal_device(self, nonce: bytes, aad_dev, pt_dev, out_dev, work, stream=None):
        if len(nonce) != AEAD_NONCE_SIZE:
            raise DecodeError(f"nonce must be {AEAD_NONCE_SIZE} bytes")
        n = pt_dev.numel()
        if out_dev.numel() < n + 16:
            raise ValueError("output buffer too small")
        aad_ptr = aad_dev.data_ptr() if aad_dev is not None and aad_dev.numel() else None
        aad_len = aad_dev.numel() if aad_dev is not None else 0
        rc = self._lib.cvb_gcm_seal_dev(self._ptr, bytes(nonce), aad_ptr, aad_len, pt_dev.data_ptr() if n else None,
                                        n, out_dev.data_ptr(), work.data_ptr(), _lib.stream_ptr(stream))
        _lib.check(rc, "gcm_seal_dev")

    def open_records_device(self, nonce: bytes, aad_dev, blob_dev, tile, labels, work, spec, stream=None):
        """Fused decrypt-and-normalise (K1b): sealed binary records -> bf16 NHWC-8 training
        tile + int32 labels in one kernel (no plaintext buffer).  ``tile`` must have been
        allocated zeroed (its pad channels are never written).  Verdict as open_device."""
        if len(nonce) != AEAD_NONCE_SIZE:
            raise DecodeError(f"nonce must be {AEAD_NONCE_SIZE} bytes")
        c, h, w = spec["c"], spec["h"], spec["w"]
        m = (ctypes.c_float * 8)(*spec["mean"])
        sd = (ctypes.c_float * 8)(*spec["std"])
        aad_ptr = aad_dev.data_ptr() if aad_dev is not None and aad_dev.numel() else None
        aad_len = aad_dev.numel() if aad_dev is not None else 0
        rc = self._lib.cvb_gcm_open_records_dev(self._ptr, bytes(nonce), aad_ptr, aad_len, blob_dev.data_ptr(),
                                                blob_dev.numel(), 1 + c * h * w, c, h * w, m, sd, tile.data_ptr(),
                                                labels.data_ptr(), work.data_ptr(), _lib.stream_ptr(stream))
        _lib.check(rc, "gcm_open_records_dev")

    @staticmethod
    def status_ok(work) -> bool:
        """Host check of the tag verdict (synchronises on the work tensor)."""
        return int(work[4].item()) == 0
