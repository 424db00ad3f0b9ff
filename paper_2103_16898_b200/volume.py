"""The reference's encrypted-volume format, read and written through the GPU AEAD.

On-disk format is byte-compatible with covault.volume (volume.py:1-13):
  manifest.json  canonical JSON (sorted keys, no whitespace, UTF-8; crypto.py:303-314)
  <hex64>        blob C || T named by SHA-256(blob)
  .lock          O_EXCL writer lock
AAD = volume_name || 0x00 || logical_path (volume.py:53-54).

``Volume.get`` keeps the reference contract -- exact bytes or AuthenticationFailure, never
partial (volume.py:185-197) -- with the AES-GCM work on the GPU.  ``Volume.get_device``
is the B200 path: ciphertext is copied once into HBM, decrypted there, and the verified
plaintext stays resident as a uint8 CUDA tensor for the training loader.
"""
from __future__ import annotations

import hashlib
import json
import os
from dataclasses import dataclass
from pathlib import Path

from . import crypto as _crypto
from .crypto import AuthenticationFailure

MANIFEST_NAME = "manifest.json"
LOCK_NAME = ".lock"

try:  # exception identity shared with the reference when installed
    from covault.volume import KeyMismatch, NotFound, VolumeError, VolumeLocked  # type: ignore
except Exception:  # pragma: no cover
    class VolumeError(Exception):
        pass

    class VolumeLocked(VolumeError):
        pass

    class KeyMismatch(VolumeError):
        pass

    class NotFound(VolumeError):
        pass


def aad_for(volume_name: str, logical_path: str) -> bytes:
    """volume.py:53-54"""
    return volume_name.encode("utf-8") + b"\x00" + logical_path.encode("utf-8")


def _check_path(logical_path: str) -> None:
    """volume.py:57-62"""
    parts = logical_path.split("/")
    if not logical_path or any(p in ("", ".", "..") for p in parts):
        raise VolumeError(f"bad logical path {logical_path!r}")
    if logical_path.startswith("/"):
        raise VolumeError("logical paths are relative")


def canonical_encode(doc) -> bytes:
    return json.dumps(doc, sort_keys=True, separators=(",", ":"), ensure_ascii=False,
                      allow_nan=False).encode("utf-8")


def key_id_hex(key) -> str:
    raw = key.reveal_bytes() if hasattr(key, "reveal_bytes") else bytes(key)
    return hashlib.sha256(raw + _crypto.KEY_COMMITMENT_TAG).hexdigest()


@dataclass(frozen=True)
class ManifestEntry:
    logical_path: str
    nonce: bytes
    ciphertext_hash: str   # lowercase hex
    plaintext_length: int


class Volume:
    def __init__(self, root: Path, volume_name: str, key_id: str, entries: dict):
        self.root = root
        self.volume_name = volume_name
        self.key_id = key_id
        self._entries = entries

    @classmethod
    def open(cls, root) -> "Volume":
        root = Path(root)
        mp = root / MANIFEST_NAME
        if not mp.exists():
            raise NotFound(f"no manifest at {root}")
        doc = json.loads(mp.read_bytes().decode("utf-8"))
        entries = {
            it["path"]: ManifestEntry(it["path"], bytes.fromhex(it["nonce"]), it["ciphertext_hash"],
                                      int(it["plaintext_length"]))
            for it in doc["entries"]
        }
        return cls(root, doc["volume_name"], doc["key_id"], entries)

    @classmethod
    def create(cls, root, volume_name: str, key) -> "Volume":
        root = Path(root)
        root.mkdir(parents=True, exist_ok=True)
        if (root / MANIFEST_NAME).exists():
            vol = cls.open(root)
            if vol.key_id != key_id_hex(key):
                raise KeyMismatch("existing volume was created under a different key")
            return vol
        vol = cls(root, volume_name, key_id_hex(key), {})
        vol._write_manifest()
        return vol

    def manifest_doc(self) -> dict:
        return {
            "volume_name": self.volume_name,
            "key_id": self.key_id,
            "entries": [
                {"path": e.logical_path, "nonce": e.nonce.hex(), "ciphertext_hash": e.ciphertext_hash,
                 "plaintext_length": e.plaintext_length}
                for e in sorted(self._entries.values(), key=lambda e: e.logical_path)
            ],
        }

    def _write_manifest(self) -> None:
        tmp = self.root / (MANIFEST_NAME + ".tmp")
        tmp.write_bytes(canonical_encode(self.manifest_doc()))
        os.replace(tmp, self.root / MANIFEST_NAME)

    def paths(self) -> list[str]:
        return sorted(self._entries)

    def entry(self, logical_path: str) -> ManifestEntry:
        e = self._entries.get(logical_path)
        if e is None:
            raise NotFound(f"{logical_path!r} not in manifest")
        return e

    def blob_path(self, logical_path: str) -> Path:
        e = self.entry(logical_path)
        p = self.root / e.ciphertext_hash
        if not p.exists():
            raise NotFound(f"blob for {logical_path!r} missing")
        return p

    # -- writer ----------------------------------------------------------------------------
    def put(self, key, logical_path: str, plaintext: bytes) -> None:
        """volume.py:161-183 with the AES-GCM seal on the GPU."""
        _check_path(logical_path)
        if key_id_hex(key) != self.key_id:
            raise KeyMismatch("key commitment does not match the volume manifest")
        try:
            fd = os.open(self.root / LOCK_NAME, os.O_CREAT | os.O_EXCL | os.O_WRONLY)
        except FileExistsError:
            raise VolumeLocked(f"another writer holds {self.root}") from None
        try:
            nonce = _crypto.fresh_nonce()
            blob = _crypto.aead_seal(key, nonce, aad_for(self.volume_name, logical_path), plaintext)
            h = hashlib.sha256(blob).hexdigest()
            (self.root / h).write_bytes(blob)
            old = self._entries.get(logical_path)
            self._entries[logical_path] = ManifestEntry(logical_path, nonce, h, len(plaintext))
            self._write_manifest()
            if old is not None and old.ciphertext_hash != h:
                (self.root / old.ciphertext_hash).unlink(missing_ok=True)
        finally:
            os.close(fd)
            (self.root / LOCK_NAME).unlink(missing_ok=True)

    # -- readers ---------------------------------------------------------------------------
    def get(self, key, logical_path: str) -> bytes:
        """Exact original bytes or AuthenticationFailure; never partial (volume.py:185-197)."""
        e = self.entry(logical_path)
        blob = self.blob_path(logical_path).read_bytes()
        pt = _crypto.aead_open(key, e.nonce, aad_for(self.volume_name, logical_path), blob)
        if len(pt) != e.plaintext_length:
            raise AuthenticationFailure("plaintext length disagrees with manifest")
        return pt

    def read_blob(self, logical_path: str) -> bytes:
        return self.blob_path(logical_path).read_bytes()

    def get_device(self, ctx: "_crypto.GcmContext", logical_path: str, stream=None, sync: bool = True):
        """Decrypt one file into HBM.  Returns (plaintext uint8 CUDA tensor, work tensor).

        With sync=True the tag verdict is checked here (raises AuthenticationFailure and
        the zeroed buffer is dropped); with sync=False the caller must check
        ``GcmContext.status_ok(work)`` before handing the buffer to training.
        """
        import torch

        e = self.entry(logical_path)
        blob = self.read_blob(logical_path)
        if len(blob) < 16 or len(blob) - 16 != e.plaintext_length:
            raise AuthenticationFailure("blob length disagrees with manifest")
        host = torch.frombuffer(bytearray(blob), dtype=torch.uint8).pin_memory()
        dev = host.to("cuda", non_blocking=True)
        aad = torch.tensor(list(aad_for(self.volume_name, logical_path)), dtype=torch.uint8, device="cuda")
        out = torch.empty(max(1, e.plaintext_length), dtype=torch.uint8, device="cuda")
        work = ctx.new_workspace()
        ctx.open_device(e.nonce, aad, dev, out, work, stream)
        if sync:
            if not ctx.status_ok(work):
                del out
                raise AuthenticationFailure("AEAD authentication failed")
        return out[: e.plaintext_length], work

    def verify(self) -> list[tuple[str, str]]:
        """Key-free integrity scan (volume.py:199-222): (kind, path) pairs."""
        violations = []
        referenced = set()
        for path, e in sorted(self._entries.items()):
            try:
                _check_path(path)
            except VolumeError:
                violations.append(("bad_path", path))
                continue
            bp = self.root / e.ciphertext_hash
            referenced.add(e.ciphertext_hash)
            if not bp.exists():
                violations.append(("missing_blob", path))
                continue
            if hashlib.sha256(bp.read_bytes()).hexdigest() != e.ciphertext_hash:
                violations.append(("hash_mismatch", path))
        for child in self.root.iterdir():
            if child.name in (MANIFEST_NAME, LOCK_NAME) or child.name.endswith(".tmp"):
                continue
            if child.name not in referenced:
                violations.append(("orphan_blob", child.name))
        return violations
