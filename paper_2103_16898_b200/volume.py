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
            # seal and blob name (SHA-256 of the sealed blob) in one device round trip
            blob, digest = _crypto.aead_seal_named(key, nonce, aad_for(self.volume_name, logical_path), plaintext)
            h = digest.hex()
            (self.root / h).write_bytes(blob)
            old = self._entries.get(logical_path)
            self._entries[logical_path] = ManifestEntry(logical_path, nonce, h, len(plaintext))
            self._write_manifest()
            if old is not None and old.ciphertext_hash != h:
                (self.root / old.ciphertext_hash).unlink(missing_ok=True)
        finally:
            os.close(fd)
            (self.root / LOCK_NAME).unlink(missing_ok=True)

    def put_sealed(self, key, logical_path: str, nonce: bytes, blob: bytes, plaintext_length: int,
                   blob_digest: bytes | None = None) -> None:
        """Install a blob already sealed under this volume's key/AAD (the GPU gate copy
        seals on the device and hashes the blob there: ``blob_digest``); same lock / naming /
        manifest discipline as put()."""
        _check_path(logical_path)
        if key_id_hex(key) != self.key_id:
            raise KeyMismatch("key commitment does not match the volume manifest")
        try:
            fd = os.open(self.root / LOCK_NAME, os.O_CREAT | os.O_EXCL | os.O_WRONLY)
        except FileExistsError:
            raise VolumeLocked(f"another writer holds {self.root}") from None
        try:
            h = (blob_digest if blob_digest is not None else _crypto.sha256_many([blob])[0]).hex()
            (self.root / h).write_bytes(blob)
            old = self._entries.get(logical_path)
            self._entries[logical_path] = ManifestEntry(logical_path, nonce, h, plaintext_length)
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
        if stream is not None:
            # the H2D copy, AAD upload and workspace zeroing above ran on the current stream
            stream.wait_stream(torch.cuda.current_stream())
        ctx.open_device(e.nonce, aad, dev, out, work, stream)
        if stream is not None:
            for t in (dev, aad, out, work):   # keep the allocator from recycling them early
                t.record_stream(stream)
        if sync:
            if stream is not None:
                stream.synchronize()   # the verdict is written on `stream`
            if not ctx.status_ok(work):
                del out
                raise AuthenticationFailure("AEAD authentication failed")
        return out[: e.plaintext_length], work

    def verify(self, batch_bytes: int = 1 << 30) -> list[tuple[str, str]]:
        """Key-free integrity scan (volume.py:199-222): (kind, path) pairs.  Blob digests are
        computed on the GPU, one launch per ~``batch_bytes`` of blobs (one thread per blob)."""
        violations = []
        referenced = set()
        pending = []          # (path, expected hex, blob bytes) awaiting a hash batch
        results = {}

        def flush():
            if pending:
                for (p, _, _), d in zip(pending, _crypto.sha256_many([b for _, _, b in pending])):
                    results[p] = d.hex()
                pending.clear()

        checks = []
        size = 0
        for path, e in sorted(self._entries.items()):
            try:
                _check_path(path)
            except VolumeError:
                checks.append(("bad_path", path, None))
                continue
            bp = self.root / e.ciphertext_hash
            referenced.add(e.ciphertext_hash)
            if not bp.exists():
                checks.append(("missing_blob", path, None))
                continue
            blob = bp.read_bytes()
            pending.append((path, e.ciphertext_hash, blob))
            checks.append(("hash", path, e.ciphertext_hash))
            size += len(blob)
            if size >= batch_bytes:
                flush()
                size = 0
        flush()
        for kind, path, want in checks:
            if kind != "hash":
                violations.append((kind, path))
            elif results[path] != want:
                violations.append(("hash_mismatch", path))
        for child in self.root.iterdir():
            if child.name in (MANIFEST_NAME, LOCK_NAME) or child.name.endswith(".tmp"):
                continue
            if child.name not in referenced:
                violations.append(("orphan_blob", child.name))
        return violations


# -- tree helpers (volume.py:239-258) and the gate's re-encryption copy
def seal_tree(volume: Volume, key, source) -> int:
    """Seal every regular file under ``source`` by its relative path (volume.py:239-247);
    the AES-GCM seal of each file runs on the GPU (Volume.put)."""
    source = Path(source)
    count = 0
    for path in sorted(source.rglob("*")):
        if path.is_file():
            volume.put(key, path.relative_to(source).as_posix(), path.read_bytes())
            count += 1
    return count


def unseal_tree(volume: Volume, key, dest) -> int:
    """volume.py:250-258 with the GPU open."""
    dest = Path(dest)
    count = 0
    for logical_path in volume.paths():
        target = dest.joinpath(*logical_path.split("/"))
        target.parent.mkdir(parents=True, exist_ok=True)
        target.write_bytes(volume.get(key, logical_path))
        count += 1
    return count


def gate_copy(source: Volume, source_key, dest: Volume, dest_key) -> list[tuple[str, str, int]]:
    """The trusted-boot gate's copy loop (gate.py:186-190) with every byte of plaintext kept in
    HBM: each source blob is copied to the device once, opened (tag verified on the device),
    re-sealed under the destination key / AAD / a fresh nonce, and both the plaintext digest
    for the copy report and the sealed blob's name are computed by the device SHA-256 -- only
    the sealed blob and two digests come back to the host.  Raises AuthenticationFailure on
    the first bad source blob (the gate maps it to "volume_auth_failure" and discards the
    staging volume, gate.py:191-192)."""
    import torch

    if key_id_hex(dest_key) != dest.key_id:
        raise KeyMismatch("key commitment does not match the destination manifest")
    src_ctx, dst_ctx = _crypto.GcmContext(source_key), _crypto.GcmContext(dest_key)
    report = []
    work_o, work_s = src_ctx.new_workspace(), dst_ctx.new_workspace()
    try:
        for logical_path in source.paths():
            e = source.entry(logical_path)
            blob = source.read_blob(logical_path)
            if len(blob) < 16 or len(blob) - 16 != e.plaintext_length:
                raise AuthenticationFailure("blob length disagrees with manifest")
            n = e.plaintext_length
            blob_dev = torch.frombuffer(bytearray(blob), dtype=torch.uint8).pin_memory().to("cuda", non_blocking=True)
            aad_s = torch.frombuffer(bytearray(aad_for(source.volume_name, logical_path)), dtype=torch.uint8).cuda()
            aad_d = torch.frombuffer(bytearray(aad_for(dest.volume_name, logical_path)), dtype=torch.uint8).cuda()
            pt = torch.empty(max(1, n), dtype=torch.uint8, device="cuda")
            work_o.zero_()
            src_ctx.open_device(e.nonce, aad_s, blob_dev, pt, work_o)
            if not src_ctx.status_ok(work_o):          # tag verdict before anything is re-sealed
                raise AuthenticationFailure("AEAD authentication failed")
            nonce = _crypto.fresh_nonce()
            sealed = torch.empty(n + 16, dtype=torch.uint8, device="cuda")
            work_s.zero_()
            dst_ctx.seal_device(nonce, aad_d, pt[:n], sealed, work_s)
            digests = _crypto.sha256_tensors([pt[:n], sealed]).cpu().numpy()   # plaintext, blob name
            pt.zero_()
            dest.put_sealed(dest_key, logical_path, nonce, sealed.cpu().numpy().tobytes(), n,
                            blob_digest=bytes(digests[1]))
            report.append((logical_path, bytes(digests[0]).hex(), n))
    finally:
        src_ctx.close()
        dst_ctx.close()
    return report
