"""B200-native encrypted-training hot path of arXiv 2103.16898 (reference: covault).

Public surface (mirrors the reference's workload-side API):
  crypto.aead_open / aead_seal / SymmetricKey / GcmContext   GPU AES-256-GCM
  volume.Volume                                              reference volume format
  workload.run_training / parse_dataset / ...                GPU fp64 reference trainer
  loader.ShardLoader                                         decrypt -> normalise in HBM
  nets / trainer                                             CNN training on tcgen05 kernels
  install()                                                  patch covault to use the GPU path
"""
from __future__ import annotations

__version__ = "0.1.0"


_SAVED: list = []


def install() -> None:
    """Route the reference package's hot-path functions to the GPU implementation.

    After this, in the running process:
      covault.crypto.aead_open / aead_seal  (crypto.py:258-272)  -> GPU AES-256-GCM
      covault.volume's AEAD + blob hashing  (volume.py:161-222)  -> GPU AES-GCM + GPU SHA-256
      covault.workload.run_training         (workload.py:48-71)  -> GPU trainer (bit-exact)
      covault.gate.gate_run                 (gate.py:148-208)    -> device-resident re-encryption
    The patched names are also replaced where other covault modules imported them by name
    (scenario.py, cli.py).  ``uninstall()`` restores the originals.
    """
    import importlib
    import sys

    import covault.crypto as cc  # type: ignore
    import covault.gate as cg  # type: ignore
    import covault.volume as cv  # type: ignore
    import covault.workload as cw  # type: ignore

    from . import crypto, gate, workload

    def hash_bytes(data: bytes):
        return cc.Digest(crypto.sha256_many([data])[0])

    patches = [(cc, "aead_open", crypto.aead_open), (cc, "aead_seal", crypto.aead_seal),
               (cv, "aead_open", crypto.aead_open), (cv, "aead_seal", crypto.aead_seal),
               (cv, "hash_bytes", hash_bytes), (cw, "run_training", workload.run_training),
               (cg, "gate_run", gate.gate_run)]
    for name in ("covault.scenario", "covault.cli"):
        mod = sys.modules.get(name) or importlib.import_module(name)
        patches.append((mod, "gate_run", gate.gate_run))
    for mod, attr, fn in patches:
        if getattr(mod, attr) is not fn:
            _SAVED.append((mod, attr, getattr(mod, attr)))
            setattr(mod, attr, fn)


def uninstall() -> None:
    """Undo install()."""
    while _SAVED:
        mod, attr, fn = _SAVED.pop()
        setattr(mod, attr, fn)
