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


def install() -> None:
    """Route the reference package's hot-path functions to the GPU implementation.

    After this, covault.crypto.aead_open/aead_seal, covault.volume's AEAD calls and
    covault.workload.run_training execute on the B200.
    """
    import covault.crypto as cc  # type: ignore
    import covault.volume as cv  # type: ignore
    import covault.workload as cw  # type: ignore

    from . import crypto, workload

    cc.aead_open = crypto.aead_open
    cc.aead_seal = crypto.aead_seal
    cv.aead_open = crypto.aead_open
    cv.aead_seal = crypto.aead_seal
    cw.run_training = workload.run_training
