"""The trusted-boot gate with its re-encryption copy on the B200.

Drop-in for covault.gate.gate_run (/root/reference/pkg/src/covault/gate.py:148-208), installed
by ``paper_2103_16898_b200.install()``.  The platform-integrity half is unchanged and runs the
reference's own code (``tpm_device.quote``, ``verify_tpm_quote``, ``replay_log``, the result and
report types); only the copy loop (gate.py:186-192) moves to the device: ``volume.gate_copy``
opens each source blob in HBM, re-seals it there and hashes both the plaintext (copy report)
and the sealed blob (its name) with the device SHA-256 -- the plaintext never reaches host
memory.  Destination publication keeps the reference's discipline: O_EXCL gate lock, a
staging volume, self-verification, atomic rename, staging removed on any failure.
"""
from __future__ import annotations

import os
import secrets
import shutil
from pathlib import Path

from .crypto import CALLS, AuthenticationFailure
from .volume import Volume, gate_copy


def gate_run(config, tpm_device, measurement_log, source_key, dest_key):
    """Verify platform integrity, then copy source files under the destination key
    (same arguments, results and exceptions as covault.gate.gate_run)."""
    import covault.gate as ref  # the reference's integrity checks, result and error types

    CALLS["gate_run"] += 1
    # integrity first: a fresh quote over exactly the expected registers (gate.py:160-168)
    qnonce = secrets.token_bytes(ref.QUOTE_NONCE_SIZE)
    quote = tpm_device.quote(sorted(config.expected_pcrs), qnonce)
    verdict = ref.verify_tpm_quote(quote, qnonce, config.tpm_root_certs, config.expected_pcrs)
    if not verdict.ok:
        return ref.GateResult(False, verdict.reason)
    want_ima = config.expected_pcrs.get(config.ima_pcr_index)
    if want_ima is None or ref.replay_log(measurement_log, config.ima_pcr_index) != want_ima:
        return ref.GateResult(False, "log_replay_mismatch")

    final = Path(config.dest_path)
    if final.exists():
        raise ref.GateError(f"destination {final} already exists")
    final.parent.mkdir(parents=True, exist_ok=True)
    lock = final.with_name(final.name + ".gate-lock")
    try:
        lock_fd = os.open(lock, os.O_CREAT | os.O_EXCL | os.O_WRONLY)
    except FileExistsError:
        raise ref.GateError(f"another gate is publishing {final}") from None
    staging = final.with_name(final.name + f".staging-{os.getpid()}")
    try:
        source = Volume.open(config.source_path)
        dest = Volume.create(staging, config.dest_volume, dest_key)
        try:
            files = gate_copy(source, source_key, dest, dest_key)
        except AuthenticationFailure:
            return ref.GateResult(False, "volume_auth_failure")
        if dest.verify():
            raise ref.GateError("staging volume failed self-verification")
        os.rename(staging, final)
        return ref.GateResult(True, report=ref.CopyReport(source_volume=config.source_volume,
                                                           dest_volume=config.dest_volume, files=tuple(files)))
    finally:
        if staging.exists():      # an aborted copy; after the rename it is gone
            shutil.rmtree(staging, ignore_errors=True)
        os.close(lock_fd)
        lock.unlink(missing_ok=True)
