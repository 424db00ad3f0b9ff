"""The reference's own test suites, run unmodified with install() active.

Suites (copied verbatim from /root/reference/pkg/tests by scripts/install_reference.sh into
baseline/_ref/ref_pkg, which travels to the GPU box):
  test_crypto.py::TestAead      (:123-154)  AEAD round trip, every-bit-flip, AAD/nonce binding
  test_volume.py                (all)        volume format, splices, corruption, key-free verify
  test_workload.py              (:26-176)    trainer digest, parse errors, attested runs
  test_acceptance.py::test_end_to_end_three_stakeholder_scenario (:197-210)
  test_gate.py                  (all but one, below)
Deselected, with the reason: test_gate.py::TestAtomicity::test_crash_at_every_file... and
test_acceptance.py::test_gate_soundness_8_cases_and_crash_atomicity inject their crash by
monkeypatching covault.volume.Volume.put, which the device gate never calls (the plaintext
never reaches the host); the same crash-atomicity property is tested against the device
gate's own write path in tests/test_gate_gpu.py.
The plugin counts the calls each GPU entry point served; the test asserts they are non-zero."""
import json
import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
REF_PKG = ROOT / "baseline" / "_ref" / "ref_pkg"


def test_reference_suites_pass_on_the_gpu_path(tmp_path):
    if not (REF_PKG / "tests").exists():
        pytest.fail("baseline/_ref/ref_pkg missing: run scripts/install_reference.sh")
    work = tmp_path / "pkg"      # hypothesis writes .hypothesis/ into the cwd: run from a copy
    shutil.copytree(REF_PKG, work)
    args = ["tests/test_crypto.py::TestAead", "tests/test_volume.py", "tests/test_workload.py", "tests/test_gate.py",
            "tests/test_acceptance.py::test_end_to_end_three_stakeholder_scenario",
            "--deselect", "tests/test_gate.py::TestAtomicity::test_crash_at_every_file_leaves_empty_or_complete"]
    calls = tmp_path / "calls.json"
    env = dict(os.environ, CVB_CALLS_OUT=str(calls),
               PYTHONPATH=os.pathsep.join([str(ROOT / "tests"), str(ROOT), str(ROOT / "baseline" / "_ref"),
                                           os.environ.get("PYTHONPATH", "")]))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "--rootdir", str(work), "-p", "no:cacheprovider",
                        "-p", "covault_gpu_plugin",
                        *args], cwd=work, env=env, capture_output=True, text=True, timeout=900)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and " failed" not in r.stdout, tail
    assert "1 deselected" in r.stdout, tail
    served = json.loads(calls.read_text())
    for entry in ("aead_open", "aead_seal", "sha256", "run_training", "gate_run"):
        assert served.get(entry, 0) > 0, (entry, served)
