"""pytest plugin that runs the reference's OWN test suites against the GPU path.

Loaded with ``-p covault_gpu_plugin`` by tests/test_reference_suites_gpu.py: it calls
``paper_2103_16898_b200.install()`` before the reference test modules are imported (so their
``from covault.crypto import aead_open`` etc. bind the GPU functions), and at session end
writes how many calls each GPU entry point served to $CVB_CALLS_OUT -- the evidence that the
suites exercised the GPU path rather than passing on the CPU reference."""
import json
import os


def pytest_configure(config):
    import paper_2103_16898_b200 as pkg

    pkg.install()


def pytest_sessionfinish(session, exitstatus):
    from paper_2103_16898_b200 import crypto

    out = os.environ.get("CVB_CALLS_OUT")
    if out:
        with open(out, "w") as f:
            json.dump(dict(crypto.CALLS), f)
