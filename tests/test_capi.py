"""The C-ABI library loads and exports every symbol include/*.h declares (no GPU needed)."""
import re
from pathlib import Path

from paper_2103_16898_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        for m in re.finditer(r"\b(cvb_[a-z0-9_]+)\s*\(", text):
            names.add(m.group(1))
    return names


def test_library_loads_and_exports_all_declared_symbols():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 12
    for n in sorted(names):
        assert hasattr(lib, n), n
        assert n in _lib.SIGNATURES, f"{n} missing from the ctypes signature table"


def test_version_and_error_string():
    lib = _lib.load()
    assert lib.cvb_version() >= 1
    assert isinstance(lib.cvb_last_error(), bytes)


def test_host_aes_key_schedule_fips197():
    # the kernels consume the host key schedule; FIPS-197 C.3 without a GPU
    import ctypes

    lib = _lib.load()
    out = ctypes.create_string_buffer(16)
    assert lib.cvb_aes256_encrypt_block_host(bytes(range(32)),
                                             bytes.fromhex("00112233445566778899aabbccddeeff"), out) == 0
    assert out.raw.hex() == "8ea2b7ca516745bfeafc49904b496089"
