"""tcgen05.mma issue rate vs operand data and concurrency: SW128 SS, M=128, one issuer, on
one SM or on every SM at once, with zero / uninitialised / random bf16 operands."""
import ctypes
import sys

sys.path.insert(0, '.')
from paper_2103_16898_b200 import _lib  # noqa: E402

L = _lib.load()
L.cvb_debug_mma_cycles.restype = ctypes.c_longlong
for bn in (64, 128, 256):
    for mode, name in ((0, "uninit"), (12, "zeros"), (11, "random"), (100, "uninit, all SMs"),
                       (112, "zeros, all SMs"), (111, "random, all SMs")):
        n = 4096
        c = L.cvb_debug_mma_cycles(n, bn, 1, mode)
        print(f"N={bn:3d} {name:18s}: {c / n:6.1f} cycles per MMA (floor {128 * bn / 256:.0f})", flush=True)

for bn in (128, 256):
    for mode, name in ((13, "wait+fence+commit/4"), (14, "commit/4"), (15, "fence/4"), (16, "wait/4")):
        n = 4096
        c = L.cvb_debug_mma_cycles(n, bn, 1, mode)
        print(f"N={bn:3d} {name:22s}: {c / n:6.1f} cycles per MMA (floor {128 * bn / 256:.0f})", flush=True)
