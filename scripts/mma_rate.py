"""Raw tcgen05.mma (SS, bf16, M=128) issue rate per N: cycles per MMA from one thread."""
import ctypes, sys
sys.path.insert(0, '.')
from paper_2103_16898_b200 import _lib
L = _lib.load()
L.cvb_debug_mma_cycles.restype = ctypes.c_longlong
for bn in (32, 64, 128, 256):
    for iss, halo in ((1, 0), (2, 0), (1, 1)):
        n = 4096
        c = L.cvb_debug_mma_cycles(n, bn, iss, halo)
        print(f"N={bn:3d} {iss} issuer(s) A={'halo/no-swizzle' if halo else 'swizzle-128B'}: {c / n:6.1f} cycles per MMA per issuer, "
              f"{c / n / iss:6.1f} per MMA overall (floor {128 * bn / 256:.0f})")
