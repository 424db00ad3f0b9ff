"""Raw tcgen05.mma (SS, bf16, M=128) issue rate per N: cycles per MMA from one thread."""
import ctypes, sys
sys.path.insert(0, '.')
from paper_2103_16898_b200 import _lib
L = _lib.load()
L.cvb_debug_mma_cycles.restype = ctypes.c_longlong
for bn in (32, 64, 128, 256):
    for iss, halo in ((1, 0), (1, 2), (3, 2), (1, 3), (1, 4), (1, 5), (1, 6), (1, 7), (1, 8), (1, 9), (1, 10)):
        n = 4096
        c = L.cvb_debug_mma_cycles(n, bn, iss, halo)
        print(f"N={bn:3d} {iss} issuer(s) A={['swizzle-128B', 'halo/no-swizzle', 'halo 3x3 sequence', 'SW128 rows, shifted 3x3', 'SW128 rows, aligned', '2 acc alternating, aligned', '2 acc alternating, shifted rows', '4 acc alternating, aligned', 'distinct tiles, aligned', 'distinct tiles, +1 row', 'halo rows pitch 16, shifted 3x3'][halo]}: {c / n:6.1f} cycles per MMA per issuer, "
              f"{c / n / min(iss, 2):6.1f} per MMA overall{' (commit every 18)' if iss == 3 else ''} (floor {128 * bn / 256:.0f})")
