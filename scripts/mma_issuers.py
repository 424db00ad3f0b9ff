"""Does a second MMA-issuing warp add tensor-core throughput?  cycles per MMA per issuer with
one vs two concurrently issuing warps (separate TMEM accumulators), per N and A layout."""
import ctypes, sys
sys.path.insert(0, '.')
from paper_2103_16898_b200 import _lib
L = _lib.load()
L.cvb_debug_mma_cycles.restype = ctypes.c_longlong
names = {0: "SW128 (4 tiles)", 2: "halo planes 3x3", 8: "distinct tiles aligned", 10: "halo rows pitch 16"}
for bn in (32, 64, 128):
    for halo in (0, 2, 8, 10):
        n = 4096
        c1 = L.cvb_debug_mma_cycles(n, bn, 1, halo) / n
        c2 = L.cvb_debug_mma_cycles(n, bn, 2, halo) / n
        print(f"N={bn:3d} A={names[halo]:24s}: 1 issuer {c1:6.1f} cyc/MMA; 2 issuers {c2:6.1f} cyc/MMA each "
              f"-> {c2 / 2:6.1f} per MMA overall")
