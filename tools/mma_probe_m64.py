"""tcgen05.mma issue rate for M = 64 vs M = 128 (kind::tf32, K-major and
MN-major operands): is an M = 64 x N = 256 MMA as cheap per flop as
M = 128 x N = 128?"""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1801_04380_b200 import _native
lib = _native.testing()
lib.sn_probe_mma_rate_m.restype = ctypes.c_longlong
lib.sn_probe_mma_rate_m.argtypes = [ctypes.c_int] * 6
iters = 4096
for kind, name in ((0, "tf32 K-major"), (2, "tf32 MN-major")):
    for m in (64, 128):
        for n in (64, 128, 192, 256):
            cyc = lib.sn_probe_mma_rate_m(m, n, kind, iters, 1, 148)
            cpm = cyc / iters
            tf = m * n * 8 * 2 / cpm * 148 * 1.965e9 / 1e12
            print(f"{name:13s} M={m:3d} N={n:3d}: {cpm:7.1f} cyc/MMA -> {tf:7.1f} TF/s", flush=True)
