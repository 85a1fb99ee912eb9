"""tcgen05.mma issue rate probe: cycles per MMA (M=128) by N, kind, and
number of interleaved accumulators."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1801_04380_b200 import _native
lib = _native.testing()
lib.sn_probe_mma_rate.restype = ctypes.c_longlong
lib.sn_probe_mma_rate.argtypes = [ctypes.c_int] * 5
iters = 4096
for kind, name in ((0, "tf32 K=8"), (2, "tf32 MN"), (1, "f16 K=16")):
    for n in (64, 128, 256):
        for accs in (1, 2):
            if accs * n > 512:
                continue
            for ctas in (148,):
                cyc = lib.sn_probe_mma_rate(n, kind, iters, accs, ctas)
                cpm = cyc / iters
                k = 16 if kind == 1 else 8
                tf = 128 * n * k * 2 / cpm * 148 * 1.965e9 / 1e12
                print(f"{name:9s} N={n:3d} accs={accs} ctas={ctas:3d}: {cpm:7.1f} cyc/MMA  -> {tf:7.1f} TF/s at 148 SMs x 1.965 GHz",
                      flush=True)
