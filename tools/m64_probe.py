"""Where does an M=64 tcgen05.mma (cta_group::1, tf32) put D in TMEM?"""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1801_04380_b200 import _native
lib = _native.testing()
lib.sn_probe_m64_layout.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int]
g = torch.Generator().manual_seed(0)
# A row r = e_r-ish so D[r][c] is identifiable: A[r][k] = (k == 0) * (r + 1), B[c][k] = (k == 0) * 1000 * (c + 1)... exact in tf32
A = torch.zeros(64, 32); B = torch.zeros(64, 32)
A[:, 0] = torch.arange(64) + 1.0
B[:, 0] = 1.0
B[:, 1] = 0.0
A[:, 1] = 1.0
B[:, 1] = (torch.arange(64) + 1.0) * 128.0   # D[r][c] = (r+1) + 128 (c+1)
for lane0 in (0, 16):
    out = torch.zeros(128, 64, device="cuda")
    rc = lib.sn_probe_m64_layout(A.cuda().data_ptr(), B.cuda().data_ptr(), out.data_ptr(), lane0)
    o = out.cpu()
    print(f"lane0={lane0} rc={rc}")
    for l in list(range(0, 128, 1)):
        row = o[l]
        if torch.isnan(row).all():
            continue
        dec = [(int(v) % 128 - 1, int(v) // 128 - 1) for v in row.tolist()[:4]] + ["..."] + \
              [(int(v) % 128 - 1, int(v) // 128 - 1) for v in row.tolist()[-2:]]
        if l % 8 == 0 or l % 16 == 15:
            print(f"  lane {l:3d}: (row, col) of cols 0..3, 62..63 = {dec}")
