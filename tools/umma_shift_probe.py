"""GPU probe: UMMA descriptors starting at a non-atom-aligned row of a
TMA-written SWIZZLE_128B tile (halo convolutions need this)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1801_04380_b200 import _native
lib = _native.testing()
lib.sn_test_umma_shift.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 3
g = torch.Generator().manual_seed(0)
B = torch.randn(64, 32, generator=g)
for mn in (0, 1):
    A = torch.randn(256, 32, generator=g) if mn == 0 else torch.randn(40, 128, generator=g)
    Ad, Bd = A.cuda(), B.cuda()
    for base_off in (0, 1):
        res = []
        for shift in range(0, 9):
            D = torch.full((128, 64), float("nan"), device="cuda")
            rc = lib.sn_test_umma_shift(Ad.data_ptr(), Bd.data_ptr(), D.data_ptr(), mn, shift, base_off)
            if mn == 0:
                ref = A[shift:shift + 128].double() @ B.double().T
            else:
                ref = A[shift:shift + 32].double().T @ B.double().T
            err = ((D.cpu().double() - ref).norm() / ref.norm()).item()
            res.append(f"{shift}:{'ok' if err < 3e-3 else 'BAD'}({err:.1e})" if rc == 0 else f"{shift}:rc{rc}")
        print(f"mn={mn} base_off={base_off}: " + " ".join(res), flush=True)
