"""Accuracy of the tcgen05 gather GEMM vs an fp64 product, per reduction
length K, in tf32 and 3xTF32 (precision 1) modes (libsntest.so hook)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_1801_04380_b200 import _native  # noqa: E402

lib = _native.testing()
lib.sn_test_gemm.restype = ctypes.c_int
lib.sn_test_gemm.argtypes = [ctypes.c_int] * 3 + [ctypes.c_void_p] * 3 + [ctypes.c_int] * 6
dev = torch.device("cuda:0")
M, N = 256, 128
for dist in ("randn", "positive"):
    for K in (32, 64, 128, 256, 512, 1024, 2048, 4096, 16384):
        g = torch.Generator().manual_seed(K)
        A = torch.randn(M, K, generator=g)
        B = torch.randn(N, K, generator=g)
        if dist == "positive":
            A, B = A.abs(), B.abs()
        ref = A.double() @ B.double().T
        row = [dist, K]
        for prec in (0, 1):
            for splits in (1, 4):
                D = torch.zeros((splits, M, N), device=dev)
                lib.sn_test_set_precision(prec)
                Ad, Bd = A.to(dev), B.to(dev)  # keep them alive across the call
                rc = lib.sn_test_gemm(0, 0, 128, Ad.data_ptr(), Bd.data_ptr(), D.data_ptr(),
                                      M, N, K, K, K, splits)
                torch.cuda.synchronize()
                lib.sn_test_set_precision(0)
                assert rc == 0
                d = D.sum(0).cpu().double()
                err = ((d - ref).norm() / ref.norm()).item()
                bias = ((d - ref).sum() / ref.abs().sum()).item()
                row += [f"p{prec}s{splits} err {err:.2e} bias {bias:+.1e}"]
        cpu = (A @ B.T).double()
        row += [f"cpu32 {((cpu - ref).norm() / ref.norm()).item():.2e}"]
        print(*row, flush=True)
