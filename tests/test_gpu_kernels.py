"""Kernel-level parity of the tcgen05 GEMM core against an fp64 torch matmul.

tf32 operands (10-bit mantissa) with fp32 accumulation: the stated tolerance
is |err| <= 2e-3 * (|A| |B|^T) element-wise bound, checked here as a relative
Frobenius error below 2e-3 plus a max-abs bound scaled by sqrt(K).
"""

import ctypes

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _lib():
    from paper_1801_04380_b200 import _native
    lib = _native.executor()
    lib.sn_test_gemm.restype = ctypes.c_int
    lib.sn_test_gemm.argtypes = [ctypes.c_int] * 3 + [ctypes.c_void_p] * 3 + [ctypes.c_int] * 6
    return lib


def _check(D, ref, K):
    err = (D.double() - ref).norm() / ref.norm().clamp_min(1e-30)
    assert err.item() < 2e-3, f"relative Frobenius error {err.item():.3e}"


@pytest.mark.parametrize("bn", [64, 128, 256])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 64, 32), (300, 200, 200), (257, 96, 1000)])
def test_tc_gemm_majors(cuda, bn, a_mn, b_mn, M, N, K):
    lib = _lib()
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N * 3 + K)
    A = torch.randn(M, K, generator=g)
    B = torch.randn(N, K, generator=g)
    ref = A.double() @ B.double().T
    Ad = (A.T.contiguous() if a_mn else A).to(cuda)
    Bd = (B.T.contiguous() if b_mn else B).to(cuda)
    lda = M if a_mn else K
    ldb = N if b_mn else K
    D = torch.full((M, N), float("nan"), device=cuda)
    rc = lib.sn_test_gemm(a_mn, b_mn, bn, Ad.data_ptr(), Bd.data_ptr(), D.data_ptr(),
                          M, N, K, lda, ldb, 1)
    assert rc == 0
    _check(D.cpu(), ref, K)


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (1, 1)])
def test_tc_gemm_split_k(cuda, a_mn, b_mn):
    lib = _lib()
    lib.sn_test_effective_splits.restype = ctypes.c_int
    M, N, K, splits = 256, 128, 4096, 8
    eff = lib.sn_test_effective_splits(K, splits)
    g = torch.Generator(device="cpu").manual_seed(5)
    A = torch.randn(M, K, generator=g)
    B = torch.randn(N, K, generator=g)
    ref = A.double() @ B.double().T
    Ad = (A.T.contiguous() if a_mn else A).to(cuda)
    Bd = (B.T.contiguous() if b_mn else B).to(cuda)
    P = torch.zeros(eff, M, N, device=cuda)
    rc = lib.sn_test_gemm(a_mn, b_mn, 128, Ad.data_ptr(), Bd.data_ptr(), P.data_ptr(),
                          M, N, K, M if a_mn else K, N if b_mn else K, splits)
    assert rc == 0
    _check(P.sum(0).cpu(), ref, K)


def test_tc_gemm_unaligned_fallback(cuda):
    """ld % 4 != 0 takes the scalar smem-store path (e.g. FC out=10)."""
    lib = _lib()
    M, N, K = 50, 10, 30
    g = torch.Generator(device="cpu").manual_seed(9)
    A = torch.randn(K, M, generator=g)   # MN-major, ld = M = 50 (not % 4)
    B = torch.randn(K, N, generator=g)   # MN-major, ld = N = 10
    ref = A.double().T @ B.double()
    D = torch.zeros(M, N, device=cuda)
    Ad, Bd = A.to(cuda), B.to(cuda)
    rc = lib.sn_test_gemm(1, 1, 64, Ad.data_ptr(), Bd.data_ptr(), D.data_ptr(), M, N, K, M, N, 1)
    assert rc == 0
    _check(D.cpu(), ref, K)
