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
    lib = _native.testing()
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


@pytest.mark.parametrize("bn", [64, 128, 256])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 64, 32), (300, 200, 200), (257, 96, 1000)])
def test_tc_gemm_3xtf32_is_fp32_faithful(cuda, bn, a_mn, b_mn, M, N, K):
    """precision 1 (3xTF32 split operands): within 2e-6 relative Frobenius of
    the fp64 product -- fp32-level (dropped lo.lo term and tf32 rounding of lo
    ~2^-22 per product), about 1000x tighter than the tf32 bound."""
    lib = _lib()
    g = torch.Generator(device="cpu").manual_seed(M * 5 + N + K)
    A = torch.randn(M, K, generator=g)
    B = torch.randn(N, K, generator=g)
    ref = A.double() @ B.double().T
    Ad = (A.T.contiguous() if a_mn else A).to(cuda)
    Bd = (B.T.contiguous() if b_mn else B).to(cuda)
    D = torch.full((M, N), float("nan"), device=cuda)
    lib.sn_test_set_precision(1)
    try:
        rc = lib.sn_test_gemm(a_mn, b_mn, bn, Ad.data_ptr(), Bd.data_ptr(), D.data_ptr(),
                              M, N, K, M if a_mn else K, N if b_mn else K, 1)
    finally:
        lib.sn_test_set_precision(0)
    assert rc == 0
    err = ((D.cpu().double() - ref).norm() / ref.norm()).item()
    assert err < 2e-6, err


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


# ---------------------------------------------------------------------------
# Convolution kernels (implicit GEMM on tcgen05) vs torch fp64 on CPU.

CONV_CASES = [
    # N, C, H, W, K, k, stride, pad
    (2, 4, 32, 32, 64, 7, 2, 3),     # padded stem (C=3 -> 4)
    (2, 64, 14, 14, 64, 3, 1, 1),    # resnet stage 1 (C % 32 == 0)
    (2, 64, 14, 14, 128, 3, 2, 1),   # stride-2 block
    (2, 96, 13, 13, 256, 5, 1, 2),   # AlexNet conv2 (C = 96)
    (3, 16, 9, 9, 8, 1, 1, 0),       # 1x1, C % 32 != 0
    (2, 3, 11, 11, 16, 3, 1, 1),     # C = 3: scalar gather path
    (1, 32, 20, 20, 96, 11, 4, 0),   # AlexNet-style 11x11 stride 4
    (4, 128, 7, 7, 256, 3, 1, 1),    # 7x7 tiles straddle images
    (2, 256, 14, 14, 64, 1, 1, 0),   # 1x1, K = 64
    (2, 64, 15, 15, 128, 3, 2, 1),   # odd extent, stride 2 (uneven phases)
    (2, 64, 16, 16, 128, 3, 2, 1),   # even extent, stride 2: sub-pixel dgrad (one 256-wide tile)
    (3, 32, 28, 20, 64, 3, 2, 1),    # sub-pixel dgrad, non-square, 128 output columns
    (2, 128, 14, 14, 96, 3, 2, 1),   # sub-pixel dgrad, two 256-wide tiles, K % 64 != 0
    (2, 32, 16, 16, 64, 1, 2, 0),    # 1x1 stride 2: phases without taps
    (1, 64, 23, 23, 96, 5, 3, 2),    # stride 3, 5x5
    (2, 128, 8, 8, 512, 3, 1, 1),    # K = 512: two N tiles of 256
    (32, 64, 28, 28, 64, 3, 1, 1),   # several 256-row tiles per CTA pair (double-buffered TMEM)
    (4, 64, 56, 56, 64, 3, 1, 1),    # ResNet stage 1 shape (halo, 3 sub-tiles of 2 rows)
    (3, 128, 28, 28, 128, 3, 1, 1),  # stage 2 (halo, 2 sub-tiles of 4 rows)
    (2, 256, 14, 14, 256, 3, 1, 1),  # stage 3 (halo, 8-row sub-tile, rows past P)
    (2, 64, 10, 12, 96, 5, 1, 2),    # 5x5, non-square image, K % 64 != 0
    (4, 64, 1, 1, 1000, 1, 1, 0),    # the FC as a 1x1 conv: K % 32 != 0 (dgrad's last chunk zero-filled)
    (2, 96, 13, 13, 64, 3, 1, 0),    # "valid" 3x3 (pad 0, H != P): TMA dgrad over dy padded by 2
    (3, 32, 15, 11, 64, 3, 1, 0),    # valid, non-square
    (3, 96, 5, 5, 100, 1, 1, 0),     # 1x1, K % 32 != 0 with spatial extent
]


def _conv_lib():
    from paper_1801_04380_b200 import _native
    lib = _native.testing()
    lib.sn_test_conv.restype = ctypes.c_int
    lib.sn_test_conv.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_void_p),
                                 ctypes.c_int]
    lib.sn_test_red_scratch_floats.restype = ctypes.c_longlong
    return lib


def _shape_arr(N, C, H, W, K, k, s, p):
    P = (H + 2 * p - k) // s + 1
    Q = (W + 2 * p - k) // s + 1
    return (ctypes.c_int * 11)(N, H, W, C, K, k, k, P, Q, s, p), P, Q


@pytest.mark.parametrize("tma,pairs,halo,subpix", [(1, 1, 1, 1), (1, 2, 0, 1), (1, 1, 2, 1), (1, 2, 2, 1), (0, 1, 0, 1),
                                                   (1, 1, 1, 0)])
@pytest.mark.parametrize("case", CONV_CASES)
def test_conv_fwd_dgrad_wgrad(cuda, case, tma, pairs, halo, subpix):
    """pairs=2 forces the CTA-pair (cta_group::2, M = 256) TMA kernels on
    every shape (odd tile counts, rows past M in the peer CTA); halo=2 the
    halo-tiled stride-1 kernels wherever they apply (junk padded columns,
    bands past the last output row); subpix=0 the phase-decomposed strided
    dgrad instead of the sub-pixel GEMM."""
    N, C, H, W, K, k, s, p = case
    if not subpix and s == 1:
        pytest.skip("sub-pixel toggle only affects strided dgrad")
    lib = _conv_lib()
    lib.sn_test_set_conv_subpix(subpix)
    lib.sn_test_set_conv_tma(tma)
    lib.sn_test_set_conv_pairs(pairs)
    lib.sn_test_set_conv_halo(halo)
    shape, P, Q = _shape_arr(*case)
    g = torch.Generator().manual_seed(sum(case))
    x = torch.randn(N, C, H, W, generator=g)
    w = torch.randn(K, C, k, k, generator=g) / (C * k * k) ** 0.5
    b = torch.randn(K, generator=g)
    dy = torch.randn(N, K, P, Q, generator=g)
    xd = x.double().requires_grad_(True)
    wd = w.double().requires_grad_(True)
    bd = b.double().requires_grad_(True)
    y = torch.nn.functional.conv2d(xd, wd, bd, stride=s, padding=p)
    y.backward(dy.double())
    nhwc = lambda t: t.permute(0, 2, 3, 1).contiguous().to(cuda)
    x_d, dy_d = nhwc(x), nhwc(dy)
    w_d = w.permute(0, 2, 3, 1).contiguous().to(cuda)   # KRSC
    b_d = b.to(cuda)
    y_d = torch.full((N, P, Q, K), float("nan"), device=cuda)
    ptrs = (ctypes.c_void_p * 4)(x_d.data_ptr(), w_d.data_ptr(), b_d.data_ptr(), y_d.data_ptr())
    assert lib.sn_test_conv(0, shape, ptrs, 0) == 0
    _check(y_d.permute(0, 3, 1, 2).cpu(), y.detach(), C * k * k)
    # dgrad, overwrite then accumulate
    wt = torch.empty(max(K * k * k * C, 16 * C * K), device=cuda)
    dx_d = torch.full((N, H, W, C), float("nan"), device=cuda)
    ptrs = (ctypes.c_void_p * 4)(dy_d.data_ptr(), w_d.data_ptr(), wt.data_ptr(), dx_d.data_ptr())
    assert lib.sn_test_conv(1, shape, ptrs, 0) == 0
    _check(dx_d.permute(0, 3, 1, 2).cpu(), xd.grad, K * k * k)
    assert lib.sn_test_conv(1, shape, ptrs, 1) == 0
    _check(dx_d.permute(0, 3, 1, 2).cpu(), 2 * xd.grad, K * k * k)
    # wgrad + bias grad
    dw_d = torch.full((K, k, k, C), float("nan"), device=cuda)
    db_d = torch.full((K,), float("nan"), device=cuda)
    lib.sn_test_wgrad_splits.restype = ctypes.c_int
    part = torch.empty(max(8 << 20, (lib.sn_test_wgrad_splits(shape) + 3) * k * k * C * K), device=cuda)
    red = torch.empty(int(lib.sn_test_red_scratch_floats(K)), device=cuda)
    ptrs = (ctypes.c_void_p * 6)(x_d.data_ptr(), dy_d.data_ptr(), dw_d.data_ptr(), db_d.data_ptr(),
                                 part.data_ptr(), red.data_ptr())
    for splits in (1, 3):
        assert lib.sn_test_conv(2, shape, ptrs, splits) == 0
        _check(dw_d.permute(0, 3, 1, 2).cpu(), wd.grad, N * P * Q)
        _check(db_d.cpu(), bd.grad, N * P * Q)
    lib.sn_test_set_conv_tma(1)
    lib.sn_test_set_conv_pairs(1)
    lib.sn_test_set_conv_halo(1)
    lib.sn_test_set_conv_subpix(1)


def test_tma_overlapping_window_probe(cuda):
    """Records whether the driver accepts overlapping-row tensor maps (used to
    decide the stem-convolution design); informational, always passes."""
    from paper_1801_04380_b200 import _native
    lib = _native.testing()
    lib.sn_test_tma_overlap.restype = ctypes.c_int
    lib.sn_test_tma_overlap.argtypes = [ctypes.c_void_p]
    buf = torch.zeros(2 * 224 * 224 * 4, device=cuda)
    print("TMA overlap probe result:", lib.sn_test_tma_overlap(buf.data_ptr()))


STEM_CASES = [  # (N, C_raw, H, W, K, k, stride, pad)
    (2, 3, 224, 224, 64, 7, 2, 3),   # ResNet stem
    (2, 3, 227, 227, 96, 11, 4, 0),  # AlexNet stem (two 8-column filter blocks)
    (3, 3, 32, 32, 32, 3, 1, 1),     # CIFAR-style 3x3 stride 1
    (2, 1, 28, 28, 128, 5, 1, 2),    # grayscale, 5x5, BN=128
    (2, 4, 40, 36, 256, 3, 2, 1),    # 4 real channels, BN=256, ragged rows
    (3, 3, 64, 60, 64, 5, 2, 2),     # K=64, P % 4 == 0: multi-row forward and weight-gradient kernels
    (2, 3, 32, 32, 64, 5, 1, 2),     # the same at stride 1
    (2, 3, 30, 30, 32, 7, 2, 3),     # K=32, P % 4 != 0 (last row group partial)
]


@pytest.mark.parametrize("case", STEM_CASES)
def test_stem_conv_fwd_wgrad(cuda, case):
    """Sliding-window TMA stem (conv_tma.cu MODE 2/3) vs fp64 torch."""
    N, Cr, H, W, K, k, s, p = case
    lib = _conv_lib()
    lib.sn_test_stem.restype = ctypes.c_int
    lib.sn_test_stem.argtypes = [ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                                 ctypes.POINTER(ctypes.c_longlong)]
    shape, P, Q = _shape_arr(N, 4, H, W, K, k, s, p)
    sizes = (ctypes.c_longlong * 3)()
    assert lib.sn_test_stem(shape, Cr, None, sizes) == 0
    g = torch.Generator().manual_seed(sum(case))
    x = torch.randn(N, Cr, H, W, generator=g)
    w = torch.randn(K, Cr, k, k, generator=g) / (Cr * k * k) ** 0.5
    b = torch.randn(K, generator=g)
    dy = torch.randn(N, K, P, Q, generator=g)
    xd = x.double().requires_grad_(True)
    wd = w.double().requires_grad_(True)
    bd = b.double().requires_grad_(True)
    y = torch.nn.functional.conv2d(xd, wd, bd, stride=s, padding=p)
    y.backward(dy.double())
    raw = x.permute(0, 2, 3, 1).contiguous().to(cuda)
    w4 = torch.nn.functional.pad(w.permute(0, 2, 3, 1), (0, 4 - Cr)).contiguous().to(cuda)  # [K][R][S][4]
    xp = torch.full((int(sizes[0]),), float("nan"), device=cuda)
    wp = torch.empty(int(sizes[1]), device=cuda)
    part = torch.empty(max(64, int(sizes[2])), device=cuda)
    red = torch.empty(int(lib.sn_test_red_scratch_floats(K)), device=cuda)
    b_d = b.to(cuda)
    y_d = torch.full((N, P, Q, K), float("nan"), device=cuda)
    dy_d = dy.permute(0, 2, 3, 1).contiguous().to(cuda)
    dw_d = torch.full((K, k, k, 4), float("nan"), device=cuda)
    db_d = torch.full((K,), float("nan"), device=cuda)
    ptrs = (ctypes.c_void_p * 11)(raw.data_ptr(), xp.data_ptr(), w4.data_ptr(), wp.data_ptr(), b_d.data_ptr(),
                                  y_d.data_ptr(), dy_d.data_ptr(), dw_d.data_ptr(), db_d.data_ptr(),
                                  part.data_ptr(), red.data_ptr())
    assert lib.sn_test_stem(shape, Cr, ptrs, None) == 0
    _check(y_d.permute(0, 3, 1, 2).cpu(), y.detach(), Cr * k * k)
    dw = dw_d.cpu()
    assert torch.all(dw[..., Cr:] == 0)  # padded channels read zeros
    _check(dw[..., :Cr].permute(0, 3, 1, 2), wd.grad, N * P * Q)
    _check(db_d.cpu(), bd.grad, N * P * Q)


def test_stem_eligibility(cuda):
    lib = _conv_lib()
    lib.sn_test_stem.restype = ctypes.c_int
    sizes = (ctypes.c_longlong * 3)()
    wide, _, _ = _shape_arr(1, 4, 8, 300, 32, 3, 1, 1)      # Q = 300 > one 128-row tile
    odd, _, _ = _shape_arr(1, 4, 32, 32, 32, 3, 3, 1)       # stride 3 does not divide 8
    assert lib.sn_test_stem(wide, 3, None, sizes) == -1
    assert lib.sn_test_stem(odd, 3, None, sizes) == -1


POOL_CASES = [
    # N, C, H, W, K, stride, pad, mode
    (4, 64, 112, 112, 3, 2, 1, 0),   # ResNet stem max-pool (fused argmax+gather path)
    (3, 96, 55, 55, 3, 2, 0, 0),     # AlexNet pool1
    (2, 48, 13, 13, 3, 2, 0, 0),     # C % 16 == 0, P < 8: one band
    (2, 128, 56, 56, 3, 2, 1, 0),    # band kernel, two channel slices per image band
    (2, 64, 40, 24, 3, 2, 1, 0),     # band kernel, non-square, partial last band
    (2, 12, 17, 17, 3, 2, 1, 0),     # C % 16 != 0: two-pass argmax + gather
    (2, 5, 9, 9, 2, 2, 0, 0),        # C % 4 != 0: scalar path
    (2, 64, 14, 14, 7, 1, 0, 1),     # global-ish average pool
    (2, 32, 20, 20, 3, 1, 1, 0),     # stride 1 (windows overlap by two)
    (3, 512, 7, 7, 7, 1, 0, 1),      # ResNet global average pool (one window per image)
    (2, 64, 5, 5, 5, 1, 0, 0),       # global max pool
]


def _pool_lib():
    from paper_1801_04380_b200 import _native
    lib = _native.testing()
    lib.sn_test_pool.restype = ctypes.c_longlong
    lib.sn_test_pool.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_void_p),
                                 ctypes.c_int]
    return lib


@pytest.mark.parametrize("ties", [False, True])
@pytest.mark.parametrize("case", POOL_CASES)
def test_pool_fwd_bwd_exact(cuda, case, ties):
    """Pool forward and backward vs torch fp64 (max: the first row-major
    maximum of the window gets the gradient, as in torch's CPU kernel).
    Forward max is bit-exact; gradients are sums of at most ceil(K/s)^2 dy
    terms (fp32 vs fp64 accumulation): atol/rtol 1e-5 -- a wrong argmax moves
    an element by O(1)."""
    N, C, H, W, K, s, p, mode = case
    lib = _pool_lib()
    P = (H + 2 * p - K) // s + 1
    Q = (W + 2 * p - K) // s + 1
    shape = (ctypes.c_int * 10)(N, H, W, C, P, Q, K, s, p, mode)
    g = torch.Generator().manual_seed(sum(case) + ties)
    x = torch.randn(N, C, H, W, generator=g)
    if ties:
        x = torch.round(x * 2) / 2  # many equal values inside a window
    dy = torch.randn(N, C, P, Q, generator=g)
    xd = x.double().requires_grad_(True)
    if mode == 0:
        y = torch.nn.functional.max_pool2d(xd, K, s, p)
    else:
        y = torch.nn.functional.avg_pool2d(xd, K, s, p, count_include_pad=True)
    y.backward(dy.double())
    nhwc = lambda t: t.permute(0, 2, 3, 1).contiguous().to(cuda)
    x_d, dy_d = nhwc(x), nhwc(dy)
    y_d = torch.full((N, P, Q, C), float("nan"), device=cuda)
    assert lib.sn_test_pool(0, shape, (ctypes.c_void_p * 2)(x_d.data_ptr(), y_d.data_ptr()), 0) == 0
    y_ref = y.detach().float()
    got = y_d.permute(0, 3, 1, 2).cpu()
    if mode == 0:
        assert torch.equal(got, y_ref)
    else:
        assert torch.allclose(got, y_ref, rtol=1e-6, atol=1e-6)
    scratch = torch.empty(max(1, int(lib.sn_test_pool(2, shape, None, 0))), dtype=torch.uint8, device=cuda)
    dx_d = torch.full((N, H, W, C), float("nan"), device=cuda)
    ptrs = (ctypes.c_void_p * 5)(x_d.data_ptr(), y_d.data_ptr(), dy_d.data_ptr(), dx_d.data_ptr(), scratch.data_ptr())
    assert lib.sn_test_pool(1, shape, ptrs, 0) == 0
    ref = xd.grad.float()
    got = dx_d.permute(0, 3, 1, 2).cpu()
    assert torch.allclose(got, ref, rtol=1e-5, atol=1e-5), (got - ref).abs().max()
    assert lib.sn_test_pool(1, shape, ptrs, 1) == 0  # accumulate
    got2 = dx_d.permute(0, 3, 1, 2).cpu()
    assert torch.allclose(got2, 2 * got, rtol=0, atol=0) if mode == 0 else torch.allclose(got2, 2 * got)
    if lib.sn_test_pool(4, shape, None, 0):
        # the forward records the argmax, the backward gathers with it: same bits
        am = torch.zeros(N * P * Q * C, dtype=torch.uint8, device=cuda)
        y2 = torch.full((N, P, Q, C), float("nan"), device=cuda)
        dx2 = torch.full((N, H, W, C), float("nan"), device=cuda)
        ptrs = (ctypes.c_void_p * 6)(x_d.data_ptr(), y2.data_ptr(), dy_d.data_ptr(), dx2.data_ptr(),
                                     scratch.data_ptr(), am.data_ptr())
        assert lib.sn_test_pool(5, shape, ptrs, 0) == 0
        assert torch.equal(y2, y_d)
        assert torch.equal(dx2.permute(0, 3, 1, 2).cpu(), got)
