// Test hook: the tcgen05 GEMM core on plain strided matrices, for the
// kernel-level parity tests (tests/test_gpu_kernels.py).  Not on the training
// path; the executor calls the same template through its conv/FC wrappers.
#include "../kernels/gemm_tc.cuh"
#include "../kernels/kernels.hpp"

namespace {

template <int BN, bool AMN, bool BMN>
cudaError_t run(const float* A, const float* B, float* D, int M, int N, int K, int lda, int ldb,
                int splits, cudaStream_t st) {
  using LA = typename std::conditional<AMN, sn::MatMNLoader<sn::kBM>, sn::MatKLoader<sn::kBM>>::type;
  using LB = typename std::conditional<BMN, sn::MatMNLoader<BN>, sn::MatKLoader<BN>>::type;
  LA la{};
  la.base = A; la.rows = M; la.K = K; la.ld = lda;
  la.fast = (reinterpret_cast<uintptr_t>(A) % 16 == 0) && lda % 4 == 0 && (AMN ? M % 4 == 0 : K % 4 == 0);
  LB lb{};
  lb.base = B; lb.rows = N; lb.K = K; lb.ld = ldb;
  lb.fast = (reinterpret_cast<uintptr_t>(B) % 16 == 0) && ldb % 4 == 0 && (BMN ? N % 4 == 0 : K % 4 == 0);
  if (splits <= 1) {
    sn::EpiRowMajor e{D, nullptr, M, N, N, 0};
    return sn::launch_tc_gemm<BN, 4, AMN, BMN>(la, lb, e, M, N, K, 1, st);
  }
  sn::EpiPartial e{D, M, N};
  return sn::launch_tc_gemm<BN, 4, AMN, BMN>(la, lb, e, M, N, K, splits, st);
}

template <int BN>
cudaError_t run_bn(int amn, int bmn, const float* A, const float* B, float* D, int M, int N, int K,
                   int lda, int ldb, int splits, cudaStream_t st) {
  if (!amn && !bmn) return run<BN, false, false>(A, B, D, M, N, K, lda, ldb, splits, st);
  if (!amn && bmn) return run<BN, false, true>(A, B, D, M, N, K, lda, ldb, splits, st);
  if (amn && !bmn) return run<BN, true, false>(A, B, D, M, N, K, lda, ldb, splits, st);
  return run<BN, true, true>(A, B, D, M, N, K, lda, ldb, splits, st);
}

}  // namespace

// A: K-major => A[m*lda + k], MN-major => A[k*lda + m]; likewise B with n.
// D: row-major M x N (splits == 1) or [splits][M][N] partials.
extern "C" int sn_test_gemm(int a_mn, int b_mn, int bn, const float* A, const float* B, float* D,
                            int M, int N, int K, int lda, int ldb, int splits) {
  cudaError_t e;
  switch (bn) {
    case 64: e = run_bn<64>(a_mn, b_mn, A, B, D, M, N, K, lda, ldb, splits, 0); break;
    case 128: e = run_bn<128>(a_mn, b_mn, A, B, D, M, N, K, lda, ldb, splits, 0); break;
    case 256: e = run_bn<256>(a_mn, b_mn, A, B, D, M, N, K, lda, ldb, splits, 0); break;
    default: return 1;
  }
  if (e != cudaSuccess) return 4;
  e = cudaDeviceSynchronize();
  return e == cudaSuccess ? 0 : 4;
}

extern "C" int sn_test_effective_splits(int K, int splits) { return sn::effective_splits(K, splits); }

// Conv kernels on caller buffers.  shape = {N,H,W,C,K,R,S,P,Q,stride,pad}.
//   op 0 forward:  p = {x, w, bias, y}
//   op 1 dgrad:    p = {dy, w, wt_scratch, dx}, flag = accumulate
//   op 2 wgrad:    p = {x, dy, dw, db, partial, red_scratch}, flag = splits (<=0: auto)
static int g_test_sync = 1;  // 0: sn_test_conv returns after the launch (timing loops)
extern "C" void sn_test_set_sync(int on) { g_test_sync = on; }

extern "C" int sn_test_conv(int op, const int* shape, void** p, int flag) {
  sn::ConvShape s{shape[0], shape[1], shape[2], shape[3], shape[4], shape[5], shape[6],
                  shape[7], shape[8], shape[9], shape[10]};
  cudaError_t e;
  if (op == 0) {
    e = sn::conv_fwd(s, (const float*)p[0], (const float*)p[1], (const float*)p[2], (float*)p[3], 0);
  } else if (op == 1) {
    e = sn::conv_dgrad(s, (const float*)p[0], (const float*)p[1], (float*)p[2], (float*)p[3], flag, 0);
  } else {
    const int splits = flag > 0 ? flag : sn::conv_wgrad_splits(s, 64ll << 20);
    e = sn::conv_wgrad(s, (const float*)p[0], (const float*)p[1], (float*)p[2], (float*)p[3], (float*)p[4],
                       splits, (float*)p[5], 0);
  }
  if (e != cudaSuccess) return 4;
  if (!g_test_sync) return 0;
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 4;
}

// Stem path on caller buffers: raw NHWC images with c_raw channels, weights
// [K][R][S][4].  shape = {N,H,W,4,K,R,S,P,Q,stride,pad}.
//   query (p == null): returns -1 if the shape is not stem-eligible, else 0 and
//   sizes[0..2] = {padded input, weight scratch, partial} floats.
//   p = {raw, xp, w, wp_scratch, bias, y, dy, dw, db, partial, red}
extern "C" int sn_test_stem(const int* shape, int c_raw, void** p, long long* sizes) {
  sn::ConvShape s{shape[0], shape[1], shape[2], shape[3], shape[4], shape[5], shape[6],
                  shape[7], shape[8], shape[9], shape[10]};
  if (!sn::conv_stem_ok(s)) return -1;
  if (!p) {
    sizes[0] = sn::stem_padded_floats(s);
    sizes[1] = sn::stem_weight_floats(s);
    sizes[2] = sn::stem_wgrad_partial_floats(s);
    return 0;
  }
  cudaError_t e = sn::stem_pad_input(s, s.H, s.W, c_raw, s.pad, (const float*)p[0], (float*)p[1], 0);
  if (e == cudaSuccess)
    e = sn::conv_stem_fwd(s, (const float*)p[1], (const float*)p[2], (float*)p[3], (const float*)p[4], (float*)p[5], nullptr, 0);
  if (e == cudaSuccess)
    e = sn::conv_stem_wgrad(s, (const float*)p[1], (const float*)p[6], (float*)p[9], (float*)p[3], (float*)p[7],
                            (float*)p[8], (float*)p[10], 0);
  if (e != cudaSuccess) return 4;
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 4;
}

extern "C" int sn_test_wgrad_splits(const int* shape) {
  sn::ConvShape s{shape[0], shape[1], shape[2], shape[3], shape[4], shape[5], shape[6],
                  shape[7], shape[8], shape[9], shape[10]};
  return sn::conv_wgrad_splits(s, 64ll << 20);
}

extern "C" long long sn_test_red_scratch_floats(int C) { return sn::red_scratch_floats(C); }

namespace sn {
int tma_probe_overlap(const float* base);
}
extern "C" int sn_test_tma_overlap(const float* base) { return sn::tma_probe_overlap(base); }

// 1: TMA-fed conv kernels where the shape allows (default), 0: cp.async gathers.
extern "C" void sn_test_set_conv_tma(int on) { sn::set_conv_tma(on); }
extern "C" void sn_test_set_conv_pairs(int mode) { sn::set_conv_pairs(mode); }
extern "C" void sn_test_set_conv_bn(int bn) { sn::set_conv_bn(bn); }
extern "C" void sn_test_set_conv_subpix(int on) { sn::set_conv_subpix(on); }
extern "C" void sn_test_set_conv_halo(int mode) { sn::set_conv_halo(mode); }

// Pool layer kernels on caller buffers.  shape = {N,H,W,C,P,Q,K,stride,pad,mode}.
//   op 0 forward:  p = {x, y}
//   op 1 backward: p = {x, y, dy, dx, scratch}, flag = accumulate
//   op 2 query:    returns pool_scratch_bytes (bytes) / 2^0 units, clipped to int
extern "C" long long sn_test_pool(int op, const int* shape, void** p, int flag) {
  sn::PoolShape s{shape[0], shape[1], shape[2], shape[3], shape[4], shape[5], shape[6], shape[7], shape[8], shape[9]};
  if (op == 2) return sn::pool_scratch_bytes(s);
  if (op == 3) return sn::pool_bwd_kernels(s);
  if (op == 4) return sn::pool_saves_argmax(s) ? 1 : 0;
  if (op == 5) {  // forward recording the argmax, then the backward using it: p = {x, y, dy, dx, scratch, argmax}
    cudaError_t e = sn::pool_fwd(s, (const float*)p[0], (float*)p[1], 0, (uint8_t*)p[5]);
    if (e == cudaSuccess)
      e = sn::pool_bwd(s, (const float*)p[0], (const float*)p[1], (const float*)p[2], (float*)p[3], flag, p[4], 0,
                       (const uint8_t*)p[5]);
    if (e != cudaSuccess) return 4;
    return cudaDeviceSynchronize() == cudaSuccess ? 0 : 4;
  }
  cudaError_t e;
  if (op == 0)
    e = sn::pool_fwd(s, (const float*)p[0], (float*)p[1], 0);
  else
    e = sn::pool_bwd(s, (const float*)p[0], (const float*)p[1], (const float*)p[2], (float*)p[3], flag, p[4], 0);
  if (e != cudaSuccess) return 4;
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 4;
}

namespace sn {
int umma_shift_probe_run(const float* A, const float* B, float* D, int mn, int shift, int base_off);
}
extern "C" int sn_test_umma_shift(const float* A, const float* B, float* D, int mn, int shift, int base_off) {
  return sn::umma_shift_probe_run(A, B, D, mn, shift, base_off);
}

// Numeric mode of the gather GEMMs for the kernel-level tests (0 tf32, 1 3xTF32).
extern "C" void sn_test_set_precision(int p) { sn::set_precision(p); }
