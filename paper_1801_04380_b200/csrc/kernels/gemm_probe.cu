// Test hook: the tcgen05 GEMM core on plain strided matrices, for the
// kernel-level parity tests (tests/test_gpu_kernels.py).  Not on the training
// path; the executor calls the same template through its conv/FC wrappers.
#include "gemm_tc.cuh"

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
