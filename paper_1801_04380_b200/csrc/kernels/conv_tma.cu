// TMA-fed tcgen05 implicit-GEMM convolutions (forward, stride-1 dgrad, wgrad).
//
// One elected thread (warp 4) drives the operand pipeline with
// cp.async.bulk.tensor: the activation operand through the TMA im2col mode
// (the hardware walks output pixels in N,P,Q order, applies stride, padding
// and the filter-tap offset, and zero-fills the halo), the other operand
// through a tiled 2-D tensor map.  One elected thread (warp 5) issues the
// tcgen05.mma chain into TMEM; warps 0-3 drain TMEM in the epilogue.
//
//   MODE 0  D[pixels][k] = im2col(x)[pixels][(r,s,c)] . w[k][(r,s,c)]^T
//           A K-major (128 pixels x 128 B per TMA, SWIZZLE_128B), B K-major
//           (forward; and stride-1 dgrad as a forward conv over dy with the
//           flipped, transposed filter and padding R-1-pad)
//   MODE 1  D[(r,s,c)][k] = sum_pixels im2col(x)[pixels][(r,s,c)] dy[pixels][k]
//           A and B MN-major: 32 pixel rows x 32 elements per TMA box with
//           SWIZZLE_128B_ATOM_32B, the tf32 MN-major UMMA layout
//           (wgrad, split-K partials reduced in a fixed order)
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "gemm_tc.cuh"
#include "kernels.hpp"

namespace sn {
namespace {

struct FastDivT {
  uint32_t mul = 1, shift = 0;
  FastDivT() = default;
  explicit FastDivT(uint32_t div) {
    uint32_t l = 0;
    while ((1ull << l) < div) ++l;
    shift = l;
    mul = static_cast<uint32_t>(((1ull << 32) * ((1ull << l) - div)) / div + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, mul) + n) >> shift; }
};

struct TmaArgs {
  int num_kb, kb_per_split;
  // MODE 0 (per k block: tap = kb / cchunks, c chunk = kb % cchunks)
  int cchunks, S, P, Q, PQ, stride, pad, pad_w;
  FastDivT fcc, fS, fPQ, fQ;
  // MODE 1
  int C, RSC, Kout, NPQ;
  FastDivT fC;
};

constexpr int kTmaThreads = 192;

template <int BN, int STAGES>
struct TmaSmem {
  static constexpr int A_BYTES = kBM * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int BAR_OFF = STAGES * (A_BYTES + B_BYTES);
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
};

// Epilogue: TMEM -> registers (+bias) -> SWIZZLE_128B smem chunks of 128 x 32
// fp32 -> one TMA bulk store per chunk (plain, reduce-add, or into the 3-D
// [split][M][N] partial tensor).  Rows/columns past the tensor are clipped by
// the TMA unit, so no predication is needed.
struct EpiArgs {
  const float* bias;  // per output column, may be null
  int N;              // valid columns
  int reduce;         // 1: out += tile (cp.reduce.async.bulk .add), 0: out = tile
  int partial3d;      // 1: tmD is [splits][M][N], coordinate z = blockIdx.z
  // Scatter mode (strided dgrad phases): GEMM row m = (n, u, v) of the phase
  // grid lands at dx[n][(u+t0)*st+ph-pad][(v+v0)*st+pw-pad][:] (direct stores).
  float* scatter;     // null: TMA store path
  int M, Uhw, Uw, t0, v0, st, ph, pw, pad, H, W;
  FastDivT fUhw, fUw;
};

template <int BN, int STAGES, int MODE>
__global__ void __launch_bounds__(kTmaThreads, (BN <= 128 ? 2 : 1))
    tc_conv_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const __grid_constant__ CUtensorMap tmD, TmaArgs a, EpiArgs e) {
  using L = TmaSmem<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * L::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * kBM, n0 = blockIdx.y * BN;
  const int kb0 = blockIdx.z * a.kb_per_split;
  const int nkb = min(a.num_kb, kb0 + a.kb_per_split) - kb0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc(tmem_slot, tmem_cols<BN>());
  if (warp == 4 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      if (MODE == 0) {
        const int n = static_cast<int>(a.fPQ.div(m0));
        const int pq = m0 - n * a.PQ;
        const int p = static_cast<int>(a.fQ.div(pq));
        const int q = pq - p * a.Q;
        const int w0 = q * a.stride - a.pad_w, h0 = p * a.stride - a.pad;
        for (int i = 0; i < nkb; ++i) {
          const int s = i % STAGES;
          if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
          const int kb = kb0 + i;
          const int tap = static_cast<int>(a.fcc.div(kb));
          const int cc = kb - tap * a.cchunks;
          const int r = static_cast<int>(a.fS.div(tap));
          const int t = tap - r * a.S;
          mbar_arrive_expect_tx(&full[s], L::A_BYTES + L::B_BYTES);
          tma_load_im2col_4d(smem_u32(sA + s * L::A_BYTES), &tmA, &full[s], cc * 32, w0, h0, n,
                             static_cast<uint16_t>(t), static_cast<uint16_t>(r));
          tma_load_2d(smem_u32(sB + s * L::B_BYTES), &tmB, &full[s], kb * kBK, n0);
        }
      } else {
        int ac[4], ar[4], as[4], na = 0;
        for (int g = 0; g < 4; ++g) {
          const int rsc0 = m0 + 32 * g;
          if (rsc0 >= a.RSC) break;
          const int tap = static_cast<int>(a.fC.div(rsc0));
          ac[g] = rsc0 - tap * a.C;
          ar[g] = static_cast<int>(a.fS.div(tap));
          as[g] = tap - ar[g] * a.S;
          ++na;
        }
        int nb = 0;
        for (int j = 0; j < BN / 32; ++j)
          if (n0 + 32 * j < a.Kout) ++nb;
        for (int i = 0; i < nkb; ++i) {
          const int s = i % STAGES;
          if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
          const int pix = (kb0 + i) * kBK;
          const int n = static_cast<int>(a.fPQ.div(pix));
          const int pq = pix - n * a.PQ;
          const int p = static_cast<int>(a.fQ.div(pq));
          const int q = pq - p * a.Q;
          const int w0 = q * a.stride - a.pad, h0 = p * a.stride - a.pad;
          mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>((na + nb) * 4096));
          for (int g = 0; g < na; ++g)
            tma_load_im2col_4d(smem_u32(sA + s * L::A_BYTES + g * 4096), &tmA, &full[s], ac[g], w0, h0, n,
                               static_cast<uint16_t>(as[g]), static_cast<uint16_t>(ar[g]));
          for (int j = 0; j < nb; ++j)
            tma_load_2d(smem_u32(sB + s * L::B_BYTES + j * 4096), &tmB, &full[s], n0 + 32 * j, pix);
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc = idesc_tf32(kBM, BN, MODE == 1, MODE == 1);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        mbar_wait(&full[s], (i / STAGES) & 1);
        tc_fence_after();
        const uint32_t a0 = smem_u32(sA + s * L::A_BYTES);
        const uint32_t b0 = smem_u32(sB + s * L::B_BYTES);
#pragma unroll
        for (int kk = 0; kk < kBK / 8; ++kk) {
          uint64_t ad, bd;
          if (MODE == 0) {
            ad = umma_desc(a0 + kk * 32, 16, 1024, kLayoutSW128);
            bd = umma_desc(b0 + kk * 32, 16, 1024, kLayoutSW128);
          } else {
            // 8 k rows = two 4-row K atoms (512 B each); MN atoms 4 KB apart
            ad = umma_desc(a0 + kk * 1024, 4096, 512, kLayoutSW128Base32);
            bd = umma_desc(b0 + kk * 1024, 4096, 512, kLayoutSW128Base32);
          }
          umma_tf32(tmem, ad, bd, idesc, (i | kk) != 0 ? 1u : 0u);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(done);
    }
  } else {
    // ---------------- epilogue (warps 0-3 own TMEM lanes 32w..32w+31) ----------------
    mbar_wait(done, 0);
    tc_fence_after();
    // All MMAs (hence all operand loads) are complete: the stage buffers are free.
    const uint32_t row = warp * 32 + lane;
    const uint32_t stage0 = smem_u32(smem);
    if (e.scatter) {
      // strided-dgrad phase: each row goes to its interleaved place in dx
      const int m = m0 + static_cast<int>(row);
      float* dst = nullptr;
      if (m < e.M) {
        const int n = static_cast<int>(e.fUhw.div(static_cast<uint32_t>(m)));
        const int uv = m - n * e.Uhw;
        const int u = static_cast<int>(e.fUw.div(static_cast<uint32_t>(uv)));
        const int v = uv - u * e.Uw;
        const int h = (u + e.t0) * e.st + e.ph - e.pad;
        const int w = (v + e.v0) * e.st + e.pw - e.pad;
        dst = e.scatter + (static_cast<size_t>(n * e.H + h) * e.W + w) * e.N;
      }
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        float v[32];
        tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(c), v);
        if (dst) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            if (n0 + c + j >= e.N) break;
            float4* p = reinterpret_cast<float4*>(dst + n0 + c + j);
            float4 o = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            if (e.reduce) {
              const float4 old = *p;
              o.x += old.x; o.y += old.y; o.z += old.z; o.w += old.w;
            }
            *p = o;
          }
        }
      }
      tc_fence_before();
    } else {
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      float v[32];
      tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(c), v);
      if (e.bias) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (n0 + c + j < e.N) v[j] += __ldg(e.bias + n0 + c + j);
      }
      const uint32_t chunk = stage0 + static_cast<uint32_t>(c / 32) * (kBM * 128);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(chunk + sw128_off(row, j)), "f"(v[4 * j]),
                     "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                     : "memory");
    }
    tc_fence_before();
    fence_proxy_async();
    named_bar(1, 128);
    if (threadIdx.x == 0) {
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        if (n0 + c >= e.N) break;
        const uint32_t chunk = stage0 + static_cast<uint32_t>(c / 32) * (kBM * 128);
        if (e.partial3d)
          tma_store_3d(&tmD, chunk, n0 + c, m0, blockIdx.z);
        else
          tma_store_2d(&tmD, chunk, n0 + c, m0, e.reduce != 0);
      }
      bulk_commit();
      bulk_wait_all();
    }
    }  // TMA store path
  }
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(tmem, tmem_cols<BN>());
  }
}

// ---------------------------------------------------------------------------
// Host: driver entry points for tensor-map encoding (no -lcuda link).

PFN_cuTensorMapEncodeTiled_v12000 g_encode_tiled = nullptr;
PFN_cuTensorMapEncodeIm2col_v12000 g_encode_im2col = nullptr;
std::once_flag g_once;

bool load_encoders() {
  std::call_once(g_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode_tiled = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode_im2col = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(fn);
  });
  return g_encode_tiled && g_encode_im2col;
}

// NHWC activation [N][H][W][C] as an im2col map.
bool make_im2col(CUtensorMap* m, const float* base, int N, int H, int W, int C, int lower_h, int lower_w, int upper_h,
                 int upper_w, int stride, int pixels, CUtensorMapSwizzle sw) {
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                        static_cast<cuuint64_t>(N)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(C) * 4, static_cast<cuuint64_t>(W) * C * 4,
                           static_cast<cuuint64_t>(H) * W * C * 4};
  int lower[2] = {lower_w, lower_h};
  int upper[2] = {upper_w, upper_h};
  cuuint32_t estr[4] = {1, static_cast<cuuint32_t>(stride), static_cast<cuuint32_t>(stride), 1};
  return g_encode_im2col(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, lower, upper,
                         32, static_cast<cuuint32_t>(pixels), estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Row-major matrix [rows][cols] with a box of {32 cols, box_rows rows}.
bool make_tiled(CUtensorMap* m, const float* base, int64_t rows, int64_t cols, int box_rows, CUtensorMapSwizzle sw) {
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 4};
  cuuint32_t box[2] = {32, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  return g_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Output [rows][cols] (2-D) or [splits][rows][cols] (3-D) store map, box 32 x 128.
bool make_store(CUtensorMap* m, float* base, int64_t rows, int64_t cols, int splits) {
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows),
                        static_cast<cuuint64_t>(splits)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(cols) * 4, static_cast<cuuint64_t>(cols) * rows * 4};
  cuuint32_t box[3] = {32, static_cast<cuuint32_t>(kBM), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return g_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, splits > 0 ? 3 : 2, base, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN>
constexpr int stages_for() {
  return BN <= 64 ? 4 : (BN <= 128 ? 3 : 4);  // BN <= 128: two CTAs per SM (96 KB each)
}

template <int BN, int MODE>
cudaError_t launch(const CUtensorMap& A, const CUtensorMap& B, const CUtensorMap& D, const TmaArgs& a,
                   const EpiArgs& e, int M, int N, int splits, cudaStream_t st) {
  constexpr int STAGES = stages_for<BN>();
  using L = TmaSmem<BN, STAGES>;
  static_assert(BN * 512 <= STAGES * (kBM * 128 + BN * 128), "epilogue staging must fit in the stage buffers");
  auto kern = tc_conv_tma_kernel<BN, STAGES, MODE>;
  static bool attr = false;
  if (!attr) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
    if (err != cudaSuccess) return err;
    attr = true;
  }
  TmaArgs args = a;
  const int kps = (a.num_kb + splits - 1) / splits;
  args.kb_per_split = kps;
  dim3 grid((M + kBM - 1) / kBM, (N + BN - 1) / BN, (a.num_kb + kps - 1) / kps);
  kern<<<grid, kTmaThreads, L::TOTAL, st>>>(A, B, D, args, e);
  return cudaGetLastError();
}

int bn_for(int n) { return n <= 64 ? 64 : (n <= 128 ? 128 : 256); }

}  // namespace

bool conv_tma_ok_fwd(const ConvShape& s) { return s.C % 32 == 0 && load_encoders(); }
bool conv_tma_ok_dgrad(const ConvShape& s) {
  return s.stride == 1 && s.K % 32 == 0 && s.H == s.P && s.W == s.Q && load_encoders();
}
bool conv_tma_ok_wgrad(const ConvShape& s) { return s.C % 32 == 0 && s.K % 32 == 0 && load_encoders(); }

cudaError_t conv_fwd_tma(const ConvShape& s, const float* x, const float* w, const float* bias, float* y,
                         cudaStream_t st) {
  const int BN = bn_for(s.K);
  CUtensorMap A, B;
  if (!make_im2col(&A, x, s.N, s.H, s.W, s.C, -s.pad, -s.pad, s.pad - (s.R - 1), s.pad - (s.S - 1), s.stride, kBM,
                   CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  const int Ktot = s.R * s.S * s.C;
  if (!make_tiled(&B, w, s.K, Ktot, BN, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
  TmaArgs a{};
  a.num_kb = Ktot / kBK;
  a.cchunks = s.C / 32;
  a.S = s.S;
  a.P = s.P;
  a.Q = s.Q;
  a.PQ = s.P * s.Q;
  a.stride = s.stride;
  a.pad = s.pad;
  a.pad_w = s.pad;
  a.fcc = FastDivT(a.cchunks);
  a.fS = FastDivT(s.S);
  a.fPQ = FastDivT(a.PQ);
  a.fQ = FastDivT(s.Q);
  const int M = s.N * s.P * s.Q;
  CUtensorMap D;
  if (!make_store(&D, y, M, s.K, 0)) return cudaErrorInvalidValue;
  const EpiArgs e{bias, s.K, 0, 0};
  switch (BN) {
    case 64: return launch<64, 0>(A, B, D, a, e, M, s.K, 1, st);
    case 128: return launch<128, 0>(A, B, D, a, e, M, s.K, 1, st);
    default: return launch<256, 0>(A, B, D, a, e, M, s.K, 1, st);
  }
}

// wt_flip[c][r][s][k] = w[k][R-1-r][S-1-s][c], written by the caller.
cudaError_t conv_dgrad_tma(const ConvShape& s, const float* dy, const float* wt_flip, float* dx, int accumulate,
                           cudaStream_t st) {
  const int BN = bn_for(s.C);
  CUtensorMap A, B;
  const int padh = s.R - 1 - s.pad, padw = s.S - 1 - s.pad;
  if (!make_im2col(&A, dy, s.N, s.P, s.Q, s.K, -padh, -padw, padh - (s.R - 1), padw - (s.S - 1), 1, kBM,
                   CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  const int Ktot = s.R * s.S * s.K;
  if (!make_tiled(&B, wt_flip, s.C, Ktot, BN, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
  TmaArgs a{};
  a.num_kb = Ktot / kBK;
  a.cchunks = s.K / 32;
  a.S = s.S;
  a.P = s.H;
  a.Q = s.W;
  a.PQ = s.H * s.W;
  a.stride = 1;
  a.pad = padh;
  a.pad_w = padw;
  a.fcc = FastDivT(a.cchunks);
  a.fS = FastDivT(s.S);
  a.fPQ = FastDivT(a.PQ);
  a.fQ = FastDivT(s.W);
  const int M = s.N * s.H * s.W;
  CUtensorMap D;
  if (!make_store(&D, dx, M, s.C, 0)) return cudaErrorInvalidValue;
  const EpiArgs e{nullptr, s.C, accumulate, 0};
  switch (BN) {
    case 64: return launch<64, 0>(A, B, D, a, e, M, s.C, 1, st);
    case 128: return launch<128, 0>(A, B, D, a, e, M, s.C, 1, st);
    default: return launch<256, 0>(A, B, D, a, e, M, s.C, 1, st);
  }
}

namespace {

// Phase (ph, pw) filter of a strided dgrad, flipped and transposed:
//   wp[c][j'][i'][k] = w[k][ph + st*(Rj-1-j')][pw + st*(Si-1-i')][c]
__global__ void phase_weights_kernel(const float* __restrict__ w, float* __restrict__ wp, int K, int R, int S, int C,
                                     int st, int ph, int pw, int Rj, int Si) {
  const int64_t total = static_cast<int64_t>(C) * Rj * Si * K;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i % K);
    int64_t t = i / K;
    const int ip = static_cast<int>(t % Si);
    t /= Si;
    const int jp = static_cast<int>(t % Rj);
    const int c = static_cast<int>(t / Rj);
    const int r = ph + st * (Rj - 1 - jp), s = pw + st * (Si - 1 - ip);
    wp[i] = w[((static_cast<int64_t>(k) * R + r) * S + s) * C + c];
  }
}

__global__ void phase_zero_kernel(float* dx, int N, int H, int W, int C, int st, int ph, int pw, int pad) {
  // rows/cols of dx in phase (ph, pw) that receive no filter tap
  const int64_t total = static_cast<int64_t>(N) * H * W * C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t t = i / C;
    const int w = static_cast<int>(t % W);
    t /= W;
    const int h = static_cast<int>(t % H);
    if (((h + pad) % st) == ph && ((w + pad) % st) == pw) dx[i] = 0.f;
  }
}

}  // namespace

bool conv_tma_ok_dgrad_strided(const ConvShape& s) {
  return s.stride > 1 && s.stride <= 4 && s.K % 32 == 0 && s.R == s.S && load_encoders();
}

// Strided dgrad as stride^2 stride-1 convolutions over dy, one per output phase
// (h + pad) % st, (w + pad) % st; each writes its interleaved rows of dx.
// wt_scratch must hold K*R*S*C floats.
cudaError_t conv_dgrad_strided_tma(const ConvShape& s, const float* dy, const float* w, float* wt_scratch, float* dx,
                                   int accumulate, cudaStream_t st) {
  const int stv = s.stride;
  const int BN = bn_for(s.C);
  int64_t woff = 0;
  for (int ph = 0; ph < stv; ++ph) {
    for (int pw = 0; pw < stv; ++pw) {
      const int Rj = ph < s.R ? (s.R - ph + stv - 1) / stv : 0;
      const int Si = pw < s.S ? (s.S - pw + stv - 1) / stv : 0;
      // phase grid: t in [t0, t1] with 0 <= t*st + ph - pad < H
      const int t0 = (s.pad - ph + stv - 1) >= 0 ? (s.pad - ph + stv - 1) / stv : 0;
      const int t1 = (s.H - 1 + s.pad - ph) >= 0 ? (s.H - 1 + s.pad - ph) / stv : -1;
      const int v0 = (s.pad - pw + stv - 1) >= 0 ? (s.pad - pw + stv - 1) / stv : 0;
      const int v1 = (s.W - 1 + s.pad - pw) >= 0 ? (s.W - 1 + s.pad - pw) / stv : -1;
      const int Uh = t1 - t0 + 1, Uw = v1 - v0 + 1;
      if (Uh <= 0 || Uw <= 0) continue;
      if (Rj == 0 || Si == 0) {
        if (!accumulate) {
          phase_zero_kernel<<<1184, 256, 0, st>>>(dx, s.N, s.H, s.W, s.C, stv, ph, pw, s.pad);
          cudaError_t e = cudaGetLastError();
          if (e != cudaSuccess) return e;
        }
        continue;
      }
      float* wp = wt_scratch + woff;
      const int64_t wn = static_cast<int64_t>(s.C) * Rj * Si * s.K;
      woff += wn;
      phase_weights_kernel<<<std::min<int64_t>(1184, (wn + 255) / 256), 256, 0, st>>>(w, wp, s.K, s.R, s.S, s.C, stv,
                                                                                      ph, pw, Rj, Si);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      // im2col over dy: window origin of phase output u is u + t0 - (Rj - 1)
      const int lower_h = t0 - (Rj - 1), lower_w = v0 - (Si - 1);
      const int upper_h = Uh - s.P + lower_h, upper_w = Uw - s.Q + lower_w;
      if (lower_h < -128 || lower_h > 127 || upper_h < -128 || upper_h > 127 || lower_w < -128 || upper_w > 127)
        return cudaErrorInvalidValue;
      CUtensorMap A, B, D;
      if (!make_im2col(&A, dy, s.N, s.P, s.Q, s.K, lower_h, lower_w, upper_h, upper_w, 1, kBM,
                       CU_TENSOR_MAP_SWIZZLE_128B))
        return cudaErrorInvalidValue;
      const int Ktot = Rj * Si * s.K;
      if (!make_tiled(&B, wp, s.C, Ktot, BN, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
      std::memset(&D, 0, sizeof D);
      TmaArgs a{};
      a.num_kb = Ktot / kBK;
      a.cchunks = s.K / 32;
      a.S = Si;
      a.P = Uh;
      a.Q = Uw;
      a.PQ = Uh * Uw;
      a.stride = 1;
      a.pad = -lower_h;
      a.pad_w = -lower_w;
      a.fcc = FastDivT(a.cchunks);
      a.fS = FastDivT(Si);
      a.fPQ = FastDivT(a.PQ);
      a.fQ = FastDivT(Uw);
      const int M = s.N * Uh * Uw;
      EpiArgs ep{};
      ep.N = s.C;
      ep.reduce = accumulate;
      ep.scatter = dx;
      ep.M = M;
      ep.Uhw = Uh * Uw;
      ep.Uw = Uw;
      ep.t0 = t0;
      ep.v0 = v0;
      ep.st = stv;
      ep.ph = ph;
      ep.pw = pw;
      ep.pad = s.pad;
      ep.H = s.H;
      ep.W = s.W;
      ep.fUhw = FastDivT(Uh * Uw);
      ep.fUw = FastDivT(Uw);
      switch (BN) {
        case 64: e = launch<64, 0>(A, B, D, a, ep, M, s.C, 1, st); break;
        case 128: e = launch<128, 0>(A, B, D, a, ep, M, s.C, 1, st); break;
        default: e = launch<256, 0>(A, B, D, a, ep, M, s.C, 1, st); break;
      }
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

cudaError_t conv_wgrad_tma(const ConvShape& s, const float* x, const float* dy, float* partial, int splits,
                           cudaStream_t st) {
  const int BN = bn_for(s.K);
  CUtensorMap A, B;
  if (!make_im2col(&A, x, s.N, s.H, s.W, s.C, -s.pad, -s.pad, s.pad - (s.R - 1), s.pad - (s.S - 1), s.stride, 32,
                   CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
    return cudaErrorInvalidValue;
  const int NPQ = s.N * s.P * s.Q;
  if (!make_tiled(&B, dy, NPQ, s.K, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) return cudaErrorInvalidValue;
  TmaArgs a{};
  a.num_kb = (NPQ + kBK - 1) / kBK;
  a.S = s.S;
  a.P = s.P;
  a.Q = s.Q;
  a.PQ = s.P * s.Q;
  a.stride = s.stride;
  a.pad = s.pad;
  a.fS = FastDivT(s.S);
  a.fPQ = FastDivT(a.PQ);
  a.fQ = FastDivT(s.Q);
  a.C = s.C;
  a.fC = FastDivT(s.C);
  a.RSC = s.R * s.S * s.C;
  a.Kout = s.K;
  a.NPQ = NPQ;
  CUtensorMap D;
  if (!make_store(&D, partial, a.RSC, s.K, splits)) return cudaErrorInvalidValue;
  const EpiArgs e{nullptr, s.K, 0, 1};
  switch (BN) {
    case 64: return launch<64, 1>(A, B, D, a, e, a.RSC, s.K, splits, st);
    case 128: return launch<128, 1>(A, B, D, a, e, a.RSC, s.K, splits, st);
    default: return launch<256, 1>(A, B, D, a, e, a.RSC, s.K, splits, st);
  }
}

}  // namespace sn
