// CONV and FC as tcgen05 GEMMs (gemm_tc.cuh) with implicit-GEMM operand
// gathers straight from the NHWC activations in the arena:
//
//   forward  D[npq][k]  = sum_{rsc} im2col(x)[npq][rsc] * w[k][rsc]      A K-major, B K-major
//   dgrad    D[nhw][c]  = sum_{rsk} dy[n, (h+pad-r)/st, (w+pad-s)/st, k]
//                                   * wt[c][rsk]                         A K-major, B K-major
//   wgrad    D[rsc][k]  = sum_{npq} im2col(x)[npq][rsc] * dy[npq][k]     A MN-major, B MN-major
//
// Padding, stride holes and tile overhang are zero-filled by cp.async with
// src-size 0, so no im2col buffer is ever materialised.  The wgrad reduction
// over N*P*Q is split across CTAs (split-K) into fp32 partials reduced in a
// fixed order by splitk_reduce (deterministic: the same split count gives
// bit-identical gradients on every replay of the schedule).
#include <algorithm>
#include <cstdlib>

#include "gemm_tc.cuh"
#include "kernels.hpp"

namespace sn {
namespace {

// n / d for n < 2^31 via multiply-high (d is a runtime constant per launch).
struct FastDiv {
  uint32_t d = 1, mul = 1, shift = 0;
  FastDiv() = default;
  explicit FastDiv(uint32_t div) : d(div) {
    uint32_t l = 0;
    while ((1ull << l) < div) ++l;
    shift = l;
    mul = static_cast<uint32_t>(((1ull << 32) * ((1ull << l) - div)) / div + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, mul) + n) >> shift; }
};

__device__ __forceinline__ void st_shared_v4(uint32_t dst, const float (&v)[4]) {
  asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(dst), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3])
               : "memory");
}

struct ConvGeomDev {
  int N, H, W, C, K, R, S, P, Q, stride, pad;
  int Ktot;  // R*S*C (fwd), R*S*K (dgrad)
  FastDiv fPQ, fQ, fC, fS, fK, fHW, fW;
};

ConvGeomDev make_geom(const ConvShape& s) {
  ConvGeomDev g;
  g.N = s.N; g.H = s.H; g.W = s.W; g.C = s.C; g.K = s.K; g.R = s.R; g.S = s.S; g.P = s.P; g.Q = s.Q;
  g.stride = s.stride; g.pad = s.pad;
  g.Ktot = s.R * s.S * s.C;
  g.fPQ = FastDiv(s.P * s.Q); g.fQ = FastDiv(s.Q); g.fC = FastDiv(s.C); g.fS = FastDiv(s.S);
  g.fK = FastDiv(s.K); g.fHW = FastDiv(s.H * s.W); g.fW = FastDiv(s.W);
  return g;
}

// ---------------------------------------------------------------------------
// forward A: rows = output pixels, k = (r, s, c)
struct FwdA {
  ConvGeomDev g;
  const float* x;
  int mode;  // 2: C % 32 == 0, 1: C % 4 == 0, 0: scalar
  int M;
  int4* rows;  // smem row table: {pixel base index n*H*W, h0, w0, valid}
  __device__ void tile_init(int m0, void* scratch, int tid) {
    rows = reinterpret_cast<int4*>(scratch);
    const int m = m0 + tid;
    int4 r = make_int4(0, -(1 << 28), -(1 << 28), 0);
    if (m < M) {
      const uint32_t n = g.fPQ.div(m);
      const uint32_t pq = m - n * (g.P * g.Q);
      const uint32_t p = g.fQ.div(pq);
      const uint32_t q = pq - p * g.Q;
      r = make_int4(static_cast<int>(n) * g.H * g.W, static_cast<int>(p) * g.stride - g.pad,
                    static_cast<int>(q) * g.stride - g.pad, 1);
    }
    rows[tid] = r;
  }
  __device__ __forceinline__ void decode(int k, int& r, int& s, int& c) const {
    const uint32_t rs = g.fC.div(k);
    c = k - static_cast<int>(rs) * g.C;
    r = static_cast<int>(g.fS.div(rs));
    s = static_cast<int>(rs) - r * g.S;
  }
  __device__ void load(uint32_t tile, int kb, int tid) {
    const int warp = tid >> 5, lane = tid & 31, chunk = lane & 7;
    const int k = kb * kBK + chunk * 4;
    if (mode >= 1) {
      int r = 0, s = 0, c = 0;
      const bool kin = k < g.Ktot;
      if (kin) decode(k, r, s, c);
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int row = warp * 32 + it * 4 + (lane >> 3);
        const int4 ri = rows[row];
        const int h = ri.y + r, w = ri.z + s;
        const bool ok = kin && ri.w && static_cast<unsigned>(h) < static_cast<unsigned>(g.H) &&
                        static_cast<unsigned>(w) < static_cast<unsigned>(g.W);
        const float* src = ok ? x + (static_cast<size_t>(ri.x + h * g.W + w) * g.C + c) : x;
        cp_async16(tile + sw128_off(row, chunk), src, ok ? 16u : 0u);
      }
    } else {
      for (int it = 0; it < 8; ++it) {
        const int row = warp * 32 + it * 4 + (lane >> 3);
        const int4 ri = rows[row];
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          v[e] = 0.f;
          if (k + e < g.Ktot && ri.w) {
            int r, s, c;
            decode(k + e, r, s, c);
            const int h = ri.y + r, w = ri.z + s;
            if (static_cast<unsigned>(h) < static_cast<unsigned>(g.H) &&
                static_cast<unsigned>(w) < static_cast<unsigned>(g.W))
              v[e] = __ldg(x + static_cast<size_t>(ri.x + h * g.W + w) * g.C + c);
          }
        }
        st_shared_v4(tile + sw128_off(row, chunk), v);
      }
    }
  }
};

// dgrad A: rows = input pixels (n, h, w), k = (r, s, kout)
struct DgradA {
  ConvGeomDev g;
  const float* dy;
  int mode;  // 1: K % 4 == 0, 0: scalar
  int M;     // N*H*W
  int4* rows;  // {n*P*Q, h+pad, w+pad, valid}
  __device__ void tile_init(int m0, void* scratch, int tid) {
    rows = reinterpret_cast<int4*>(scratch);
    const int m = m0 + tid;
    int4 r = make_int4(0, -(1 << 28), -(1 << 28), 0);
    if (m < M) {
      const uint32_t n = g.fHW.div(m);
      const uint32_t hw = m - n * (g.H * g.W);
      const uint32_t h = g.fW.div(hw);
      const uint32_t w = hw - h * g.W;
      r = make_int4(static_cast<int>(n) * g.P * g.Q, static_cast<int>(h) + g.pad, static_cast<int>(w) + g.pad, 1);
    }
    rows[tid] = r;
  }
  __device__ __forceinline__ bool tap(const int4& ri, int r, int s, int& pix) const {
    const int ph = ri.y - r, pw = ri.z - s;
    if (!ri.w || ph < 0 || pw < 0) return false;
    int p = ph, q = pw;
    if (g.stride != 1) {
      if (ph % g.stride || pw % g.stride) return false;
      p = ph / g.stride;
      q = pw / g.stride;
    }
    if (p >= g.P || q >= g.Q) return false;
    pix = ri.x + p * g.Q + q;
    return true;
  }
  __device__ __forceinline__ void decode(int k, int& r, int& s, int& ko) const {
    const uint32_t rs = g.fK.div(k);
    ko = k - static_cast<int>(rs) * g.K;
    r = static_cast<int>(g.fS.div(rs));
    s = static_cast<int>(rs) - r * g.S;
  }
  __device__ void load(uint32_t tile, int kb, int tid) {
    const int warp = tid >> 5, lane = tid & 31, chunk = lane & 7;
    const int k = kb * kBK + chunk * 4;
    const int Ktot = g.R * g.S * g.K;
    if (mode == 1) {
      int r = 0, s = 0, ko = 0;
      const bool kin = k < Ktot;
      if (kin) decode(k, r, s, ko);
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int row = warp * 32 + it * 4 + (lane >> 3);
        int pix = 0;
        const bool ok = kin && tap(rows[row], r, s, pix);
        const float* src = ok ? dy + (static_cast<size_t>(pix) * g.K + ko) : dy;
        cp_async16(tile + sw128_off(row, chunk), src, ok ? 16u : 0u);
      }
    } else {
      for (int it = 0; it < 8; ++it) {
        const int row = warp * 32 + it * 4 + (lane >> 3);
        const int4 ri = rows[row];
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          v[e] = 0.f;
          int r, s, ko, pix;
          if (k + e < Ktot) {
            decode(k + e, r, s, ko);
            if (tap(ri, r, s, pix)) v[e] = __ldg(dy + static_cast<size_t>(pix) * g.K + ko);
          }
        }
        st_shared_v4(tile + sw128_off(row, chunk), v);
      }
    }
  }
};

// wgrad A (MN-major): k rows = output pixels, mn = (r, s, c)
struct WgradA {
  ConvGeomDev g;
  const float* x;
  int mode;   // 1: C % 4 == 0, 0: scalar
  int NPQ, RSC;
  int m0;
  __device__ void tile_init(int m0_, void*, int) { m0 = m0_; }
  __device__ void load(uint32_t tile, int kb, int tid) {
    const int warp = tid >> 5, lane = tid & 31;
    const int m = m0 + lane * 4;  // this thread's 4 consecutive rsc
    int r = 0, s = 0, c = 0;
    const bool min_ok = m < RSC;
    if (min_ok) {
      const uint32_t rs = g.fC.div(m);
      c = m - static_cast<int>(rs) * g.C;
      r = static_cast<int>(g.fS.div(rs));
      s = static_cast<int>(rs) - r * g.S;
    }
#pragma unroll 2
    for (int i = 0; i < 8; ++i) {
      const int krow = warp + 4 * i;
      const int pix = kb * kBK + krow;
      const uint32_t dst = tile + mn_tile_off<kBM>(krow, lane);
      int n = 0, h0 = 0, w0 = 0;
      const bool pix_ok = pix < NPQ;
      if (pix_ok) {
        n = static_cast<int>(g.fPQ.div(pix));
        const int pq = pix - n * g.P * g.Q;
        const int p = static_cast<int>(g.fQ.div(pq));
        const int q = pq - p * g.Q;
        h0 = p * g.stride - g.pad;
        w0 = q * g.stride - g.pad;
      }
      if (mode == 1) {
        const int h = h0 + r, w = w0 + s;
        const bool ok = pix_ok && min_ok && static_cast<unsigned>(h) < static_cast<unsigned>(g.H) &&
                        static_cast<unsigned>(w) < static_cast<unsigned>(g.W);
        const float* src = ok ? x + (static_cast<size_t>((n * g.H + h) * g.W + w) * g.C + c) : x;
        cp_async16(dst, src, ok ? 16u : 0u);
      } else {
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          v[e] = 0.f;
          const int me = m + e;
          if (pix_ok && me < RSC) {
            const uint32_t rs = g.fC.div(me);
            const int ce = me - static_cast<int>(rs) * g.C;
            const int re = static_cast<int>(g.fS.div(rs));
            const int se = static_cast<int>(rs) - re * g.S;
            const int h = h0 + re, w = w0 + se;
            if (static_cast<unsigned>(h) < static_cast<unsigned>(g.H) &&
                static_cast<unsigned>(w) < static_cast<unsigned>(g.W))
              v[e] = __ldg(x + static_cast<size_t>((n * g.H + h) * g.W + w) * g.C + ce);
          }
        }
        st_shared_v4(dst, v);
      }
    }
  }
};

// D[M][N] = sum_split P[split][M][N] (+bias[n]) (+D if accumulate); optionally
// written transposed (D^T[N][M], for wgrad partials laid out [rsc][k]).
// Stage 1 of a wide split-K reduction: group g of `per` consecutive splits is
// summed (in split order) into its first split's slot, in place (each element
// is read and written by one thread only).
__global__ void splitk_group_kernel(float* P, int splits, int per, int64_t MN) {
  const int g = blockIdx.y;
  const int s0 = g * per, s1 = min(splits, s0 + per);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < MN;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float* p = P + static_cast<size_t>(s0) * MN + e;
    float acc = *p;
    int s = s0 + 1;
    // 8 loads in flight, summed in split order
    for (; s + 7 < s1; s += 8) {
      float a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = P[static_cast<size_t>(s + u) * MN + e];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += a[u];
    }
    for (; s < s1; ++s) acc += P[static_cast<size_t>(s) * MN + e];
    *p = acc;
  }
}

// sstride: distance between consecutive summed slices, in slices (1, or the
// group size after splitk_group_kernel).  A 32 x 32 output tile per block of
// 32 x 8 threads, 4 elements per thread (rows ty, ty+8, ty+16, ty+24), every
// element's slices summed from +0 in split order (the same additions as one
// thread per element).  The reduction is a chain of L2 / DRAM loads, so what
// matters is how many are in flight per SM: 4 elements x 4 slices per step
// (one element per thread and 1024-thread blocks took 29 us for the two
// 9.4 MB slices of a ResNet stage-4 3x3 weight gradient: 8 waves of blocks
// that each waited for one load round trip).
constexpr int kRedTileRows = 8;
__global__ void __launch_bounds__(32 * kRedTileRows) splitk_reduce_kernel(const float* __restrict__ P, int splits,
                                                                          int M, int N, float* D, const float* bias,
                                                                          int accumulate, int transpose, int sstride) {
  __shared__ float tile[32][33];
  const int m0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  constexpr int E = 32 / kRedTileRows;           // elements per thread
  const size_t stride = static_cast<size_t>(M) * N * sstride;
  const int n = n0 + tx;
  const float* p[E];
  bool ok[E];
  float acc[E];
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const int m = m0 + ty + kRedTileRows * j;
    ok[j] = m < M && n < N;
    p[j] = P + (ok[j] ? static_cast<size_t>(m) * N + n : 0);
    acc[j] = 0.f;
  }
  int s = 0;
  for (; s + 3 < splits; s += 4) {
    float a[E][4];
#pragma unroll
    for (int j = 0; j < E; ++j)
#pragma unroll
      for (int u = 0; u < 4; ++u) a[j][u] = ok[j] ? p[j][(s + u) * stride] : 0.f;
#pragma unroll
    for (int j = 0; j < E; ++j)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[j] += a[j][u];
  }
  for (; s < splits; ++s)
#pragma unroll
    for (int j = 0; j < E; ++j)
      if (ok[j]) acc[j] += p[j][s * stride];
#pragma unroll
  for (int j = 0; j < E; ++j) {
    if (ok[j] && bias) acc[j] += bias[n];
    tile[ty + kRedTileRows * j][tx] = acc[j];
  }
  if (!transpose) {
#pragma unroll
    for (int j = 0; j < E; ++j) {
      if (!ok[j]) continue;
      float* d = D + static_cast<size_t>(m0 + ty + kRedTileRows * j) * N + n;
      *d = accumulate ? *d + acc[j] : acc[j];
    }
    return;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const int nn = n0 + ty + kRedTileRows * j, m = m0 + tx;
    if (m < M && nn < N) {
      float* d = D + static_cast<size_t>(nn) * M + m;
      const float v = tile[tx][ty + kRedTileRows * j];
      *d = accumulate ? *d + v : v;
    }
  }
}

cudaError_t splitk_reduce_impl(const float* P, int splits, int M, int N, float* D, const float* bias, int accumulate,
                          int transpose, cudaStream_t st) {
  dim3 grid((N + 31) / 32, (M + 31) / 32), block(32, kRedTileRows);
  // Few output tiles and many splits: first sum groups of splits with the whole
  // GPU (in place), then reduce the group sums in order.
  const int64_t MN = static_cast<int64_t>(M) * N;
  const int64_t tiles = static_cast<int64_t>(grid.x) * grid.y;
  if (splits >= 16 && tiles < 4 * 148) {
    int groups = static_cast<int>(std::min<int64_t>(splits / 4, (4 * 148 + tiles - 1) / tiles));
    groups = std::max(groups, 2);
    const int per = (splits + groups - 1) / groups;
    groups = (splits + per - 1) / per;
    // one element per thread (the grid is small next to a wave only for tiny MN)
    const int bx = static_cast<int>(std::min<int64_t>((MN + 255) / 256, 65535));
    if (xskip(32)) return cudaSuccess;
    splitk_group_kernel<<<dim3(bx, groups), 256, 0, st>>>(const_cast<float*>(P), splits, per, MN);
    splitk_reduce_kernel<<<grid, block, 0, st>>>(P, groups, M, N, D, bias, accumulate, transpose, per);
    return cudaGetLastError();
  }
  if (xskip(32)) return cudaSuccess;
  splitk_reduce_kernel<<<grid, block, 0, st>>>(P, splits, M, N, D, bias, accumulate, transpose, 1);
  return cudaGetLastError();
}

// wt[c][rs'][k] = w[k][rs][c] with rs' = rs (flip = 0) or RS-1-rs (flip = 1,
// the rotated filter of the stride-1 dgrad-as-forward-convolution).
__global__ void transpose_w_kernel(const float* __restrict__ w, float* __restrict__ wt, int K, int RS, int C,
                                   int flip) {
  __shared__ float tile[32][33];
  const int rs_in = blockIdx.z;
  const int rs = flip ? RS - 1 - rs_in : rs_in;
  const int k0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int k = k0 + i, c = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (k < K && c < C) ? w[(static_cast<size_t>(k) * RS + rs_in) * C + c] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int c = c0 + i, k = k0 + threadIdx.x;
    if (k < K && c < C) wt[(static_cast<size_t>(c) * RS + rs) * K + k] = tile[threadIdx.x][i];
  }
}

template <int BN>
cudaError_t conv_fwd_bn(const ConvShape& s, const float* x, const float* w, const float* bias, float* y,
                        cudaStream_t st) {
  const ConvGeomDev g = make_geom(s);
  FwdA la{g, x, (s.C % 32 == 0) ? 2 : (s.C % 4 == 0 ? 1 : 0), s.N * s.P * s.Q, nullptr};
  MatKLoader<BN> lb{};
  lb.base = w; lb.rows = s.K; lb.K = g.Ktot; lb.ld = g.Ktot; lb.fast = (g.Ktot % 4 == 0);
  EpiStore e{y, bias, la.M, s.K, s.K, 0};
  return launch_tc_gemm<BN, 4, false, false>(la, lb, e, la.M, s.K, g.Ktot, 1, st);
}

template <int BN>
cudaError_t conv_dgrad_bn(const ConvShape& s, const float* dy, const float* wt, float* dx, int accumulate,
                          cudaStream_t st) {
  const ConvGeomDev g = make_geom(s);
  const int Ktot = s.R * s.S * s.K;
  DgradA la{g, dy, (s.K % 4 == 0) ? 1 : 0, s.N * s.H * s.W, nullptr};
  MatKLoader<BN> lb{};
  lb.base = wt; lb.rows = s.C; lb.K = Ktot; lb.ld = Ktot; lb.fast = (Ktot % 4 == 0);
  EpiStore e{dx, nullptr, la.M, s.C, s.C, accumulate};
  return launch_tc_gemm<BN, 4, false, false>(la, lb, e, la.M, s.C, Ktot, 1, st);
}

template <int BN>
cudaError_t conv_wgrad_bn(const ConvShape& s, const float* x, const float* dy, float* partial, int splits,
                          cudaStream_t st) {
  const ConvGeomDev g = make_geom(s);
  const int NPQ = s.N * s.P * s.Q, RSC = s.R * s.S * s.C;
  WgradA la{g, x, (s.C % 4 == 0) ? 1 : 0, NPQ, RSC, 0};
  MatMNLoader<BN> lb{};
  lb.base = dy; lb.rows = s.K; lb.K = NPQ; lb.ld = s.K; lb.fast = (s.K % 4 == 0);
  EpiPartial e{partial, RSC, s.K};
  return launch_tc_gemm<BN, 4, true, true>(la, lb, e, RSC, s.K, NPQ, splits, st);
}

template <int BN>
cudaError_t fc_gemm_bn(int a_mn, int b_mn, const float* A, int lda, const float* B, int ldb, int M, int N, int K,
                       float* partial, int splits, cudaStream_t st) {
  EpiPartial e{partial, M, N};
  auto setK = [](auto& l, const float* p, int rows, int KK, int ld) {
    l.base = p; l.rows = rows; l.K = KK; l.ld = ld;
    l.fast = (reinterpret_cast<uintptr_t>(p) % 16 == 0) && ld % 4 == 0 && KK % 4 == 0;
  };
  auto setMN = [](auto& l, const float* p, int rows, int KK, int ld) {
    l.base = p; l.rows = rows; l.K = KK; l.ld = ld;
    l.fast = (reinterpret_cast<uintptr_t>(p) % 16 == 0) && ld % 4 == 0 && rows % 4 == 0;
  };
  if (!a_mn && !b_mn) {
    MatKLoader<kBM> la{}; MatKLoader<BN> lb{};
    setK(la, A, M, K, lda); setK(lb, B, N, K, ldb);
    return launch_tc_gemm<BN, 4, false, false>(la, lb, e, M, N, K, splits, st);
  }
  if (!a_mn && b_mn) {
    MatKLoader<kBM> la{}; MatMNLoader<BN> lb{};
    setK(la, A, M, K, lda); setMN(lb, B, N, K, ldb);
    return launch_tc_gemm<BN, 4, false, true>(la, lb, e, M, N, K, splits, st);
  }
  MatMNLoader<kBM> la{}; MatMNLoader<BN> lb{};
  setMN(la, A, M, K, lda); setMN(lb, B, N, K, ldb);
  return launch_tc_gemm<BN, 4, true, true>(la, lb, e, M, N, K, splits, st);
}

cudaError_t fc_gemm(int a_mn, int b_mn, const float* A, int lda, const float* B, int ldb, int M, int N, int K,
                    float* partial, int splits, cudaStream_t st) {
  if (N <= 64) return fc_gemm_bn<64>(a_mn, b_mn, A, lda, B, ldb, M, N, K, partial, splits, st);
  if (N <= 128 || gemm_precision() == 1) return fc_gemm_bn<128>(a_mn, b_mn, A, lda, B, ldb, M, N, K, partial, splits, st);
  return fc_gemm_bn<256>(a_mn, b_mn, A, lda, B, ldb, M, N, K, partial, splits, st);
}

// tile width of the gather GEMMs; the fp32-faithful mode stays at <= 128, where
// two TMEM partial accumulators fit beside the running sum (gemm_tc.cuh)
int bn_for(int n) { return n <= 64 ? 64 : ((n <= 128 || gemm_precision() == 1) ? 128 : 256); }

}  // namespace

cudaError_t splitk_reduce(const float* P, int splits, int M, int N, float* D, const float* bias, int accumulate,
                          int transpose, cudaStream_t st) {
  return splitk_reduce_impl(P, splits, M, N, D, bias, accumulate, transpose, st);
}

static int g_use_tma = -1;  // SN_CONV_TMA=0 forces the cp.async gather path (tests, A/B)
static int g_precision = 0;  // 0 tf32, 1 fp32-faithful 3xTF32 (gather kernels only)
int gemm_precision() { return g_precision; }
void set_precision(int p) { g_precision = p ? 1 : 0; }
int precision() { return g_precision; }
bool use_tma() {
  if (g_use_tma < 0) {
    const char* v = std::getenv("SN_CONV_TMA");
    g_use_tma = (v && v[0] == '0') ? 0 : 1;
  }
  // the 3xTF32 split lives in the generic gather kernel (gemm_tc.cuh): the
  // fp32-faithful mode routes every CONV / FC through it
  return g_use_tma == 1 && g_precision == 0;
}
void set_conv_tma(int on) { g_use_tma = on ? 1 : 0; }

cudaError_t conv_fwd(const ConvShape& s, const float* x, const float* w, const float* bias, float* y,
                     cudaStream_t st, float* stats) {
  if (use_tma() && s.stride <= 2 && conv_halo_variant(s.N, s.H, s.W, s.C, s.K, s.R, s.S, s.pad, s.P, s.Q, s.stride))
    return conv_halo(s.N, s.H, s.W, s.C, s.K, s.R, s.S, s.pad, s.P, s.Q, x, w, bias, y, 0, stats, st, s.stride);
  if (use_tma() && conv_tma_ok_fwd(s)) return conv_fwd_tma(s, x, w, bias, y, stats, st);
  if (stats) return cudaErrorInvalidValue;  // only the TMA kernels emit BN tile statistics
  switch (bn_for(s.K)) {
    case 64: return conv_fwd_bn<64>(s, x, w, bias, y, st);
    case 128: return conv_fwd_bn<128>(s, x, w, bias, y, st);
    default: return conv_fwd_bn<256>(s, x, w, bias, y, st);
  }
}

namespace {
int g_subpix = 1;
bool use_subpix(const ConvShape& s) { return g_subpix && use_tma() && conv_dgrad_subpix_ok(s); }
}  // namespace

void set_conv_subpix(int on) { g_subpix = on; }
int conv_subpix_mode() { return g_subpix; }

ConvKnobs conv_knobs() { return ConvKnobs{conv_halo_mode(), conv_pairs_mode(), conv_bn_force(), conv_subpix_mode()}; }
void set_conv_knobs(const ConvKnobs& k) {
  set_conv_halo(k.halo);
  set_conv_pairs(k.pairs);
  set_conv_bn(k.bn);
  set_conv_subpix(k.subpix);
}

int conv_dgrad_launches(const ConvShape& s, int prepped) {
  if (use_subpix(s)) return prepped ? 1 : 2;
  if (use_tma() && conv_tma_ok_dgrad_strided(s)) return 2 * s.stride * s.stride;
  return prepped ? 1 : 2;
}

bool conv_dgrad_prep_job(const ConvShape& s, const float* w, float* wt, DgradPrepJob* job) {
  const bool sub = use_subpix(s);
  if (!sub && use_tma() && conv_tma_ok_dgrad_strided(s)) return false;
  const bool tma = use_tma() && conv_tma_ok_dgrad(s);
  *job = DgradPrepJob{w, wt, s.K, s.R * s.S, s.C, tma ? 1 : 0, sub ? 1 : 0};
  return true;
}

int64_t conv_dgrad_scratch_floats(const ConvShape& s) {
  const int64_t base = static_cast<int64_t>(s.K) * s.R * s.S * s.C;
  return conv_dgrad_subpix_ok(s) ? std::max<int64_t>(base, 16ll * s.C * s.K) : base;
}

cudaError_t conv_dgrad(const ConvShape& s, const float* dy, const float* w, float* wt, float* dx, int accumulate,
                       cudaStream_t st, int prepped) {
  if (use_subpix(s)) return conv_dgrad_subpix_tma(s, dy, w, wt, dx, accumulate, st, prepped);
  if (use_tma() && conv_tma_ok_dgrad_strided(s)) return conv_dgrad_strided_tma(s, dy, w, wt, dx, accumulate, st);
  const bool tma = use_tma() && conv_tma_ok_dgrad(s);
  if (xskip(64)) return cudaSuccess;
  if (!prepped) {
    dim3 grid((s.C + 31) / 32, (s.K + 31) / 32, s.R * s.S), block(32, 8);
    transpose_w_kernel<<<grid, block, 0, st>>>(w, wt, s.K, s.R * s.S, s.C, tma ? 1 : 0);
    if (xskip(1024)) transpose_w_kernel<<<grid, block, 0, st>>>(w, wt, s.K, s.R * s.S, s.C, tma ? 1 : 0);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (tma) {
    // stride-1 dgrad = stride-1 conv of dy with the flipped filter, padding R-1-pad
    const int pd = s.R - 1 - s.pad;
    if (s.R == s.S && conv_halo_variant(s.N, s.P, s.Q, s.K, s.C, s.R, s.S, pd, s.H, s.W))
      return conv_halo(s.N, s.P, s.Q, s.K, s.C, s.R, s.S, pd, s.H, s.W, dy, wt, nullptr, dx, accumulate, nullptr, st);
    return conv_dgrad_tma(s, dy, wt, dx, accumulate, st);
  }
  switch (bn_for(s.C)) {
    case 64: return conv_dgrad_bn<64>(s, dy, wt, dx, accumulate, st);
    case 128: return conv_dgrad_bn<128>(s, dy, wt, dx, accumulate, st);
    default: return conv_dgrad_bn<256>(s, dy, wt, dx, accumulate, st);
  }
}

bool conv_wgrad_splits_fixed(const ConvShape& s) {
  return use_tma() && s.stride == 1 &&
         (conv_halo_wgrad128_ok(s.N, s.H, s.W, s.C, s.K, s.R, s.S, s.pad, s.P, s.Q) ||
          conv_halo_wgrad_ok(s.N, s.H, s.W, s.C, s.K, s.R, s.S, s.pad, s.P, s.Q));
}

int conv_wgrad_splits(const ConvShape& s, int64_t partial_floats_cap) {
  // the halo weight-gradient kernels write one partial slice per CTA (per job)
  if (use_tma() && s.stride == 1 && conv_halo_wgrad128_ok(s.N, s.H, s.W, s.C, s.K, s.R, s.S, s.pad, s.P, s.Q))
    return conv_halo_wgrad128_splits(s.C, s.K, s.R);
  if (use_tma() && s.stride == 1 && conv_halo_wgrad_ok(s.N, s.H, s.W, s.C, s.K, s.R, s.S, s.pad, s.P, s.Q))
    return conv_halo_wgrad_splits();
  const int64_t RSC = static_cast<int64_t>(s.R) * s.S * s.C;
  const int bn = bn_for(s.K);
  const int64_t tiles = ((RSC + kBM - 1) / kBM) * ((s.K + bn - 1) / bn);
  const int64_t NPQ = static_cast<int64_t>(s.N) * s.P * s.Q;
  const int64_t nkb = (NPQ + kBK - 1) / kBK;
  // Split count with the best wave fill of the persistent grid (2 resident CTAs
  // per SM for N tiles <= 128), fewest splits on ties: 54 tiles at 2 splits
  // left 40 of 148 SMs idle (Inception-style 384->384 wgrad, 73 % fill).
  const int64_t slots = 148 * (bn <= 128 ? 2 : 1);
  const int64_t per = RSC * s.K;
  auto search = [&](int64_t limit, int64_t& want, double& best) {
    const int64_t smax = std::max<int64_t>(
        1, std::min<int64_t>({limit, std::max<int64_t>(1, nkb / 8), std::max<int64_t>(1, partial_floats_cap / per)}));
    want = 1;
    best = 0.0;
    for (int64_t sp = 1; sp <= smax; ++sp) {
      const int64_t items = tiles * sp, waves = (items + slots - 1) / slots;
      const double fill = static_cast<double>(items) / static_cast<double>(waves * slots);
      if (fill > best + 0.02) {
        best = fill;
        want = sp;
      }
    }
  };
  int64_t want = 1;
  double best = 0.0;
  search(16, want, best);
  // few output tiles (a stride-2 3x3 wgrad of 64 -> 128 channels has 5): up to
  // 16 splits leave most slots idle (80 of 296 CTAs, 34 % tensor pipe) -- go
  // to 64 splits there (the partials stay a few MB)
  if (best < 0.6) search(64, want, best);
  // a single output tile (Inception's 3x3/2 stem on the 4-channel image: 36 x 32
  // weights over 2.8 M output pixels) fills at most 64 of 296 slots even then:
  // one split per slot (partials 296 x 36 x 32 floats)
  if (best < 0.6) search(slots, want, best);
  return effective_splits(static_cast<int>(NPQ), static_cast<int>(want));
}

int splitk_reduce_launches(int splits, int M, int N) {
  const int64_t tiles = static_cast<int64_t>((N + 31) / 32) * ((M + 31) / 32);
  return (splits >= 16 && tiles < 4 * 148) ? 2 : 1;  // mirrors splitk_reduce_impl
}

int conv_wgrad_launches(const ConvShape& s, int splits, bool bias) {
  const int nb = bias ? 2 : 0;  // bias_grad: column-reduction stage 1 + finish
  const int RSC = s.R * s.S * s.C;
  if (use_tma() && s.stride == 1 && conv_halo_wgrad128_ok(s.N, s.H, s.W, s.C, s.K, s.R, s.S, s.pad, s.P, s.Q))
    return 1 + splitk_reduce_launches(conv_halo_wgrad128_splits(s.C, s.K, s.R), RSC, s.K) + nb;
  if (use_tma() && s.stride == 1 && conv_halo_wgrad_ok(s.N, s.H, s.W, s.C, s.K, s.R, s.S, s.pad, s.P, s.Q))
    return (s.C / 64) * (s.K / 64) + splitk_reduce_launches(conv_halo_wgrad_splits(), RSC, s.K) + nb;
  return 1 + splitk_reduce_launches(effective_splits(s.N * s.P * s.Q, splits), RSC, s.K) + nb;
}

cudaError_t conv_wgrad(const ConvShape& s, const float* x, const float* dy, float* dw, float* db, float* partial,
                       int splits, float* red_scratch, cudaStream_t st) {
  cudaError_t e;
  splits = effective_splits(s.N * s.P * s.Q, splits);  // the count the launch will really use
  if (use_tma() && s.stride == 1 && conv_halo_wgrad128_ok(s.N, s.H, s.W, s.C, s.K, s.R, s.S, s.pad, s.P, s.Q)) {
    e = conv_halo_wgrad128(s.N, s.H, s.W, s.C, s.K, s.R, s.S, s.pad, s.P, s.Q, x, dy, partial, dw, st);
    if (e != cudaSuccess) return e;
    if (!db) return cudaSuccess;
    return bias_grad(dy, static_cast<int64_t>(s.N) * s.P * s.Q, s.K, db, red_scratch, st);
  }
  if (use_tma() && s.stride == 1 && conv_halo_wgrad_ok(s.N, s.H, s.W, s.C, s.K, s.R, s.S, s.pad, s.P, s.Q)) {
    e = conv_halo_wgrad(s.N, s.H, s.W, s.C, s.K, s.R, s.S, s.pad, s.P, s.Q, x, dy, partial, dw, st);
    if (e != cudaSuccess) return e;
    if (!db) return cudaSuccess;
    return bias_grad(dy, static_cast<int64_t>(s.N) * s.P * s.Q, s.K, db, red_scratch, st);
  }
  if (use_tma() && conv_tma_ok_wgrad(s)) {
    e = conv_wgrad_tma(s, x, dy, partial, splits, st);
  } else {
    switch (bn_for(s.K)) {
      case 64: e = conv_wgrad_bn<64>(s, x, dy, partial, splits, st); break;
      case 128: e = conv_wgrad_bn<128>(s, x, dy, partial, splits, st); break;
      default: e = conv_wgrad_bn<256>(s, x, dy, partial, splits, st); break;
    }
  }
  if (e != cudaSuccess) return e;
  const int RSC = s.R * s.S * s.C;
  e = splitk_reduce_impl(partial, splits, RSC, s.K, dw, nullptr, 0, 1, st);
  if (e != cudaSuccess) return e;
  if (!db) return cudaSuccess;  // bias gradient fused into the consuming BN's backward
  return bias_grad(dy, static_cast<int64_t>(s.N) * s.P * s.Q, s.K, db, red_scratch, st);
}

int fc_splits(int B, int I, int O, int64_t partial_floats_cap) {
  // forward: M=B, N=O, K=I ; dgrad: M=B, N=I, K=O.  Same split count for both.
  const int64_t tiles = static_cast<int64_t>((B + kBM - 1) / kBM) * ((std::max(I, O) + 255) / 256);
  const int64_t nkb = (std::min(I, O) + kBK - 1) / kBK;
  int64_t want = (2 * 148 + tiles - 1) / tiles;
  want = std::min<int64_t>(want, std::max<int64_t>(1, nkb / 4));
  want = std::min<int64_t>(want, std::max<int64_t>(1, partial_floats_cap / (static_cast<int64_t>(B) * std::max(I, O))));
  return static_cast<int>(std::max<int64_t>(1, want));
}

namespace {
// FC forward as a 1x1 convolution over B "images" of one pixel: the TMA
// im2col kernel (K-major x and w straight from HBM, bias in the epilogue, no
// split-K partials); 32 us + a 7 us reduction -> one ~8 us launch for 512->1000
ConvShape fc_as_conv(int B, int I, int O) {
  ConvShape cs{};
  cs.N = B; cs.H = 1; cs.W = 1; cs.C = I; cs.K = O; cs.R = 1; cs.S = 1; cs.P = 1; cs.Q = 1; cs.stride = 1; cs.pad = 0;
  return cs;
}
bool fc_fwd_tma_ok(int B, int I, int O) { return use_tma() && conv_tma_ok_fwd(fc_as_conv(B, I, O)) && O % 4 == 0; }
}  // namespace

int fc_fwd_launches(int B, int I, int O) { return fc_fwd_tma_ok(B, I, O) ? 1 : 2; }

cudaError_t fc_fwd(int B, int I, int O, const float* x, const float* w, const float* bias, float* y, float* partial,
                   int splits, cudaStream_t st) {
  if (fc_fwd_tma_ok(B, I, O)) return conv_fwd_tma(fc_as_conv(B, I, O), x, w, bias, y, nullptr, st);
  const int eff = effective_splits(I, splits);
  cudaError_t e = fc_gemm(0, 0, x, I, w, I, B, O, I, partial, eff, st);
  if (e != cudaSuccess) return e;
  return splitk_reduce_impl(partial, eff, B, O, y, bias, 0, 0, st);
}

cudaError_t fc_dgrad(int B, int I, int O, const float* dy, const float* w, float* dx, int accumulate, float* partial,
                     int splits, cudaStream_t st, float* wt_scratch) {
  // as the dgrad of the 1x1 convolution (w transposed once, TMA kernel, no split-K)
  const ConvShape cs = fc_as_conv(B, I, O);
  if (wt_scratch && use_tma() && conv_tma_ok_dgrad(cs)) return conv_dgrad(cs, dy, w, wt_scratch, dx, accumulate, st);
  // dx[b][i] = sum_o dy[b][o] w[o][i]: A = dy (K-major, ld O), B[i][o] = w[o][i] (MN-major, ld I)
  const int eff = effective_splits(O, splits);
  cudaError_t e = fc_gemm(0, 1, dy, O, w, I, B, I, O, partial, eff, st);
  if (e != cudaSuccess) return e;
  return splitk_reduce_impl(partial, eff, B, I, dx, nullptr, accumulate, 0, st);
}

int fc_bwd_launches(int B, int I, int O, int wsplits, bool dgrad) {
  int n = 0;
  const ConvShape cs = fc_as_conv(B, I, O);
  if (wsplits > 0 && use_tma() && conv_tma_ok_wgrad(cs)) {
    const int sp = effective_splits(B, wsplits);
    const int64_t tiles = static_cast<int64_t>((O + 31) / 32) * ((I + 31) / 32);
    n += 1 + ((sp >= 16 && tiles < 4 * 148) ? 2 : 1) + 2;  // wgrad, split-K reduction, bias (colred)
  } else {
    n += 1 + 2;  // tc_gemm wgrad, bias (colred)
  }
  if (dgrad) n += 2;  // transpose + TMA dgrad, or tc_gemm + reduction
  return n;
}

int fc_wgrad_splits(int B, int I, int O, int64_t partial_floats_cap) {
  const ConvShape cs = fc_as_conv(B, I, O);
  return (use_tma() && conv_tma_ok_wgrad(cs)) ? conv_wgrad_splits(cs, partial_floats_cap) : 0;
}

cudaError_t fc_wgrad(int B, int I, int O, const float* x, const float* dy, float* dw, float* db, float* red_scratch,
                     cudaStream_t st, float* partial, int splits) {
  // as the weight gradient of the 1x1 convolution (TMA kernel, split-K over the batch)
  const ConvShape cs = fc_as_conv(B, I, O);
  if (partial && splits > 0 && use_tma() && conv_tma_ok_wgrad(cs))
    return conv_wgrad(cs, x, dy, dw, db, partial, splits, red_scratch, st);
  // dw[o][i] = sum_b dy[b][o] x[b][i]: A[o][b] = dy (MN-major, ld O), B[i][b] = x (MN-major, ld I)
  EpiStore e{dw, nullptr, O, I, I, 0};
  MatMNLoader<kBM> la{};
  la.base = dy; la.rows = O; la.K = B; la.ld = O;
  la.fast = (reinterpret_cast<uintptr_t>(dy) % 16 == 0) && O % 4 == 0;
  cudaError_t err;
  if (I <= 64) {
    MatMNLoader<64> lb{};
    lb.base = x; lb.rows = I; lb.K = B; lb.ld = I; lb.fast = (reinterpret_cast<uintptr_t>(x) % 16 == 0) && I % 4 == 0;
    err = launch_tc_gemm<64, 4, true, true>(la, lb, e, O, I, B, 1, st);
  } else if (I <= 128 || gemm_precision() == 1) {
    MatMNLoader<128> lb{};
    lb.base = x; lb.rows = I; lb.K = B; lb.ld = I; lb.fast = (reinterpret_cast<uintptr_t>(x) % 16 == 0) && I % 4 == 0;
    err = launch_tc_gemm<128, 4, true, true>(la, lb, e, O, I, B, 1, st);
  } else {
    MatMNLoader<256> lb{};
    lb.base = x; lb.rows = I; lb.K = B; lb.ld = I; lb.fast = (reinterpret_cast<uintptr_t>(x) % 16 == 0) && I % 4 == 0;
    err = launch_tc_gemm<256, 4, true, true>(la, lb, e, O, I, B, 1, st);
  }
  if (err != cudaSuccess) return err;
  return bias_grad(dy, B, O, db, red_scratch, st);
}

}  // namespace sn
