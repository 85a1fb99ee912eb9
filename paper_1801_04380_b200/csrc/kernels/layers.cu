// Memory-bound layer kernels of the training step (HBM roofline): BN, ReLU,
// POOL, LRN, DROPOUT, SOFTMAX+CE, JOIN, gradient copies and the SGD update.
// NHWC fp32; float4 paths whenever the channel count allows.  Every reduction
// is two-stage with a fixed combination order, so a replayed (recomputed)
// forward and every feature set produce bit-identical values.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "bn_math.cuh"
#include "kernels.hpp"
#include "tc_common.cuh"

namespace sn {
namespace {

constexpr int kThreads = 256;

inline int blocks_for(int64_t n, int per_block = kThreads, int cap = 148 * 16) {
  int64_t b = (n + per_block - 1) / per_block;
  if (b < 1) b = 1;
  return static_cast<int>(b < cap ? b : cap);
}

// ---------------------------------------------------------------------------
// Deterministic per-channel column sums over a [rows][C] matrix.
// Stage 1: block b reduces rows [b*chunk, (b+1)*chunk) into part[b][2][C]
// (doubles); stage 2 sums the blocks in order.  Two sums per channel:
// f1 and f2 of the functor.

__device__ __forceinline__ float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float4 zero4() { return make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ void add4(float4& a, const float4& b) {
  a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
}
__device__ __forceinline__ float relu1(float v) { return v > 0.f ? v : 0.f; }
__device__ __forceinline__ float4 relu4(const float4& v) {
  return make_float4(relu1(v.x), relu1(v.y), relu1(v.z), relu1(v.w));
}

// BN normalisation, written with explicit-rounding intrinsics so that the
// forward, its replays and the ReLU mask recomputed in the fused backward are
// bit-identical (no compiler FMA contraction choices).

struct Bn4 {
  float4 m, is, g, b;
};
__device__ __forceinline__ Bn4 bn_params4(const float* stats, const float* gamma, const float* beta, int c, int C) {
  return Bn4{ld4(stats + c), ld4(stats + C + c), ld4(gamma + c), beta ? ld4(beta + c) : zero4()};
}
__device__ __forceinline__ float4 bn_affine4(const float4& v, const Bn4& p) {
  return make_float4(bn_affine(v.x, p.m.x, p.is.x, p.g.x, p.b.x), bn_affine(v.y, p.m.y, p.is.y, p.g.y, p.b.y),
                     bn_affine(v.z, p.m.z, p.is.z, p.g.z, p.b.z), bn_affine(v.w, p.m.w, p.is.w, p.g.w, p.b.w));
}

// Element loops keep kUnroll independent 16-byte loads in flight per thread
// (grid-stride loop unrolled by hand, loads before math): with ~2k threads per
// SM that is enough outstanding bytes to cover HBM latency.
constexpr int kUnroll = 4;
constexpr int kEltBlocks = 148 * 8;  // 2048 threads per SM

inline int elt_blocks(int64_t n4, int min_threads = 1) {
  int64_t b = (n4 + kThreads - 1) / kThreads;
  b = b < 1 ? 1 : (b > kEltBlocks ? kEltBlocks : b);
  const int64_t need = (min_threads + kThreads - 1) / kThreads;
  return static_cast<int>(b > need ? b : need);
}

// Per-channel loops: the stride is a multiple of C/4, so each thread's channel
// quad is fixed and its per-channel parameters stay in registers.
struct ChanLoop {
  int64_t S, start;
  int c;
  bool active;
};
__device__ __forceinline__ ChanLoop chan_loop(int C4) {
  const int64_t T = static_cast<int64_t>(gridDim.x) * blockDim.x;
  ChanLoop L;
  L.S = (T / C4) * C4;
  L.start = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  L.active = L.start < L.S;
  L.c = static_cast<int>(L.start % C4) * 4;
  return L;
}

// Reduction operands: load() issues the raw 16-byte loads of one row (all of
// them before any math, so kUnroll rows x operands are in flight per thread),
// comp() turns them into the two summands.
struct RedBiasOp {  // f1 = dy
  const float* dy;
  struct P {};
  struct R {
    float4 g;
  };
  __device__ P prep4(int, int) const { return P{}; }
  __device__ void eval(int64_t row, int c, int C, float& a, float& b) const {
    a = dy[row * C + c];
    b = 0.f;
  }
  __device__ R load(int64_t off) const { return R{ld4(dy + off)}; }
  __device__ void side(int64_t, const R&) const {}
  __device__ void comp(const P&, const R& r, float4& a, float4& b) const {
    a = r.g;
    b = zero4();
  }
};
struct RedBnStatsOp {  // f1 = x - x[0][c], f2 = (x - x[0][c])^2
  const float* x;
  struct P {
    float4 s;
  };
  struct R {
    float4 v;
  };
  __device__ P prep4(int c, int) const { return P{ld4(x + c)}; }
  __device__ void eval(int64_t row, int c, int C, float& a, float& b) const {
    const float d = x[row * C + c] - x[c];
    a = d;
    b = d * d;
  }
  __device__ R load(int64_t off) const { return R{ld4(x + off)}; }
  __device__ void side(int64_t, const R&) const {}
  __device__ void comp(const P& p, const R& r, float4& a, float4& b) const {
    a = make_float4(r.v.x - p.s.x, r.v.y - p.s.y, r.v.z - p.s.z, r.v.w - p.s.w);
    b = make_float4(a.x * a.x, a.y * a.y, a.z * a.z, a.w * a.w);
  }
};
// f1 = g, f2 = g * xhat with g = dy, or (relu: the fused ReLU backward) g = dy
// where the recomputed BN output is positive, else 0.
struct RedBnBwdOp {
  const float* x;
  const float* dy;
  const float* stats;  // mean[C], invstd[C]
  const float* gamma;
  const float* beta;
  int relu;
  // fused JOIN backward: the raw dy (the JOIN's gradient) is also written
  // (or added) into the JOIN's other input's gradient buffer
  float* copy_dst;
  int copy_acc;
  float* copy2;  // optional second (plain) copy of dy: the dx pass reads it
  using P = Bn4;
  struct R {
    float4 g, v;
  };
  __device__ P prep4(int c, int C) const { return bn_params4(stats, gamma, beta, c, C); }
  __device__ void eval(int64_t row, int c, int C, float& a, float& b) const {
    const float v = x[row * C + c];
    float g = dy[row * C + c];
    if (relu && !(bn_affine(v, stats[c], stats[C + c], gamma[c], beta[c]) > 0.f)) g = 0.f;
    a = g;
    b = g * bn_xhat(v, stats[c], stats[C + c]);
  }
  __device__ R load(int64_t off) const { return R{ld4(dy + off), ld4(x + off)}; }
  __device__ void side(int64_t off, const R& r) const {
    if (copy2) *reinterpret_cast<float4*>(copy2 + off) = r.g;
    if (!copy_dst) return;
    float4* d = reinterpret_cast<float4*>(copy_dst + off);
    if (copy_acc) {
      const float4 o = *d;
      *d = make_float4(o.x + r.g.x, o.y + r.g.y, o.z + r.g.z, o.w + r.g.w);
    } else {
      *d = r.g;
    }
  }
  __device__ void comp(const P& p, const R& r, float4& a, float4& b) const {
    float4 g = r.g;
    const float4 v = r.v;
    if (relu) {
      const float4 y = bn_affine4(v, p);
      g = make_float4(y.x > 0.f ? g.x : 0.f, y.y > 0.f ? g.y : 0.f, y.z > 0.f ? g.z : 0.f, y.w > 0.f ? g.w : 0.f);
    }
    a = g;
    b = make_float4(g.x * bn_xhat(v.x, p.m.x, p.is.x), g.y * bn_xhat(v.y, p.m.y, p.is.y),
                    g.z * bn_xhat(v.z, p.m.z, p.is.z), g.w * bn_xhat(v.w, p.m.w, p.is.w));
  }
};

// Stage 1, float4 variant for C % 4 == 0: block b reduces rows [b*chunk,
// (b+1)*chunk) into part[b][2][C] (doubles).  A thread owns 4 adjacent
// channels and walks its rows with kUnroll independent accumulators (fixed
// per-thread order, fixed merge).
constexpr int kRedThreads = 512;
template <class Op, int kUo = 0, int MINB = 2>
__global__ void __launch_bounds__(kRedThreads, MINB) colred_stage1_v4(Op op, int64_t rows, int C, int64_t chunk,
                                                                   double* part) {
  __shared__ float4 s1[kRedThreads], s2[kRedThreads];
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t r1 = r0 + chunk < rows ? r0 + chunk : rows;
  const int C4 = C / 4;
  const int cb = C4 < kRedThreads ? C4 : kRedThreads;
  const int lanes = kRedThreads / cb;
  const int t = threadIdx.x;
  const int lane = t / cb, cc = t % cb;
  for (int c0 = 0; c0 < C4; c0 += cb) {
    const int c4 = c0 + cc;
    // one accumulator pair (the kU rows' loads are what must overlap, not
    // the adds): 2 blocks of 512 threads per SM instead of 1 at 127 registers
    constexpr int kU = kUo ? kUo : kUnroll;
    float4 a = zero4(), b = a;
    if (lane < lanes && c4 < C4) {
      const typename Op::P p = op.prep4(c4 * 4, C);
      int64_t r = r0 + lane;
      for (; r + (kU - 1) * lanes < r1; r += kU * lanes) {
        typename Op::R raw[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) raw[u] = op.load((r + u * lanes) * C + c4 * 4);
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          op.side((r + u * lanes) * C + c4 * 4, raw[u]);
          float4 fa, fb;
          op.comp(p, raw[u], fa, fb);
          add4(a, fa);
          add4(b, fb);
        }
      }
      for (; r < r1; r += lanes) {
        float4 fa, fb;
        const typename Op::R raw1 = op.load(r * C + c4 * 4);
        op.side(r * C + c4 * 4, raw1);
        op.comp(p, raw1, fa, fb);
        add4(a, fa);
        add4(b, fb);
      }
    }
    s1[t] = a;
    s2[t] = b;
    __syncthreads();
    if (lane == 0 && c4 < C4) {
      double A[4] = {0, 0, 0, 0}, Bv[4] = {0, 0, 0, 0};
      for (int l = 0; l < lanes; ++l) {
        const float4 x = s1[l * cb + cc], y = s2[l * cb + cc];
        A[0] += x.x; A[1] += x.y; A[2] += x.z; A[3] += x.w;
        Bv[0] += y.x; Bv[1] += y.y; Bv[2] += y.z; Bv[3] += y.w;
      }
      double* pa = part + (static_cast<size_t>(blockIdx.x) * 2) * C + c4 * 4;
      double* pb = part + (static_cast<size_t>(blockIdx.x) * 2 + 1) * C + c4 * 4;
      for (int e = 0; e < 4; ++e) {
        pa[e] = A[e];
        pb[e] = Bv[e];
      }
    }
    __syncthreads();
  }
}

template <class Op>
__global__ void colred_stage1(Op op, int64_t rows, int C, int64_t chunk, double* part) {
  __shared__ double s1[kThreads], s2[kThreads];
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t r1 = r0 + chunk < rows ? r0 + chunk : rows;
  const int cb = C < kThreads ? C : kThreads;  // channels covered per pass
  const int lanes = kThreads / cb;             // row lanes
  const int t = threadIdx.x;
  const int lane = t / cb, cc = t % cb;
  for (int c0 = 0; c0 < C; c0 += cb) {
    const int c = c0 + cc;
    float a = 0.f, b = 0.f;
    if (lane < lanes && c < C) {
      for (int64_t r = r0 + lane; r < r1; r += lanes) {
        float fa, fb;
        op.eval(r, c, C, fa, fb);
        a += fa;
        b += fb;
      }
    }
    s1[t] = a;
    s2[t] = b;
    __syncthreads();
    if (lane == 0 && c < C) {
      double A = 0.0, B = 0.0;
      for (int l = 0; l < lanes; ++l) {
        A += s1[l * cb + cc];
        B += s2[l * cb + cc];
      }
      part[(static_cast<size_t>(blockIdx.x) * 2) * C + c] = A;
      part[(static_cast<size_t>(blockIdx.x) * 2 + 1) * C + c] = B;
    }
    __syncthreads();
  }
}

// Stage 2: 8 channels per block x 128 partial lanes (thread = channel + 8 *
// lane, so a warp reads 4 stage-1 rows x 8 adjacent channels); each lane sums
// stage-1 blocks lane, lane + 128, ... (4 loads in flight per operand), then
// the lanes are combined 8 at a time and the 16 group sums in order -- a fixed
// order, so the result is deterministic -- and handed to the finaliser.  More
// blocks and shorter chains than one block per 32 channels (C = 64 ran on 2 SMs).
constexpr int kStage2Threads = 1024;
constexpr int kStage2Chan = 8, kStage2Lanes = kStage2Threads / kStage2Chan;
inline int stage2_blocks(int C) { return (C + kStage2Chan - 1) / kStage2Chan; }
template <class Fin>
__global__ void __launch_bounds__(kStage2Threads) colred_stage2(const double* __restrict__ part, int nblocks, int C,
                                                                Fin fin) {
  __shared__ double sa[kStage2Lanes][kStage2Chan], sb[kStage2Lanes][kStage2Chan];
  __shared__ double ga[16][kStage2Chan], gb[16][kStage2Chan];
  const int cl = threadIdx.x % kStage2Chan, pl = threadIdx.x / kStage2Chan;
  const int c = blockIdx.x * kStage2Chan + cl;
  double A = 0.0, B = 0.0;
  if (c < C) {
    int b = pl;
    for (; b + 3 * kStage2Lanes < nblocks; b += 4 * kStage2Lanes) {
      double va[4], vb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        va[u] = part[(static_cast<size_t>(b + kStage2Lanes * u) * 2) * C + c];
        vb[u] = part[(static_cast<size_t>(b + kStage2Lanes * u) * 2 + 1) * C + c];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        A += va[u];
        B += vb[u];
      }
    }
    for (; b < nblocks; b += kStage2Lanes) {
      A += part[(static_cast<size_t>(b) * 2) * C + c];
      B += part[(static_cast<size_t>(b) * 2 + 1) * C + c];
    }
  }
  sa[pl][cl] = A;
  sb[pl][cl] = B;
  __syncthreads();
  if (pl < 16) {
    double a = 0.0, b = 0.0;
    for (int i = 0; i < kStage2Lanes / 16; ++i) {
      a += sa[pl * (kStage2Lanes / 16) + i][cl];
      b += sb[pl * (kStage2Lanes / 16) + i][cl];
    }
    ga[pl][cl] = a;
    gb[pl][cl] = b;
  }
  __syncthreads();
  if (pl == 0 && c < C) {
    double a = 0.0, b = 0.0;
    for (int i = 0; i < 16; ++i) {
      a += ga[i][cl];
      b += gb[i][cl];
    }
    fin(c, a, b);
  }
}

// BN backward statistics (RedBnBwdOp), bulk-copy pipelined: block b owns the
// contiguous rows [b*chunk, (b+1)*chunk) of dy and x; one producer thread
// streams them through a kCbStages-deep shared-memory ring with 1D bulk
// copies (8 KB per operand per stage), 8 consumer warps reduce from shared
// memory.  The loop-carried load latency the register version exposes (one
// 512-thread block per SM, loads then math per iteration: ~3 TB/s) is gone.
// Position e of a stage always holds channel quad e % C4 (stages hold whole
// numbers of rows' worth of quads: 512 % C4 == 0), consumer t reads positions
// t and t + 256; per-position float sums, then per quad in position order in
// double: a fixed order.
constexpr int kCbConsumers = 256;
constexpr int kCbThreads = kCbConsumers + 32;
constexpr int kCbStageF4 = 512;
constexpr int kCbStages = 6;
constexpr int kCbBlocks = 2 * 148;  // one wave at 2 blocks / SM
static_assert(kCbBlocks <= kRedChunks, "partials fit the reduction scratch");
constexpr int kCbSmem = kCbStages * 2 * kCbStageF4 * 16;

// Float4 positions per ring stage: a whole number of rows' worth of channel
// quads (512 when C/4 divides it, else the largest multiple of C/4 below 512:
// Inception's C = 96, 224, 384 ... -- position e of every stage then holds quad
// e % C4 and each consumer keeps one accumulator pair per position).
__host__ __device__ inline int bulk_stage_f4(int C4) { return (kCbStageF4 / C4) * C4; }

// Row chunks of colred_bulk_bn_bwd: block b owns rows [b*ck, (b+1)*ck), at
// least 8 ring stages per block, at most one wave.
int64_t bulk_chunk(int64_t rows, int C, int* nblocks) {
  int64_t nbb = (rows * (C / 4) + kCbStageF4 * 8 - 1) / (kCbStageF4 * 8);
  nbb = nbb < 1 ? 1 : (nbb > kCbBlocks ? kCbBlocks : nbb);
  const int64_t ck = (rows + nbb - 1) / nbb;
  *nblocks = static_cast<int>((rows + ck - 1) / ck);
  return ck;
}

bool colred_bulk_ok(int C) {
  const int C4 = C / 4;
  return C % 4 == 0 && C4 >= 1 && C4 <= kCbStageF4;
}

__global__ void __launch_bounds__(kCbThreads, 2)
    colred_bulk_bn_bwd(RedBnBwdOp op, int64_t rows, int C, int64_t chunk, double* part) {
  extern __shared__ __align__(128) float4 ring[];  // [stage][dy, x][kCbStageF4]
  __shared__ uint64_t full[kCbStages], empty[kCbStages];
  const int C4 = C / 4;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t r1 = r0 + chunk < rows ? r0 + chunk : rows;
  const int64_t f0 = r0 * C4, nf = (r1 - r0) * C4;  // float4 range of this block
  const int sf4 = bulk_stage_f4(C4);  // positions per stage
  const int nst = static_cast<int>((nf + sf4 - 1) / sf4);
  const int t = threadIdx.x, warp = t >> 5;
  if (t == 0) {
    for (int i = 0; i < kCbStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kCbConsumers / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const float4* dy4 = reinterpret_cast<const float4*>(op.dy);
  const float4* x4 = reinterpret_cast<const float4*>(op.x);
  float4 a0 = zero4(), b0 = zero4(), a1 = zero4(), b1 = zero4();
  // distinct quads per consumer: positions t and t + 256 share a quad when
  // C4 divides 256 (one accumulator pair), else each keeps its own
  const int nq = (C4 > kCbConsumers || kCbConsumers % C4 != 0) ? 2 : 1;
  if (warp == kCbConsumers / 32) {
    if (t == kCbConsumers) {
      for (int it = 0; it < nst; ++it) {
        const int s = it % kCbStages;
        if (it >= kCbStages) mbar_wait(&empty[s], ((it / kCbStages) - 1) & 1);
        const int64_t off = f0 + static_cast<int64_t>(it) * sf4;
        const int n = static_cast<int>(nf - static_cast<int64_t>(it) * sf4 < sf4 ? nf - static_cast<int64_t>(it) * sf4
                                                                                  : sf4);
        mbar_arrive_expect_tx(&full[s], 2u * n * 16u);
        bulk_load_1d(ring + (s * 2) * kCbStageF4, dy4 + off, n * 16u, &full[s]);
        bulk_load_1d(ring + (s * 2 + 1) * kCbStageF4, x4 + off, n * 16u, &full[s]);
      }
    }
  } else {
    const typename RedBnBwdOp::P p0 = op.prep4((t % C4) * 4, C);
    const typename RedBnBwdOp::P p1 = op.prep4(((t + kCbConsumers) % C4) * 4, C);
    for (int it = 0; it < nst; ++it) {
      const int s = it % kCbStages;
      mbar_wait(&full[s], (it / kCbStages) & 1);
      const int64_t off = f0 + static_cast<int64_t>(it) * sf4;
      const int64_t left = nf - static_cast<int64_t>(it) * sf4;
      const int n = static_cast<int>(left < sf4 ? left : sf4);
      if (t < n) {
        const RedBnBwdOp::R r{ring[(s * 2) * kCbStageF4 + t], ring[(s * 2 + 1) * kCbStageF4 + t]};
        op.side((off + t) * 4, r);
        float4 fa, fb;
        op.comp(p0, r, fa, fb);
        add4(a0, fa);
        add4(b0, fb);
      }
      const int e = t + kCbConsumers;
      if (e < n) {
        const RedBnBwdOp::R r{ring[(s * 2) * kCbStageF4 + e], ring[(s * 2 + 1) * kCbStageF4 + e]};
        op.side((off + e) * 4, r);
        float4 fa, fb;
        op.comp(p1, r, fa, fb);
        if (nq == 2) {
          add4(a1, fa);
          add4(b1, fb);
        } else {
          add4(a0, fa);
          add4(b0, fb);
        }
      }
      __syncwarp();
      if ((t & 31) == 0) mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();  // the ring is free: reuse it for the per-position sums
  float4* sa = ring;                        // [nq * 256]
  float4* sb = ring + 2 * kCbConsumers;     // [nq * 256]
  if (t < kCbConsumers) {
    sa[t] = a0;
    sb[t] = b0;
    if (nq == 2) {
      sa[t + kCbConsumers] = a1;
      sb[t + kCbConsumers] = b1;
    }
  }
  __syncthreads();
  const int ne = nq * kCbConsumers;
  for (int q = t; q < C4; q += blockDim.x) {
    double A[4] = {0, 0, 0, 0}, Bv[4] = {0, 0, 0, 0};
    for (int e = q; e < ne; e += C4) {
      const float4 u = sa[e], v = sb[e];
      A[0] += u.x; A[1] += u.y; A[2] += u.z; A[3] += u.w;
      Bv[0] += v.x; Bv[1] += v.y; Bv[2] += v.z; Bv[3] += v.w;
    }
    double* pa = part + (static_cast<size_t>(blockIdx.x) * 2) * C + q * 4;
    double* pb = pa + C;
    for (int i = 0; i < 4; ++i) {
      pa[i] = A[i];
      pb[i] = Bv[i];
    }
  }
}

// The same bulk-copy ring for the single-operand reductions (BN forward
// statistics of an input no CONV epilogue summed -- DenseNet's JOIN outputs --
// and a CONV bias gradient no BN dx pass summed): one 8 KB stream per stage
// instead of two; the register version (colred_stage1_v4) ran them at 2-3 TB/s.
template <class Op>
__global__ void __launch_bounds__(kCbThreads, 2)
    colred_bulk1(Op op, const float4* __restrict__ src, int64_t rows, int C, int64_t chunk, double* part) {
  extern __shared__ __align__(128) float4 ring[];  // [stage][kCbStageF4]
  __shared__ uint64_t full[kCbStages], empty[kCbStages];
  const int C4 = C / 4;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t r1 = r0 + chunk < rows ? r0 + chunk : rows;
  const int64_t f0 = r0 * C4, nf = (r1 - r0) * C4;
  const int sf4 = bulk_stage_f4(C4);
  const int nst = static_cast<int>((nf + sf4 - 1) / sf4);
  const int t = threadIdx.x, warp = t >> 5;
  if (t == 0) {
    for (int i = 0; i < kCbStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kCbConsumers / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  float4 a0 = zero4(), b0 = zero4(), a1 = zero4(), b1 = zero4();
  const int nq = (C4 > kCbConsumers || kCbConsumers % C4 != 0) ? 2 : 1;
  if (warp == kCbConsumers / 32) {
    if (t == kCbConsumers) {
      for (int it = 0; it < nst; ++it) {
        const int s = it % kCbStages;
        if (it >= kCbStages) mbar_wait(&empty[s], ((it / kCbStages) - 1) & 1);
        const int64_t left = nf - static_cast<int64_t>(it) * sf4;
        const int n = static_cast<int>(left < sf4 ? left : sf4);
        mbar_arrive_expect_tx(&full[s], n * 16u);
        bulk_load_1d(ring + s * kCbStageF4, src + f0 + static_cast<int64_t>(it) * sf4, n * 16u, &full[s]);
      }
    }
  } else {
    const typename Op::P p0 = op.prep4((t % C4) * 4, C);
    const typename Op::P p1 = op.prep4(((t + kCbConsumers) % C4) * 4, C);
    for (int it = 0; it < nst; ++it) {
      const int s = it % kCbStages;
      mbar_wait(&full[s], (it / kCbStages) & 1);
      const int64_t left = nf - static_cast<int64_t>(it) * sf4;
      const int n = static_cast<int>(left < sf4 ? left : sf4);
      if (t < n) {
        const typename Op::R r{ring[s * kCbStageF4 + t]};
        float4 fa, fb;
        op.comp(p0, r, fa, fb);
        add4(a0, fa);
        add4(b0, fb);
      }
      const int e = t + kCbConsumers;
      if (e < n) {
        const typename Op::R r{ring[s * kCbStageF4 + e]};
        float4 fa, fb;
        op.comp(p1, r, fa, fb);
        if (nq == 2) {
          add4(a1, fa);
          add4(b1, fb);
        } else {
          add4(a0, fa);
          add4(b0, fb);
        }
      }
      __syncwarp();
      if ((t & 31) == 0) mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();
  float4* sa = ring;
  float4* sb = ring + 2 * kCbConsumers;
  if (t < kCbConsumers) {
    sa[t] = a0;
    sb[t] = b0;
    if (nq == 2) {
      sa[t + kCbConsumers] = a1;
      sb[t + kCbConsumers] = b1;
    }
  }
  __syncthreads();
  const int ne = nq * kCbConsumers;
  for (int q = t; q < C4; q += blockDim.x) {
    double A[4] = {0, 0, 0, 0}, Bv[4] = {0, 0, 0, 0};
    for (int e = q; e < ne; e += C4) {
      const float4 u = sa[e], v = sb[e];
      A[0] += u.x; A[1] += u.y; A[2] += u.z; A[3] += u.w;
      Bv[0] += v.x; Bv[1] += v.y; Bv[2] += v.z; Bv[3] += v.w;
    }
    double* pa = part + (static_cast<size_t>(blockIdx.x) * 2) * C + q * 4;
    double* pb = pa + C;
    for (int i = 0; i < 4; ++i) {
      pa[i] = A[i];
      pb[i] = Bv[i];
    }
  }
}
constexpr int kCb1Smem = kCbStages * kCbStageF4 * 16;

// Blocks of stage 1: enough rows per thread (>= ~64 float4 per operand) that
// the double partials stay small next to the input, at most kRedChunks.
template <class Op, class Fin>
cudaError_t colred(Op op, Fin fin, int64_t rows, int C, float* scratch_f, cudaStream_t st) {
  double* part = reinterpret_cast<double*>(scratch_f);
  const bool v4 = C % 4 == 0;
  const int64_t per_block = v4 ? static_cast<int64_t>(kRedThreads) * 64 * 4 : static_cast<int64_t>(kThreads) * 64;
  int64_t nb = (rows * C + per_block - 1) / per_block;
  nb = nb < 148 ? 148 : (nb > kRedChunks ? kRedChunks : nb);
  if (nb > rows) nb = rows;
  if (nb < 1) nb = 1;
  const int64_t chunk = (rows + nb - 1) / nb;
  nb = (rows + chunk - 1) / chunk;
  if (nb < 1) nb = 1;
  if constexpr (std::is_same<Op, RedBnBwdOp>::value) {
    if (colred_bulk_ok(C)) {
      int nbb = 0;
      const int64_t ck = bulk_chunk(rows, C, &nbb);
      const cudaError_t ea = cudaFuncSetAttribute(colred_bulk_bn_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  kCbSmem);
      if (ea != cudaSuccess) return ea;
      if (!xskip(4)) colred_bulk_bn_bwd<<<static_cast<int>(nbb), kCbThreads, kCbSmem, st>>>(op, rows, C, ck, part);
      if (!xskip(1)) colred_stage2<<<stage2_blocks(C), kStage2Threads, 0, st>>>(part, static_cast<int>(nbb), C, fin);
      if (xskip(512)) colred_stage2<<<stage2_blocks(C), kStage2Threads, 0, st>>>(part, static_cast<int>(nbb), C, fin);
      return cudaGetLastError();
    }
  }
  if constexpr (std::is_same<Op, RedBnStatsOp>::value || std::is_same<Op, RedBiasOp>::value) {
    if (colred_bulk_ok(C)) {
      int nbb = 0;
      const int64_t ck = bulk_chunk(rows, C, &nbb);
      const cudaError_t ea = cudaFuncSetAttribute(colred_bulk1<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  kCb1Smem);
      if (ea != cudaSuccess) return ea;
      const float* src;
      if constexpr (std::is_same<Op, RedBnStatsOp>::value) src = op.x; else src = op.dy;
      colred_bulk1<Op><<<static_cast<int>(nbb), kCbThreads, kCb1Smem, st>>>(
          op, reinterpret_cast<const float4*>(src), rows, C, ck, part);
      colred_stage2<<<stage2_blocks(C), kStage2Threads, 0, st>>>(part, static_cast<int>(nbb), C, fin);
      return cudaGetLastError();
    }
  }
  // RedBnBwdOp (two operands + side copies per row): one 512-thread block per
  // SM without a register cap beats two capped ones (eager A/B over the step:
  // 9.47 vs 9.52 ms, SN_COLRED_ROWS experiment)
  if (v4 && std::is_same<Op, RedBnBwdOp>::value)
    colred_stage1_v4<Op, 4, 1><<<static_cast<int>(nb), kRedThreads, 0, st>>>(op, rows, C, chunk, part);
  else if (v4)
    colred_stage1_v4<<<static_cast<int>(nb), kRedThreads, 0, st>>>(op, rows, C, chunk, part);
  else
    colred_stage1<<<static_cast<int>(nb), kThreads, 0, st>>>(op, rows, C, chunk, part);
  colred_stage2<<<stage2_blocks(C), kStage2Threads, 0, st>>>(part, static_cast<int>(nb), C, fin);
  return cudaGetLastError();
}

struct BiasFin {
  float* db;
  __device__ void operator()(int c, double a, double) const { db[c] = static_cast<float>(a); }
};

struct BnStatsFin {
  const float* x;
  int64_t rows;
  int C;
  float eps, momentum;
  float* stats;
  float* running;
  __device__ void operator()(int c, double s1, double s2) const {
    const double n = static_cast<double>(rows);
    const double m1 = s1 / n;
    double var = s2 / n - m1 * m1;
    if (var < 0.0) var = 0.0;
    const double mean = static_cast<double>(x[c]) + m1;
    stats[c] = static_cast<float>(mean);
    stats[C + c] = static_cast<float>(1.0 / sqrt(var + static_cast<double>(eps)));
    if (running) {
      const double unbiased = rows > 1 ? var * n / (n - 1.0) : var;
      running[c] = static_cast<float>((1.0 - momentum) * running[c] + momentum * mean);
      running[C + c] = static_cast<float>((1.0 - momentum) * running[C + c] + momentum * unbiased);
    }
  }
};

struct BnBwdFin {
  int C;
  float* dgamma;
  float* dbeta;
  float* coef;  // {sum g, sum g*xhat} as floats for the dx pass
  __device__ void operator()(int c, double s1, double s2) const {
    dbeta[c] = static_cast<float>(s1);
    dgamma[c] = static_cast<float>(s2);
    coef[c] = static_cast<float>(s1);
    coef[C + c] = static_cast<float>(s2);
  }
};

__global__ void bn_apply_scalar(const float* __restrict__ x, int64_t n, int C, const float* __restrict__ gamma,
                                const float* __restrict__ beta, const float* __restrict__ stats, float* __restrict__ y) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const int c = static_cast<int>(i % C);
    y[i] = bn_affine(x[i], stats[c], stats[C + c], gamma[c], beta[c]);
  }
}

// BN apply (C % 4 == 0), optionally fused with the ReLU that consumes it:
// y = bn(x) (skipped when null), yr = relu(y) (skipped when null).
// y = bn(x), yr = relu(y), yj = relu(y) + add (the 2-input JOIN fed by the
// ReLU; a + b == b + a in IEEE arithmetic, so the JOIN's input order does not
// matter).  Null outputs are skipped.
__global__ void bn_apply_v4(const float4* __restrict__ x, int64_t n4, int C, const float* __restrict__ gamma,
                            const float* __restrict__ beta, const float* __restrict__ stats, float4* __restrict__ y,
                            float4* __restrict__ yr, const float4* __restrict__ add, float4* __restrict__ yj) {
  const ChanLoop L = chan_loop(C / 4);
  if (!L.active) return;
  const Bn4 p = bn_params4(stats, gamma, beta, L.c, C);
  for (int64_t i0 = L.start; i0 < n4; i0 += kUnroll * L.S) {
    float4 v[kUnroll], w[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      v[u] = i0 + u * L.S < n4 ? x[i0 + u * L.S] : zero4();
      w[u] = (yj && i0 + u * L.S < n4) ? add[i0 + u * L.S] : zero4();
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t i = i0 + u * L.S;
      if (i < n4) {
        const float4 o = bn_affine4(v[u], p);
        if (y) y[i] = o;
        const float4 r = relu4(o);
        if (yr) yr[i] = r;
        if (yj) {
          float4 j = r;
          add4(j, w[u]);
          yj[i] = j;
        }
      }
    }
  }
}

// JOIN backward for two destinations: one read of dy.
__global__ void grad_copy2_kernel(const float4* __restrict__ src, float4* d1, int acc1, float4* d2, int acc2,
                                  int64_t n4) {
  const int64_t T = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i0 < n4; i0 += kUnroll * T) {
    float4 v[kUnroll], o1[kUnroll], o2[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t i = i0 + u * T;
      v[u] = i < n4 ? src[i] : zero4();
      o1[u] = (acc1 && i < n4) ? d1[i] : zero4();
      o2[u] = (acc2 && i < n4) ? d2[i] : zero4();
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t i = i0 + u * T;
      if (i < n4) {
        float4 a = v[u], b = v[u];
        if (acc1) add4(a, o1[u]);
        if (acc2) add4(b, o2[u]);
        d1[i] = a;
        d2[i] = b;
      }
    }
  }
}


// dx (+)= gamma*invstd*(g - sum(g)/m - xhat*sum(g*xhat)/m), g = dy or the
// ReLU-masked dy (relu: mask recomputed from x, see RedBnBwdOp).
__global__ void bn_dx_scalar(const float* __restrict__ x, const float* __restrict__ dy, int64_t n, int64_t rows, int C,
                             const float* __restrict__ gamma, const float* __restrict__ beta,
                             const float* __restrict__ stats, const float* __restrict__ coef, float* dx,
                             int accumulate, int relu) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const float inv_m = 1.0f / static_cast<float>(rows);
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < n; j += stride) {
    const int c = static_cast<int>(j % C);
    float g = dy[j];
    if (relu && !(bn_affine(x[j], stats[c], stats[C + c], gamma[c], beta[c]) > 0.f)) g = 0.f;
    const float xh = bn_xhat(x[j], stats[c], stats[C + c]);
    (void)xh;
    const float v = bn_dx_elem(g, x[j], stats[c], stats[C + c], gamma[c] * stats[C + c], coef[c] * inv_m,
                               coef[C + c] * inv_m);
    dx[j] = accumulate ? dx[j] + v : v;
  }
}

// Block-level combination of per-thread channel-quad sums (threads t and
// t + C/4 share a quad; 256 % (C/4) == 0) in thread order, into
// part[blockIdx.x][0][C] (doubles) and a zero second plane.
__device__ void bias_block_reduce(const float4& v, int C, double* part) {
  __shared__ float4 sb[kThreads];
  sb[threadIdx.x] = v;
  __syncthreads();
  const int C4 = C / 4;
  for (int c4 = threadIdx.x; c4 < C4; c4 += blockDim.x) {
    double a[4] = {0, 0, 0, 0};
    // the block's first thread need not sit on quad 0: thread t holds quad (base + t) % C4
    const int base = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x) % C4);
    const int t0 = (c4 - base + C4) % C4;
    for (int t = t0; t < static_cast<int>(blockDim.x); t += C4) {
      const float4 w = sb[t];
      a[0] += w.x; a[1] += w.y; a[2] += w.z; a[3] += w.w;
    }
    double* p0 = part + static_cast<size_t>(blockIdx.x) * 2 * C + c4 * 4;
    double* p1 = p0 + C;
    for (int e = 0; e < 4; ++e) {
      p0[e] = a[e];
      p1[e] = 0.0;
    }
  }
}

// dbias (optional, 256 % (C/4) == 0): also the column sums of this pass's dx
// contribution -- the bias gradient of the CONV producing x, whose only
// consumer this BN is (its gradient buffer holds nothing else) -- as per-block partials part[block][2][C] (doubles; second plane 0) for
// colred_stage2: a fixed thread -> (channel quad, row lane) map, so the sums
// are deterministic.
__global__ void __launch_bounds__(kThreads, 4) bn_dx_v4(const float4* __restrict__ x, const float4* __restrict__ dy, int64_t n4, int64_t rows,
                         int C, const float* __restrict__ gamma, const float* __restrict__ beta,
                         const float* __restrict__ stats, const float* __restrict__ coef, float4* dx, int accumulate,
                         int relu, double* dbias_part) {
  const ChanLoop L = chan_loop(C / 4);
  float4 bsum = zero4();
  if (!L.active) {
    if (dbias_part) bias_block_reduce(bsum, C, dbias_part);
    return;
  }
  const float inv_m = 1.0f / static_cast<float>(rows);
  const Bn4 p = bn_params4(stats, gamma, beta, L.c, C);
  const float4 c1 = ld4(coef + L.c), c2 = ld4(coef + C + L.c);
  const float k1[4] = {c1.x * inv_m, c1.y * inv_m, c1.z * inv_m, c1.w * inv_m};
  const float k2[4] = {c2.x * inv_m, c2.y * inv_m, c2.z * inv_m, c2.w * inv_m};
  const float gs[4] = {p.g.x * p.is.x, p.g.y * p.is.y, p.g.z * p.is.z, p.g.w * p.is.w};
  const float m[4] = {p.m.x, p.m.y, p.m.z, p.m.w}, is[4] = {p.is.x, p.is.y, p.is.z, p.is.w};
  // 2 rows per thread in flight (x, dy[, dx]) at <= 64 registers: 4 blocks per SM
  constexpr int U = 2;
  for (int64_t i0 = L.start; i0 < n4; i0 += U * L.S) {
    float4 xv[U], gv[U], ov[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * L.S;
      xv[u] = i < n4 ? x[i] : zero4();
      gv[u] = i < n4 ? dy[i] : zero4();
      ov[u] = (accumulate && i < n4) ? dx[i] : zero4();
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * L.S;
      if (i >= n4) break;
      if (relu) {
        const float4 y = bn_affine4(xv[u], p);
        gv[u] = make_float4(y.x > 0.f ? gv[u].x : 0.f, y.y > 0.f ? gv[u].y : 0.f, y.z > 0.f ? gv[u].z : 0.f,
                            y.w > 0.f ? gv[u].w : 0.f);
      }
      const float xs[4] = {xv[u].x, xv[u].y, xv[u].z, xv[u].w}, gg[4] = {gv[u].x, gv[u].y, gv[u].z, gv[u].w};
      float r[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) r[e] = bn_dx_elem(gg[e], xs[e], m[e], is[e], gs[e], k1[e], k2[e]);
      float4 o = make_float4(r[0], r[1], r[2], r[3]);
      if (dbias_part) add4(bsum, o);
      if (accumulate) add4(o, ov[u]);
      dx[i] = o;
    }
  }
  if (dbias_part) bias_block_reduce(bsum, C, dbias_part);
}

// ---------------------------------------------------------------------------
__global__ void relu_fwd_kernel(const float4* __restrict__ x, float4* __restrict__ y, int64_t n4) {
  const int64_t T = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i0 < n4; i0 += kUnroll * T) {
    float4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) v[u] = i0 + u * T < n4 ? x[i0 + u * T] : zero4();
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (i0 + u * T < n4) y[i0 + u * T] = relu4(v[u]);
  }
}
__global__ void relu_fwd_tail(const float* x, float* y, int64_t from, int64_t n) {
  const int64_t i = from + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) y[i] = x[i] > 0.f ? x[i] : 0.f;
}
__global__ void relu_bwd_kernel(const float4* __restrict__ y, float4* g, int64_t n4) {
  const int64_t T = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i0 < n4; i0 += kUnroll * T) {
    float4 yy[kUnroll], v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t i = i0 + u * T;
      yy[u] = i < n4 ? y[i] : zero4();
      v[u] = i < n4 ? g[i] : zero4();
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t i = i0 + u * T;
      if (i < n4)
        g[i] = make_float4(yy[u].x > 0.f ? v[u].x : 0.f, yy[u].y > 0.f ? v[u].y : 0.f, yy[u].z > 0.f ? v[u].z : 0.f,
                           yy[u].w > 0.f ? v[u].w : 0.f);
    }
  }
}
__global__ void relu_bwd_tail(const float* y, float* g, int64_t from, int64_t n) {
  const int64_t i = from + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) g[i] = y[i] > 0.f ? g[i] : 0.f;
}

// ---------------------------------------------------------------------------
__global__ void pool_fwd_kernel(PoolShape s, const float* __restrict__ x, float* __restrict__ y, int64_t total) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total; i += stride) {
    const int c = static_cast<int>(i % s.C);
    int64_t t = i / s.C;
    const int q = static_cast<int>(t % s.Q);
    t /= s.Q;
    const int p = static_cast<int>(t % s.P);
    const int n = static_cast<int>(t / s.P);
    const int h0 = p * s.stride - s.pad, w0 = q * s.stride - s.pad;
    float acc = s.mode == 0 ? -FLT_MAX : 0.f;
    bool any = false;
    for (int r = 0; r < s.K; ++r) {
      const int h = h0 + r;
      if (h < 0 || h >= s.H) continue;
      for (int u = 0; u < s.K; ++u) {
        const int w = w0 + u;
        if (w < 0 || w >= s.W) continue;
        const float v = x[((static_cast<int64_t>(n) * s.H + h) * s.W + w) * s.C + c];
        if (s.mode == 0) {
          if (!any || v > acc) acc = v;
          any = true;
        } else {
          acc += v;
        }
      }
    }
    y[i] = s.mode == 0 ? acc : acc / static_cast<float>(s.K * s.K);
  }
}

// float4 over channels (C % 4 == 0); 32-bit index math (tensors < 2^31 elements).
// KC: compile-time window (0 = runtime s.K); with it the window's loads are
// unrolled and in flight together (the max / sum order is the same row-major
// order either way, so replays and both variants are bit-identical).
template <int KC>
__global__ void pool_fwd_v4_kernel(PoolShape s, const float4* __restrict__ x, float4* __restrict__ y, int total4) {
  const int C4 = s.C >> 2;
  const float inv = 1.0f / static_cast<float>(s.K * s.K);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total4; i += gridDim.x * blockDim.x) {
    const int c4 = i % C4;
    int t = i / C4;
    const int q = t % s.Q;
    t /= s.Q;
    const int p = t % s.P;
    const int n = t / s.P;
    const int h0 = p * s.stride - s.pad, w0 = q * s.stride - s.pad;
    const float4* xb = x + static_cast<size_t>(n) * s.H * s.W * C4 + c4;
    float4 acc;
    if constexpr (KC > 0) {
      float4 v[KC * KC];
      bool in[KC * KC];
#pragma unroll
      for (int r = 0; r < KC; ++r)
#pragma unroll
        for (int u = 0; u < KC; ++u) {
          const int h = h0 + r, w = w0 + u;
          in[r * KC + u] = h >= 0 && h < s.H && w >= 0 && w < s.W;
          v[r * KC + u] = in[r * KC + u] ? xb[(h * s.W + w) * C4] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      if (s.mode == 0) {
        bool have = false;
#pragma unroll
        for (int k = 0; k < KC * KC; ++k) {
          if (!in[k]) continue;
          if (!have) {
            acc = v[k];
            have = true;
          } else {
            acc.x = v[k].x > acc.x ? v[k].x : acc.x;
            acc.y = v[k].y > acc.y ? v[k].y : acc.y;
            acc.z = v[k].z > acc.z ? v[k].z : acc.z;
            acc.w = v[k].w > acc.w ? v[k].w : acc.w;
          }
        }
      } else {
        acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k = 0; k < KC * KC; ++k)
          if (in[k]) {
            acc.x += v[k].x; acc.y += v[k].y; acc.z += v[k].z; acc.w += v[k].w;
          }
        acc.x *= inv; acc.y *= inv; acc.z *= inv; acc.w *= inv;
      }
    } else {
      const int hb = h0 < 0 ? 0 : h0, he = min(h0 + s.K, s.H);
      const int wb = w0 < 0 ? 0 : w0, we = min(w0 + s.K, s.W);
      if (s.mode == 0) {
        acc = xb[(hb * s.W + wb) * C4];
        for (int h = hb; h < he; ++h)
          for (int w = wb; w < we; ++w) {
            const float4 v = xb[(h * s.W + w) * C4];
            acc.x = v.x > acc.x ? v.x : acc.x;
            acc.y = v.y > acc.y ? v.y : acc.y;
            acc.z = v.z > acc.z ? v.z : acc.z;
            acc.w = v.w > acc.w ? v.w : acc.w;
          }
      } else {
        acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int h = hb; h < he; ++h)
          for (int w = wb; w < we; ++w) {
            const float4 v = xb[(h * s.W + w) * C4];
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
          }
        acc.x *= inv; acc.y *= inv; acc.z *= inv; acc.w *= inv;
      }
    }
    y[i] = acc;
  }
}

// One block per output row (n, p) for the common small-window case: the only
// per-element index math left is one division by C/4.
//
// BNR: the input is a BN input; BN (batch statistics) + ReLU are applied on
// load (bn_affine4 / relu4, bit-identical to bn_apply_v4).  yr (optional)
// receives the ReLU output, each element written by the one window that owns
// it (rows/cols 2p, 2p+1: needs pad 1, H = 2P, W = 2Q; pool_fwd_bn_relu_ok).
constexpr int kPoolBnMaxC4 = 128;
template <int KC, int SC, bool BNR>
__global__ void __launch_bounds__(256) pool_fwd_rows_kernel(PoolShape s, const float4* __restrict__ x,
                                                            float4* __restrict__ y, uchar4* __restrict__ arg,
                                                            const float* __restrict__ stats,
                                                            const float* __restrict__ gamma,
                                                            const float* __restrict__ beta, float4* __restrict__ yr) {
  const int C4 = s.C >> 2;
  const int p = blockIdx.x, n = blockIdx.y;
  __shared__ Bn4 bp[BNR ? kPoolBnMaxC4 : 1];
  if constexpr (BNR) {
    for (int c = threadIdx.x; c < C4; c += blockDim.x) bp[c] = bn_params4(stats, gamma, beta, 4 * c, s.C);
    __syncthreads();
  }
  const int h0 = p * SC - s.pad;
  const float inv = 1.0f / static_cast<float>(KC * KC);
  const float4* xb = x + static_cast<size_t>(n) * s.H * s.W * C4;
  float4* yrow = y + (static_cast<size_t>(n) * s.P + p) * s.Q * C4;
  for (int i = threadIdx.x; i < s.Q * C4; i += blockDim.x) {
    const int q = i / C4, c4 = i - q * C4;
    const int w0 = q * SC - s.pad;
    float4 v[KC * KC];
    bool in[KC * KC];
#pragma unroll
    for (int r = 0; r < KC; ++r)
#pragma unroll
      for (int u = 0; u < KC; ++u) {
        const int h = h0 + r, w = w0 + u;
        in[r * KC + u] = h >= 0 && h < s.H && w >= 0 && w < s.W;
        v[r * KC + u] = in[r * KC + u] ? xb[(h * s.W + w) * C4 + c4] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    if constexpr (BNR) {
      const Bn4 bq = bp[c4];
#pragma unroll
      for (int r = 0; r < KC; ++r)
#pragma unroll
        for (int u = 0; u < KC; ++u) {
          if (!in[r * KC + u]) continue;
          v[r * KC + u] = relu4(bn_affine4(v[r * KC + u], bq));
          if (yr && r >= 1 && u >= 1)
            yr[static_cast<size_t>(n) * s.H * s.W * C4 + ((h0 + r) * s.W + (w0 + u)) * C4 + c4] = v[r * KC + u];
        }
    }
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (s.mode == 0) {
      // max and the first (row-major) position holding it, for the backward
      bool have = false;
      int a0 = 255, a1 = 255, a2 = 255, a3 = 255;
#pragma unroll
      for (int k = 0; k < KC * KC; ++k) {
        if (!in[k]) continue;
        if (!have) {
          acc = v[k];
          a0 = a1 = a2 = a3 = k;
          have = true;
        } else {
          if (v[k].x > acc.x) { acc.x = v[k].x; a0 = k; }
          if (v[k].y > acc.y) { acc.y = v[k].y; a1 = k; }
          if (v[k].z > acc.z) { acc.z = v[k].z; a2 = k; }
          if (v[k].w > acc.w) { acc.w = v[k].w; a3 = k; }
        }
      }
      if (arg) arg[(static_cast<size_t>(n) * s.P + p) * s.Q * C4 + i] = make_uchar4(a0, a1, a2, a3);
    } else {
#pragma unroll
      for (int k = 0; k < KC * KC; ++k)
        if (in[k]) {
          acc.x += v[k].x; acc.y += v[k].y; acc.z += v[k].z; acc.w += v[k].w;
        }
      acc.x *= inv; acc.y *= inv; acc.z *= inv; acc.w *= inv;
    }
    yrow[i] = acc;
  }
}

// 3x3 / stride 2 / pad 1 max pool over an even input (H = 2P, W = 2Q), the
// shape after a stride-2 stem: block = (band of PB output rows, image), thread
// = (output column q, channel quad); each thread walks its band keeping input
// row 2p-1 from the previous output row in registers, so it loads 6 of the 9
// window elements per output (the columns 2q-1 are also its left neighbour's:
// L1/L2 hits) and the input leaves HBM once.  Same window order, comparisons
// and argmax encoding as pool_fwd_rows_kernel.  BNR as there.
// Row partial of a 3-wide window row: the max per component and the first
// column holding it, as the window index k = 3*r + u (strict > keeps the first).
struct RowMax {
  float4 v;
  int a0, a1, a2, a3;
};
__device__ __forceinline__ void rowmax_take(RowMax& m, const float4& v, int k) {
  if (v.x > m.v.x) { m.v.x = v.x; m.a0 = k; }
  if (v.y > m.v.y) { m.v.y = v.y; m.a1 = k; }
  if (v.z > m.v.z) { m.v.z = v.z; m.a2 = k; }
  if (v.w > m.v.w) { m.v.w = v.w; m.a3 = k; }
}
__device__ __forceinline__ void rowmax_take(RowMax& m, const RowMax& o) {
  if (o.v.x > m.v.x) { m.v.x = o.v.x; m.a0 = o.a0; }
  if (o.v.y > m.v.y) { m.v.y = o.v.y; m.a1 = o.a1; }
  if (o.v.z > m.v.z) { m.v.z = o.v.z; m.a2 = o.a2; }
  if (o.v.w > m.v.w) { m.v.w = o.v.w; m.a3 = o.a3; }
}

template <bool BNR>
__global__ void __launch_bounds__(448, 2) pool_fwd_k3s2_band_kernel(PoolShape s, int PB, int CS, const float4* __restrict__ x,
                                                                  float4* __restrict__ y, uchar4* __restrict__ arg,
                                                                  const float* __restrict__ stats,
                                                                  const float* __restrict__ gamma,
                                                                  const float* __restrict__ beta,
                                                                  float4* __restrict__ yr) {
  const int C4 = s.C >> 2;
  const int n = blockIdx.y;
  const int q = threadIdx.x / CS, c4 = blockIdx.z * CS + threadIdx.x - q * CS;  // CS channel quads per block
  __shared__ Bn4 bp[BNR ? kPoolBnMaxC4 : 1];
  if constexpr (BNR) {
    for (int c = threadIdx.x; c < C4; c += blockDim.x) bp[c] = bn_params4(stats, gamma, beta, 4 * c, s.C);
    __syncthreads();
  }
  if (q >= s.Q) return;
  const bool left = q > 0;  // column 2q-1 inside the image
  const int rs = s.W * C4;  // input row stride (float4)
  // element (h, 2q-1+u) of this image: xi[h*rs + col + u*C4]
  const float4* xi = x + static_cast<size_t>(n) * s.H * rs;
  float4* yri = BNR && yr ? yr + static_cast<size_t>(n) * s.H * rs : nullptr;
  const int col = (2 * q - 1) * C4 + c4;
  auto load3 = [&](int h, float4* v) {
    const int o = h * rs + col;
    v[0] = left ? xi[o] : make_float4(0.f, 0.f, 0.f, 0.f);
    v[1] = xi[o + C4];
    v[2] = xi[o + 2 * C4];
  };
  // BN+ReLU (BNR) and the row partial of one loaded window triple
  auto reduce3 = [&](int h, float4* v, int kr, bool own) -> RowMax {
    if constexpr (BNR) {
      const Bn4 b = bp[c4];
#pragma unroll
      for (int u = 0; u < 3; ++u) v[u] = relu4(bn_affine4(v[u], b));
      if (yri && own) {
        const int o = h * rs + col;
        yri[o + C4] = v[1];
        yri[o + 2 * C4] = v[2];
      }
    }
    RowMax m;
    if (left) {
      m.v = v[0];
      m.a0 = m.a1 = m.a2 = m.a3 = kr;
      rowmax_take(m, v[1], kr + 1);
    } else {
      m.v = v[1];
      m.a0 = m.a1 = m.a2 = m.a3 = kr + 1;
    }
    rowmax_take(m, v[2], kr + 2);
    return m;
  };
  const int p0 = blockIdx.x * PB, p1 = min(s.P, p0 + PB);
  RowMax top{};
  if (p0 > 0) {
    float4 t[3];
    load3(2 * p0 - 1, t);
    top = reduce3(2 * p0 - 1, t, 0, false);
  }
  for (int p = p0; p < p1; ++p) {
    float4 a[3], b[3];
    load3(2 * p, a);  // all six loads in flight before any math
    load3(2 * p + 1, b);
    const RowMax m0 = reduce3(2 * p, a, 3, true);
    const RowMax m1 = reduce3(2 * p + 1, b, 6, true);
    RowMax acc;
    if (p > 0) {
      acc = top;
      rowmax_take(acc, m0);
    } else {
      acc = m0;
    }
    rowmax_take(acc, m1);
    // the bottom row's partial is the next window's top row, with k shifted by 6
    top = m1;
    top.a0 -= 6; top.a1 -= 6; top.a2 -= 6; top.a3 -= 6;
    const size_t o = ((static_cast<size_t>(n) * s.P + p) * s.Q + q) * C4 + c4;
    if (arg) arg[o] = make_uchar4(acc.a0, acc.a1, acc.a2, acc.a3);
    y[o] = acc.v;
  }
}

// Global pool (one output pixel per image, window = the whole image, pad 0):
// block = (image, 128 channels); 8 pixel lanes x 32 channel quads, each lane
// reduces pixels lane, lane+8, ... and the lanes are combined in lane order.
// Same row-major order per lane for max; avg sums in that fixed order.
__global__ void __launch_bounds__(256) pool_global_kernel(PoolShape s, const float4* __restrict__ x,
                                                          float4* __restrict__ y) {
  __shared__ float4 part[8][32];
  const int C4 = s.C >> 2;
  const int cq = threadIdx.x & 31, pl = threadIdx.x >> 5;
  const int c4 = blockIdx.x * 32 + cq;
  const int n = blockIdx.y;
  const int HW = s.H * s.W;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  bool have = false;
  if (c4 < C4) {
    const float4* xb = x + static_cast<size_t>(n) * HW * C4 + c4;
    for (int i = pl; i < HW; i += 8) {
      const float4 v = xb[static_cast<size_t>(i) * C4];
      if (s.mode == 0) {
        if (!have) {
          acc = v;
          have = true;
        } else {
          acc.x = v.x > acc.x ? v.x : acc.x;
          acc.y = v.y > acc.y ? v.y : acc.y;
          acc.z = v.z > acc.z ? v.z : acc.z;
          acc.w = v.w > acc.w ? v.w : acc.w;
        }
      } else {
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
    }
  }
  part[pl][cq] = acc;
  __syncthreads();
  if (pl == 0 && c4 < C4) {
    float4 r = part[0][cq];
    for (int l = 1; l < 8 && l < HW; ++l) {
      const float4 v = part[l][cq];
      if (s.mode == 0) {
        r.x = v.x > r.x ? v.x : r.x;
        r.y = v.y > r.y ? v.y : r.y;
        r.z = v.z > r.z ? v.z : r.z;
        r.w = v.w > r.w ? v.w : r.w;
      } else {
        r.x += v.x; r.y += v.y; r.z += v.z; r.w += v.w;
      }
    }
    if (s.mode == 1) {
      const float inv = 1.0f / static_cast<float>(s.K * s.K);
      r.x *= inv; r.y *= inv; r.z *= inv; r.w *= inv;
    }
    y[static_cast<size_t>(n) * C4 + c4] = r;
  }
}

__global__ void pool_bwd_kernel(PoolShape s, const float* __restrict__ x, const float* __restrict__ y,
                                const float* __restrict__ dy, float* dx, int accumulate, int64_t total) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const float inv = 1.0f / static_cast<float>(s.K * s.K);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total; i += stride) {
    const int c = static_cast<int>(i % s.C);
    int64_t t = i / s.C;
    const int w = static_cast<int>(t % s.W);
    t /= s.W;
    const int h = static_cast<int>(t % s.H);
    const int n = static_cast<int>(t / s.H);
    // output rows/cols whose window covers (h, w)
    int plo = h + s.pad - s.K + 1, qlo = w + s.pad - s.K + 1;
    plo = plo <= 0 ? 0 : (plo + s.stride - 1) / s.stride;
    qlo = qlo <= 0 ? 0 : (qlo + s.stride - 1) / s.stride;
    int phi = (h + s.pad) / s.stride, qhi = (w + s.pad) / s.stride;
    if (phi > s.P - 1) phi = s.P - 1;
    if (qhi > s.Q - 1) qhi = s.Q - 1;
    float acc = 0.f;
    for (int p = plo; p <= phi; ++p) {
      for (int q = qlo; q <= qhi; ++q) {
        const int64_t o = ((static_cast<int64_t>(n) * s.P + p) * s.Q + q) * s.C + c;
        if (s.mode == 1) {
          acc += dy[o] * inv;
          continue;
        }
        // first position of the window (row-major) holding the maximum
        const float m = y[o];
        const int h0 = p * s.stride - s.pad, w0 = q * s.stride - s.pad;
        int fh = -1, fw = -1;
        for (int r = 0; r < s.K && fh < 0; ++r) {
          const int hh = h0 + r;
          if (hh < 0 || hh >= s.H) continue;
          for (int u = 0; u < s.K; ++u) {
            const int ww = w0 + u;
            if (ww < 0 || ww >= s.W) continue;
            if (x[((static_cast<int64_t>(n) * s.H + hh) * s.W + ww) * s.C + c] == m) {
              fh = hh;
              fw = ww;
              break;
            }
          }
        }
        if (fh == h && fw == w) acc += dy[o];
      }
    }
    dx[i] = accumulate ? dx[i] + acc : acc;
  }
}

// Max-pool backward, pass 1: for every output, the window offset r*K+s of the
// first element (row-major) equal to the forward maximum y (255: none).
// Vectorised over 4 channels.
__global__ void pool_argmax_kernel(PoolShape s, const float* __restrict__ x, const float* __restrict__ y,
                                   uchar4* __restrict__ arg, int total4) {
  const int stride = gridDim.x * blockDim.x;
  const int C4 = s.C / 4;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total4; i += stride) {
    const int c4 = i % C4;
    int t = i / C4;
    const int q = static_cast<int>(t % s.Q);
    t /= s.Q;
    const int p = static_cast<int>(t % s.P);
    const int n = static_cast<int>(t / s.P);
    const float4 m = reinterpret_cast<const float4*>(y)[i];
    const int h0 = p * s.stride - s.pad, w0 = q * s.stride - s.pad;
    int a0 = 255, a1 = 255, a2 = 255, a3 = 255;
    for (int r = 0; r < s.K; ++r) {
      const int h = h0 + r;
      if (h < 0 || h >= s.H) continue;
      for (int u = 0; u < s.K; ++u) {
        const int w = w0 + u;
        if (w < 0 || w >= s.W) continue;
        const float4 v = reinterpret_cast<const float4*>(x)[((static_cast<int64_t>(n) * s.H + h) * s.W + w) * C4 + c4];
        const int off = r * s.K + u;
        if (a0 == 255 && v.x == m.x) a0 = off;
        if (a1 == 255 && v.y == m.y) a1 = off;
        if (a2 == 255 && v.z == m.z) a2 = off;
        if (a3 == 255 && v.w == m.w) a3 = off;
      }
    }
    arg[i] = make_uchar4(a0, a1, a2, a3);
  }
}

// Pass 2 (and the whole of avg-pool backward): gather over the <= ceil(K/s)^2
// windows covering each input element.
__global__ void pool_gather_kernel(PoolShape s, const uchar4* __restrict__ arg, const float* __restrict__ dy,
                                   float* dx, int accumulate, int total4) {
  const int stride = gridDim.x * blockDim.x;
  const int C4 = s.C / 4;
  const float inv = 1.0f / static_cast<float>(s.K * s.K);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total4; i += stride) {
    const int c4 = i % C4;
    int t = i / C4;
    const int w = static_cast<int>(t % s.W);
    t /= s.W;
    const int h = static_cast<int>(t % s.H);
    const int n = static_cast<int>(t / s.H);
    int plo = h + s.pad - s.K + 1, qlo = w + s.pad - s.K + 1;
    plo = plo <= 0 ? 0 : (plo + s.stride - 1) / s.stride;
    qlo = qlo <= 0 ? 0 : (qlo + s.stride - 1) / s.stride;
    int phi = (h + s.pad) / s.stride, qhi = (w + s.pad) / s.stride;
    if (phi > s.P - 1) phi = s.P - 1;
    if (qhi > s.Q - 1) qhi = s.Q - 1;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int p = plo; p <= phi; ++p) {
      for (int q = qlo; q <= qhi; ++q) {
        const int64_t o = ((static_cast<int64_t>(n) * s.P + p) * s.Q + q) * C4 + c4;
        const float4 g = reinterpret_cast<const float4*>(dy)[o];
        if (s.mode == 1) {
          acc.x += g.x * inv; acc.y += g.y * inv; acc.z += g.z * inv; acc.w += g.w * inv;
          continue;
        }
        const int off = (h - (p * s.stride - s.pad)) * s.K + (w - (q * s.stride - s.pad));
        const uchar4 a = arg[o];
        if (a.x == off) acc.x += g.x;
        if (a.y == off) acc.y += g.y;
        if (a.z == off) acc.z += g.z;
        if (a.w == off) acc.w += g.w;
      }
    }
    float4* d = reinterpret_cast<float4*>(dx) + i;
    if (accumulate) {
      const float4 o = *d;
      acc.x += o.x; acc.y += o.y; acc.z += o.z; acc.w += o.w;
    }
    *d = acc;
  }
}

// Max-pool backward, fused (argmax + gather, one pass over x, y, dy, dx).
// Block = (16-channel chunk, band of PB output rows, image).  The block owns the
// input rows h whose floor((h + pad) / stride) lies in its band; phase 1
// computes, for every window covering those rows, the first (row-major)
// position holding the forward maximum y and stages it with dy in shared
// memory; phase 2 gathers each owned input element from the <= ceil(K/s)^2
// windows covering it.  Windows on a band edge are evaluated by both
// neighbouring blocks (cheap) so that no element has two writers.
constexpr int kPoolCv = 4;  // float4s per pixel chunk (16 channels)

// KC / SC = compile-time window size and stride (0: runtime s.K / s.stride):
// the window's loads are unrolled and all in flight at once, and the index
// arithmetic is shifts.  Threads map to (column lane = tid / 4, 16-byte
// channel quad = tid % 4) and walk rows / columns in nested loops, so no
// per-element divisions remain (the kernel was issue-bound on them).
template <int KC, int SC>
__global__ void __launch_bounds__(256) pool_max_bwd_fused(PoolShape s, const float4* __restrict__ x,
                                                          const float4* __restrict__ y,
                                                          const float4* __restrict__ dy, float4* dx,
                                                          int accumulate, int PB, int WR,
                                                          const uchar4* __restrict__ saved) {
  extern __shared__ float4 psm[];
  const int K = KC > 0 ? KC : s.K, ST = SC > 0 ? SC : s.stride;
  float4* sdy = psm;                                                  // [WR][Q][kPoolCv]
  uchar4* sarg = reinterpret_cast<uchar4*>(psm + WR * s.Q * kPoolCv);  // [WR][Q][kPoolCv]
  const int C4 = s.C / 4;
  const int c4 = blockIdx.x * kPoolCv;
  const int band = blockIdx.y, n = blockIdx.z;
  int h_lo = band * PB * ST - s.pad;
  int h_hi = (band + 1) * PB * ST - s.pad - 1;
  if (band == 0) h_lo = 0;
  if (band == gridDim.y - 1) h_hi = s.H - 1;
  if (h_lo < 0) h_lo = 0;
  if (h_hi > s.H - 1) h_hi = s.H - 1;
  const int t = h_lo + s.pad - K + 1;
  const int pl = t <= 0 ? 0 : (t + ST - 1) / ST;
  int ph = (h_hi + s.pad) / ST;
  if (ph > s.P - 1) ph = s.P - 1;
  const int cv = threadIdx.x & 3, lane = threadIdx.x >> 2;
  const float4* xn = x + static_cast<int64_t>(n) * s.H * s.W * C4 + c4 + cv;
  // phase 1: argmax (first row-major match) and dy of every window touching the band
  for (int p = pl; p <= ph; ++p) {
    const int h0 = p * ST - s.pad;
    const int64_t orow = (static_cast<int64_t>(n) * s.P + p) * s.Q;
    for (int q = lane; q < s.Q; q += 64) {
      const int64_t o = (orow + q) * C4 + c4 + cv;
      const float4 g = dy[o];
      if (saved) {  // argmax recorded by the forward: no x / y reads
        const int j = ((p - pl) * s.Q + q) * kPoolCv + cv;
        sarg[j] = saved[o];
        sdy[j] = g;
        continue;
      }
      const float4 m = y[o];
      const int w0 = q * ST - s.pad;
      int a0 = 255, a1 = 255, a2 = 255, a3 = 255;
      if constexpr (KC > 0) {
        float4 v[KC * KC];
#pragma unroll
        for (int r = 0; r < KC; ++r)
#pragma unroll
          for (int u = 0; u < KC; ++u) {
            const int h = h0 + r, w = w0 + u;
            const bool in = h >= 0 && h < s.H && w >= 0 && w < s.W;
            // out-of-image taps can never equal the maximum: NaN
            v[r * KC + u] = in ? xn[(static_cast<int64_t>(h) * s.W + w) * C4] : make_float4(NAN, NAN, NAN, NAN);
          }
#pragma unroll
        for (int k = KC * KC - 1; k >= 0; --k) {  // descending: the first (row-major) match wins
          if (v[k].x == m.x) a0 = k;
          if (v[k].y == m.y) a1 = k;
          if (v[k].z == m.z) a2 = k;
          if (v[k].w == m.w) a3 = k;
        }
      } else {
        for (int r = 0; r < K; ++r) {
          const int h = h0 + r;
          if (h < 0 || h >= s.H) continue;
          for (int u = 0; u < K; ++u) {
            const int w = w0 + u;
            if (w < 0 || w >= s.W) continue;
            const float4 v = xn[(static_cast<int64_t>(h) * s.W + w) * C4];
            const int off = r * K + u;
            if (a0 == 255 && v.x == m.x) a0 = off;
            if (a1 == 255 && v.y == m.y) a1 = off;
            if (a2 == 255 && v.z == m.z) a2 = off;
            if (a3 == 255 && v.w == m.w) a3 = off;
          }
        }
      }
      const int j = ((p - pl) * s.Q + q) * kPoolCv + cv;
      sarg[j] = make_uchar4(a0, a1, a2, a3);
      sdy[j] = g;
    }
  }
  __syncthreads();
  // phase 2: gather each input element of the band from the windows covering it
  float4* dxn = dx + static_cast<int64_t>(n) * s.H * s.W * C4 + c4 + cv;
  for (int h = h_lo; h <= h_hi; ++h) {
    int plo = h + s.pad - K + 1;
    plo = plo <= 0 ? 0 : (plo + ST - 1) / ST;
    int phi = (h + s.pad) / ST;
    if (phi > s.P - 1) phi = s.P - 1;
    for (int w = lane; w < s.W; w += 64) {
      int qlo = w + s.pad - K + 1;
      qlo = qlo <= 0 ? 0 : (qlo + ST - 1) / ST;
      int qhi = (w + s.pad) / ST;
      if (qhi > s.Q - 1) qhi = s.Q - 1;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int p = plo; p <= phi; ++p) {
        const int roff = (h - (p * ST - s.pad)) * K;
        for (int q = qlo; q <= qhi; ++q) {
          const int j = ((p - pl) * s.Q + q) * kPoolCv + cv;
          const int off = roff + (w - (q * ST - s.pad));
          const uchar4 a = sarg[j];
          const float4 g = sdy[j];
          if (a.x == off) acc.x += g.x;
          if (a.y == off) acc.y += g.y;
          if (a.z == off) acc.z += g.z;
          if (a.w == off) acc.w += g.w;
        }
      }
      float4* d = dxn + (static_cast<int64_t>(h) * s.W + w) * C4;
      if (accumulate) {
        const float4 o = *d;
        acc.x += o.x; acc.y += o.y; acc.z += o.z; acc.w += o.w;
      }
      *d = acc;
    }
  }
}

// Max-pool 3x3 / stride 2 / pad 1 backward with the forward's saved argmax, for
// H = 2P, W = 2Q: one thread per 2 x 2 block of input pixels (rows 2m, 2m+1,
// columns 2k, 2k+1) and channel quad.  The four windows (m|m+1, k|k+1) that can
// cover the block are read once; input (2m+dh, 2k+dw) sits at window offset
// (dh+1, dw+1) of window (m, k) and (dh-1, dw-1) of window (m+1, k+1), etc.
// Contributions are summed in window order (m,k), (m,k+1), (m+1,k), (m+1,k+1)
// -- the ascending (p, q) order of the general kernel, so the bits agree.
__global__ void __launch_bounds__(256) pool_max_bwd_k3s2(PoolShape s, const uchar4* __restrict__ arg,
                                                         const float4* __restrict__ dy, float4* dx, int accumulate,
                                                         int64_t total) {
  const int C4 = s.C >> 2;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c4 = static_cast<int>(i % C4);
    int64_t t = i / C4;
    const int k = static_cast<int>(t % s.Q);
    t /= s.Q;
    const int m = static_cast<int>(t % s.P);
    const int n = static_cast<int>(t / s.P);
    const int64_t wbase = (static_cast<int64_t>(n) * s.P + m) * s.Q + k;  // window (m, k)
    const bool k1 = k + 1 < s.Q, m1 = m + 1 < s.P;
    const uchar4 a00 = arg[wbase * C4 + c4];
    const float4 g00 = dy[wbase * C4 + c4];
    const uchar4 a01 = k1 ? arg[(wbase + 1) * C4 + c4] : make_uchar4(255, 255, 255, 255);
    const float4 g01 = k1 ? dy[(wbase + 1) * C4 + c4] : make_float4(0.f, 0.f, 0.f, 0.f);
    const uchar4 a10 = m1 ? arg[(wbase + s.Q) * C4 + c4] : make_uchar4(255, 255, 255, 255);
    const float4 g10 = m1 ? dy[(wbase + s.Q) * C4 + c4] : make_float4(0.f, 0.f, 0.f, 0.f);
    const uchar4 a11 = (k1 && m1) ? arg[(wbase + s.Q + 1) * C4 + c4] : make_uchar4(255, 255, 255, 255);
    const float4 g11 = (k1 && m1) ? dy[(wbase + s.Q + 1) * C4 + c4] : make_float4(0.f, 0.f, 0.f, 0.f);
    // out[dh][dw]: (window, offset) pairs in window order
    float4 o[4];
#define SN_PICK(A, G, OFF, ACC)                    \
  ACC.x += (A.x == (OFF)) ? G.x : 0.f;             \
  ACC.y += (A.y == (OFF)) ? G.y : 0.f;             \
  ACC.z += (A.z == (OFF)) ? G.z : 0.f;             \
  ACC.w += (A.w == (OFF)) ? G.w : 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) o[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    SN_PICK(a00, g00, 4, o[0]);                                          // (0,0)
    SN_PICK(a00, g00, 5, o[1]); SN_PICK(a01, g01, 3, o[1]);              // (0,1)
    SN_PICK(a00, g00, 7, o[2]); SN_PICK(a10, g10, 1, o[2]);              // (1,0)
    SN_PICK(a00, g00, 8, o[3]); SN_PICK(a01, g01, 6, o[3]);              // (1,1)
    SN_PICK(a10, g10, 2, o[3]); SN_PICK(a11, g11, 0, o[3]);
#undef SN_PICK
    const int64_t r0 = ((static_cast<int64_t>(n) * s.H + 2 * m) * s.W + 2 * k) * C4 + c4;
    const int64_t r1 = r0 + static_cast<int64_t>(s.W) * C4;
    float4* d[4] = {dx + r0, dx + r0 + C4, dx + r1, dx + r1 + C4};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (accumulate) {
        const float4 old = *d[q];
        o[q].x += old.x; o[q].y += old.y; o[q].z += old.z; o[q].w += old.w;
      }
      *d[q] = o[q];
    }
  }
}

// ---------------------------------------------------------------------------
__device__ __forceinline__ float lrn_scale(const float* xp, int c, int C, int lo, int hi, float alpha_n, float k) {
  float s = 0.f;
  for (int j = c - lo; j <= c + hi; ++j)
    if (j >= 0 && j < C) s += xp[j] * xp[j];
  return k + alpha_n * s;
}

__global__ void lrn_fwd_kernel(const float* __restrict__ x, float* __restrict__ y, int64_t total, int C, int size,
                               float alpha, float beta, float k) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int lo = size / 2, hi = (size - 1) / 2;
  const float an = alpha / static_cast<float>(size);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total; i += stride) {
    const int c = static_cast<int>(i % C);
    const float* xp = x + (i - c);
    const float s = lrn_scale(xp, c, C, lo, hi, an, k);
    y[i] = x[i] / powf(s, beta);
  }
}

__global__ void lrn_bwd_kernel(const float* __restrict__ x, const float* __restrict__ y, const float* __restrict__ dy,
                               float* dx, int64_t total, int C, int size, float alpha, float beta, float k,
                               int accumulate) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int lo = size / 2, hi = (size - 1) / 2;
  const float an = alpha / static_cast<float>(size);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total; i += stride) {
    const int ci = static_cast<int>(i % C);
    const int64_t base = i - ci;
    const float* xp = x + base;
    const float si = lrn_scale(xp, ci, C, lo, hi, an, k);
    float acc = 0.f;
    // channels c whose window [c-lo, c+hi] contains ci
    for (int c = ci - hi; c <= ci + lo; ++c) {
      if (c < 0 || c >= C) continue;
      const float sc = lrn_scale(xp, c, C, lo, hi, an, k);
      acc += dy[base + c] * y[base + c] / sc;
    }
    const float v = dy[i] / powf(si, beta) - 2.f * an * beta * x[i] * acc;
    dx[i] = accumulate ? dx[i] + v : v;
  }
}

// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t mix32(uint32_t v) {
  v ^= v >> 16;
  v *= 0x7feb352dU;
  v ^= v >> 15;
  v *= 0x846ca68bU;
  v ^= v >> 16;
  return v;
}
__device__ __forceinline__ bool drop_keep(uint64_t seed, int layer, uint32_t iter, uint32_t idx, uint32_t thresh) {
  const uint32_t key = mix32(static_cast<uint32_t>(seed) ^ mix32(static_cast<uint32_t>(seed >> 32) ^
                                                               mix32(iter * 0x9E3779B9U + static_cast<uint32_t>(layer))));
  return mix32(idx ^ key) >= thresh;
}

__global__ void dropout_fwd_kernel(const float* __restrict__ x, float* __restrict__ y, int64_t n, uint32_t thresh,
                                   float scale, uint64_t seed, int layer, const uint32_t* iteration) {
  const uint32_t it = *iteration;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    y[i] = drop_keep(seed, layer, it, static_cast<uint32_t>(i), thresh) ? x[i] * scale : 0.f;
}
__global__ void dropout_bwd_kernel(float* g, int64_t n, uint32_t thresh, float scale, uint64_t seed, int layer,
                                   const uint32_t* iteration) {
  const uint32_t it = *iteration;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    g[i] = drop_keep(seed, layer, it, static_cast<uint32_t>(i), thresh) ? g[i] * scale : 0.f;
}

// ---------------------------------------------------------------------------
// One warp per row.
__global__ void softmax_fwd_kernel(const float* __restrict__ x, float* __restrict__ y, int B, int F,
                                   const int32_t* __restrict__ labels, float* loss_rows) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= B) return;
  const float* xr = x + static_cast<int64_t>(warp) * F;
  float m = -FLT_MAX;
  for (int f = lane; f < F; f += 32) m = fmaxf(m, xr[f]);
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float s = 0.f;
  for (int f = lane; f < F; f += 32) s += expf(xr[f] - m);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float inv = 1.f / s;
  float* yr = y + static_cast<int64_t>(warp) * F;
  for (int f = lane; f < F; f += 32) yr[f] = expf(xr[f] - m) * inv;
  if (lane == 0 && loss_rows) {
    int lab = labels[warp];
    lab = lab < 0 ? 0 : (lab >= F ? F - 1 : lab);
    loss_rows[warp] = logf(s) - (xr[lab] - m);
  }
}

__global__ void softmax_bwd_kernel(const float* __restrict__ y, const int32_t* __restrict__ labels, float* dx, int B,
                                   int F, int accumulate) {
  const int64_t total = static_cast<int64_t>(B) * F;
  const float invb = 1.f / static_cast<float>(B);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total; i += stride) {
    const int b = static_cast<int>(i / F), f = static_cast<int>(i % F);
    int lab = labels[b];
    lab = lab < 0 ? 0 : (lab >= F ? F - 1 : lab);
    const float v = (y[i] - (f == lab ? 1.f : 0.f)) * invb;
    dx[i] = accumulate ? dx[i] + v : v;
  }
}

__global__ void loss_reduce_kernel(const float* loss_rows, int B, float* loss) {
  __shared__ double part[256];
  double a = 0.0;
  for (int i = threadIdx.x; i < B; i += 256) a += loss_rows[i];
  part[threadIdx.x] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < 256; ++i) s += part[i];
    *loss = static_cast<float>(s / B);
  }
}

// ---------------------------------------------------------------------------
// Two-input joins (the residual add) read both operands with kUnroll loads in
// flight; wider joins walk the inputs in order.
__global__ void join_fwd_kernel(const float* const* __restrict__ in, int n_in, float* __restrict__ y, int64_t n) {
  const int64_t T = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t n4 = n / 4;
  const float4* a = reinterpret_cast<const float4*>(in[0]);
  if (n_in == 2) {
    const float4* b = reinterpret_cast<const float4*>(in[1]);
    for (int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i0 < n4; i0 += kUnroll * T) {
      float4 va[kUnroll], vb[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t i = i0 + u * T;
        va[u] = i < n4 ? a[i] : zero4();
        vb[u] = i < n4 ? b[i] : zero4();
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t i = i0 + u * T;
        if (i < n4) {
          add4(va[u], vb[u]);
          reinterpret_cast<float4*>(y)[i] = va[u];
        }
      }
    }
  } else {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4; i += T) {
      float4 acc = a[i];
      for (int k = 1; k < n_in; ++k) add4(acc, reinterpret_cast<const float4*>(in[k])[i]);
      reinterpret_cast<float4*>(y)[i] = acc;
    }
  }
  for (int64_t i = n4 * 4 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += T) {
    float acc = in[0][i];
    for (int k = 1; k < n_in; ++k) acc += in[k][i];
    y[i] = acc;
  }
}

__global__ void grad_copy_kernel(const float* __restrict__ src, float* dst, int64_t n, int accumulate) {
  const int64_t T = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t n4 = n / 4;
  const float4* s4 = reinterpret_cast<const float4*>(src);
  float4* d4 = reinterpret_cast<float4*>(dst);
  for (int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i0 < n4; i0 += kUnroll * T) {
    float4 v[kUnroll], o[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t i = i0 + u * T;
      v[u] = i < n4 ? s4[i] : zero4();
      o[u] = (accumulate && i < n4) ? d4[i] : zero4();
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t i = i0 + u * T;
      if (i < n4) {
        if (accumulate) add4(v[u], o[u]);
        d4[i] = v[u];
      }
    }
  }
  for (int64_t i = n4 * 4 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += T)
    dst[i] = accumulate ? dst[i] + src[i] : src[i];
}

__global__ void sgd_kernel(float* p, const float* __restrict__ g, int64_t n, float lr, float scale) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    p[i] -= lr * (g[i] * scale);
}

// The data-parallel per-bucket update: skipped when *flag == 0 (a step
// without update); same arithmetic as sgd_kernel.
__global__ void sgd_flagged_kernel(float* p, const float* __restrict__ g, int64_t n, float lr, float scale,
                                   const int* flag) {
  if (*flag == 0) return;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    p[i] -= lr * (g[i] * scale);
}

__global__ void bump_kernel(uint32_t* it) { *it += 1; }

__global__ void zero_kernel(float* p, int64_t n) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) p[i] = 0.f;
}

}  // namespace

int64_t red_scratch_floats(int C) {
  // kRedChunks*2*C partial doubles + 2*C float coefficients (+ pad), then the
  // fused bias-gradient partials of bn_bwd: kEltBlocks*2*C doubles
  return static_cast<int64_t>(kRedChunks) * 2 * C * 2 + 2 * C + 64 + static_cast<int64_t>(kEltBlocks) * 2 * C * 2;
}

cudaError_t bias_grad_from_partials(const double* part, int nblocks, int C, float* db, cudaStream_t st) {
  colred_stage2<<<stage2_blocks(C), kStage2Threads, 0, st>>>(part, nblocks, C, BiasFin{db});
  return cudaGetLastError();
}

float* bn_coef_ptr(float* red_scratch, int C) { return red_scratch + static_cast<int64_t>(kRedChunks) * 2 * C * 2; }

cudaError_t bias_grad(const float* dy, int64_t rows, int C, float* db, float* red_scratch, cudaStream_t st) {
  return colred(RedBiasOp{dy}, BiasFin{db}, rows, C, red_scratch, st);
}

cudaError_t bn_fwd(const float* x, int64_t rows, int C, const float* gamma, const float* beta, float* y, float* stats,
                   float* running, float eps, float momentum, int compute_stats, float* red_scratch, cudaStream_t st) {
  cudaError_t e;
  if (compute_stats) {
    e = colred(RedBnStatsOp{x}, BnStatsFin{x, rows, C, eps, momentum, stats, running}, rows, C, red_scratch, st);
    if (e != cudaSuccess) return e;
  }
  if (!y) return cudaGetLastError();  // statistics only (apply fused downstream)
  const int64_t n = rows * C;
  if (C % 4 == 0)
    bn_apply_v4<<<elt_blocks(n / 4, C / 4), kThreads, 0, st>>>(reinterpret_cast<const float4*>(x), n / 4, C, gamma,
                                                                beta, stats, reinterpret_cast<float4*>(y), nullptr,
                                                                nullptr, nullptr);
  else
    bn_apply_scalar<<<blocks_for(n), kThreads, 0, st>>>(x, n, C, gamma, beta, stats, y);
  return cudaGetLastError();
}

namespace {

// Stage 1 over the convolution's tile partials: block b combines tiles
// [b*chunk, (b+1)*chunk) into {sum(y - x0), sum((y - x0)^2)} (doubles) about the
// global shift x0 = x[0][c]:  with d = shift_t - x0,
//   sum(y - x0)     = S1_t + n_t d
//   sum((y - x0)^2) = S2_t + 2 d S1_t + n_t d^2.
// Block = (chunk of tiles, 64 channels); 4 tile lanes x 64 channels per block,
// each lane walks its tiles with 4 independent accumulator pairs (loads in
// flight), lanes and accumulators merged in a fixed order.  ~2 blocks per SM
// (a 25-block grid for stage 3 took 13 us of pure latency).
constexpr int kTsChan = 64, kTsLanes = kThreads / kTsChan;
__global__ void __launch_bounds__(kThreads) tile_stats_stage1(const float* __restrict__ tiles, int ntiles,
                                                              int tile_rows, int64_t rows, int C,
                                                              const float* __restrict__ x, int chunk, double* part) {
  __shared__ double s1[kThreads], s2[kThreads];
  const int t0 = blockIdx.x * chunk;
  const int t1 = min(ntiles, t0 + chunk);
  const int lane = threadIdx.x / kTsChan;
  const int c = blockIdx.y * kTsChan + threadIdx.x % kTsChan;
  const int planes = tile_rows > 0 ? 3 : 4;
  double a[4] = {0, 0, 0, 0}, b[4] = {0, 0, 0, 0};
  if (c < C) {
    const double x0 = x[c];
    int t = t0 + lane;
    for (; t < t1; t += 4 * kTsLanes) {
      float sh[4], f1[4], f2[4], cnt[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int tu = t + u * kTsLanes;
        const float* p = tiles + static_cast<size_t>(tu < t1 ? tu : t0) * planes * C + c;
        sh[u] = p[0];
        f1[u] = p[C];
        f2[u] = p[2 * C];
        cnt[u] = tile_rows > 0 ? 0.f : p[3 * C];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int tu = t + u * kTsLanes;
        if (tu >= t1) continue;
        const int64_t left = rows - static_cast<int64_t>(tu) * tile_rows;
        const double n = tile_rows > 0 ? static_cast<double>(left < tile_rows ? left : tile_rows)
                                       : static_cast<double>(cnt[u]);
        if (n <= 0.0) continue;  // a tile past the last output row (its shift is not a value)
        const double d = static_cast<double>(sh[u]) - x0;
        const double S1 = f1[u], S2 = f2[u];
        a[u] += S1 + n * d;
        b[u] += S2 + 2.0 * d * S1 + n * d * d;
      }
    }
  }
  s1[threadIdx.x] = (a[0] + a[1]) + (a[2] + a[3]);
  s2[threadIdx.x] = (b[0] + b[1]) + (b[2] + b[3]);
  __syncthreads();
  if (lane == 0 && c < C) {
    double A = 0.0, B = 0.0;
    for (int l = 0; l < kTsLanes; ++l) {
      A += s1[l * kTsChan + threadIdx.x];
      B += s2[l * kTsChan + threadIdx.x];
    }
    part[(static_cast<size_t>(blockIdx.x) * 2) * C + c] = A;
    part[(static_cast<size_t>(blockIdx.x) * 2 + 1) * C + c] = B;
  }
}

}  // namespace

cudaError_t bn_stats_from_tiles(const float* tiles, int ntiles, int tile_rows, const float* x, int64_t rows, int C,
                                float* stats, float* running, float eps, float momentum, float* red_scratch,
                                cudaStream_t st) {
  double* part = reinterpret_cast<double*>(red_scratch);
  const int cgroups = (C + kTsChan - 1) / kTsChan;
  int nb = (2 * 148 + cgroups - 1) / cgroups;  // ~2 blocks per SM in total
  nb = std::max(1, std::min({nb, (ntiles + 3) / 4, kRedChunks}));
  const int chunk = (ntiles + nb - 1) / nb;
  nb = (ntiles + chunk - 1) / chunk;
  if (xskip(128)) return cudaSuccess;
  tile_stats_stage1<<<dim3(nb, cgroups), kThreads, 0, st>>>(tiles, ntiles, tile_rows, rows, C, x, chunk, part);
  colred_stage2<<<stage2_blocks(C), kStage2Threads, 0, st>>>(part, nb, C,
                                                          BnStatsFin{x, rows, C, eps, momentum, stats, running});
  if (xskip(512))
  colred_stage2<<<stage2_blocks(C), kStage2Threads, 0, st>>>(part, nb, C,
                                                          BnStatsFin{x, rows, C, eps, momentum, stats, running});
  return cudaGetLastError();
}

cudaError_t bn_apply_relu(const float* x, int64_t rows, int C, const float* gamma, const float* beta,
                          const float* stats, float* y, float* y_relu, cudaStream_t st, const float* join_other,
                          float* y_join) {
  const int64_t n4 = rows * C / 4;
  bn_apply_v4<<<elt_blocks(n4, C / 4), kThreads, 0, st>>>(
      reinterpret_cast<const float4*>(x), n4, C, gamma, beta, stats, reinterpret_cast<float4*>(y),
      reinterpret_cast<float4*>(y_relu), reinterpret_cast<const float4*>(join_other),
      reinterpret_cast<float4*>(y_join));
  return cudaGetLastError();
}

cudaError_t grad_copy2(const float* src, float* d1, int acc1, float* d2, int acc2, int64_t n, cudaStream_t st) {
  grad_copy2_kernel<<<elt_blocks(n / 4), kThreads, 0, st>>>(reinterpret_cast<const float4*>(src),
                                                            reinterpret_cast<float4*>(d1), acc1,
                                                            reinterpret_cast<float4*>(d2), acc2, n / 4);
  return cudaGetLastError();
}

int xskip(int bit) {
  static int mask = -1;
  if (mask < 0) {
    const char* v = std::getenv("SN_XSKIP");
    mask = v ? std::atoi(v) : 0;
  }
  return (mask & bit) != 0;
}

bool bn_bwd_bias_ok(int C) { return C % 4 == 0 && kThreads % (C / 4) == 0; }

cudaError_t bn_bwd_dx(const float* x, const float* dy, int64_t rows, int C, const float* gamma, const float* beta,
                      const float* stats, int relu, float* dx, int accumulate, float* red_scratch, cudaStream_t st,
                      float* dbias) {
  const float* coef = bn_coef_ptr(red_scratch, C);
  const int64_t n = rows * C;
  if (dbias && (!dx || !bn_bwd_bias_ok(C))) return cudaErrorInvalidValue;
  if (!dx) return cudaSuccess;
  if (C % 4 == 0) {
    const int nb = elt_blocks(n / 4, C / 4);
    // bias partials past the colred partials and coef (see red_scratch_floats)
    double* part = dbias ? reinterpret_cast<double*>(red_scratch + static_cast<int64_t>(kRedChunks) * 2 * C * 2 +
                                                     ((2 * C + 63) / 64) * 64)
                         : nullptr;
    if (!xskip(8)) bn_dx_v4<<<nb, kThreads, 0, st>>>(reinterpret_cast<const float4*>(x), reinterpret_cast<const float4*>(dy), n / 4,
                                      rows, C, gamma, beta, stats, coef, reinterpret_cast<float4*>(dx), accumulate,
                                      relu, part);
    if (dbias && !xskip(2)) colred_stage2<<<stage2_blocks(C), kStage2Threads, 0, st>>>(part, nb, C, BiasFin{dbias});
  } else {
    bn_dx_scalar<<<blocks_for(n), kThreads, 0, st>>>(x, dy, n, rows, C, gamma, beta, stats, coef, dx, accumulate,
                                                     relu);
  }
  return cudaGetLastError();
}

cudaError_t bn_bwd(const float* x, const float* dy, int64_t rows, int C, const float* gamma, const float* beta,
                   const float* stats, int relu, float* dx, int accumulate, float* dgamma, float* dbeta,
                   float* red_scratch, cudaStream_t st, float* dbias, float* copy_dst, int copy_acc,
                   float* copy2) {
  float* coef = bn_coef_ptr(red_scratch, C);
  if ((copy_dst || copy2) && C % 4 != 0) return cudaErrorInvalidValue;
  if (dbias && (!dx || !bn_bwd_bias_ok(C))) return cudaErrorInvalidValue;
  cudaError_t e = colred(RedBnBwdOp{x, dy, stats, gamma, beta, relu, copy_dst, copy_acc, copy2},
                         BnBwdFin{C, dgamma, dbeta, coef}, rows, C, red_scratch, st);
  if (e != cudaSuccess) return e;
  if (copy2) dy = copy2;  // the dx pass reads the copy (the original may be overwritten by dx)
  return bn_bwd_dx(x, dy, rows, C, gamma, beta, stats, relu, dx, accumulate, red_scratch, st, dbias);
}

// ---------------------------------------------------------------------------
// BN backward statistics of a BN whose ReLU output feeds a 3x3 / stride 2 /
// pad 1 max pool with saved argmax (H = 2P, W = 2Q) -- the stem's: one pass
// over 2 x 2 pixel blocks (thread item = a run of kPbRun blocks along a pool
// row x channel quad; windows two neighbouring blocks share load once) taking dy either gathered from the pool output's
// gradient and the argmax (GATHER: the pool backward fused in, its output
// never written) or read from the materialised pool-input gradient.  The
// gathered values are the same picks, summed from +0 in the same order, as
// pool_max_bwd_k3s2 writes, so both variants give the same bits.  Per-thread
// sums (a fixed channel quad: the grid stride is a multiple of C/4) are
// combined per block in thread order into part[block][2][C] doubles, then by
// colred_stage2 in block order (deterministic).
constexpr int kPbThreads = 256;

constexpr int kPbRun = 8;  // 2 x 2 blocks per thread item (a run along the pool row)
constexpr int kPbBlocks = 2 * 148;  // one wave on a B200 at 2 blocks / SM (fixed: it sets the summation order)
static_assert(kPbBlocks <= kRedChunks, "partials fit the reduction scratch");

template <bool GATHER>
__global__ void __launch_bounds__(kPbThreads, 2) pool_bn_stats_kernel(  // kPbBlocks: one wave
    // (3 or 4 blocks per SM cap the registers and spill: 260 / 408 vs 228 us)
    PoolShape s, const uchar4* __restrict__ arg, const float4* __restrict__ dyp, const float4* __restrict__ dym,
    const float4* __restrict__ x, const float* __restrict__ stats, const float* __restrict__ gamma,
    const float* __restrict__ beta, int relu, int items, double* part) {
  __shared__ float4 sh[kPbThreads];
  const int C4 = s.C >> 2;
  const int runs = (s.Q + kPbRun - 1) / kPbRun;
  const int stride = gridDim.x * blockDim.x;  // a multiple of C4
  const int i0 = blockIdx.x * blockDim.x + threadIdx.x;
  const int c4 = i0 % C4;
  const RedBnBwdOp op{nullptr, nullptr, stats, gamma, beta, relu, nullptr, 0, nullptr};
  const Bn4 p = op.prep4(c4 * 4, s.C);
  float4 a = zero4(), b = zero4();
  const uchar4 none = make_uchar4(255, 255, 255, 255);
  for (int i = i0; i < items; i += stride) {
    int t = i / C4;
    const int run = t % runs;
    t /= runs;
    const int m = t % s.P;
    const int n = t / s.P;
    const int k0 = run * kPbRun, k1e = min(s.Q, k0 + kPbRun);
    const bool m1 = m + 1 < s.P;
    const int64_t wrow = (static_cast<int64_t>(n) * s.P + m) * s.Q;  // window (m, 0)
    // windows (m, k), (m + 1, k) carried from the previous block's right-hand pair
    uchar4 a00 = none, a10 = none;
    float4 g00 = zero4(), g10 = zero4();
    if (GATHER) {
      a00 = arg[(wrow + k0) * C4 + c4];
      g00 = dyp[(wrow + k0) * C4 + c4];
      if (m1) {
        a10 = arg[(wrow + s.Q + k0) * C4 + c4];
        g10 = dyp[(wrow + s.Q + k0) * C4 + c4];
      }
    }
    static_assert(kPbRun == 8, "the unrolled run");
#pragma unroll 4
    for (int k = k0; k < k1e; ++k) {
      float4 o[4];
      const int64_t r0 = ((static_cast<int64_t>(n) * s.H + 2 * m) * s.W + 2 * k) * C4 + c4;
      const int64_t r1 = r0 + static_cast<int64_t>(s.W) * C4;
      if (GATHER) {
        const bool k1 = k + 1 < s.Q;
        uchar4 a01 = none, a11 = none;
        float4 g01 = zero4(), g11 = zero4();
        if (k1) {
          a01 = arg[(wrow + k + 1) * C4 + c4];
          g01 = dyp[(wrow + k + 1) * C4 + c4];
          if (m1) {
            a11 = arg[(wrow + s.Q + k + 1) * C4 + c4];
            g11 = dyp[(wrow + s.Q + k + 1) * C4 + c4];
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) o[q] = zero4();
#define SN_PICK(A, G, OFF, ACC)        \
  ACC.x += (A.x == (OFF)) ? G.x : 0.f; \
  ACC.y += (A.y == (OFF)) ? G.y : 0.f; \
  ACC.z += (A.z == (OFF)) ? G.z : 0.f; \
  ACC.w += (A.w == (OFF)) ? G.w : 0.f;
        SN_PICK(a00, g00, 4, o[0]);
        SN_PICK(a00, g00, 5, o[1]); SN_PICK(a01, g01, 3, o[1]);
        SN_PICK(a00, g00, 7, o[2]); SN_PICK(a10, g10, 1, o[2]);
        SN_PICK(a00, g00, 8, o[3]); SN_PICK(a01, g01, 6, o[3]);
        SN_PICK(a10, g10, 2, o[3]); SN_PICK(a11, g11, 0, o[3]);
#undef SN_PICK
        a00 = a01, g00 = g01, a10 = a11, g10 = g11;
      } else {
        o[0] = dym[r0];
        o[1] = dym[r0 + C4];
        o[2] = dym[r1];
        o[3] = dym[r1 + C4];
      }
      const float4 xv[4] = {x[r0], x[r0 + C4], x[r1], x[r1 + C4]};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float4 fa, fb;
        op.comp(p, RedBnBwdOp::R{o[q], xv[q]}, fa, fb);
        add4(a, fa);
        add4(b, fb);
      }
    }
  }
  // block combination: thread t holds quad t % C4 (kPbThreads % C4 == 0)
  for (int plane = 0; plane < 2; ++plane) {
    sh[threadIdx.x] = plane ? b : a;
    __syncthreads();
    for (int q = threadIdx.x; q < C4; q += blockDim.x) {
      double acc[4] = {0, 0, 0, 0};
      for (int tt = q; tt < static_cast<int>(blockDim.x); tt += C4) {
        const float4 w = sh[tt];
        acc[0] += w.x; acc[1] += w.y; acc[2] += w.z; acc[3] += w.w;
      }
      double* dst = part + (static_cast<size_t>(blockIdx.x) * 2 + plane) * s.C + q * 4;
      for (int e = 0; e < 4; ++e) dst[e] = acc[e];
    }
    __syncthreads();
  }
}

bool pool_bn_stats_ok(const PoolShape& ps, int bn_C) {
  return pool_bwd_argmax_only(ps) && ps.C == bn_C && ps.C % 4 == 0 && kPbThreads % (ps.C / 4) == 0 &&
         static_cast<int64_t>(ps.N) * ps.P * ((ps.Q + kPbRun - 1) / kPbRun) * (ps.C / 4) < (int64_t(1) << 31);
}

cudaError_t bn_bwd_pool_stats(const PoolShape& ps, const uint8_t* argmax, const float* dy_pool, const float* dy_mat,
                              const float* x, int C, const float* gamma, const float* beta, const float* stats,
                              int relu, float* dgamma, float* dbeta, float* red_scratch, cudaStream_t st) {
  if (!pool_bn_stats_ok(ps, C)) return cudaErrorInvalidValue;
  const int items = ps.N * ps.P * ((ps.Q + kPbRun - 1) / kPbRun) * (C / 4);
  const int nb = (items + kPbThreads - 1) / kPbThreads;
  const int grid = nb < 1 ? 1 : (nb > kPbBlocks ? kPbBlocks : nb);
  double* part = reinterpret_cast<double*>(red_scratch);
  float* coef = bn_coef_ptr(red_scratch, C);
  const uchar4* arg = reinterpret_cast<const uchar4*>(argmax);
  if (dy_mat) {
    pool_bn_stats_kernel<false><<<grid, kPbThreads, 0, st>>>(ps, arg, nullptr, reinterpret_cast<const float4*>(dy_mat),
                                   reinterpret_cast<const float4*>(x), stats, gamma, beta, relu, items, part);
  } else {
    if (!argmax || !dy_pool) return cudaErrorInvalidValue;
    pool_bn_stats_kernel<true><<<grid, kPbThreads, 0, st>>>(ps, arg, reinterpret_cast<const float4*>(dy_pool), nullptr,
                                   reinterpret_cast<const float4*>(x), stats, gamma, beta, relu, items, part);
  }
  colred_stage2<<<stage2_blocks(C), kStage2Threads, 0, st>>>(part, grid, C, BnBwdFin{C, dgamma, dbeta, coef});
  if (xskip(512)) colred_stage2<<<stage2_blocks(C), kStage2Threads, 0, st>>>(part, grid, C, BnBwdFin{C, dgamma, dbeta, coef});
  return cudaGetLastError();
}

cudaError_t relu_fwd(const float* x, float* y, int64_t n, cudaStream_t st) {
  const int64_t n4 = n / 4;
  if (n4) relu_fwd_kernel<<<elt_blocks(n4), kThreads, 0, st>>>(reinterpret_cast<const float4*>(x),
                                                                   reinterpret_cast<float4*>(y), n4);
  if (n % 4) relu_fwd_tail<<<1, 4, 0, st>>>(x, y, n4 * 4, n);
  return cudaGetLastError();
}

__global__ void relu_bwd_to_kernel(const float* __restrict__ y, const float* __restrict__ dy, float* dx, int64_t n,
                                   int accumulate) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const float v = y[i] > 0.f ? dy[i] : 0.f;
    dx[i] = accumulate ? dx[i] + v : v;
  }
}

cudaError_t relu_bwd_to(const float* y, const float* dy, float* dx, int64_t n, int accumulate, cudaStream_t st) {
  relu_bwd_to_kernel<<<blocks_for(n), kThreads, 0, st>>>(y, dy, dx, n, accumulate);
  return cudaGetLastError();
}

cudaError_t relu_bwd_inplace(const float* y, float* g, int64_t n, cudaStream_t st) {
  const int64_t n4 = n / 4;
  if (n4) relu_bwd_kernel<<<elt_blocks(n4), kThreads, 0, st>>>(reinterpret_cast<const float4*>(y),
                                                                   reinterpret_cast<float4*>(g), n4);
  if (n % 4) relu_bwd_tail<<<1, 4, 0, st>>>(y, g, n4 * 4, n);
  return cudaGetLastError();
}

// channel quads per block of the band kernel: the largest divisor of C/4 with
// Q * CS <= 448 threads (0: not applicable)
static int pool_k3s2_band_cs(const PoolShape& s) {
  if (!(s.mode == 0 && s.K == 3 && s.stride == 2 && s.pad == 1 && s.H == 2 * s.P && s.W == 2 * s.Q && s.C % 4 == 0))
    return 0;
  const int C4 = s.C / 4;
  for (int cs = C4; cs >= 1; --cs)
    if (C4 % cs == 0 && s.Q * cs <= 448) return s.Q * cs >= 128 ? cs : 0;
  return 0;
}
static bool pool_k3s2_band_ok(const PoolShape& s) { return pool_k3s2_band_cs(s) > 0; }
static void pool_k3s2_band(const PoolShape& s, bool bnr, const float* x, float* y, uint8_t* argmax,
                           const float* stats, const float* gamma, const float* beta, float* y_relu,
                           cudaStream_t st) {
  // 14 output rows per block (ResNet stem: 4 bands per image): 195 vs 221 us
  // at 4 rows (fewer halo-row reloads and block starts; 14, 28 tie)
  const int PB = 14, CS = pool_k3s2_band_cs(s);
  const dim3 grid((s.P + PB - 1) / PB, s.N, s.C / 4 / CS);
  auto k = bnr ? pool_fwd_k3s2_band_kernel<true> : pool_fwd_k3s2_band_kernel<false>;
  k<<<grid, s.Q * CS, 0, st>>>(s, PB, CS, reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y),
                               reinterpret_cast<uchar4*>(argmax), stats, gamma, beta,
                               reinterpret_cast<float4*>(y_relu));
}

cudaError_t pool_fwd(const PoolShape& s, const float* x, float* y, cudaStream_t st, uint8_t* argmax) {
  const int64_t total = static_cast<int64_t>(s.N) * s.P * s.Q * s.C;
  if (s.C % 4 == 0 && static_cast<int64_t>(s.N) * s.H * s.W * s.C < (1ll << 31)) {
    if (s.P == 1 && s.Q == 1 && s.pad == 0 && s.K == s.H && s.K == s.W) {
      dim3 grid((s.C / 4 + 31) / 32, s.N);
      pool_global_kernel<<<grid, 256, 0, st>>>(s, reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y));
      return cudaGetLastError();
    }
    if (pool_k3s2_band_ok(s)) {
      pool_k3s2_band(s, false, x, y, argmax, nullptr, nullptr, nullptr, nullptr, st);
      return cudaGetLastError();
    }
    if (s.K == 3 && s.stride == 2) {
      pool_fwd_rows_kernel<3, 2, false><<<dim3(s.P, s.N), 256, 0, st>>>(
          s, reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y), reinterpret_cast<uchar4*>(argmax),
          nullptr, nullptr, nullptr, nullptr);
      return cudaGetLastError();
    }
    const int total4 = static_cast<int>(total / 4);
    auto k = s.K == 3 ? pool_fwd_v4_kernel<3> : (s.K == 2 ? pool_fwd_v4_kernel<2> : pool_fwd_v4_kernel<0>);
    k<<<blocks_for(total4), kThreads, 0, st>>>(s, reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y),
                                               total4);
    return cudaGetLastError();
  }
  pool_fwd_kernel<<<blocks_for(total), kThreads, 0, st>>>(s, x, y, total);
  return cudaGetLastError();
}

static bool pool_fused_ok(const PoolShape& s, int* PB, int* WR, size_t* smem) {
  if (s.mode != 0 || s.C % (4 * kPoolCv) != 0 || s.K * s.K >= 255 || s.stride < 1) return false;
  // band of PB output rows: enough windows per block to amortise the edge re-evaluation
  *PB = s.P >= 8 ? 4 : s.P;
  *WR = *PB + (s.K - 1) / s.stride + 1;
  *smem = static_cast<size_t>(*WR) * s.Q * kPoolCv * (sizeof(float4) + sizeof(uchar4));
  return *smem <= 48 * 1024;
}

int pool_bwd_kernels(const PoolShape& s) {
  int PB, WR;
  size_t smem;
  if (pool_fused_ok(s, &PB, &WR, &smem)) return 1;
  return (s.C % 4 == 0 && s.mode == 0 && s.K * s.K < 255) ? 2 : 1;
}

int64_t pool_scratch_bytes(const PoolShape& s) {
  if (pool_bwd_kernels(s) == 1) return 0;
  return (s.C % 4 == 0 && s.mode == 0 && s.K * s.K < 255) ? static_cast<int64_t>(s.N) * s.P * s.Q * s.C : 0;
}

bool pool_saves_argmax(const PoolShape& s) {
  int PB, WR;
  size_t smem;
  return s.mode == 0 && s.K == 3 && s.stride == 2 && s.C % 4 == 0 && !(s.P == 1 && s.Q == 1) &&
         static_cast<int64_t>(s.N) * s.H * s.W * s.C < (1ll << 31) && pool_fused_ok(s, &PB, &WR, &smem);
}

bool pool_bwd_argmax_only(const PoolShape& s) {
  return pool_saves_argmax(s) && s.pad == 1 && s.H == 2 * s.P && s.W == 2 * s.Q;
}

bool pool_fwd_bn_relu_ok(const PoolShape& s) { return pool_bwd_argmax_only(s) && s.C / 4 <= kPoolBnMaxC4; }

cudaError_t pool_fwd_bn_relu(const PoolShape& s, const float* x, const float* gamma, const float* beta,
                             const float* stats, float* y_relu, float* y, uint8_t* argmax, cudaStream_t st) {
  if (!pool_fwd_bn_relu_ok(s) || !argmax) return cudaErrorInvalidValue;
  if (pool_k3s2_band_ok(s)) {
    pool_k3s2_band(s, true, x, y, argmax, stats, gamma, beta, y_relu, st);
    return cudaGetLastError();
  }
  pool_fwd_rows_kernel<3, 2, true><<<dim3(s.P, s.N), 256, 0, st>>>(
      s, reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y), reinterpret_cast<uchar4*>(argmax), stats,
      gamma, beta, reinterpret_cast<float4*>(y_relu));
  return cudaGetLastError();
}

cudaError_t pool_bwd(const PoolShape& s, const float* x, const float* y, const float* dy, float* dx, int accumulate,
                     void* scratch, cudaStream_t st, const uint8_t* argmax) {
  if (argmax && pool_bwd_argmax_only(s)) {
    const int64_t total = static_cast<int64_t>(s.N) * s.P * s.Q * (s.C / 4);
    pool_max_bwd_k3s2<<<blocks_for(total, kThreads, 148 * 32), kThreads, 0, st>>>(
        s, reinterpret_cast<const uchar4*>(argmax), reinterpret_cast<const float4*>(dy), reinterpret_cast<float4*>(dx),
        accumulate, total);
    return cudaGetLastError();
  }
  int PB, WR;
  size_t smem;
  if (pool_fused_ok(s, &PB, &WR, &smem)) {
    dim3 grid(s.C / (4 * kPoolCv), (s.P + PB - 1) / PB, s.N);
    auto k = (s.K == 3 && s.stride == 2)   ? pool_max_bwd_fused<3, 2>
             : (s.K == 2 && s.stride == 2) ? pool_max_bwd_fused<2, 2>
             : s.K == 3                    ? pool_max_bwd_fused<3, 0>
                                           : pool_max_bwd_fused<0, 0>;
    k<<<grid, 256, smem, st>>>(s, reinterpret_cast<const float4*>(x), reinterpret_cast<const float4*>(y),
                               reinterpret_cast<const float4*>(dy), reinterpret_cast<float4*>(dx), accumulate, PB,
                               WR, reinterpret_cast<const uchar4*>(argmax));
    return cudaGetLastError();
  }
  if (s.C % 4 == 0 && (s.mode == 1 || (scratch && s.K * s.K < 255))) {
    const int in4 = static_cast<int>(static_cast<int64_t>(s.N) * s.H * s.W * s.C / 4);
    const int out4 = static_cast<int>(static_cast<int64_t>(s.N) * s.P * s.Q * s.C / 4);
    uchar4* arg = reinterpret_cast<uchar4*>(scratch);
    if (s.mode == 0) pool_argmax_kernel<<<blocks_for(out4), kThreads, 0, st>>>(s, x, y, arg, out4);
    pool_gather_kernel<<<blocks_for(in4), kThreads, 0, st>>>(s, arg, dy, dx, accumulate, in4);
    return cudaGetLastError();
  }
  const int64_t total = static_cast<int64_t>(s.N) * s.H * s.W * s.C;
  pool_bwd_kernel<<<blocks_for(total), kThreads, 0, st>>>(s, x, y, dy, dx, accumulate, total);
  return cudaGetLastError();
}

cudaError_t lrn_fwd(const float* x, float* y, int64_t pixels, int C, int size, float alpha, float beta, float k,
                    cudaStream_t st) {
  const int64_t total = pixels * C;
  lrn_fwd_kernel<<<blocks_for(total), kThreads, 0, st>>>(x, y, total, C, size, alpha, beta, k);
  return cudaGetLastError();
}

cudaError_t lrn_bwd(const float* x, const float* y, const float* dy, float* dx, int64_t pixels, int C, int size,
                    float alpha, float beta, float k, int accumulate, cudaStream_t st) {
  const int64_t total = pixels * C;
  lrn_bwd_kernel<<<blocks_for(total), kThreads, 0, st>>>(x, y, dy, dx, total, C, size, alpha, beta, k, accumulate);
  return cudaGetLastError();
}

static uint32_t drop_thresh(float rate) {
  double t = static_cast<double>(rate) * 4294967296.0;
  if (t < 0) t = 0;
  if (t > 4294967295.0) t = 4294967295.0;
  return static_cast<uint32_t>(t);
}

cudaError_t dropout_fwd(const float* x, float* y, int64_t n, float rate, uint64_t seed, int layer,
                        const uint32_t* iteration, cudaStream_t st) {
  dropout_fwd_kernel<<<blocks_for(n), kThreads, 0, st>>>(x, y, n, drop_thresh(rate), 1.0f / (1.0f - rate), seed, layer,
                                                         iteration);
  return cudaGetLastError();
}

__global__ void dropout_bwd_to_kernel(const float* __restrict__ dy, float* dx, int64_t n, uint32_t thresh, float scale,
                                      uint64_t seed, int layer, const uint32_t* iteration, int accumulate) {
  const uint32_t it = *iteration;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const float v = drop_keep(seed, layer, it, static_cast<uint32_t>(i), thresh) ? dy[i] * scale : 0.f;
    dx[i] = accumulate ? dx[i] + v : v;
  }
}

cudaError_t dropout_bwd_to(const float* dy, float* dx, int64_t n, float rate, uint64_t seed, int layer,
                           const uint32_t* iteration, int accumulate, cudaStream_t st) {
  dropout_bwd_to_kernel<<<blocks_for(n), kThreads, 0, st>>>(dy, dx, n, drop_thresh(rate), 1.0f / (1.0f - rate), seed,
                                                            layer, iteration, accumulate);
  return cudaGetLastError();
}

cudaError_t dropout_bwd_inplace(float* g, int64_t n, float rate, uint64_t seed, int layer, const uint32_t* iteration,
                                cudaStream_t st) {
  dropout_bwd_kernel<<<blocks_for(n), kThreads, 0, st>>>(g, n, drop_thresh(rate), 1.0f / (1.0f - rate), seed, layer,
                                                         iteration);
  return cudaGetLastError();
}

cudaError_t softmax_fwd(const float* x, float* y, int B, int F, const int32_t* labels, float* loss_rows,
                        cudaStream_t st) {
  const int threads = 256;
  softmax_fwd_kernel<<<(B * 32 + threads - 1) / threads, threads, 0, st>>>(x, y, B, F, labels, loss_rows);
  return cudaGetLastError();
}

cudaError_t softmax_ce_bwd(const float* y, const int32_t* labels, float* dx, int B, int F, int accumulate,
                           cudaStream_t st) {
  softmax_bwd_kernel<<<blocks_for(static_cast<int64_t>(B) * F), kThreads, 0, st>>>(y, labels, dx, B, F, accumulate);
  return cudaGetLastError();
}

cudaError_t loss_reduce(const float* loss_rows, int B, float* loss, cudaStream_t st) {
  loss_reduce_kernel<<<1, 256, 0, st>>>(loss_rows, B, loss);
  return cudaGetLastError();
}

cudaError_t join_fwd(const float* const* inputs, int n_in, float* y, int64_t n, cudaStream_t st) {
  join_fwd_kernel<<<elt_blocks(n / 4 + 1), kThreads, 0, st>>>(inputs, n_in, y, n);
  return cudaGetLastError();
}

namespace {
// k-way JOIN backward: one read of dy, every destination written (or added,
// old + dy as grad_copy does) in the same pass
constexpr int kMultiDst = 8;
struct MultiDst {
  float4* d[kMultiDst];
  int acc[kMultiDst];
  int k;
};
__global__ void grad_copy_multi_kernel(const float4* __restrict__ src, MultiDst md, int64_t n4) {
  const int64_t T = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i0 < n4; i0 += 2 * T) {
    float4 v[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) v[u] = i0 + u * T < n4 ? src[i0 + u * T] : zero4();
    for (int t = 0; t < md.k; ++t) {
      float4* d = md.d[t];
      float4 o[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) o[u] = (md.acc[t] && i0 + u * T < n4) ? d[i0 + u * T] : zero4();
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (i0 + u * T >= n4) continue;
        float4 w = v[u];
        if (md.acc[t]) add4(w, o[u]);
        d[i0 + u * T] = w;
      }
    }
  }
}
// One step of a dense JOIN chain's backward (the executor's dense_chain): the
// running sum r (+)= dy, then every destination d (+)= r.  The additions are
// the ones the per-destination JOIN backward would make, in the same order.
__global__ void grad_prefix_kernel(const float4* __restrict__ src, float4* r, int acc_r, MultiDst md, int64_t n4) {
  const int64_t T = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i0 < n4; i0 += 2 * T) {
    float4 v[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t i = i0 + u * T;
      v[u] = i < n4 ? src[i] : zero4();
      if (acc_r && i < n4) add4(v[u], r[i]);
      if (i < n4) r[i] = v[u];
    }
    for (int t = 0; t < md.k; ++t) {
      float4* d = md.d[t];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int64_t i = i0 + u * T;
        if (i >= n4) continue;
        float4 w = v[u];
        if (md.acc[t]) add4(w, d[i]);
        d[i] = w;
      }
    }
  }
}
}  // namespace

int grad_prefix_launches(int k) { return 1 + (k > kMultiDst ? grad_copy_multi_launches(k - kMultiDst) : 0); }

cudaError_t grad_prefix(const float* src, float* r, int acc_r, float* const* dsts, const int* accs, int k, int64_t n,
                        cudaStream_t st) {
  if (n % 4 != 0) return cudaErrorInvalidValue;
  MultiDst md{};
  md.k = std::min(kMultiDst, k);
  for (int t = 0; t < md.k; ++t) {
    md.d[t] = reinterpret_cast<float4*>(dsts[t]);
    md.acc[t] = accs[t];
  }
  grad_prefix_kernel<<<elt_blocks(n / 4), kThreads, 0, st>>>(reinterpret_cast<const float4*>(src),
                                                            reinterpret_cast<float4*>(r), acc_r, md, n / 4);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || k <= kMultiDst) return e;
  return grad_copy_multi(r, dsts + kMultiDst, accs + kMultiDst, k - kMultiDst, n, st);
}

int grad_copy_multi_launches(int k) { return (k + kMultiDst - 1) / kMultiDst; }

cudaError_t grad_copy_multi(const float* src, float* const* dsts, const int* accs, int k, int64_t n, cudaStream_t st) {
  if (n % 4 != 0) return cudaErrorInvalidValue;
  for (int t0 = 0; t0 < k; t0 += kMultiDst) {
    MultiDst md{};
    md.k = std::min(kMultiDst, k - t0);
    for (int t = 0; t < md.k; ++t) {
      md.d[t] = reinterpret_cast<float4*>(dsts[t0 + t]);
      md.acc[t] = accs[t0 + t];
    }
    grad_copy_multi_kernel<<<elt_blocks(n / 4), kThreads, 0, st>>>(reinterpret_cast<const float4*>(src), md, n / 4);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t grad_copy(const float* src, float* dst, int64_t n, int accumulate, cudaStream_t st) {
  grad_copy_kernel<<<elt_blocks(n / 4 + 1), kThreads, 0, st>>>(src, dst, n, accumulate);
  return cudaGetLastError();
}

cudaError_t sgd_update(float* params, const float* grads, int64_t n, float lr, float grad_scale, cudaStream_t st) {
  sgd_kernel<<<blocks_for(n), kThreads, 0, st>>>(params, grads, n, lr, grad_scale);
  return cudaGetLastError();
}

__global__ void pad_channels_kernel(const float* __restrict__ raw, int C_raw, float* __restrict__ out, int Cs,
                                    int64_t total) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total; i += stride) {
    const int c = static_cast<int>(i % Cs);
    out[i] = c < C_raw ? raw[(i / Cs) * C_raw + c] : 0.f;
  }
}

cudaError_t pad_channels(const float* raw, int C_raw, float* out, int Cs, int64_t pixels, cudaStream_t st) {
  pad_channels_kernel<<<blocks_for(pixels * Cs), kThreads, 0, st>>>(raw, C_raw, out, Cs, pixels * Cs);
  return cudaGetLastError();
}

cudaError_t sgd_update_flagged(float* params, const float* grads, int64_t n, float lr, float grad_scale,
                               const int* flag, cudaStream_t st) {
  sgd_flagged_kernel<<<blocks_for(n), kThreads, 0, st>>>(params, grads, n, lr, grad_scale, flag);
  return cudaGetLastError();
}

cudaError_t bump_iteration(uint32_t* iteration, cudaStream_t st) {
  bump_kernel<<<1, 1, 0, st>>>(iteration);
  return cudaGetLastError();
}

cudaError_t fill_zero(float* p, int64_t n, cudaStream_t st) {
  zero_kernel<<<blocks_for(n), kThreads, 0, st>>>(p, n);
  return cudaGetLastError();
}

}  // namespace sn
