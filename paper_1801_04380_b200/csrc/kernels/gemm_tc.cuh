// Warp-specialised tcgen05 (kind::tf32) GEMM core used by every dense
// contraction of the training step: CONV forward / dgrad / wgrad as
// implicit GEMMs and the FC layers as plain GEMMs.
//
//   D[M x N] (+)= A[M x K] . B[N x K]^T          fp32 in HBM, tf32 MMA, fp32 acc
//
// One CTA computes one BM=128 x BN tile for a range of K blocks (split-K over
// gridDim.z).  Warps 0-3 are producers (cp.async 16 B into SWIZZLE_128B smem
// stages, zero fill for padding / out-of-range rows) and afterwards the
// epilogue (tcgen05.ld of the TMEM accumulator); warp 4 allocates TMEM and one
// elected lane issues the tcgen05.mma chain.  Operands are either K-major
// (128-byte rows hold 32 consecutive k of one row) or MN-major (128-byte rows
// hold 32 consecutive rows of one k), so transposed operands (dgrad/wgrad) are
// fed directly from their NHWC layout without a transpose pass.
//
// fp32-faithful mode (SPLIT3, "3xTF32"): after a stage lands, the producers
// split every operand element in place into hi = tf32_rn(x) and a residual
// lo = x - hi (exact in fp32) written to a twin buffer of the same swizzled
// layout, and the issuer accumulates hi.hi + hi.lo + lo.hi per K = 8 step.
// The dropped lo.lo term and the tf32 rounding of lo are ~2^-22 relative:
// fp32-level products, at 3x the MMA work and half the pipeline depth (the
// twins double the smem per stage).  The tensor core's accumulation into TMEM
// is not round-to-nearest: measured (tools/precision_probe.py) it loses about
// 2^-25 of the running sum per MMA, toward zero, so a long K chain drifts
// (K = 2048: 2.3e-5 on positive data), and that drift is biased, so it
// compounds through a deep network.  SPLIT3 therefore restarts the TMEM
// accumulator every split3_group() k blocks: the producer warps add each
// group's partial into a running sum in TMEM (fp32 round-to-nearest on the
// CUDA cores) and the epilogue adds the last group -- the drift is bounded by
// one group's 12 * group MMAs whatever K is.  With BN <= 128 two partial
// accumulators alternate (one k block per group, drained while the tensor
// core fills the other); BN = 256 has room for one (4 blocks per group, the
// MMA waits for each drain).  lo is rounded to tf32 explicitly, so the
// hardware's own operand conversion drops nothing (unbiased).
//
// The operand gathers are policy objects (see conv loaders in conv_tc.cu):
//   struct Loader { __device__ void tile_init(int r0, void* scratch, int tid);
//                   __device__ void load(uint32_t smem_tile, int kb, int tid); };
#pragma once
#include "tc_common.cuh"

namespace sn {

constexpr int kBM = 128;     // MMA M (rows of the tile, TMEM lanes)
constexpr int kBK = 32;      // fp32 elements per k block (= one 128 B swizzle row)
constexpr int kProducers = 128;
constexpr int kGemmThreads = 160;
constexpr int kScratchBytes = 4096;  // per-operand tile_init scratch (row tables)

template <int BN, int STAGES, bool SPLIT3 = false>
struct GemmSmem {
  static constexpr int A_BYTES = kBM * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int STAGE_BYTES = (A_BYTES + B_BYTES) * (SPLIT3 ? 2 : 1);
  static constexpr int LO_OFF = STAGES * (A_BYTES + B_BYTES);  // SPLIT3: lo twins of every stage
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int SCRATCH_OFF = BAR_OFF + 256;
  static constexpr int TOTAL = SCRATCH_OFF + 2 * kScratchBytes + 1024;  // +1024 alignment slack
};

template <int BN>
__host__ __device__ constexpr uint32_t tmem_cols() {
  return BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
}
// SPLIT3 accumulation: partial accumulators in TMEM and k blocks per group
template <int BN>
constexpr int split3_accs() {
  return BN <= 128 ? 2 : 1;
}
template <int BN>
constexpr int split3_group() {
  return split3_accs<BN>() == 2 ? 1 : 4;
}

// MN-major tile of 32 k-rows x R mn-elements in the SWIZZLE_128B_BASE32B
// canonical layout: MN atoms (32 elements x 4 k rows = 512 B) are adjacent
// (LBO = 512), K atoms (4 k rows) are R*16 B apart (SBO).
template <int R>
struct MNTile {
  static constexpr uint32_t LBO = 512;
  static constexpr uint32_t SBO = (R / 32) * 512;
};
template <int R>
__device__ __forceinline__ uint32_t mn_tile_off(uint32_t krow, uint32_t mchunk) {
  const uint32_t r4 = krow & 3u;
  const uint32_t c16 = mchunk & 7u;
  return (krow >> 2) * MNTile<R>::SBO + (mchunk >> 3) * MNTile<R>::LBO + (r4 << 7) +
         ((((c16 >> 1) ^ r4) & 3u) << 5) + ((c16 & 1u) << 4);
}

// hi = x rounded to tf32 (low 13 mantissa bits zero), lo = x - hi (exact).
__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// Split a tile of `bytes` (a multiple of 128 * 16) in place: tile -> hi, twin -> lo.
template <int BYTES>
__device__ __forceinline__ void split3_tile(uint8_t* tile, uint8_t* twin, int tid) {
#pragma unroll 4
  for (int off = tid * 16; off < BYTES; off += kProducers * 16) {
    float4 v = *reinterpret_cast<const float4*>(tile + off);
    const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
    *reinterpret_cast<float4*>(tile + off) = h;
    *reinterpret_cast<float4*>(twin + off) =
        make_float4(tf32_hi(v.x - h.x), tf32_hi(v.y - h.y), tf32_hi(v.z - h.z), tf32_hi(v.w - h.w));
  }
}

template <int BN, int STAGES, bool A_MN, bool B_MN, class LA, class LB, class EPI, bool SPLIT3 = false>
__global__ void __launch_bounds__(kGemmThreads, 1)
    tc_gemm_kernel(LA la, LB lb, EPI epi, int num_kb, int kb_per_split) {
  using L = GemmSmem<BN, STAGES, SPLIT3>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * L::A_BYTES;
  uint8_t* sA_lo = smem + L::LO_OFF;  // SPLIT3 only
  uint8_t* sB_lo = sA_lo + STAGES * L::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint64_t* drain_full = done + 1;   // SPLIT3 [2]: a group's partial is complete in TMEM
  uint64_t* drain_empty = done + 3;  // SPLIT3 [2]: ... and folded into the running sum
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 5);
  uint8_t* scratch_a = smem + L::SCRATCH_OFF;
  uint8_t* scratch_b = scratch_a + kScratchBytes;

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int m0 = blockIdx.x * kBM;
  const int n0 = blockIdx.y * BN;
  const int kb0 = blockIdx.z * kb_per_split;
  const int kb1 = min(num_kb, kb0 + kb_per_split);
  const int nkb = kb1 - kb0;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], kProducers);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    for (int a = 0; a < 2; ++a) {
      mbar_init(&drain_full[a], 1);
      mbar_init(&drain_empty[a], kProducers);
    }
    fence_mbar_init();
  }
  constexpr int kAcc = SPLIT3 ? split3_accs<BN>() : 1;
  constexpr int kG = split3_group<BN>();
  // SPLIT3: kAcc partial accumulators + the running sum (a power of two of columns)
  constexpr uint32_t kTmemCols = tmem_cols<BN>() * (SPLIT3 ? (kAcc == 2 ? 4 : 2) : 1);
  if (warp == 4) tmem_alloc(tmem_slot, kTmemCols);
  if (tid < kProducers) {
    la.tile_init(m0, scratch_a, tid);
    lb.tile_init(n0, scratch_b, tid);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int last_group = (nkb - 1) / kG;  // SPLIT3 accumulation groups 0 .. last_group
  if (warp < 4) {
    // ---------------- producers ----------------
    constexpr int LAG = STAGES - 1;
    // a landed stage: (SPLIT3) every producer's copies are in, split it, then
    // publish it to the tensor core
    auto publish = [&](int j) {
      const int s = j % STAGES;
      if constexpr (SPLIT3) {
        named_bar(1, kProducers);
        split3_tile<L::A_BYTES>(sA + s * L::A_BYTES, sA_lo + s * L::A_BYTES, tid);
        split3_tile<L::B_BYTES>(sB + s * L::B_BYTES, sB_lo + s * L::B_BYTES, tid);
      }
      fence_proxy_async();
      mbar_arrive(&full[s]);
    };
    const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
    const uint32_t run_col = tmem_cols<BN>() * kAcc;
    // SPLIT3: fold group d's TMEM partial into the running sum (RN adds).  With
    // two accumulators this runs after the first block of group d + 1 is
    // published, so the tensor core fills the other one meanwhile.
    auto drain_after = [&](int j) {
      if constexpr (SPLIT3) {
        const int d = (j + 1 - kAcc) / kG;  // candidate group finished by publishing j
        if (j + 1 - kAcc < 0 || (j + 1 - kAcc) % kG != kG - 1 || d >= last_group) return;
        const int a = d % kAcc;
        mbar_wait(&drain_full[a], (d / kAcc) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          float v[32];
          tmem_ld32(tmem + lane_base + static_cast<uint32_t>(a * tmem_cols<BN>() + c), v);
          if (d > 0) {
            float r[32];
            tmem_ld32(tmem + lane_base + run_col + static_cast<uint32_t>(c), r);
#pragma unroll
            for (int q = 0; q < 32; ++q) v[q] += r[q];
          }
          tmem_st32(tmem + lane_base + run_col + static_cast<uint32_t>(c), v);
        }
        tc_fence_before();
        mbar_arrive(&drain_empty[a]);
      }
    };
    for (int i = 0; i < nkb; ++i) {
      const int s = i % STAGES;
      if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
      la.load(smem_u32(sA + s * L::A_BYTES), kb0 + i, tid);
      lb.load(smem_u32(sB + s * L::B_BYTES), kb0 + i, tid);
      cp_async_commit();
      if (i >= LAG) {
        cp_async_wait<LAG>();
        publish(i - LAG);
        drain_after(i - LAG);
      }
    }
    cp_async_wait<0>();
    for (int j = (nkb > LAG ? nkb - LAG : 0); j < nkb; ++j) {
      publish(j);
      drain_after(j);
    }

    // ---------------- epilogue ----------------
    mbar_wait(done, 0);
    tc_fence_after();
    const int row = warp * 32 + lane;
    const bool drained = SPLIT3 && last_group > 0;
    const uint32_t acc_col = SPLIT3 ? static_cast<uint32_t>((last_group % kAcc) * tmem_cols<BN>()) : 0u;
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      float v[32];
      tmem_ld32(tmem + lane_base + acc_col + static_cast<uint32_t>(c), v);
      if (drained) {
        float r[32];
        tmem_ld32(tmem + lane_base + run_col + static_cast<uint32_t>(c), r);
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] += r[q];
      }
      epi.store(m0 + row, n0 + c, v, blockIdx.z);
    }
    tc_fence_before();
  } else if (lane == 0) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc = idesc_tf32(kBM, BN, A_MN, B_MN);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % STAGES;
      // SPLIT3: group g accumulates from zero into accumulator g % kAcc once
      // that accumulator's previous group has been folded into the running sum
      const int g = i / kG;
      const bool fresh = SPLIT3 ? (i % kG == 0) : (i == 0);
      const uint32_t dtm = tmem + (SPLIT3 ? static_cast<uint32_t>((g % kAcc) * tmem_cols<BN>()) : 0u);
      if (SPLIT3 && fresh && g >= kAcc) {
        mbar_wait(&drain_empty[g % kAcc], ((g - kAcc) / kAcc) & 1);
        tc_fence_after();
      }
      mbar_wait(&full[s], (i / STAGES) & 1);
      tc_fence_after();
      const uint32_t a0 = smem_u32(sA + s * L::A_BYTES);
      const uint32_t b0 = smem_u32(sB + s * L::B_BYTES);
#pragma unroll
      for (int kk = 0; kk < kBK / 8; ++kk) {
        // One MMA consumes K = 8: 32 B of each K-major row, or two 4-row K
        // atoms of an MN-major tile.
        const uint64_t ad =
            A_MN ? umma_desc(a0 + kk * 2 * MNTile<kBM>::SBO, MNTile<kBM>::LBO, MNTile<kBM>::SBO,
                             kLayoutSW128Base32)
                 : umma_desc(a0 + kk * 32, 16, 1024, kLayoutSW128);
        const uint64_t bd =
            B_MN ? umma_desc(b0 + kk * 2 * MNTile<BN>::SBO, MNTile<BN>::LBO, MNTile<BN>::SBO,
                             kLayoutSW128Base32)
                 : umma_desc(b0 + kk * 32, 16, 1024, kLayoutSW128);
        umma_tf32(dtm, ad, bd, idesc, (fresh && kk == 0) ? 0u : 1u);
        if constexpr (SPLIT3) {
          // the twins sit at a fixed offset with the same 1024-aligned swizzle
          // phase: the descriptors differ only in their start address (16 B units)
          constexpr uint64_t kLoA = static_cast<uint64_t>(L::LO_OFF) >> 4;
          umma_tf32(dtm, ad, bd + kLoA, idesc, 1u);
          umma_tf32(dtm, ad + kLoA, bd, idesc, 1u);
        }
      }
      umma_commit(&empty[s]);
      if (SPLIT3 && (i % kG == kG - 1) && g < last_group) umma_commit(&drain_full[g % kAcc]);
    }
    umma_commit(done);
  }
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

// Numeric mode of the gather GEMMs (set_precision in kernels.hpp): 0 tf32,
// 1 fp32-faithful 3xTF32 (SPLIT3).
int gemm_precision();

template <int BN, int STAGES, bool A_MN, bool B_MN, bool SPLIT3, class LA, class LB, class EPI>
inline cudaError_t launch_tc_gemm_impl(const LA& la, const LB& lb, const EPI& epi, int M, int N, int K,
                                       int splits, cudaStream_t stream) {
  using L = GemmSmem<BN, STAGES, SPLIT3>;
  auto kern = tc_gemm_kernel<BN, STAGES, A_MN, B_MN, LA, LB, EPI, SPLIT3>;
  static bool attr_set = false;  // per template instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int num_kb = (K + kBK - 1) / kBK;
  if (splits < 1) splits = 1;
  if (splits > num_kb) splits = num_kb;
  const int kps = (num_kb + splits - 1) / splits;
  splits = (num_kb + kps - 1) / kps;  // every split owns >= 1 k block
  dim3 grid((M + kBM - 1) / kBM, (N + BN - 1) / BN, splits);
  kern<<<grid, kGemmThreads, L::TOTAL, stream>>>(la, lb, epi, num_kb, kps);
  return cudaGetLastError();
}

// 3xTF32 stage depth: the lo twins double the smem of a stage
template <int BN>
constexpr int split3_stages() {
  return BN >= 256 ? 2 : (BN >= 128 ? 3 : 4);
}

template <int BN, int STAGES, bool A_MN, bool B_MN, class LA, class LB, class EPI>
inline cudaError_t launch_tc_gemm(const LA& la, const LB& lb, const EPI& epi, int M, int N, int K,
                                  int splits, cudaStream_t stream) {
  if (gemm_precision() == 1)
    return launch_tc_gemm_impl<BN, split3_stages<BN>(), A_MN, B_MN, true>(la, lb, epi, M, N, K, splits, stream);
  return launch_tc_gemm_impl<BN, STAGES, A_MN, B_MN, false>(la, lb, epi, M, N, K, splits, stream);
}

// Split count actually used by launch_tc_gemm for a requested count.
inline int effective_splits(int K, int splits) {
  const int num_kb = (K + kBK - 1) / kBK;
  if (splits < 1) splits = 1;
  if (splits > num_kb) splits = num_kb;
  const int kps = (num_kb + splits - 1) / splits;
  return (num_kb + kps - 1) / kps;
}

// ===========================================================================
// Generic strided-matrix loaders (FC layers, tests).
// ===========================================================================

// K-major operand: element (r, k) at base[r * ld + k], R rows per tile.
template <int R>
struct MatKLoader {
  const float* base;
  int rows, K, ld;
  int fast;  // base 16 B aligned and ld % 4 == 0 and K % 4 == 0
  int r0;
  __device__ void tile_init(int r0_, void*, int) { r0 = r0_; }
  __device__ void load(uint32_t tile, int kb, int tid) {
    const int warp = tid >> 5, lane = tid & 31;
    const int chunk = lane & 7;
    const int k = kb * kBK + chunk * 4;
#pragma unroll 4
    for (int it = 0; it < R / 16; ++it) {
      const int row = warp * (R / 4) + it * 4 + (lane >> 3);
      const int r = r0 + row;
      const uint32_t dst = tile + sw128_off(row, chunk);
      if (fast) {
        const bool ok = (r < rows) && (k < K);
        cp_async16(dst, ok ? base + static_cast<size_t>(r) * ld + k : base, ok ? 16u : 0u);
      } else {
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
          v[e] = (r < rows && k + e < K) ? __ldg(base + static_cast<size_t>(r) * ld + k + e) : 0.f;
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(dst), "f"(v[0]), "f"(v[1]),
                     "f"(v[2]), "f"(v[3])
                     : "memory");
      }
    }
  }
};

// MN-major operand: element (r, k) at base[k * ld + r], R rows per tile.
template <int R>
struct MatMNLoader {
  const float* base;
  int rows, K, ld;
  int fast;  // base 16 B aligned and ld % 4 == 0 and rows % 4 == 0
  int r0;
  __device__ void tile_init(int r0_, void*, int) { r0 = r0_; }
  __device__ void load(uint32_t tile, int kb, int tid) {
    constexpr int CPR = R / 4;             // 16-byte chunks per k row
    constexpr int TOTAL = 32 * CPR;        // chunks per tile
#pragma unroll 4
    for (int f = tid; f < TOTAL; f += kProducers) {
      const int krow = f / CPR, mc = f % CPR;
      const int k = kb * kBK + krow;
      const int r = r0 + mc * 4;
      const uint32_t dst = tile + mn_tile_off<R>(krow, mc);
      if (fast) {
        const bool ok = (k < K) && (r < rows);
        cp_async16(dst, ok ? base + static_cast<size_t>(k) * ld + r : base, ok ? 16u : 0u);
      } else {
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
          v[e] = (k < K && r + e < rows) ? __ldg(base + static_cast<size_t>(k) * ld + r + e) : 0.f;
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(dst), "f"(v[0]), "f"(v[1]),
                     "f"(v[2]), "f"(v[3])
                     : "memory");
      }
    }
  }
};

// Row-major output D[m * ldd + n] = alpha*acc + (beta ? D : 0) + bias[n].
struct EpiRowMajor {
  float* D;
  const float* bias;  // may be null
  int M, N, ldd;
  int accumulate;     // 1: D += acc, 0: D = acc
  __device__ void store(int m, int n0, const float* v, int) const {
    if (m >= M) return;
    float* d = D + static_cast<size_t>(m) * ldd;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int n = n0 + j;
      if (n < N) {
        float x = v[j];
        if (bias) x += __ldg(bias + n);
        d[n] = accumulate ? d[n] + x : x;
      }
    }
  }
};

// Row-major epilogue with per-column bias and optional accumulate.
struct EpiStore {
  float* D;
  const float* bias;
  int M, N, ldd, accumulate;
  __device__ void store(int m, int n0, const float* v, int) const {
    if (m >= M) return;
    float* d = D + static_cast<size_t>(m) * ldd;
    if ((N & 3) == 0 && n0 + 32 <= N) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float4 o = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        if (bias) {
          const float4 b = *reinterpret_cast<const float4*>(bias + n0 + j);
          o.x += b.x; o.y += b.y; o.z += b.z; o.w += b.w;
        }
        float4* dp = reinterpret_cast<float4*>(d + n0 + j);
        if (accumulate) {
          const float4 old = *dp;
          o.x += old.x; o.y += old.y; o.z += old.z; o.w += old.w;
        }
        *dp = o;
      }
      return;
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int n = n0 + j;
      if (n < N) {
        float o = v[j];
        if (bias) o += bias[n];
        d[n] = accumulate ? d[n] + o : o;
      }
    }
  }
};

// Split-K partial store: P[split][m][n] (no bias, no accumulation).
struct EpiPartial {
  float* P;
  int M, N;
  __device__ void store(int m, int n0, const float* v, int split) const {
    if (m >= M) return;
    float* d = P + (static_cast<size_t>(split) * M + m) * N;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (n0 + j < N) d[n0 + j] = v[j];
  }
};

}  // namespace sn
