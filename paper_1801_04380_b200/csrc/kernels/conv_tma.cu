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
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "gemm_tc.cuh"
#include "bn_math.cuh"
#include "kernels.hpp"
#include "tma_host.hpp"

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
  // MODE 2/3 (stem over a padded C=4 input, sliding-window view): k block =
  // (filter row r, block b of 8 filter columns x 4 channels); M tile = one
  // output row (fwd) / 4 k-atoms (wgrad); qblocks = ceil(Q / 32).
  int sblocks, shift, qblocks, R;
  FastDivT fsb, fqb, fP;
};

constexpr int kTmaThreads = 192;

// Persistent schedule: one CTA per SM walks tiles t = blockIdx.x, +gridDim.x,
// ... (tile = m-tile fastest, then n-tile, then split).  The TMA producer runs
// ahead across tile boundaries, the MMA issuer alternates between two TMEM
// accumulators (2 x BN columns), so tile i's epilogue overlaps tile i+1's MMAs.
//
// CG = 2 (CTA pair, cluster of 2 on one TPC): the pair computes a 256 x BN
// tile with tcgen05.mma.cta_group::2 issued by the even CTA; each CTA stages
// its own 128 A rows and HALF of B (BN/2 rows), so the per-SM operand traffic
// from L2 drops from (128 + BN) to (128 + BN/2) rows per k block -- the
// im2col conv kernels are bound by that traffic (~12 TB/s chip-wide).
template <int BN, int STAGES, int CG = 1>
struct TmaSmem {
  static constexpr int A_BYTES = kBM * 128;
  static constexpr int B_BYTES = (BN / CG) * 128;
  static constexpr int EPI_OFF = STAGES * (A_BYTES + B_BYTES);   // 2 x 16 KB store staging
  static constexpr int BAR_OFF = EPI_OFF + 2 * kBM * 128;
  static constexpr int STATS_OFF = BAR_OFF + 512;  // [4 warps][32 columns][2] floats
  static constexpr int TOTAL = STATS_OFF + 1024 + 1024;
};

// Epilogue: TMEM -> registers (+bias) -> SWIZZLE_128B smem chunk of 128 x 32
// fp32 (double-buffered) -> one TMA bulk store per chunk (plain, reduce-add, or
// into the 3-D [split][M][N] partial tensor).  Rows/columns past the tensor are
// clipped by the TMA unit, so no predication is needed.
struct EpiArgs {
  const float* bias;  // per output column, may be null
  int N;              // valid columns
  int reduce;         // 1: out += tile (cp.reduce.async.bulk .add), 0: out = tile
  int partial3d;      // 1: tmD is [splits][M][N], coordinate z = split
  // Scatter mode (strided dgrad phases): GEMM row m = (n, u, v) of the phase
  // grid lands at dx[n][(u+t0)*st+ph-pad][(v+v0)*st+pw-pad][:] (direct stores).
  float* scatter;     // null: TMA store path
  int M, Uhw, Uw, t0, v0, st, ph, pw, pad, H, W;
  FastDivT fUhw, fUw;
  // Sub-pixel strided dgrad (subpix = C): GEMM row m = (n, u, v) of dy's grid,
  // column (a*2 + b)*C + c lands at dx[n][2u+a][2v+b][c].
  int subpix;
  // BatchNorm statistics of the output (forward; the consumer is a BN):
  // per M tile and column, {shift = tile row 0, sum(y - shift), sum((y - shift)^2)}
  // over the tile's valid rows, into stats[tile][3][N] (see bn_stats_from_tiles).
  float* stats;
};

struct TileGrid {
  int m_tiles, n_tiles, tiles;
};

template <int BN, int STAGES, int MODE, int CG = 1>
__global__ void __launch_bounds__(kTmaThreads, 1)
    tc_conv_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const __grid_constant__ CUtensorMap tmD, TmaArgs a, EpiArgs e, TileGrid tg) {
  static_assert(CG == 1 || MODE <= 1, "CTA pairs: forward / dgrad (MODE 0) and wgrad (MODE 1) only");
  using L = TmaSmem<BN, STAGES, CG>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * L::A_BYTES;
  const uint32_t sEpi = smem_u32(smem + L::EPI_OFF);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2] accumulator ready
  uint64_t* tempty = tfull + 2;       // [2] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t kCols = tmem_cols<2 * BN>();

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 128 * CG);  // both CTAs' epilogues drain the pair's accumulator
    }
    fence_mbar_init();
  }
  if (warp == 5) {
    if constexpr (CG == 1) {
      tmem_alloc(tmem_slot, kCols);
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(kCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
  }
  if (warp == 4 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (!e.scatter) tma_prefetch(&tmD);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync_all();  // the peer's barriers are initialised before any remote signal
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int rank = CG == 2 ? static_cast<int>(cluster_rank()) : 0;
  const int unit = blockIdx.x / CG, units = gridDim.x / CG;  // CTA pair (or CTA) index / count

  // m0: this CTA's first A row (the pair's tile is 128*CG rows, rank r owns
  // rows [128 r, 128 r + 128)); n0: the tile's first column (rank r stages B
  // columns [n0 + r BN/CG, n0 + (r+1) BN/CG)).
  auto tile_coords = [&](int t, int& m0, int& n0, int& kb0, int& nkb, int& split) {
    const int mt = t % tg.m_tiles;
    const int rest = t / tg.m_tiles;
    const int nt = rest % tg.n_tiles;
    split = rest / tg.n_tiles;
    m0 = mt * kBM * CG + rank * kBM;
    n0 = nt * BN;
    kb0 = split * a.kb_per_split;
    nkb = min(a.num_kb, kb0 + a.kb_per_split) - kb0;
  };
  constexpr int BH = BN / CG;  // B columns staged by this CTA

  if (warp == 4) {
    {
      // ---------------- TMA producer (whole warp, elected lane issues) ----------------
      uint32_t g = 0;  // k blocks issued by this CTA (stage ring position)
      for (int t = unit; t < tg.tiles; t += units) {
        int m0, n0, kb0, nkb, split;
        tile_coords(t, m0, n0, kb0, nkb, split);
        if (MODE == 0) {
          const int n = static_cast<int>(a.fPQ.div(m0));
          const int pq = m0 - n * a.PQ;
          const int p = static_cast<int>(a.fQ.div(pq));
          const int q = pq - p * a.Q;
          const int w0 = q * a.stride - a.pad_w, h0 = p * a.stride - a.pad;
          for (int i = 0; i < nkb; ++i, ++g) {
            const int s = g % STAGES;
            if (g >= STAGES) mbar_wait(&empty[s], ((g / STAGES) - 1) & 1);
            const int kb = kb0 + i;
            const int tap = static_cast<int>(a.fcc.div(kb));
            const int cc = kb - tap * a.cchunks;
            const int r = static_cast<int>(a.fS.div(tap));
            const int tt = tap - r * a.S;
            if (elect_one()) {
            if constexpr (CG == 1) {
              mbar_arrive_expect_tx(&full[s], L::A_BYTES + L::B_BYTES);
              tma_load_im2col_4d(smem_u32(sA + s * L::A_BYTES), &tmA, &full[s], cc * 32, w0, h0, n,
                                 static_cast<uint16_t>(tt), static_cast<uint16_t>(r));
              tma_load_2d(smem_u32(sB + s * L::B_BYTES), &tmB, &full[s], kb * kBK, n0);
            } else {
              // both CTAs' loads complete on the leader's full barrier
              if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * (L::A_BYTES + L::B_BYTES));
              const uint32_t cb = mapa_u32(&full[s], 0);
              tma2_load_im2col_4d(smem_u32(sA + s * L::A_BYTES), &tmA, cb, cc * 32, w0, h0, n,
                                  static_cast<uint16_t>(tt), static_cast<uint16_t>(r));
              tma2_load_2d(smem_u32(sB + s * L::B_BYTES), &tmB, cb, kb * kBK, n0 + rank * BH);
            }
            }
            __syncwarp();
          }
        } else if (MODE == 2) {
          // stem forward: the M tile is output row (n, p); window of output q
          // starts at padded column stride*q + 8b (view dim1 step = stride pixels)
          const int mt = m0 / kBM;
          const int n = static_cast<int>(a.fP.div(mt));
          const int p = mt - n * a.P;
          for (int i = 0; i < nkb; ++i, ++g) {
            const int s = g % STAGES;
            if (g >= STAGES) mbar_wait(&empty[s], ((g / STAGES) - 1) & 1);
            const int kb = kb0 + i;
            const int r = static_cast<int>(a.fsb.div(kb));
            const int b = kb - r * a.sblocks;
            if (elect_one()) {
              mbar_arrive_expect_tx(&full[s], L::A_BYTES + L::B_BYTES);
              tma_load_4d(smem_u32(sA + s * L::A_BYTES), &tmA, &full[s], 0, b * a.shift, p * a.stride + r, n);
              tma_load_2d(smem_u32(sB + s * L::B_BYTES), &tmB, &full[s], kb * kBK, n0);
            }
            __syncwarp();
          }
        } else if (MODE == 3) {
          // stem wgrad: 4 k-atoms (r, b) per M tile; k block = 32 output columns of one row
          int ar[4], ab[4], na = 0;
          for (int q4 = 0; q4 < 4; ++q4) {
            const int atom = m0 / 32 + q4;
            const int r = static_cast<int>(a.fsb.div(atom));
            if (r >= a.R) break;
            ar[q4] = r;
            ab[q4] = atom - r * a.sblocks;
            ++na;
          }
          int nb = 0;
          for (int j = 0; j < BN / 32; ++j)
            if (n0 + 32 * j < a.Kout) ++nb;
          for (int i = 0; i < nkb; ++i, ++g) {
            const int s = g % STAGES;
            if (g >= STAGES) mbar_wait(&empty[s], ((g / STAGES) - 1) & 1);
            const int kb = kb0 + i;
            const int row = static_cast<int>(a.fqb.div(kb));
            const int qb = kb - row * a.qblocks;
            const int n = static_cast<int>(a.fP.div(row));
            const int p = row - n * a.P;
            if (elect_one()) {
              mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>((na + nb) * 4096));
              for (int q4 = 0; q4 < na; ++q4)
                tma_load_4d(smem_u32(sA + s * L::A_BYTES + q4 * 4096), &tmA, &full[s], 0,
                            qb * 32 + ab[q4] * a.shift, p * a.stride + ar[q4], n);
              for (int j = 0; j < nb; ++j)
                tma_load_4d(smem_u32(sB + s * L::B_BYTES + j * 4096), &tmB, &full[s], n0 + 32 * j, qb * 32, p, n);
            }
            __syncwarp();
          }
        } else {
          int ac[4], ar[4], as[4], na = 0;
          for (int q4 = 0; q4 < 4; ++q4) {
            const int rsc0 = m0 + 32 * q4;
            if (rsc0 >= a.RSC) break;
            const int tap = static_cast<int>(a.fC.div(rsc0));
            ac[q4] = rsc0 - tap * a.C;
            ar[q4] = static_cast<int>(a.fS.div(tap));
            as[q4] = tap - ar[q4] * a.S;
            ++na;
          }
          const int nbase = n0 + rank * BH;
          int nb = 0;
          for (int j = 0; j < BH / 32; ++j)
            if (nbase + 32 * j < a.Kout) ++nb;
          // the pair's total (leader's expect_tx): the other CTA's boxes
          int pair_boxes = na + nb;
          if constexpr (CG == 2) {
            const int om0 = m0 + (rank == 0 ? kBM : -kBM), onb0 = n0 + (rank == 0 ? BH : 0);
            for (int q4 = 0; q4 < 4; ++q4)
              if (om0 + 32 * q4 < a.RSC) ++pair_boxes;
            for (int j = 0; j < BH / 32; ++j)
              if (onb0 + 32 * j < a.Kout) ++pair_boxes;
          }
          for (int i = 0; i < nkb; ++i, ++g) {
            const int s = g % STAGES;
            if (g >= STAGES) mbar_wait(&empty[s], ((g / STAGES) - 1) & 1);
            const int pix = (kb0 + i) * kBK;
            const int n = static_cast<int>(a.fPQ.div(pix));
            const int pq = pix - n * a.PQ;
            const int p = static_cast<int>(a.fQ.div(pq));
            const int q = pq - p * a.Q;
            const int w0 = q * a.stride - a.pad, h0 = p * a.stride - a.pad;
            if (elect_one()) {
            if constexpr (CG == 1) {
              mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>((na + nb) * 4096));
              for (int q4 = 0; q4 < na; ++q4)
                tma_load_im2col_4d(smem_u32(sA + s * L::A_BYTES + q4 * 4096), &tmA, &full[s], ac[q4], w0, h0, n,
                                   static_cast<uint16_t>(as[q4]), static_cast<uint16_t>(ar[q4]));
              for (int j = 0; j < nb; ++j)
                tma_load_2d(smem_u32(sB + s * L::B_BYTES + j * 4096), &tmB, &full[s], nbase + 32 * j, pix);
            } else {
              if (rank == 0) mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(pair_boxes * 4096));
              const uint32_t cb = mapa_u32(&full[s], 0);
              for (int q4 = 0; q4 < na; ++q4)
                tma2_load_im2col_4d(smem_u32(sA + s * L::A_BYTES + q4 * 4096), &tmA, cb, ac[q4], w0, h0, n,
                                    static_cast<uint16_t>(as[q4]), static_cast<uint16_t>(ar[q4]));
              for (int j = 0; j < nb; ++j)
                tma2_load_2d(smem_u32(sB + s * L::B_BYTES + j * 4096), &tmB, cb, nbase + 32 * j, pix);
            }
            }
            __syncwarp();
          }
        }
      }
    }
  } else if (warp == 5) {
    if (rank == 0) {
      // ---------------- MMA issuer (the pair leader for CG = 2; whole warp, elected lane issues) ----------------
      constexpr bool kMN = (MODE == 1 || MODE == 3);  // wgrad: both operands MN-major
      constexpr uint32_t idesc = idesc_tf32(kBM * CG, BN, kMN, kMN);
      // The issue loop is kept to a handful of instructions per MMA: with
      // descriptors built per MMA the single issuing thread, not the tensor
      // core, set the pace (~150-200 cycles per MMA vs the 55 / 64 / 128 cycle
      // hardware floor at N = 64 / 128 / 256; tools/mma_probe.py).  The stage
      // descriptors are one base descriptor plus the stage offset (address
      // field in 16-byte units), the k step within a stage a constant.
      //   K-major SW128: 8 k = 32 B;  MN-major SW128_BASE32B: 8 k rows = 1024 B
      constexpr uint32_t KSTEP = kMN ? (1024u >> 4) : (32u >> 4);
      const uint64_t adesc0 = kMN ? umma_desc(smem_u32(sA), 4096, 512, kLayoutSW128Base32)
                                  : umma_desc(smem_u32(sA), 16, 1024, kLayoutSW128);
      const uint64_t bdesc0 = kMN ? umma_desc(smem_u32(sB), 4096, 512, kLayoutSW128Base32)
                                  : umma_desc(smem_u32(sB), 16, 1024, kLayoutSW128);
      auto mma = [&](uint32_t d, uint64_t ad, uint64_t bd, uint32_t accum) {
        if constexpr (CG == 1)
          umma_tf32(d, ad, bd, idesc, accum);
        else
          umma2_tf32(d, ad, bd, idesc, accum);
      };
      uint32_t s = 0, ph = 0;  // stage ring position and parity
      int local = 0;
      for (int t = unit; t < tg.tiles; t += units, ++local) {
        int m0, n0, kb0, nkb, split;
        tile_coords(t, m0, n0, kb0, nkb, split);
        const int acc = local & 1;
        if (local >= 2) mbar_wait(&tempty[acc], ((local >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + static_cast<uint32_t>(acc * BN);
        for (int i = 0; i < nkb; ++i) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t ad = adesc0 + s * (L::A_BYTES >> 4), bd = bdesc0 + s * (L::B_BYTES >> 4);
          if (elect_one()) {
            mma(d, ad, bd, i != 0 ? 1u : 0u);
#pragma unroll
            for (int kk = 1; kk < kBK / 8; ++kk) mma(d, ad + kk * KSTEP, bd + kk * KSTEP, 1u);
            if constexpr (CG == 1)
              umma_commit(&empty[s]);
            else
              umma2_commit(&empty[s]);
          }
          __syncwarp();
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        if (elect_one()) {
          if constexpr (CG == 1)
            umma_commit(&tfull[acc]);
          else
            umma2_commit(&tfull[acc]);
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------- epilogue (warps 0-3 own TMEM lanes 32w..32w+31) ----------------
    const uint32_t row = warp * 32 + lane;
    int local = 0;
    uint32_t chunk_no = 0;  // store-staging double-buffer position
    const uint32_t tempty_leader[2] = {CG == 2 ? mapa_u32(&tempty[0], 0) : 0u, CG == 2 ? mapa_u32(&tempty[1], 0) : 0u};
    for (int t = unit; t < tg.tiles; t += units, ++local) {
      int m0, n0, kb0, nkb, split;
      tile_coords(t, m0, n0, kb0, nkb, split);
      const int acc = local & 1;
      mbar_wait(&tfull[acc], (local >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem + static_cast<uint32_t>(acc * BN) + (static_cast<uint32_t>(warp * 32) << 16);
      if (e.scatter) {
        // strided-dgrad phase: each row goes to its interleaved place in dx
        const int m = m0 + static_cast<int>(row);
        float* dst = nullptr;
        if (m < e.M) {
          const int n = static_cast<int>(e.fUhw.div(static_cast<uint32_t>(m)));
          const int uv = m - n * e.Uhw;
          const int u = static_cast<int>(e.fUw.div(static_cast<uint32_t>(uv)));
          const int v = uv - u * e.Uw;
          if (e.subpix) {  // the 2x2 block (2u, 2v) of dx; columns pick the phase below
            dst = e.scatter + (static_cast<size_t>(n * e.H + 2 * u) * e.W + 2 * v) * e.subpix;
          } else {
            const int h = (u + e.t0) * e.st + e.ph - e.pad;
            const int w = (v + e.v0) * e.st + e.pw - e.pad;
            dst = e.scatter + (static_cast<size_t>(n * e.H + h) * e.W + w) * e.N;
          }
        }
        // Each row's 32-column chunk is 128 contiguous bytes of dx: stage the
        // warp's 32 rows in shared memory (16-byte units XOR-swizzled by row)
        // and write them back 4 rows x 128 B per warp instruction (coalesced),
        // each lane taking its row's base pointer from the owning lane.
        const uint32_t wbuf = sEpi + static_cast<uint32_t>(warp) * 4096u;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          float v[32];
          tmem_ld32(tbase + static_cast<uint32_t>(c), v);
          float* dchunk = dst ? dst + n0 + c : nullptr;
          if (dst && e.subpix) {
            const int col = n0 + c, ab = col / e.subpix;
            dchunk = dst + ((ab >> 1) * e.W + (ab & 1)) * e.subpix + (col - ab * e.subpix);
          }
#pragma unroll
          for (int j = 0; j < 8; ++j)
            asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(wbuf + lane * 128u + ((j ^ (lane & 7)) << 4)),
                         "f"(v[4 * j]), "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                         : "memory");
          __syncwarp();
          const unsigned long long mine = reinterpret_cast<unsigned long long>(dchunk);
          const int q = lane & 7;
          const bool col_ok = n0 + c + 4 * q < e.N;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = 4 * i + (lane >> 3);
            float* rp = reinterpret_cast<float*>(__shfl_sync(0xffffffffu, mine, r));
            float4 o;
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                         : "=f"(o.x), "=f"(o.y), "=f"(o.z), "=f"(o.w)
                         : "r"(wbuf + static_cast<uint32_t>(r) * 128u + ((q ^ (r & 7)) << 4))
                         : "memory");
            if (rp && col_ok) {
              float4* p = reinterpret_cast<float4*>(rp + 4 * q);
              if (e.reduce) {
                const float4 old = *p;
                o.x += old.x; o.y += old.y; o.z += old.z; o.w += old.w;
              }
              *p = o;
            }
          }
          __syncwarp();
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < BN; c += 32, ++chunk_no) {
          if (n0 + c >= e.N) break;
          float v[32];
          tmem_ld32(tbase + static_cast<uint32_t>(c), v);
          if (e.bias) {
            if (n0 + c + 32 <= e.N) {  // 16-byte loads (parameter slices are 256-byte aligned)
              const float4* b4 = reinterpret_cast<const float4*>(e.bias + n0 + c);
#pragma unroll
              for (int q4 = 0; q4 < 8; ++q4) {
                const float4 bq = __ldg(b4 + q4);
                v[4 * q4] += bq.x; v[4 * q4 + 1] += bq.y; v[4 * q4 + 2] += bq.z; v[4 * q4 + 3] += bq.w;
              }
            } else {
#pragma unroll
              for (int q = 0; q < 32; ++q)
                if (n0 + c + q < e.N) v[q] += __ldg(e.bias + n0 + c + q);
            }
          }
          const uint32_t buf = sEpi + (chunk_no & 1u) * (kBM * 128);
          // the store issued two chunks ago from this buffer must have read it
          if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          named_bar(1, 128);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(buf + sw128_off(row, j)), "f"(v[4 * j]),
                         "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                         : "memory");
          fence_proxy_async();
          named_bar(1, 128);
          if (threadIdx.x == 0) {
            if (MODE == 2) {  // tile = output row (n, p): [N][P][Q][K] store, q >= Q clipped
              const int mt = m0 / kBM;
              const int n = static_cast<int>(a.fP.div(mt));
              tma_store_4d(&tmD, buf, n0 + c, 0, mt - n * a.P, n);
            } else if (e.partial3d)
              tma_store_3d(&tmD, buf, n0 + c, m0, split);
            else
              tma_store_2d(&tmD, buf, n0 + c, m0, e.reduce != 0);
            bulk_commit();
          }
          if (e.stats) {
            const int nv = MODE == 2 ? a.Q : min(kBM, e.M - m0);
            const uint8_t* sb = smem + L::EPI_OFF + (chunk_no & 1u) * (kBM * 128);
            float shift, t1, t2;
            chunk_column_stats(sb, [&](int r) { return r < nv; }, reinterpret_cast<float*>(smem + L::STATS_OFF),
                               shift, t1, t2);
            if (warp == 0 && n0 + c + lane < e.N) {
              float* out = e.stats + static_cast<size_t>(m0 / kBM) * 3 * e.N + n0 + c + lane;
              out[0] = shift;
              out[e.N] = t1;
              out[2 * static_cast<size_t>(e.N)] = t2;
            }
          }
        }
      }
      tc_fence_before();
      if constexpr (CG == 1)
        mbar_arrive(&tempty[acc]);
      else
        mbar_arrive_cluster(tempty_leader[acc]);
    }
    if (threadIdx.x == 0) bulk_wait_all();
  }
  __syncthreads();
  if constexpr (CG == 2) cluster_sync_all();  // no CTA leaves while its peer may still signal it
  if (warp == 5) {
    tc_fence_after();
    if constexpr (CG == 1)
      tmem_dealloc(tmem, kCols);
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols) : "memory");
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
  // one persistent CTA per SM: as many stages as fit next to the 32 KB store staging
  return BN <= 64 ? 8 : (BN <= 128 ? 5 : 4);
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

template <int BN, int CG = 1>
constexpr int stages_for2() {
  // one persistent CTA per SM: as many stages as fit next to the 32 KB store staging
  return (227 * 1024 - 2 * kBM * 128 - 3 * 1024) / (kBM * 128 + (BN / CG) * 128);
}

template <int BN, int MODE, int CG = 1>
cudaError_t launch(const CUtensorMap& A, const CUtensorMap& B, const CUtensorMap& D, const TmaArgs& a,
                   const EpiArgs& e, int M, int N, int splits, cudaStream_t st) {
  constexpr int STAGES = CG == 1 ? stages_for<BN>() : stages_for2<BN, CG>();
  using L = TmaSmem<BN, STAGES, CG>;
  static_assert(L::TOTAL <= 227 * 1024, "shared memory budget");
  auto kern = tc_conv_tma_kernel<BN, STAGES, MODE, CG>;
  static bool attr = false;
  if (!attr) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
    if (err != cudaSuccess) return err;
    if (CG == 2) {
      err = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
      (void)err;
    }
    attr = true;
  }
  TmaArgs args = a;
  const int kps = (a.num_kb + splits - 1) / splits;
  args.kb_per_split = kps;
  TileGrid tg;
  tg.m_tiles = (M + kBM * CG - 1) / (kBM * CG);
  tg.n_tiles = (N + BN - 1) / BN;
  tg.tiles = tg.m_tiles * tg.n_tiles * ((a.num_kb + kps - 1) / kps);
  const int sms = num_sms();
  if constexpr (CG == 1) {
    const int grid = std::min(tg.tiles, sms);
    kern<<<grid, kTmaThreads, L::TOTAL, st>>>(A, B, D, args, e, tg);
    return cudaGetLastError();
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * std::min(tg.tiles, sms / 2));
    cfg.blockDim = dim3(kTmaThreads);
    cfg.dynamicSmemBytes = L::TOTAL;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, A, B, D, args, e, tg);
  }
}

// CTA pairs (SN_CONV_PAIRS=0 disables): MODE 0 always when the tile count
// keeps the pairs busy; MODE 1 (wgrad, M = R*S*C) when 256-row tiles waste
// no more than 128-row ones.
// 0 off, 1 by size (default), 2 always (tests)
int g_pairs = -1;
int pairs_mode() {
  if (g_pairs < 0) {
    const char* v = std::getenv("SN_CONV_PAIRS");
    g_pairs = (v && v[0] == '0') ? 0 : 1;
  }
  return g_pairs;
}
bool use_pairs(int64_t rows) { return pairs_mode() == 2 || (pairs_mode() == 1 && rows >= 2 * kBM * 148); }

int bn_for(int n) { return n <= 64 ? 64 : (n <= 128 ? 128 : 256); }

// Single-CTA tile width by wave fill: 128-wide tiles run the tensor pipe at the
// same rate as 256-wide ones (64 vs 128 cycles per k step, tools/mma_probe.py),
// so when the 256-wide tile count leaves the last wave of the persistent grid
// much emptier (ResNet stage 4: 196 tiles = 1.32 waves), halve the width.
// Tile shape (CTA group, tile width) of the im2col kernels.  Large M: pairs of
// 256-wide tiles (use_pairs).  Small M with >= 256 output columns (ResNet stage
// 4, M = 12544): 256-wide tiles fill 1.32 waves; pairs of 128-wide tiles fill
// 2.65 and share the B tile across the pair (conv_bench: 101 -> 90 us fwd).
struct TileCfg {
  int cg, bn;
};
TileCfg tile_cfg(int64_t M, int n, int kdim = 1 << 30);
int g_bn_force = 0;  // A/B knob (conv_bench --bn): 0 = policy, else the tile width when it fits
int bn_for_waves(int64_t M, int n) {
  const int bn = bn_for(n);
  if (g_bn_force > 0) return g_bn_force < bn ? g_bn_force : bn;
  if (bn != 256) return bn;
  const int64_t mt = (M + kBM - 1) / kBM;
  auto fill = [](int64_t tiles) {
    const int64_t waves = (tiles + 147) / 148;
    return static_cast<double>(tiles) / static_cast<double>(waves * 148);
  };
  const double f256 = fill(mt * ((n + 255) / 256)), f128 = fill(mt * ((n + 127) / 128));
  return f128 > f256 + 0.1 ? 128 : 256;
}

}  // namespace

bool tma_encoders_ok() { return load_encoders(); }

bool tma_map_nhwc(CUtensorMap* m, const float* base, int N, int H, int W, int C, int box_w, int box_h, int swz,
                  int es) {
  if (!load_encoders()) return false;
  if (es < 1 || es > 8 || box_w * es > 256 || box_h * es > 256) return false;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                        static_cast<cuuint64_t>(N)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(C) * 4, static_cast<cuuint64_t>(W) * C * 4,
                           static_cast<cuuint64_t>(H) * W * C * 4};
  // with element strides the box spans es x the elements it loads (TMA traversal stride)
  cuuint32_t box[4] = {32, static_cast<cuuint32_t>(box_w * es), static_cast<cuuint32_t>(box_h * es), 1};
  cuuint32_t estr[4] = {1, static_cast<cuuint32_t>(es), static_cast<cuuint32_t>(es), 1};
  return g_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swz ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool tma_map_2d(CUtensorMap* m, const float* base, int64_t rows, int64_t cols, int box_rows, int swz) {
  if (!load_encoders()) return false;
  return make_tiled(m, base, rows, cols, box_rows,
                    swz ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B);
}

bool conv_tma_ok_fwd(const ConvShape& s) { return s.C % 32 == 0 && load_encoders(); }

namespace {
// kdim: the GEMM reduction length.  At <= 128 (a 1x1 convolution over <= 128
// channels: 4 k blocks per tile) the tile is a short load -> store pass and
// CTA pairs only add cluster handshakes: single CTAs (conv_bench, 1x1 64->64
// at 56x56 b256: fwd 113 -> 75 us, dgrad 115 -> 82 us; 128->128 at 28x28:
// 50 -> 40 us, 53 -> 45 us -- DenseNet-style bottleneck convolutions).
TileCfg tile_cfg(int64_t M, int n, int kdim) {
  if (kdim <= 128 && pairs_mode() == 1 && !g_bn_force) return {1, bn_for_waves(M, n)};
  if (use_pairs(M)) return {2, g_bn_force ? bn_for_waves(M, n) : bn_for(n)};
  if (pairs_mode() == 1 && !g_bn_force && bn_for(n) == 256) return {2, 128};
  return {1, bn_for_waves(M, n)};
}
}  // namespace

void set_conv_pairs(int mode) { g_pairs = mode; }
void set_conv_bn(int bn) { g_bn_force = bn; }
int conv_bn_force() { return g_bn_force; }
int conv_pairs_mode() { return pairs_mode(); }

constexpr int kStemRT = 4;  // stem forward: output rows per tile
// the stem forward's rows kernel: <= 64 channels, one 8-tap block per filter row, R <= 8
bool stem_rows_fwd_ok(const ConvShape& s) { return s.K <= 64 && (s.S + 7) / 8 == 1 && s.R <= 8; }

int conv_fwd_stats_tiles(const ConvShape& s, bool stem, int* tile_rows) {
  if (stem) {
    if (stem_rows_fwd_ok(s)) {  // one tile per kStemRT output rows (contiguous: P % kStemRT == 0)
      if (s.P % kStemRT != 0) return 0;
      *tile_rows = kStemRT * s.Q;
      return s.N * s.P / kStemRT;
    }
    *tile_rows = s.Q;  // generic path: one 128-row tile per output row
    return s.N * s.P;
  }
  if (!use_tma()) return 0;
  if (s.stride <= 2) {
    const int ht = conv_halo_stats_tiles(s.N, s.H, s.W, s.C, s.K, s.R, s.S, s.pad, s.P, s.Q, s.stride);
    if (ht > 0) {
      *tile_rows = 0;
      return ht;
    }
  }
  if (!conv_tma_ok_fwd(s)) return 0;
  *tile_rows = kBM;
  return (s.N * s.P * s.Q + kBM - 1) / kBM;
}

bool conv_tma_ok_dgrad(const ConvShape& s) {
  // a 1x1 filter may have K % 32 != 0 (the FC dgrad): the last channel chunk
  // reads past K, which both tensor maps zero-fill (one tap: no neighbour to hit)
  const bool kok = s.K % 32 == 0 || (s.R == 1 && s.S == 1 && s.K % 4 == 0);
  // any stride-1 geometry (the dgrad is the full correlation of dy padded by
  // R-1-pad: "valid" convolutions too), as long as that padding is >= 0
  const bool geom = s.H == s.P + s.R - 1 - 2 * s.pad && s.W == s.Q + s.S - 1 - 2 * s.pad && s.pad <= s.R - 1 &&
                    s.pad <= s.S - 1;
  return s.stride == 1 && kok && geom && load_encoders();
}
bool conv_tma_ok_wgrad(const ConvShape& s) {
  // 1x1 with K % 32 != 0 (the FC): dy's last column box and the partial store
  // run past K (zero fill / clipped)
  const bool kok = s.K % 32 == 0 || (s.R == 1 && s.S == 1 && s.K % 4 == 0);
  return s.C % 32 == 0 && kok && load_encoders();
}

cudaError_t conv_fwd_tma(const ConvShape& s, const float* x, const float* w, const float* bias, float* y,
                         float* stats, cudaStream_t st) {
  CUtensorMap A, B;
  if (!make_im2col(&A, x, s.N, s.H, s.W, s.C, -s.pad, -s.pad, s.pad - (s.R - 1), s.pad - (s.S - 1), s.stride, kBM,
                   CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  const int Ktot = s.R * s.S * s.C;
  const int M = s.N * s.P * s.Q;
  const TileCfg tc = tile_cfg(M, s.K, Ktot);
  const int CG = tc.cg, BN = tc.bn;
  if (!make_tiled(&B, w, s.K, Ktot, BN / CG, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
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
  CUtensorMap D;
  if (!make_store(&D, y, M, s.K, 0)) return cudaErrorInvalidValue;
  EpiArgs e{bias, s.K, 0, 0};
  e.M = M;
  e.stats = stats;
  if (CG == 2) {
    switch (BN) {
      case 64: return launch<64, 0, 2>(A, B, D, a, e, M, s.K, 1, st);
      case 128: return launch<128, 0, 2>(A, B, D, a, e, M, s.K, 1, st);
      default: return launch<256, 0, 2>(A, B, D, a, e, M, s.K, 1, st);
    }
  }
  switch (BN) {
    case 64: return launch<64, 0>(A, B, D, a, e, M, s.K, 1, st);
    case 128: return launch<128, 0>(A, B, D, a, e, M, s.K, 1, st);
    default: return launch<256, 0>(A, B, D, a, e, M, s.K, 1, st);
  }
}

// wt_flip[c][r][s][k] = w[k][R-1-r][S-1-s][c], written by the caller.
cudaError_t conv_dgrad_tma(const ConvShape& s, const float* dy, const float* wt_flip, float* dx, int accumulate,
                           cudaStream_t st) {
  CUtensorMap A, B;
  const int padh = s.R - 1 - s.pad, padw = s.S - 1 - s.pad;
  if (!make_im2col(&A, dy, s.N, s.P, s.Q, s.K, -padh, -padw, padh - (s.R - 1), padw - (s.S - 1), 1, kBM,
                   CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  const int Ktot = s.R * s.S * s.K;
  const int M = s.N * s.H * s.W;
  const TileCfg tc = tile_cfg(M, s.C, Ktot);
  const int CG = tc.cg, BN = tc.bn;
  if (!make_tiled(&B, wt_flip, s.C, Ktot, BN / CG, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
  TmaArgs a{};
  a.num_kb = (Ktot + kBK - 1) / kBK;
  a.cchunks = (s.K + 31) / 32;
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
  CUtensorMap D;
  if (!make_store(&D, dx, M, s.C, 0)) return cudaErrorInvalidValue;
  const EpiArgs e{nullptr, s.C, accumulate, 0};
  if (CG == 2) {
    switch (BN) {
      case 64: return launch<64, 0, 2>(A, B, D, a, e, M, s.C, 1, st);
      case 128: return launch<128, 0, 2>(A, B, D, a, e, M, s.C, 1, st);
      default: return launch<256, 0, 2>(A, B, D, a, e, M, s.C, 1, st);
    }
  }
  switch (BN) {
    case 64: return launch<64, 0>(A, B, D, a, e, M, s.C, 1, st);
    case 128: return launch<128, 0>(A, B, D, a, e, M, s.C, 1, st);
    default: return launch<256, 0>(A, B, D, a, e, M, s.C, 1, st);
  }
}

// ---------------------------------------------------------------------------
// Stem convolution (input = the executor's spatially padded C=4 image buffer).
// For a fixed filter row r the 8 filter columns x 4 channels a window needs are
// 32 consecutive floats of one padded input row, and consecutive output
// columns' windows start `stride` pixels apart: a tiled tensor map whose dim-1
// stride (16*stride bytes) is smaller than its 128-byte inner extent presents
// exactly those overlapping windows, so the whole K block of an output row is
// ONE TMA box -- no im2col gather, no per-element padding logic.

namespace {

struct StemGeom {
  int N, Hp, Wp, R, S, P, Q, K, stride, sblocks, shift, Qv, qblocks;
};

StemGeom stem_geom(const ConvShape& s) {
  StemGeom g;
  g.N = s.N;
  g.R = s.R;
  g.S = s.S;
  g.P = s.P;
  g.Q = s.Q;
  g.K = s.K;
  g.stride = s.stride;
  g.sblocks = (s.S + 7) / 8;
  g.shift = 8 / s.stride;
  g.Qv = s.Q + (g.sblocks - 1) * g.shift;
  g.qblocks = (s.Q + 31) / 32;
  g.Hp = s.H + 2 * s.pad;
  g.Wp = std::max(s.W + 2 * s.pad, s.stride * (g.Qv - 1) + 8);
  return g;
}

// One thread per padded pixel: reads the C_raw (<= 4) image channels, writes
// one float4 (zeros in the border and the padding channels).
__global__ void stem_pad_kernel(const float* __restrict__ raw, int C_raw, float4* __restrict__ xp, int N, int H, int W,
                                int Hp, int Wp, int pad) {
  const int64_t total = static_cast<int64_t>(N) * Hp * Wp;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int w = static_cast<int>(i % Wp) - pad;
    const int64_t t = i / Wp;
    const int h = static_cast<int>(t % Hp) - pad;
    const int n = static_cast<int>(t / Hp);
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (h >= 0 && h < H && w >= 0 && w < W) {
      const float* src = raw + ((static_cast<int64_t>(n) * H + h) * W + w) * C_raw;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (c < C_raw) v[c] = __ldg(src + c);
    }
    xp[i] = make_float4(v[0], v[1], v[2], v[3]);
  }
}

// wp[k][r][s'][c] (s' < 8*sblocks) <-> w[k][r][s][c]; to_padded selects the direction.
__global__ void stem_weights_kernel(float* __restrict__ w, float* __restrict__ wp, int K, int R, int S, int Sp,
                                    int to_padded) {
  const int64_t total = static_cast<int64_t>(K) * R * Sp * 4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % 4);
    int64_t t = i / 4;
    const int sp = static_cast<int>(t % Sp);
    t /= Sp;
    const int r = static_cast<int>(t % R);
    const int k = static_cast<int>(t / R);
    const int64_t src = ((static_cast<int64_t>(k) * R + r) * S + sp) * 4 + c;
    if (to_padded)
      wp[i] = sp < S ? w[src] : 0.f;
    else if (sp < S)
      w[src] = wp[i];
  }
}

// Overlapping sliding-window view of the padded input: [N][Hp][Qv windows][32 floats].
bool make_stem_view(CUtensorMap* m, const float* xp, const StemGeom& g, int box_q, CUtensorMapSwizzle sw) {
  cuuint64_t dims[4] = {32, static_cast<cuuint64_t>(g.Qv), static_cast<cuuint64_t>(g.Hp),
                        static_cast<cuuint64_t>(g.N)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(g.stride) * 16, static_cast<cuuint64_t>(g.Wp) * 16,
                           static_cast<cuuint64_t>(g.Hp) * g.Wp * 16};
  cuuint32_t box[4] = {32, static_cast<cuuint32_t>(box_q), 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return g_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(xp), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// NHWC [N][P][Q][K] as a 4-D tiled map with box {32 channels, box_q columns, 1, 1}.
bool make_nhwc4(CUtensorMap* m, const float* base, int N, int P, int Q, int K, int box_q, CUtensorMapSwizzle sw) {
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(Q), static_cast<cuuint64_t>(P),
                        static_cast<cuuint64_t>(N)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(K) * 4, static_cast<cuuint64_t>(Q) * K * 4,
                           static_cast<cuuint64_t>(P) * Q * K * 4};
  cuuint32_t box[4] = {32, static_cast<cuuint32_t>(box_q), 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return g_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool conv_stem_ok(const ConvShape& s) {
  return s.C == 4 && s.stride >= 1 && s.stride <= 8 && 8 % s.stride == 0 && s.S <= 32 && s.K % 32 == 0 &&
         s.Q <= kBM && load_encoders();
}

int64_t stem_padded_floats(const ConvShape& s) {
  const StemGeom g = stem_geom(s);
  return static_cast<int64_t>(g.N) * g.Hp * g.Wp * 4 + 64;
}

int64_t stem_weight_floats(const ConvShape& s) {
  return static_cast<int64_t>(s.K) * s.R * ((s.S + 7) / 8) * 8 * 4;
}

cudaError_t stem_pad_input(const ConvShape& s, int H_raw, int W_raw, int C_raw, int pad, const float* raw, float* xp,
                           cudaStream_t st) {
  const StemGeom g = stem_geom(s);
  if (C_raw > 4) return cudaErrorInvalidValue;
  stem_pad_kernel<<<148 * 8, 256, 0, st>>>(raw, C_raw, reinterpret_cast<float4*>(xp), s.N, H_raw, W_raw, g.Hp, g.Wp,
                                           pad);
  return cudaGetLastError();
}

namespace {

// Stem forward, RT output rows per tile (one 128-row accumulator each): the
// whole filter (R k-blocks of 64 x 32, <= 64 output channels) is loaded into
// SMEM once per CTA, and the sliding-window view of each padded input row
// (one TMA box) is loaded once per tile and feeds every output row of the tile
// that uses it -- (RT-1)*stride + R row loads per RT output rows instead of
// R per row, and no per-tile weight traffic (the 1-row kernel was bound by
// its L2 -> SMEM operand traffic).
constexpr int kStemRing = 6;
constexpr int kStemThreads = 320;  // producer (warp 4), MMA (warp 5), two epilogue groups (warps 0-3, 6-9)
struct StemRowsArgs {
  int N, P, Q, R, stride, K, rows_in;  // rows_in = (RT-1)*stride + R input rows per tile
  int tiles;                           // N * ceil(P / RT)
  const float* bias;
  float* stats;                        // [N*P/RT][3][K] tile statistics (tile = RT output rows), or null
  float* y;                            // output [N][P][Q][K]
};

__global__ void __launch_bounds__(kStemThreads, 1)
    stem_rows_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW,
                     const __grid_constant__ CUtensorMap tmD, StemRowsArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  constexpr int A_BYTES = kBM * 128, W_BYTES = 64 * 128;
  uint8_t* sA = smem;                                  // kStemRing input-row views
  uint8_t* sW = sA + kStemRing * A_BYTES;              // R weight k-blocks (resident)
  uint8_t* sEpi = sW + a.R * W_BYTES;                  // 2 groups x 2 x 16 KB store staging
  uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + 4 * kBM * 128);
  uint64_t* empty = full + kStemRing;
  uint64_t* wbar = empty + kStemRing;
  uint64_t* tfull = wbar + 1;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* sred = reinterpret_cast<float*>(tmem_slot + 4);
  sred += (4u - ((smem_u32(sred) >> 2) & 3u)) & 3u;  // 16-byte aligned (float4 shift stores)
  float* sbias = sred + 1152 + ((4u - ((smem_u32(sred + 1152) >> 2) & 3u)) & 3u);  // [64], 16-byte aligned
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bands = (a.P + kStemRT - 1) / kStemRT;
  if (a.bias && threadIdx.x < 64) sbias[threadIdx.x] = threadIdx.x < a.K ? a.bias[threadIdx.x] : 0.f;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStemRing; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(wbar, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 256);
    }
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    if (elect_one()) {
      mbar_arrive_expect_tx(wbar, a.R * W_BYTES);
      for (int r = 0; r < a.R; ++r) tma_load_2d(smem_u32(sW + r * W_BYTES), &tmW, wbar, r * 32, 0);
    }
    __syncwarp();
    uint32_t s = 0, ph = 0;
    bool wrap = false;
    for (int t = blockIdx.x; t < a.tiles; t += gridDim.x) {
      const int n = t / bands, p0 = (t - n * bands) * kStemRT;
      for (int j = 0; j < a.rows_in; ++j) {
        if (wrap) mbar_wait(&empty[s], ph ^ 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&full[s], A_BYTES);
          tma_load_4d(smem_u32(sA + s * A_BYTES), &tmA, &full[s], 0, 0, p0 * a.stride + j, n);
        }
        __syncwarp();
        if (++s == kStemRing) {
          s = 0;
          ph ^= 1;
          wrap = true;
        }
      }
    }
  } else if (warp == 5) {
    constexpr uint32_t idesc = idesc_tf32(kBM, 64, false, false);
    const uint64_t ad0 = umma_desc(smem_u32(sA), 16, 1024, kLayoutSW128);
    const uint64_t wd0 = umma_desc(smem_u32(sW), 16, 1024, kLayoutSW128);
    mbar_wait(wbar, 0);
    uint32_t s = 0, ph = 0;
    int local = 0;
    for (int t = blockIdx.x; t < a.tiles; t += gridDim.x, ++local) {
      const int acc = local & 1;
      if (local >= 2) mbar_wait(&tempty[acc], ((local >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t d0 = tmem + static_cast<uint32_t>(acc * kStemRT * 64);
      for (int j = 0; j < a.rows_in; ++j) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t ad = ad0 + s * (A_BYTES >> 4);
#pragma unroll
          for (int i = 0; i < kStemRT; ++i) {
            const int r = j - i * a.stride;  // filter row this input row is for output row p0 + i
            if (r < 0 || r >= a.R) continue;
            const uint64_t wd = wd0 + static_cast<uint32_t>(r) * (W_BYTES >> 4);
#pragma unroll
            for (int kk = 0; kk < kBK / 8; ++kk)
              umma_tf32(d0 + i * 64, ad + kk * 2, wd + kk * 2, idesc, (r | kk) != 0 ? 1u : 0u);
          }
          umma_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == kStemRing) {
          s = 0;
          ph ^= 1;
        }
      }
      if (elect_one()) umma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else {
    // two epilogue groups (warps 0-3, 6-9); group g drains output channels
    // 32g .. 32g+31 of every row of the tile.  Per row: TMEM -> registers ->
    // swizzled staging (one barrier), then thread (cq = t & 7, rg = t >> 3)
    // reads back column quad cq of rows 8rg .. 8rg+7 and uses each value twice:
    // a coalesced global store (a warp instruction writes 4 whole 128-byte
    // rows) and the BN statistics, accumulated in registers over the tile's
    // kStemRT output rows against the tile's first pixel (the shift).  The
    // four warps' partials meet in one of two sred slots once per tile; warp 0
    // combines them after the next barrier.  No async-proxy fence, no
    // bulk-store wait, one barrier per staged chunk.
    const int grp = warp >= 6 ? 1 : 0, q4 = warp & 3;
    const uint32_t row = q4 * 32 + lane;
    const uint32_t bar_id = 1 + grp;
    const int et = q4 * 32 + lane, cq = et & 7, rg = et >> 3;
    const int c = 32 * grp;
    uint8_t* sEpiG = sEpi + grp * 2 * (kBM * 128);
    float* sredG = sred + grp * 576;  // [2 slots][4 warps x 32 columns x 2 partials, 32 shifts]
    const bool col_ok = c + 4 * cq < a.K;
    int local = 0;
    uint32_t chunk_no = 0;
    bool pend = false;  // the previous tile's statistics still to be combined by warp 0
    int pt = 0, pslot = 0;
    auto finish_stats = [&](uint32_t slot, int tile) {
      if (q4 != 0) return;
      const float* sr = sredG + slot * 288;
      float t1 = sr[lane * 2], t2 = sr[lane * 2 + 1];
      for (int w = 1; w < 4; ++w) {
        t1 += sr[(w * 32 + lane) * 2];
        t2 += sr[(w * 32 + lane) * 2 + 1];
      }
      if (c + lane < a.K) {
        float* out = a.stats + static_cast<size_t>(tile) * 3 * a.K + c + lane;
        out[0] = sr[256 + lane];
        out[a.K] = t1;
        out[2 * static_cast<size_t>(a.K)] = t2;
      }
    };
    for (int t = blockIdx.x; t < a.tiles; t += gridDim.x, ++local) {
      const int n = t / bands, p0 = (t - n * bands) * kStemRT;
      const int acc = local & 1;
      mbar_wait(&tfull[acc], (local >> 1) & 1);
      tc_fence_after();
      if (c >= a.K) {  // this group has no channels: release the accumulator
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
        continue;
      }
      float4 sh = make_float4(0.f, 0.f, 0.f, 0.f), sa = sh, sq = sh;
      for (int i = 0; i < kStemRT; ++i) {
        const int p = p0 + i;
        float v[32];
        tmem_ld32(tmem + static_cast<uint32_t>((acc * kStemRT + i) * 64 + c) + (static_cast<uint32_t>(q4 * 32) << 16),
                  v);
        if (i == kStemRT - 1) {  // the accumulator is drained: the MMA may reuse it
          tc_fence_before();
          mbar_arrive(&tempty[acc]);
        }
        if (a.bias) {  // staged in shared memory (zero past K)
          const float4* b4 = reinterpret_cast<const float4*>(sbias + c);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 bq = b4[q];
            v[4 * q] += bq.x; v[4 * q + 1] += bq.y; v[4 * q + 2] += bq.z; v[4 * q + 3] += bq.w;
          }
        }
        const uint32_t slot = chunk_no & 1u;
        uint8_t* sb = sEpiG + slot * (kBM * 128);
        const uint32_t buf = smem_u32(sb);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(buf + sw128_off(row, q)), "f"(v[4 * q]),
                       "f"(v[4 * q + 1]), "f"(v[4 * q + 2]), "f"(v[4 * q + 3])
                       : "memory");
        // staged; the previous tile's statistics partials are visible; the
        // buffer written two chunks ago is no longer read
        named_bar(bar_id, 128);
        if (pend) finish_stats(pslot, pt);
        pend = false;
        ++chunk_no;
        if (p >= a.P) continue;
        float4 u[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) u[j] = *reinterpret_cast<const float4*>(sb + sw128_off(rg * 8 + j, cq));
        if (i == 0) sh = *reinterpret_cast<const float4*>(sb + sw128_off(0, cq));
        float* yrow = a.y + ((static_cast<size_t>(n) * a.P + p) * a.Q) * a.K + c + 4 * cq;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int r = rg * 8 + j;
          if (r < a.Q) {
            if (col_ok) *reinterpret_cast<float4*>(yrow + static_cast<size_t>(r) * a.K) = u[j];
            const float d0 = u[j].x - sh.x, d1 = u[j].y - sh.y, d2 = u[j].z - sh.z, d3 = u[j].w - sh.w;
            sa.x += d0; sa.y += d1; sa.z += d2; sa.w += d3;
            sq.x = fmaf(d0, d0, sq.x); sq.y = fmaf(d1, d1, sq.y); sq.z = fmaf(d2, d2, sq.z); sq.w = fmaf(d3, d3, sq.w);
          }
        }
      }
      if (a.stats) {
#pragma unroll
        for (int off = 8; off <= 16; off <<= 1) {
          sa.x += __shfl_xor_sync(0xffffffffu, sa.x, off); sa.y += __shfl_xor_sync(0xffffffffu, sa.y, off);
          sa.z += __shfl_xor_sync(0xffffffffu, sa.z, off); sa.w += __shfl_xor_sync(0xffffffffu, sa.w, off);
          sq.x += __shfl_xor_sync(0xffffffffu, sq.x, off); sq.y += __shfl_xor_sync(0xffffffffu, sq.y, off);
          sq.z += __shfl_xor_sync(0xffffffffu, sq.z, off); sq.w += __shfl_xor_sync(0xffffffffu, sq.w, off);
        }
        if (lane < 8) {
          float* o = sredG + (local & 1) * 288 + (q4 * 32 + 4 * cq) * 2;
          o[0] = sa.x; o[1] = sq.x; o[2] = sa.y; o[3] = sq.y; o[4] = sa.z; o[5] = sq.z; o[6] = sa.w; o[7] = sq.w;
          if (q4 == 0) *reinterpret_cast<float4*>(sredG + (local & 1) * 288 + 256 + 4 * cq) = sh;
        }
        pend = true;
        pt = t;
        pslot = local & 1;
      }
    }
    named_bar(bar_id, 128);
    if (pend) finish_stats(pslot, pt);
  }
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace

cudaError_t conv_stem_fwd(const ConvShape& s, const float* xp, const float* w, float* wp_scratch, const float* bias,
                          float* y, float* stats, cudaStream_t st) {
  const StemGeom g = stem_geom(s);
  const int Sp = g.sblocks * 8;
  stem_weights_kernel<<<148, 256, 0, st>>>(const_cast<float*>(w), wp_scratch, s.K, s.R, s.S, Sp, 1);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  if (stem_rows_fwd_ok(s)) {
    CUtensorMap A, W, D;
    if (!make_stem_view(&A, xp, g, kBM, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
    if (!make_tiled(&W, wp_scratch, s.K, s.R * Sp * 4, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
    if (!make_nhwc4(&D, y, s.N, s.P, s.Q, s.K, kBM, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
    StemRowsArgs ra{};
    ra.N = s.N;
    ra.P = s.P;
    ra.Q = s.Q;
    ra.R = s.R;
    ra.stride = s.stride;
    ra.K = s.K;
    ra.rows_in = (kStemRT - 1) * s.stride + s.R;
    ra.tiles = s.N * ((s.P + kStemRT - 1) / kStemRT);
    ra.bias = bias;
    ra.stats = stats;
    ra.y = y;
    const int smem = kStemRing * kBM * 128 + s.R * 64 * 128 + 4 * kBM * 128 + 512 + 4608 + 272 + 1024;
    static int attr_smem = 0;  // the filter's share depends on R: raise the opt-in when a larger one comes
    if (smem > attr_smem) {
      err = cudaFuncSetAttribute(stem_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (err != cudaSuccess) return err;
      attr_smem = smem;
    }
    stem_rows_kernel<<<std::min(ra.tiles, num_sms()), kStemThreads, smem, st>>>(A, W, D, ra);
    return cudaGetLastError();
  }
  const int BN = bn_for(s.K);
  CUtensorMap A, B, D;
  if (!make_stem_view(&A, xp, g, kBM, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
  const int Ktot = s.R * Sp * 4;
  if (!make_tiled(&B, wp_scratch, s.K, Ktot, BN, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
  if (!make_nhwc4(&D, y, s.N, s.P, s.Q, s.K, kBM, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
  TmaArgs a{};
  a.num_kb = s.R * g.sblocks;
  a.P = s.P;
  a.stride = s.stride;
  a.sblocks = g.sblocks;
  a.shift = g.shift;
  a.fsb = FastDivT(g.sblocks);
  a.fP = FastDivT(s.P);
  a.Q = s.Q;
  EpiArgs e{bias, s.K, 0, 0};
  e.stats = stats;
  const int M = s.N * s.P * kBM;  // one 128-row tile per output row
  switch (BN) {
    case 64: return launch<64, 2>(A, B, D, a, e, M, s.K, 1, st);
    case 128: return launch<128, 2>(A, B, D, a, e, M, s.K, 1, st);
    default: return launch<256, 2>(A, B, D, a, e, M, s.K, 1, st);
  }
}

int conv_stem_wgrad_splits(const ConvShape& s) {
  const StemGeom g = stem_geom(s);
  const int M = s.R * g.sblocks * 32;
  const int bn = bn_for(s.K);
  const int tiles = ((M + kBM - 1) / kBM) * ((s.K + bn - 1) / bn);
  const int nkb = s.N * s.P * g.qblocks;
  int want = std::max(1, 148 / tiles);
  want = std::min(want, std::max(1, nkb / 8));
  const int kps = (nkb + want - 1) / want;
  return (nkb + kps - 1) / kps;
}

int64_t stem_wgrad_partial_floats(const ConvShape& s) {
  const StemGeom g = stem_geom(s);
  const int64_t rows = static_cast<int64_t>(s.R) * g.sblocks * 32 * s.K;
  return std::max<int64_t>(conv_stem_wgrad_splits(s), num_sms()) * rows;
}

namespace {

// Stem weight gradient, 2 output rows per k block: the sliding-window views of
// input rows 2p .. 2p+9 (10 boxes of 32 windows) serve output rows p, p+1 --
// row p+g's filter-row atoms r = 0..7 are boxes 2g .. 2g+7, consecutive, so the
// A operand of either 128-row M tile is a uniform-stride run of boxes -- and
// both M tiles (filter rows 0-3, 4-7; row 7 is padding) share every dy box.
// Each CTA accumulates a contiguous range of units (image, 2-row group,
// 32-column block) and writes one [256][64] partial slice.
//
// Warps 0-7 see every dy tile before the tensor core does: they sum the conv
// bias gradient from it (fixed order: thread = channel quad x 2 x 2 pixel blocks),
// and with FUSED the tile is not dy at all but the stem BN's own dy g, which
// they turn into the BN's dx in place from the BN input x (loaded beside it)
// and the BN statistics -- the BN backward's dx pass fused into its only
// consumer, dx never written to HBM.  Both paths compute dx with the same
// element function (bn_dx_elem) and sum in the same order, so they are
// bit-identical.
//
// MODE 2 (the BN's output feeds a ReLU and a 3x3 / s2 / p1 max pool with
// saved argmax) goes one step further back: g is not read either but gathered
// from the pool output's gradient and the argmax -- for the k block's 2 x 32
// pixels, the pool windows (rows p0/2, p0/2 + 1; columns qb*16 .. qb*16+16)
// arrive as one TMA box each (out-of-range windows zero-filled: a zero pick),
// and each pixel sums its picks from +0 in pool_max_bwd_k3s2's order -- so the
// pool backward never runs and neither g nor dx is written.  The x tiles land
// in the B slots and are overwritten by dx in place.
constexpr int kSwG = 2;  // output rows per k block
constexpr int kSwStages = 3;
constexpr int kSwConv = 8;                                   // converter / epilogue warps
constexpr int kSwThreads = (kSwConv + 2) * 32;               // + TMA producer + MMA issuer
constexpr int kSwWin = 17;                                   // pool windows per k block row (32 pixels + 1)
constexpr int kSwGatherDy = 2 * kSwWin * 64 * 4;             // [2][17][64] fp32
constexpr int kSwGatherAm = 2 * kSwWin * 64;                 // [2][17][64] u8
constexpr int kSwGather = ((kSwGatherDy + kSwGatherAm + 1023) / 1024) * 1024;
struct StemWgArgs {
  int N, P, Q, groups, qblocks, units, stride;
  int M;           // valid rows R * 32 (the rest of the second M tile is the padding atom)
  float* partial;  // [gridDim.x][M][64]
  double* dbias_part;  // [gridDim.x][2][64] conv bias gradient partials (plane 1 zero), or null
  // FUSED: the stem BN's backward (its statistics pass has run)
  const float* stats;  // BN mean[64], invstd[64]
  const float* gamma;
  const float* beta;
  const float* coef;   // sum(g), sum(g xhat) [2][64]
  float inv_m;
  int relu;
};

template <int MODE>
__global__ void __launch_bounds__(kSwThreads, 1)
    stem_wgrad_rows_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                           const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmG,
                           const __grid_constant__ CUtensorMap tmM, StemWgArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  constexpr bool FUSED = MODE >= 1, GATHER = MODE == 2;
  static_assert(kSwG == 2, "warps 0-3 walk the k block's 2 rows as 2 x 2 pixel blocks");
  // box slots per stage (stride <= 2); GATHER: x in the B slots, then the pool windows
  constexpr int NA = 2 * kSwG + 6, NB = 2 * kSwG, NX = MODE == 1 ? 2 * kSwG : 0;
  const int na = a.stride * (kSwG - 1) + 8;  // input rows the output rows need (8 = R padded)
  constexpr uint32_t STAGE = (NA + NB + NX) * 4096 + (GATHER ? kSwGather : 0);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSwStages * STAGE);
  uint64_t* conv = full + kSwStages;   // warps 0-3 are done with the dy tile
  uint64_t* empty = conv + kSwStages;
  uint64_t* done = empty + kSwStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  float4* sred = reinterpret_cast<float4*>(smem + kSwStages * STAGE + 128);  // kSwConv * 32 float4
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSwStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&conv[i], kSwConv * 32);
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == kSwConv + 1) tmem_alloc(tmem_slot, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int per = (a.units + gridDim.x - 1) / gridDim.x;
  const int u0 = min(a.units, static_cast<int>(blockIdx.x) * per), u1 = min(a.units, u0 + per);
  auto unit = [&](int u, int& n, int& p0, int& qb) {
    qb = u % a.qblocks;
    const int r = u / a.qblocks;
    p0 = (r % a.groups) * kSwG;
    n = r / a.groups;
  };
  if (warp == kSwConv) {
    uint32_t s = 0, ph = 0;
    bool wrap = false;
    for (int u = u0; u < u1; ++u) {
      int n, p0, qb;
      unit(u, n, p0, qb);
      if (wrap) mbar_wait(&empty[s], ph ^ 1);
      if (elect_one()) {
        uint8_t* st = smem + s * STAGE;
        mbar_arrive_expect_tx(&full[s], (na + NB + NX) * 4096 + (GATHER ? kSwGatherDy + kSwGatherAm : 0));
        for (int j = 0; j < na; ++j)
          tma_load_4d(smem_u32(st + j * 4096), &tmA, &full[s], 0, qb * 32, p0 * a.stride + j, n);
        for (int g = 0; g < kSwG; ++g)
          for (int kc = 0; kc < 2; ++kc) {
            tma_load_4d(smem_u32(st + (NA + 2 * g + kc) * 4096), GATHER ? &tmX : &tmB, &full[s], kc * 32, qb * 32,
                        p0 + g, n);
            if (MODE == 1)
              tma_load_4d(smem_u32(st + (NA + NB + 2 * g + kc) * 4096), &tmX, &full[s], kc * 32, qb * 32, p0 + g, n);
          }
        if (GATHER) {
          uint8_t* gw = st + (NA + NB) * 4096;
          tma_load_4d(smem_u32(gw), &tmG, &full[s], 0, qb * 16, p0 >> 1, n);
          tma_load_4d(smem_u32(gw + kSwGatherDy), &tmM, &full[s], 0, qb * 16, p0 >> 1, n);
        }
      }
      __syncwarp();
      if (++s == kSwStages) {
        s = 0;
        ph ^= 1;
        wrap = true;
      }
    }
  } else if (warp == kSwConv + 1) {
    constexpr uint32_t idesc = idesc_tf32(kBM, 64, true, true);
    const uint64_t a0 = umma_desc(smem_u32(smem), 4096, 512, kLayoutSW128Base32);
    const uint64_t b0 = umma_desc(smem_u32(smem + NA * 4096), 4096, 512, kLayoutSW128Base32);
    uint32_t s = 0, ph = 0;
    bool first = true;
    for (int u = u0; u < u1; ++u) {
      mbar_wait(&conv[s], ph);
      tc_fence_after();
      if (elect_one()) {
        const uint64_t ad = a0 + s * (STAGE >> 4), bd = b0 + s * (STAGE >> 4);
#pragma unroll
        for (int g = 0; g < kSwG; ++g)
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              umma_tf32(tmem + mt * 64, ad + (a.stride * g + 4 * mt) * 256 + kk * 64, bd + g * 512 + kk * 64, idesc,
                        (first && g == 0 && kk == 0) ? 0u : 1u);
        umma_commit(&empty[s]);
      }
      __syncwarp();
      first = false;
      if (++s == kSwStages) {
        s = 0;
        ph ^= 1;
      }
    }
    if (elect_one()) umma_commit(done);
    __syncwarp();
  } else {
    // ---- dy tiles: bias-gradient sums, FUSED: g -> dx in place ----
    // thread = channel quad cq (kc = cq / 8, 16-byte chunk cq % 8 of the
    // 128-byte k-rows) x 2 x 2 pixel block cb (k-rows 2cb, 2cb+1 of both
    // output rows)
    static_assert(kSwConv == 8, "16 channel quads x 16 pixel blocks");
    const int t = threadIdx.x, cq = t & 15, cb = t >> 4, kc = cq >> 3, mc = cq & 7;
    const int c0 = cq * 4;
    float4 bsum = make_float4(0.f, 0.f, 0.f, 0.f);
    float gm[4] = {0, 0, 0, 0}, gi[4] = {0, 0, 0, 0}, gga[4] = {0, 0, 0, 0}, gbe[4] = {0, 0, 0, 0};
    float gs[4] = {0, 0, 0, 0}, k1[4] = {0, 0, 0, 0}, k2[4] = {0, 0, 0, 0};
    if (FUSED) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        gm[e] = a.stats[c0 + e];
        gi[e] = a.stats[64 + c0 + e];
        gga[e] = a.gamma[c0 + e];
        gbe[e] = a.beta[c0 + e];
        gs[e] = gga[e] * gi[e];
        k1[e] = a.coef[c0 + e] * a.inv_m;
        k2[e] = a.coef[64 + c0 + e] * a.inv_m;
      }
    }
    uint32_t s = 0, ph = 0;
    for (int u = u0; u < u1; ++u) {
      int n, p0, qb;
      unit(u, n, p0, qb);
      (void)n;
      (void)p0;
      const int qvalid = a.Q - qb * 32;  // k-rows (output columns) beyond Q are zero-filled padding
      mbar_wait(&full[s], ph);
      uint8_t* st = smem + s * STAGE;
      {
        const int c = cb;
        float4 o[4];
        if (GATHER) {
          // the block's pixels (dh, dw) from windows (r, c), (r, c + 1) of the
          // box, picks in pool_max_bwd_k3s2's order
          const float4* gd = reinterpret_cast<const float4*>(st + (NA + NB) * 4096);
          const uchar4* gm4 = reinterpret_cast<const uchar4*>(st + (NA + NB) * 4096 + kSwGatherDy);
          const int w00 = c * 16 + cq, w01 = w00 + 16, w10 = w00 + kSwWin * 16, w11 = w10 + 16;
          const uchar4 a00 = gm4[w00], a01 = gm4[w01], a10 = gm4[w10], a11 = gm4[w11];
          const float4 g00 = gd[w00], g01 = gd[w01], g10 = gd[w10], g11 = gd[w11];
#pragma unroll
          for (int q = 0; q < 4; ++q) o[q] = make_float4(0.f, 0.f, 0.f, 0.f);
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
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int dh = q >> 1, krow = 2 * c + (q & 1);
          uint8_t* bbox = st + (NA + 2 * dh + kc) * 4096;
          const uint8_t* xbox = GATHER ? bbox : st + (NA + NB + 2 * dh + kc) * 4096;
          const uint32_t off = mn_tile_off<32>(static_cast<uint32_t>(krow), static_cast<uint32_t>(mc));
          float4 v = GATHER ? o[q] : *reinterpret_cast<const float4*>(bbox + off);
          if (FUSED) {
            const float4 xv = *reinterpret_cast<const float4*>(xbox + off);
            const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
            float gg[4] = {v.x, v.y, v.z, v.w}, r[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              if (a.relu && !(bn_affine(xs[e], gm[e], gi[e], gga[e], gbe[e]) > 0.f)) gg[e] = 0.f;
              r[e] = krow < qvalid ? bn_dx_elem(gg[e], xs[e], gm[e], gi[e], gs[e], k1[e], k2[e]) : 0.f;
            }
            v = make_float4(r[0], r[1], r[2], r[3]);
            *reinterpret_cast<float4*>(bbox + off) = v;
          }
          bsum.x += v.x;
          bsum.y += v.y;
          bsum.z += v.z;
          bsum.w += v.w;
        }
      }
      if (FUSED) fence_proxy_async();
      mbar_arrive(&conv[s]);
      if (++s == kSwStages) {
        s = 0;
        ph ^= 1;
      }
    }
    // conv bias gradient partial of this CTA: the 16 pixel-block columns of
    // each channel quad in order, in double
    if (a.dbias_part) {
      sred[t] = bsum;
      named_bar(1, kSwConv * 32);
      if (t < 16) {
        double acc[4] = {0, 0, 0, 0};
        for (int j = 0; j < 16; ++j) {
          const float4 w = sred[j * 16 + t];
          acc[0] += w.x; acc[1] += w.y; acc[2] += w.z; acc[3] += w.w;
        }
        double* p = a.dbias_part + static_cast<size_t>(blockIdx.x) * 128 + t * 4;
        for (int e = 0; e < 4; ++e) {
          p[e] = acc[e];
          p[64 + e] = 0.0;
        }
      }
    }
    // epilogue: warp w drains M tile w / 4, TMEM lanes 32 (w % 4) ..
    const int lane = threadIdx.x & 31, mt = warp >> 2, wl = warp & 3;
    float* out = a.partial + static_cast<size_t>(blockIdx.x) * a.M * 64;
    const int row = mt * 128 + wl * 32 + lane;
    float4* dst = reinterpret_cast<float4*>(out + row * 64);
    if (u0 >= u1) {
      if (row < a.M)
        for (int q = 0; q < 16; ++q) dst[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      mbar_wait(done, 0);
      tc_fence_after();
      for (int c = 0; c < 64; c += 32) {
        float v[32];
        tmem_ld32(tmem + static_cast<uint32_t>(mt * 64 + c) + (static_cast<uint32_t>(wl * 32) << 16), v);
        if (row < a.M) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            dst[c / 4 + q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kSwConv + 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 128);
  }
}

}  // namespace

bool conv_stem_wgrad_rows_ok(const ConvShape& s) {
  const StemGeom g = stem_geom(s);
  return s.K == 64 && g.sblocks == 1 && s.R <= 8 && s.P % kSwG == 0 && s.stride <= 2;
}

bool stem_pool_gather_ok(const ConvShape& s, int pool_P, int pool_Q) {
  return conv_stem_wgrad_rows_ok(s) && s.P == 2 * pool_P && s.Q == 2 * pool_Q;
}

cudaError_t conv_stem_wgrad(const ConvShape& s, const float* xp, const float* dy, float* partial, float* wp_scratch,
                            float* dw, float* db, float* red, cudaStream_t st, const StemBnFuse* fuse) {
  const StemGeom g = stem_geom(s);
  const int Sp = g.sblocks * 8;
  const int M = s.R * g.sblocks * 32;
  cudaError_t err;
  if (conv_stem_wgrad_rows_ok(s)) {
    CUtensorMap A, B, X, G, Am;
    const int mode = !fuse ? 0 : fuse->dy_pool ? 2 : 1;
    if (mode == 2 && !stem_pool_gather_ok(s, fuse->pool_P, fuse->pool_Q)) return cudaErrorInvalidValue;
    const float* bsrc = mode == 0 ? dy : mode == 1 ? fuse->g : fuse->x;
    if (!make_stem_view(&A, xp, g, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) return cudaErrorInvalidValue;
    if (!make_nhwc4(&B, bsrc, s.N, s.P, s.Q, s.K, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) return cudaErrorInvalidValue;
    if (!make_nhwc4(&X, fuse ? fuse->x : bsrc, s.N, s.P, s.Q, s.K, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
      return cudaErrorInvalidValue;
    G = X;
    Am = X;
    if (mode == 2) {  // pool windows [N][P/2][Q/2][64]: boxes {64, 17, 2, 1}, zero-filled past the edges
      const cuuint64_t P2 = static_cast<cuuint64_t>(fuse->pool_P), Q2 = static_cast<cuuint64_t>(fuse->pool_Q);
      cuuint64_t dims[4] = {64, Q2, P2, static_cast<cuuint64_t>(s.N)};
      cuuint32_t box[4] = {64, kSwWin, 2, 1};
      cuuint32_t estr[4] = {1, 1, 1, 1};
      cuuint64_t sf[3] = {64 * 4, Q2 * 64 * 4, P2 * Q2 * 64 * 4};
      cuuint64_t sb[3] = {64, Q2 * 64, P2 * Q2 * 64};
      if (g_encode_tiled(&G, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(fuse->dy_pool), dims, sf, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
          g_encode_tiled(&Am, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<uint8_t*>(fuse->argmax), dims, sb, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    }
    StemWgArgs wa{};
    wa.N = s.N;
    wa.P = s.P;
    wa.Q = s.Q;
    wa.groups = s.P / kSwG;
    wa.qblocks = g.qblocks;
    wa.units = s.N * wa.groups * wa.qblocks;
    wa.stride = s.stride;
    wa.M = M;
    wa.partial = partial;
    wa.dbias_part = db ? reinterpret_cast<double*>(red) : nullptr;
    if (fuse) {
      wa.stats = fuse->stats;
      wa.gamma = fuse->gamma;
      wa.beta = fuse->beta;
      wa.coef = fuse->coef;
      wa.inv_m = 1.0f / static_cast<float>(fuse->rows);
      wa.relu = fuse->relu;
    }
    const int grid = num_sms();
    const int nbox = 2 * kSwG + 6 + 2 * kSwG + (mode == 1 ? 2 * kSwG : 0);
    const int smem = kSwStages * (nbox * 4096 + (mode == 2 ? kSwGather : 0)) + 128 + kSwConv * 32 * 16 + 1024;
    auto kern = mode == 2   ? stem_wgrad_rows_kernel<2>
                : mode == 1 ? stem_wgrad_rows_kernel<1>
                            : stem_wgrad_rows_kernel<0>;
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    kern<<<grid, kSwThreads, smem, st>>>(A, B, X, G, Am, wa);
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    // rows (r, s', c) of the [256][64] slices; rows >= R*32 are the padding atom
    err = splitk_reduce(partial, grid, M, s.K, wp_scratch, nullptr, 0, 1, st);
    if (err != cudaSuccess) return err;
    stem_weights_kernel<<<148, 256, 0, st>>>(dw, wp_scratch, s.K, s.R, s.S, Sp, 0);
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    if (!db) return cudaSuccess;
    return bias_grad_from_partials(reinterpret_cast<const double*>(red), grid, s.K, db, st);
  }
  if (fuse) return cudaErrorInvalidValue;  // the fused BN dx exists only in the rows kernel
  const int splits = conv_stem_wgrad_splits(s);
  const int BN = bn_for(s.K);
  CUtensorMap A, B, D;
  if (!make_stem_view(&A, xp, g, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) return cudaErrorInvalidValue;
  if (!make_nhwc4(&B, dy, s.N, s.P, s.Q, s.K, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) return cudaErrorInvalidValue;
  if (!make_store(&D, partial, M, s.K, splits)) return cudaErrorInvalidValue;
  TmaArgs a{};
  a.num_kb = s.N * s.P * g.qblocks;
  a.P = s.P;
  a.stride = s.stride;
  a.sblocks = g.sblocks;
  a.shift = g.shift;
  a.qblocks = g.qblocks;
  a.R = s.R;
  a.Kout = s.K;
  a.fsb = FastDivT(g.sblocks);
  a.fqb = FastDivT(g.qblocks);
  a.fP = FastDivT(s.P);
  const EpiArgs e{nullptr, s.K, 0, 1};
  switch (BN) {
    case 64: err = launch<64, 3>(A, B, D, a, e, M, s.K, splits, st); break;
    case 128: err = launch<128, 3>(A, B, D, a, e, M, s.K, splits, st); break;
    default: err = launch<256, 3>(A, B, D, a, e, M, s.K, splits, st); break;
  }
  if (err != cudaSuccess) return err;
  err = splitk_reduce(partial, splits, M, s.K, wp_scratch, nullptr, 0, 1, st);  // -> [K][R][Sp][4]
  if (err != cudaSuccess) return err;
  stem_weights_kernel<<<148, 256, 0, st>>>(dw, wp_scratch, s.K, s.R, s.S, Sp, 0);
  err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  if (!db) return cudaSuccess;  // bias gradient fused into the consuming BN's backward
  return bias_grad(dy, static_cast<int64_t>(s.N) * s.P * s.Q, s.K, db, red, st);
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

// Sub-pixel form of the 3x3 / stride-2 / pad-1 dgrad over an even input: dx
// pixel (2u+a, 2v+b) only sees dy pixels (u+dr, v+ds), dr, ds in {0, 1}, through
// filter tap (a - 2dr + 1, b - 2ds + 1) -- one GEMM over dy's grid with a 2x2
// window and 4C output columns (a, b, c), instead of four phase GEMMs that each
// re-read dy with 64..256-wide tiles and 4..16 k blocks.  7 of the 16 (tap,
// phase) weight blocks are zero (56% useful MMA work, at the full 256-wide rate).
// wsub[(a*2+b)*C + c][(dr*2+ds)*K + k] = w[k][a-2dr+1][b-2ds+1][c] or 0.
__device__ void subpix_weights_range(const float* __restrict__ w, float* __restrict__ wsub, int K, int C, int64_t i0,
                                     int64_t step) {
  const int64_t total = static_cast<int64_t>(16) * C * K;
  for (int64_t i = i0; i < total; i += step) {
    const int k = static_cast<int>(i % K);
    int64_t t = i / K;
    const int tap = static_cast<int>(t % 4);
    t /= 4;
    const int c = static_cast<int>(t % C);
    const int ab = static_cast<int>(t / C);
    const int r = (ab >> 1) - 2 * (tap >> 1) + 1, q = (ab & 1) - 2 * (tap & 1) + 1;
    wsub[i] = (r >= 0 && q >= 0) ? w[((static_cast<int64_t>(k) * 3 + r) * 3 + q) * C + c] : 0.f;
  }
}
__global__ void subpix_weights_kernel(const float* __restrict__ w, float* __restrict__ wsub, int K, int C) {
  subpix_weights_range(w, wsub, K, C, blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x,
                       static_cast<int64_t>(gridDim.x) * blockDim.x);
}

bool conv_dgrad_subpix_ok(const ConvShape& s) {
  return s.R == 3 && s.S == 3 && s.stride == 2 && s.pad == 1 && s.H == 2 * s.P && s.W == 2 * s.Q &&
         s.C % 32 == 0 && s.K % 32 == 0 && load_encoders();
}

cudaError_t conv_dgrad_subpix_tma(const ConvShape& s, const float* dy, const float* w, float* wt_scratch, float* dx,
                                  int accumulate, cudaStream_t st, int prepped) {
  if (!conv_dgrad_subpix_ok(s)) return cudaErrorInvalidValue;
  if (!prepped) {
    const int64_t wn = static_cast<int64_t>(16) * s.C * s.K;
    subpix_weights_kernel<<<std::min<int64_t>(1184, (wn + 255) / 256), 256, 0, st>>>(w, wt_scratch, s.K, s.C);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  // im2col over dy (P x Q grid), window 2x2 at (u, v); row/col P, Q read as 0
  CUtensorMap A, B, D;
  if (!make_im2col(&A, dy, s.N, s.P, s.Q, s.K, 0, 0, 0, 0, 1, kBM, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  const int Ncols = 4 * s.C, Ktot = 4 * s.K;
  const int M = s.N * s.P * s.Q;
  // pairs halve each CTA's share of the (large, 16CK) weight tile stream; small
  // M keeps single CTAs (conv_bench, stage 4: 84 us single vs 93 us pairs of 128)
  const TileCfg tc = use_pairs(M) ? tile_cfg(M, Ncols) : TileCfg{1, bn_for_waves(M, Ncols)};
  const int CG = tc.cg, BN = tc.bn;
  if (!make_tiled(&B, wt_scratch, Ncols, Ktot, BN / CG, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
  std::memset(&D, 0, sizeof D);
  TmaArgs a{};
  a.num_kb = Ktot / kBK;
  a.cchunks = s.K / 32;
  a.S = 2;
  a.P = s.P;
  a.Q = s.Q;
  a.PQ = s.P * s.Q;
  a.stride = 1;
  a.pad = 0;
  a.pad_w = 0;
  a.fcc = FastDivT(a.cchunks);
  a.fS = FastDivT(2);
  a.fPQ = FastDivT(a.PQ);
  a.fQ = FastDivT(s.Q);
  EpiArgs ep{};
  ep.N = Ncols;
  ep.reduce = accumulate;
  ep.scatter = dx;
  ep.M = M;
  ep.Uhw = s.P * s.Q;
  ep.Uw = s.Q;
  ep.H = s.H;
  ep.W = s.W;
  ep.fUhw = FastDivT(s.P * s.Q);
  ep.fUw = FastDivT(s.Q);
  ep.subpix = s.C;
  if (CG == 2) {
    switch (BN) {
      case 64: return launch<64, 0, 2>(A, B, D, a, ep, M, Ncols, 1, st);
      case 128: return launch<128, 0, 2>(A, B, D, a, ep, M, Ncols, 1, st);
      default: return launch<256, 0, 2>(A, B, D, a, ep, M, Ncols, 1, st);
    }
  }
  switch (BN) {
    case 64: return launch<64, 0>(A, B, D, a, ep, M, Ncols, 1, st);
    case 128: return launch<128, 0>(A, B, D, a, ep, M, Ncols, 1, st);
    default: return launch<256, 0>(A, B, D, a, ep, M, Ncols, 1, st);
  }
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
  // pairs when 256-row tiles cover R*S*C as tightly as 128-row ones
  const bool pair = pairs_mode() == 2 ||
                    (pairs_mode() == 1 && (a.RSC + 2 * kBM - 1) / (2 * kBM) * 2 == (a.RSC + kBM - 1) / kBM);
  if (pair) {
    switch (BN) {
      case 64: return launch<64, 1, 2>(A, B, D, a, e, a.RSC, s.K, splits, st);
      case 128: return launch<128, 1, 2>(A, B, D, a, e, a.RSC, s.K, splits, st);
      default: return launch<256, 1, 2>(A, B, D, a, e, a.RSC, s.K, splits, st);
    }
  }
  switch (BN) {
    case 64: return launch<64, 1>(A, B, D, a, e, a.RSC, s.K, splits, st);
    case 128: return launch<128, 1>(A, B, D, a, e, a.RSC, s.K, splits, st);
    default: return launch<256, 1>(A, B, D, a, e, a.RSC, s.K, splits, st);
  }
}


// Every layer's dgrad weight transform of a step in one launch: block row y =
// job y, blocks along x walk that job's 32 x 32 transpose tiles (the same
// element map as transpose_w_kernel in gemm_ops.cu) or its sub-pixel elements.
__global__ void __launch_bounds__(256) dgrad_prep_batch_kernel(const DgradPrepJob* __restrict__ jobs) {
  __shared__ float tile[32][33];
  const DgradPrepJob j = jobs[blockIdx.y];
  const int tid = threadIdx.y * 32 + threadIdx.x;
  if (j.subpix) {
    subpix_weights_range(j.w, j.wt, j.K, j.C, static_cast<int64_t>(blockIdx.x) * 256 + tid,
                         static_cast<int64_t>(gridDim.x) * 256);
    return;
  }
  const int tcx = (j.C + 31) / 32, tky = (j.K + 31) / 32;
  const int nt = tcx * tky * j.RS;
  for (int t = blockIdx.x; t < nt; t += gridDim.x) {
    const int rs_in = t / (tcx * tky);
    const int rem = t - rs_in * tcx * tky;
    const int c0 = (rem % tcx) * 32, k0 = (rem / tcx) * 32;
    const int rs = j.flip ? j.RS - 1 - rs_in : rs_in;
    for (int i = threadIdx.y; i < 32; i += 8) {
      const int k = k0 + i, c = c0 + threadIdx.x;
      tile[i][threadIdx.x] = (k < j.K && c < j.C) ? j.w[(static_cast<size_t>(k) * j.RS + rs_in) * j.C + c] : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += 8) {
      const int c = c0 + i, k = k0 + threadIdx.x;
      if (k < j.K && c < j.C) j.wt[(static_cast<size_t>(c) * j.RS + rs) * j.K + k] = tile[threadIdx.x][i];
    }
    __syncthreads();
  }
}

cudaError_t conv_dgrad_prep_batch(const DgradPrepJob* jobs, int njobs, cudaStream_t st) {
  if (njobs <= 0) return cudaSuccess;
  dgrad_prep_batch_kernel<<<dim3(64, njobs), dim3(32, 8), 0, st>>>(jobs);
  return cudaGetLastError();
}

}  // namespace sn
