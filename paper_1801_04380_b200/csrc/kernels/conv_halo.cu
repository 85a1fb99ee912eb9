// Halo-tiled implicit-GEMM convolution (stride 1) on tcgen05/TMEM.
//
// The im2col kernels (conv_tma.cu) load every input pixel once per filter tap
// (R*S times) from L2; on B200 those kernels are bound by the L2 -> SMEM
// operand traffic (~12 TB/s chip-wide), not by the tensor cores.  Here the
// output is enumerated on the *padded* grid: output position m = (n, y, x'),
// x' in [0, Wp) with Wp = W + 2*pad, of which x' < Q are real (the rest are
// junk rows of the GEMM, clipped by the TMA store).  On that grid every tap
// (r, s) is a uniform shift of r*Wp + s rows, so one TMA box per 32-channel
// chunk -- TR*MT + R - 1 padded input rows x Wp columns, zero-filled out of
// range -- serves all R*S taps: the UMMA A descriptor simply starts r*Wp + s
// rows into the halo (the SWIZZLE_128B pattern is a function of the absolute
// shared-memory address, so any 128-byte row offset is a valid operand start;
// tools/umma_shift_probe.py).
//
// One persistent CTA per SM walks tiles (n, band of TR*MT output rows, BN
// output channels); MT sub-tiles of TR rows (TR*Wp <= 128 GEMM rows each) share
// every weight tile, so a weight k-block feeds MT MMAs.  Two operand rings:
// halos (one per channel chunk) and weight tiles (one per tap and chunk).
// Warp roles as in conv_tma.cu: warp 4 = TMA producer, warp 5 = MMA issuer,
// warps 0-3 = epilogue (TMEM -> regs (+bias, +BN statistics) -> smem -> TMA
// store of a {32 ch, Wp, TR} box, columns >= Q and rows >= P clipped).
//
// Dgrad (stride 1) runs the same kernel over dy with the flipped, transposed
// filter and padding R-1-pad.
//
// Stride 2 (phase mode): output (p, q) tap (r, s) reads padded input pixel
// (2p + r, 2q + s), i.e. pixel (p + r/2, q + s/2) of the phase image
// (r % 2, s % 2) = padded input rows / columns of one parity.  A strided TMA
// box (elementStrides 2 along W and H) loads one phase image of the band per
// 32-channel chunk -- TR*MT + (R-1)/2 phase rows x Wp = Q + (S-1)/2 columns --
// and on the output grid (p, q'), q' < Wp, every tap of that phase is again a
// uniform row shift ((r/2) Wp + s/2) of it.  Four phase boxes per chunk read
// the input about once (the im2col kernel reads it R*S/4 = 2.25x and was
// bound by that L2 -> SMEM traffic: 41 % tensor pipe on ResNet conv_s2b1).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "gemm_tc.cuh"
#include "kernels.hpp"
#include "tma_host.hpp"

namespace sn {
namespace {

constexpr int kHaloThreads = 192;   // weight-gradient kernel: 4 epilogue warps + producer + MMA
constexpr int kHaloFwdThreads = 320;  // forward / dgrad: two epilogue groups (warps 0-3, 6-9)

struct HaloArgs {
  int Wp, TR, MT, R, S, pad, P, Q, cchunks, bands, n_tiles, tiles;
  int halo_rows;       // TR*MT + R - 1
  uint32_t halo_bytes; // TMA bytes of one halo box
  uint32_t halo_slot;  // smem stride between halo ring slots (1024-aligned, with read slack)
  const float* bias;
  int N;               // output channels (valid columns)
  int reduce;          // dgrad accumulate: TMA reduce-add store
  float* stats;        // BN statistics per sub-tile: [tile*MT + j][4][N] {shift, S1, S2, count}
  int phase;           // 1: stride-2 phase mode (four phase boxes per chunk, see above)
};

// EB: store-staging buffers per epilogue group (2: double-buffered; 1 frees
// 32 KB for a deeper operand ring, the group waits for its previous store's read)
template <int BN, int MT, int HST, int BST, int CG = 1, int EB = 2>
struct HaloSmem {
  static constexpr int B_BYTES = (BN / CG) * 128;  // CTA pairs: each CTA stages half of the weight rows
  static constexpr int EPI_BYTES = 2 * EB * kBM * 128;  // two epilogue groups x EB 16 KB chunks
  // halo ring first (dynamic size), then the fixed tail (barriers, TMEM slot, 2 x 1 KB statistics scratch)
  static constexpr int tail() { return BST * B_BYTES + EPI_BYTES + 512 + 2048 + 1024; }
};

// CG = 2: CTA pair (cluster of 2): the pair's tile is 2 x TR*MT output rows,
// rank r owns rows [r TR*MT, (r+1) TR*MT) of it (its own halo boxes, its own
// TMEM accumulators) and stages half of every weight tile; the even CTA issues
// tcgen05.mma.cta_group::2 with M = 256 (as conv_tma.cu CG = 2).
template <int BN, int MT, int HST, int BST, int CG = 1, int EB = 2>
__global__ void __launch_bounds__(kHaloFwdThreads, 1)
    tc_conv_halo_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                        const __grid_constant__ CUtensorMap tmY, HaloArgs a) {
  using L = HaloSmem<BN, MT, HST, BST, CG, EB>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* sH = smem;                                   // HST halo slots
  uint8_t* sB = smem + HST * a.halo_slot;               // BST weight tiles
  uint8_t* sEpi = sB + BST * L::B_BYTES;                // 2 x 16 KB store staging
  uint64_t* hfull = reinterpret_cast<uint64_t*>(sEpi + L::EPI_BYTES);
  uint64_t* hempty = hfull + HST;
  uint64_t* bfull = hempty + HST;
  uint64_t* bempty = bfull + BST;
  uint64_t* tfull = bempty + BST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* sred0 = reinterpret_cast<float*>(tmem_slot + 4);  // per epilogue group [4 warps][32][2]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t kCols = tmem_cols<2 * MT * BN>();

  if (threadIdx.x == 0) {
    for (int i = 0; i < HST; ++i) {
      mbar_init(&hfull[i], 1);
      mbar_init(&hempty[i], 1);
    }
    for (int i = 0; i < BST; ++i) {
      mbar_init(&bfull[i], 1);
      mbar_init(&bempty[i], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 256 * CG);  // both epilogue groups of both CTAs drain the accumulator
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
    tma_prefetch(&tmX);
    tma_prefetch(&tmW);
    tma_prefetch(&tmY);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int rank = CG == 2 ? static_cast<int>(cluster_rank()) : 0;
  const int unit = blockIdx.x / CG, units = gridDim.x / CG;

  // tile t -> (image n, band b, output-channel tile nt); band = CG*TR*MT output
  // rows, this CTA's part starts at y0
  auto coords = [&](int t, int& n, int& y0, int& n0) {
    const int nt = t % a.n_tiles;
    const int rest = t / a.n_tiles;
    const int b = rest % a.bands;
    n = rest / a.bands;
    y0 = (b * CG + rank) * a.TR * MT;
    n0 = nt * BN;
  };

  if (warp == 4) {
    {
      // ---------------- TMA producer (whole warp; the elected lane issues) ----------------
      uint32_t hs = 0, hph = 0, bs = 0, bph = 0;
      bool hwrap = false, bwrap = false;  // ring slots reused: wait for their release
      for (int t = unit; t < a.tiles; t += units) {
        int n, y0, n0;
        coords(t, n, y0, n0);
        for (int cc = 0; cc < a.cchunks; ++cc) {
         for (int ph = 0; ph < (a.phase ? 4 : 1); ++ph) {
          const int rho = ph >> 1, phi = ph & 1;
          if (rho >= a.R || phi >= a.S) continue;  // a phase without taps (1-wide filter)
          const int cx = a.phase ? phi - a.pad : -a.pad;
          const int cy = a.phase ? 2 * y0 + rho - a.pad : y0 - a.pad;
          if (hwrap) mbar_wait(&hempty[hs], hph ^ 1);
          if (elect_one()) {
            if constexpr (CG == 1) {
              mbar_arrive_expect_tx(&hfull[hs], a.halo_bytes);
              tma_load_4d(smem_u32(sH + hs * a.halo_slot), &tmX, &hfull[hs], cc * 32, cx, cy, n);
            } else {
              if (rank == 0) mbar_arrive_expect_tx(&hfull[hs], 2 * a.halo_bytes);
              tma2_load_4d(smem_u32(sH + hs * a.halo_slot), &tmX, mapa_u32(&hfull[hs], 0), cc * 32, cx, cy, n);
            }
          }
          __syncwarp();
          if (++hs == HST) {
            hs = 0;
            hph ^= 1;
            hwrap = true;
          }
          const int tstep = a.phase ? 2 : 1;
          for (int r = a.phase ? rho : 0; r < a.R; r += tstep)
          for (int sx = a.phase ? phi : 0; sx < a.S; sx += tstep) {
            const int tap = r * a.S + sx;
            if (bwrap) mbar_wait(&bempty[bs], bph ^ 1);
            if (elect_one()) {
              if constexpr (CG == 1) {
                mbar_arrive_expect_tx(&bfull[bs], L::B_BYTES);
                tma_load_2d(smem_u32(sB + bs * L::B_BYTES), &tmW, &bfull[bs], (tap * a.cchunks + cc) * 32, n0);
              } else {
                if (rank == 0) mbar_arrive_expect_tx(&bfull[bs], 2 * L::B_BYTES);
                tma2_load_2d(smem_u32(sB + bs * L::B_BYTES), &tmW, mapa_u32(&bfull[bs], 0),
                             (tap * a.cchunks + cc) * 32, n0 + rank * (BN / CG));
              }
            }
            __syncwarp();
            if (++bs == BST) {
              bs = 0;
              bph ^= 1;
              bwrap = true;
            }
          }
         }
        }
      }
    }
  } else if (warp == 5) {
    if (rank == 0) {
      // ---------------- MMA issuer (whole warp; the elected lane issues; pair leader for CG = 2) ----------------
      constexpr uint32_t idesc = idesc_tf32(kBM * CG, BN, false, false);
      // lean issue loop (see conv_tma.cu): base descriptors + offsets in 16-byte units
      const uint64_t hdesc0 = umma_desc(smem_u32(sH), 16, 1024, kLayoutSW128);
      const uint64_t bdesc0 = umma_desc(smem_u32(sB), 16, 1024, kLayoutSW128);
      const uint32_t jstep = static_cast<uint32_t>(a.TR * a.Wp) * 8u;  // sub-tile rows * 128 B / 16
      uint32_t hs = 0, hph = 0, bs = 0, bph = 0;
      int local = 0;
      for (int t = unit; t < a.tiles; t += units, ++local) {
        const int acc = local & 1;
        if (local >= 2) mbar_wait(&tempty[acc], ((local >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d0 = tmem + static_cast<uint32_t>(acc * MT * BN);
        bool first_mma = true;
        for (int cc = 0; cc < a.cchunks; ++cc) {
         for (int ph = 0; ph < (a.phase ? 4 : 1); ++ph) {
          const int rho = ph >> 1, phi = ph & 1;
          if (rho >= a.R || phi >= a.S) continue;
          mbar_wait(&hfull[hs], hph);
          const uint64_t h0 = hdesc0 + hs * (a.halo_slot >> 4);
          const int tstep = a.phase ? 2 : 1, sh = a.phase ? 1 : 0;
          for (int r = a.phase ? rho : 0; r < a.R; r += tstep)
          for (int sx = a.phase ? phi : 0; sx < a.S; sx += tstep) {
            mbar_wait(&bfull[bs], bph);
            tc_fence_after();
            const uint64_t ad = h0 + static_cast<uint32_t>((r >> sh) * a.Wp + (sx >> sh)) * 8u;
            const uint64_t bd = bdesc0 + bs * (L::B_BYTES >> 4);
            const uint32_t first = first_mma ? 0u : 1u;
            first_mma = false;
            if (elect_one()) {
              // sub-tiles innermost: consecutive MMAs feed different accumulators
#pragma unroll
              for (int kk = 0; kk < kBK / 8; ++kk)
#pragma unroll
                for (int j = 0; j < MT; ++j) {
                  if constexpr (CG == 1)
                    umma_tf32(d0 + j * BN, ad + j * jstep + kk * 2, bd + kk * 2, idesc, kk ? 1u : first);
                  else
                    umma2_tf32(d0 + j * BN, ad + j * jstep + kk * 2, bd + kk * 2, idesc, kk ? 1u : first);
                }
              if constexpr (CG == 1)
                umma_commit(&bempty[bs]);
              else
                umma2_commit(&bempty[bs]);
            }
            __syncwarp();
            if (++bs == BST) {
              bs = 0;
              bph ^= 1;
            }
          }
          if (elect_one()) {
            if constexpr (CG == 1)
              umma_commit(&hempty[hs]);
            else
              umma2_commit(&hempty[hs]);
          }
          __syncwarp();
          if (++hs == HST) {
            hs = 0;
            hph ^= 1;
          }
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
    // ---------------- epilogue: two groups of 4 warps (0-3, 6-9); warp w owns TMEM
    // lanes 32 (w % 4) ..; group g drains the chunks (sub-tile, 32 columns) of
    // parity g, with its own staging buffers, named barrier and leader thread
    const int grp = warp >= 6 ? 1 : 0, q4 = warp & 3;
    const uint32_t row = q4 * 32 + lane;
    const bool leader = q4 == 0 && lane == 0;
    const uint32_t bar_id = 1 + grp;
    uint8_t* sEpiG = sEpi + grp * EB * (kBM * 128);
    float* sred = sred0 + grp * 256;
    int local = 0;
    uint32_t chunk_no = 0;
    const uint32_t tempty_leader[2] = {CG == 2 ? mapa_u32(&tempty[0], 0) : 0u, CG == 2 ? mapa_u32(&tempty[1], 0) : 0u};
    for (int t = unit; t < a.tiles; t += units, ++local) {
      int n, y0, n0;
      coords(t, n, y0, n0);
      const int acc = local & 1;
      mbar_wait(&tfull[acc], (local >> 1) & 1);
      tc_fence_after();
      int ci = 0;  // chunk index within the tile (group = ci & 1)
      for (int j = 0; j < MT; ++j) {
        const int ys = y0 + j * a.TR;  // first output row of the sub-tile
        const uint32_t tbase = tmem + static_cast<uint32_t>(acc * MT * BN + j * BN) +
                               (static_cast<uint32_t>(q4 * 32) << 16);
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          if (n0 + c >= a.N) break;
          if ((ci++ & 1) != grp) continue;
          float v[32];
          tmem_ld32(tbase + static_cast<uint32_t>(c), v);
          if (a.bias) {
            if (n0 + c + 32 <= a.N) {  // 16-byte loads (parameter slices are 256-byte aligned)
              const float4* b4 = reinterpret_cast<const float4*>(a.bias + n0 + c);
#pragma unroll
              for (int q4 = 0; q4 < 8; ++q4) {
                const float4 bq = __ldg(b4 + q4);
                v[4 * q4] += bq.x; v[4 * q4 + 1] += bq.y; v[4 * q4 + 2] += bq.z; v[4 * q4 + 3] += bq.w;
              }
            } else {
#pragma unroll
              for (int q = 0; q < 32; ++q)
                if (n0 + c + q < a.N) v[q] += __ldg(a.bias + n0 + c + q);
            }
          }
          const uint32_t buf = smem_u32(sEpiG) + (EB == 2 ? (chunk_no & 1u) : 0u) * (kBM * 128);
          if (leader) {
            if constexpr (EB == 2)
              asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            else
              asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
          named_bar(bar_id, 128);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(buf + sw128_off(row, q)), "f"(v[4 * q]),
                         "f"(v[4 * q + 1]), "f"(v[4 * q + 2]), "f"(v[4 * q + 3])
                         : "memory");
          fence_proxy_async();
          named_bar(bar_id, 128);
          if (leader) {
            if (a.reduce)
              asm volatile(
                  "cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4, %5}], "
                  "[%1];" ::"l"(reinterpret_cast<uint64_t>(&tmY)),
                  "r"(buf), "r"(n0 + c), "r"(0), "r"(ys), "r"(n)
                  : "memory");
            else
              tma_store_4d(&tmY, buf, n0 + c, 0, ys, n);
            bulk_commit();
          }
          if (a.stats) {
            // junk rows (padded columns x' >= Q, rows past P) are skipped; the
            // shift is the sub-tile's row 0 (real unless the whole sub-tile lies
            // past P, then its count is 0 and the reduction skips it)
            const uint8_t* sb = sEpiG + (EB == 2 ? (chunk_no & 1u) : 0u) * (kBM * 128);
            const int Wp = a.Wp, TR = a.TR, Q = a.Q, rows_left = a.P - ys;
            float shift, t1, t2;
            chunk_column_stats(
                sb,
                [=](int rr) {
                  const int yy = rr / Wp, xx = rr - yy * Wp;
                  return yy < TR && xx < Q && yy < rows_left;
                },
                sred, shift, t1, t2, bar_id);
            if (q4 == 0 && n0 + c + lane < a.N) {
              const int rows_valid = max(0, min(a.TR, a.P - ys)) * a.Q;
              const size_t tile = ((static_cast<size_t>(t / a.n_tiles) * CG + rank) * MT + j);
              float* out = a.stats + tile * 4 * a.N + n0 + c + lane;
              out[0] = shift;
              out[a.N] = t1;
              out[2 * static_cast<size_t>(a.N)] = t2;
              out[3 * static_cast<size_t>(a.N)] = static_cast<float>(rows_valid);
            }
          }
          ++chunk_no;
        }
      }
      tc_fence_before();
      if constexpr (CG == 1)
        mbar_arrive(&tempty[acc]);
      else
        mbar_arrive_cluster(tempty_leader[acc]);
    }
    if (leader) bulk_wait_all();
  }
  __syncthreads();
  if constexpr (CG == 2) cluster_sync_all();
  if (warp == 5) {
    tc_fence_after();
    if constexpr (CG == 1)
      tmem_dealloc(tmem, kCols);
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols) : "memory");
  }
}

int num_sms_h() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

// Geometry for a stride-1 conv over an [N][H][W][C] input with R x S filter and
// padding pad (output P x Q): TR rows per 128-row sub-tile, MT sub-tiles.
struct HaloGeom {
  int Wp, TR, MT, halo_rows;
  uint32_t halo_bytes, halo_slot;
};

// Stride 2 (phase mode): Wp = Q + (S-1)/2 phase columns, TR*MT + (R-1)/2
// phase rows per box (the strided box spans twice that many input rows).
template <int BN, int MT>
bool halo_geom(int H, int W, int R, int S, int pad, int P, HaloGeom* g, int stride = 1, int Q = 0) {
  g->Wp = stride == 1 ? W + 2 * pad : Q + (S - 1) / 2;
  if (g->Wp > kBM || g->Wp > 256) return false;
  g->TR = std::min(kBM / g->Wp, P);
  g->MT = MT;
  g->halo_rows = stride == 1 ? g->TR * MT + R - 1 : g->TR * MT + (R - 1) / 2;
  if (g->halo_rows * stride > 256) return false;
  g->halo_bytes = static_cast<uint32_t>(g->halo_rows) * g->Wp * 128;
  // the last sub-tile's junk GEMM rows (TR*Wp .. 127) read past the halo box
  const int over = std::max(0, kBM + S - g->TR * g->Wp);
  const uint32_t need = g->halo_bytes + static_cast<uint32_t>(over) * 128;
  g->halo_slot = (need + 1023) / 1024 * 1024;
  (void)H;
  return true;
}

template <int BN, int MT, int HST, int BST, int CG, int EB = 2>
cudaError_t launch_halo(const CUtensorMap& X, const CUtensorMap& Wm, const CUtensorMap& Y, HaloArgs a,
                        const HaloGeom& g, cudaStream_t st) {
  using L = HaloSmem<BN, MT, HST, BST, CG, EB>;
  const int smem = static_cast<int>(HST * g.halo_slot) + L::tail();
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  auto kern = tc_conv_halo_kernel<BN, MT, HST, BST, CG, EB>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (err != cudaSuccess) return err;
  if constexpr (CG == 1) {
    const int grid = std::min(a.tiles, num_sms_h());
    kern<<<grid, kHaloFwdThreads, smem, st>>>(X, Wm, Y, a);
    return cudaGetLastError();
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * std::min(a.tiles, num_sms_h() / 2));
    cfg.blockDim = dim3(kHaloFwdThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, X, Wm, Y, a);
  }
}

// Variant table: (BN, MT, halo stages, weight stages, CTA group) fitting 227 KB.
template <int BN, int MT, int HST, int BST, int CG = 1, int EB = 2>
bool halo_fits(const HaloGeom& g) {
  return static_cast<int>(HST * g.halo_slot) + HaloSmem<BN, MT, HST, BST, CG, EB>::tail() <= 227 * 1024;
}

// variant id -> (BN, MT, CG): 1-3 single CTA BN 64/128/256, 4-6 the same as
// CTA pairs; 7-12 the stride-2 phase-mode kernels (three halo stages: a phase
// box feeds only 1-4 taps, so the ring turns over four times per chunk)
constexpr int kVarBN[13] = {0, 64, 128, 256, 64, 128, 256, 64, 128, 256, 64, 128, 256};
constexpr int kVarMT[13] = {0, 3, 2, 1, 3, 2, 1, 3, 2, 1, 3, 2, 1};
constexpr int kVarCG[13] = {0, 1, 1, 1, 2, 2, 2, 1, 1, 1, 2, 2, 2};

template <int BN, int MT>
bool geom_for(int v, int H, int W, int R, int S, int pad, int P, int Q, HaloGeom* g) {
  return halo_geom<BN, MT>(H, W, R, S, pad, P, g, v >= 7 ? 2 : 1, Q);
}
bool geom_any(int v, int H, int W, int R, int S, int pad, int P, int Q, HaloGeom* g) {
  switch (kVarBN[v]) {
    case 64: return geom_for<64, 3>(v, H, W, R, S, pad, P, Q, g);
    case 128: return geom_for<128, 2>(v, H, W, R, S, pad, P, Q, g);
    default: return geom_for<256, 1>(v, H, W, R, S, pad, P, Q, g);
  }
}

}  // namespace

// Which variant a shape runs (0: none).  Stride 1 or 2, C % 32 == 0,
// K % 32 == 0, padded rows fit one 128-row sub-tile, and the im2col kernel
// would re-read the input R*S > 1 times (stride 2: R*S/4 > 1).
int g_halo = -1;  // 0 off, 1 by shape (default; env SN_CONV_HALO=0 turns it off), 2 whenever legal (tests)
int halo_mode() {
  if (g_halo < 0) {
    const char* v = std::getenv("SN_CONV_HALO");
    g_halo = (v && v[0] == '0') ? 0 : 1;
  }
  return g_halo;
}

int conv_halo_mode() { return halo_mode(); }

int conv_halo_variant(int N, int H, int W, int C, int K, int R, int S, int pad, int P, int Q, int stride) {
  if (halo_mode() == 0 || C % 32 != 0 || K % 32 != 0 || R * S <= 1 || !tma_encoders_ok()) return 0;
  if (stride != 1 && stride != 2) return 0;
  static const int s2_off = std::getenv("SN_CONV_HALO_S2") && std::getenv("SN_CONV_HALO_S2")[0] == '0';
  if (stride == 2 && s2_off && halo_mode() == 1) return 0;  // A/B knob: the im2col kernel for stride 2
  if (pad < 0 || P != (H + 2 * pad - R) / stride + 1 || Q != (W + 2 * pad - S) / stride + 1) return 0;
  if (stride == 1 && (P != H + 2 * pad - R + 1 || Q != W + 2 * pad - S + 1)) return 0;
  // stride 2: every phase image has taps (a 1-wide filter has none in the odd phases)
  if (stride == 2 && (R < 2 || S < 2)) return 0;
  // by shape: real output rows must fill >= 3/4 of each 128-row sub-tile, and
  // K <= 128 (profiles/r01_conv_bench_halopair.txt, ResNet b256, CTA pairs:
  // stage 1 161 -> 118 us, stage 2 102 -> 94 us; at K = 256 the im2col
  // kernel's wider N amortises its operand traffic better: 80 vs 98 us)
  const int Wp = stride == 1 ? W + 2 * pad : Q + (S - 1) / 2;
  if (halo_mode() == 1 && (Wp > kBM || std::min(kBM / Wp, P) * Q * 4 < 3 * kBM || K > 128)) return 0;
  HaloGeom g;
  const int bn = K <= 64 ? 64 : (K <= 128 ? 128 : 256);
  const int base = stride == 2 ? 6 : 0;
  // CTA pairs halve the per-SM weight traffic; they need >= 148 pair tiles
  const int pm = conv_pairs_mode();
  int v = 0;
  if (!geom_any(base + (bn == 64 ? 1 : bn == 128 ? 2 : 3), H, W, R, S, pad, P, Q, &g)) return 0;
  if (stride == 1) {
    if (bn == 64) {
      v = halo_fits<64, 3, 2, 4>(g) ? 1 : 0;
      if (pm != 0 && halo_fits<64, 3, 2, 8, 2>(g)) v = 4;
    } else if (bn == 128) {
      v = halo_fits<128, 2, 2, 4>(g) ? 2 : 0;
      if (pm != 0 && halo_fits<128, 2, 2, 8, 2>(g)) v = 5;
    } else {
      v = halo_fits<256, 1, 2, 3>(g) ? 3 : 0;
      if (pm != 0 && halo_fits<256, 1, 2, 6, 2>(g)) v = 6;
    }
  } else {
    if (bn == 64) {
      v = halo_fits<64, 3, 2, 4>(g) ? 7 : 0;
      if (pm != 0 && halo_fits<64, 3, 2, 8, 2>(g)) v = 10;
    } else if (bn == 128) {
      v = halo_fits<128, 2, 3, 3>(g) ? 8 : 0;
      if (pm != 0 && halo_fits<128, 2, 3, 6, 2>(g)) v = 11;
    } else {
      v = halo_fits<256, 1, 3, 3>(g) ? 9 : 0;
      if (pm != 0 && halo_fits<256, 1, 3, 6, 2>(g)) v = 12;
    }
  }
  if (v && kVarCG[v] == 2 && pm == 1) {
    const int bands2 = (P + g.TR * g.MT * 2 - 1) / (g.TR * g.MT * 2);
    if (static_cast<int64_t>(N) * bands2 * ((K + bn - 1) / bn) < num_sms_h() / 2) v -= 3;
  }
  return v;
}

int conv_halo_stats_tiles(int N, int H, int W, int C, int K, int R, int S, int pad, int P, int Q, int stride) {
  const int v = conv_halo_variant(N, H, W, C, K, R, S, pad, P, Q, stride);
  if (!v) return 0;
  const int MT = kVarMT[v], CG = kVarCG[v];
  const int Wp = stride == 1 ? W + 2 * pad : Q + (S - 1) / 2;
  const int TR = std::min(kBM / Wp, P);
  const int bands = (P + TR * MT * CG - 1) / (TR * MT * CG);
  return N * bands * CG * MT;
}

// y[N][P][Q][K] (+)= conv(x[N][H][W][C], w[K][R][S][C]) + bias, stride 1 or 2.
cudaError_t conv_halo(int N, int H, int W, int C, int K, int R, int S, int pad, int P, int Q, const float* x,
                      const float* w, const float* bias, float* y, int accumulate, float* stats, cudaStream_t st,
                      int stride) {
  const int v = conv_halo_variant(N, H, W, C, K, R, S, pad, P, Q, stride);
  if (!v) return cudaErrorInvalidValue;
  HaloGeom g;
  const int BN = kVarBN[v], MT = kVarMT[v], CG = kVarCG[v];
  geom_any(v, H, W, R, S, pad, P, Q, &g);
  CUtensorMap X, Wm, Y;
  if (!tma_map_nhwc(&X, x, N, H, W, C, g.Wp, g.halo_rows, 0, stride)) return cudaErrorInvalidValue;
  if (!tma_map_2d(&Wm, w, K, static_cast<int64_t>(R) * S * C, BN / CG, 0)) return cudaErrorInvalidValue;
  if (!tma_map_nhwc(&Y, y, N, P, Q, K, g.Wp, g.TR, 0)) return cudaErrorInvalidValue;
  HaloArgs a{};
  a.Wp = g.Wp;
  a.TR = g.TR;
  a.MT = MT;
  a.R = R;
  a.S = S;
  a.pad = pad;
  a.P = P;
  a.Q = Q;
  a.cchunks = C / 32;
  a.bands = (P + g.TR * MT * CG - 1) / (g.TR * MT * CG);
  a.n_tiles = (K + BN - 1) / BN;
  a.tiles = N * a.bands * a.n_tiles;
  a.halo_rows = g.halo_rows;
  a.halo_bytes = g.halo_bytes;
  a.halo_slot = g.halo_slot;
  a.bias = bias;
  a.N = K;
  a.reduce = accumulate;
  a.stats = stats;
  a.phase = stride == 2 ? 1 : 0;
  switch (v) {
    case 1: return launch_halo<64, 3, 2, 4, 1>(X, Wm, Y, a, g, st);
    case 2: return launch_halo<128, 2, 2, 4, 1>(X, Wm, Y, a, g, st);
    case 3: return launch_halo<256, 1, 2, 3, 1>(X, Wm, Y, a, g, st);
    case 4: return launch_halo<64, 3, 2, 8, 2>(X, Wm, Y, a, g, st);
    case 5: return launch_halo<128, 2, 2, 8, 2>(X, Wm, Y, a, g, st);
    case 6: return launch_halo<256, 1, 2, 6, 2>(X, Wm, Y, a, g, st);
    case 7: return launch_halo<64, 3, 2, 4, 1>(X, Wm, Y, a, g, st);
    case 8: return launch_halo<128, 2, 3, 3, 1>(X, Wm, Y, a, g, st);
    case 9: return launch_halo<256, 1, 3, 3, 1>(X, Wm, Y, a, g, st);
    case 10: return launch_halo<64, 3, 2, 8, 2>(X, Wm, Y, a, g, st);
    case 11: return launch_halo<128, 2, 3, 6, 2>(X, Wm, Y, a, g, st);
    default: return launch_halo<256, 1, 3, 6, 2>(X, Wm, Y, a, g, st);
  }
}

}  // namespace sn

namespace sn {
void set_conv_halo(int mode) { g_halo = mode; }
}  // namespace sn

// ---------------------------------------------------------------------------
// Halo-tiled weight gradient for C = K = 64, R x S taps, stride 1:
//   dW_tap[c][k] = sum over output positions p of x[p + shift(tap)][c] dy[p][k]
// on the padded grid (dy is zero at the junk columns x' >= Q: TMA zero fill).
// The GEMM K dimension is the position; per band of TR padded output rows one
// x halo box per 32-channel chunk (MN-major, SWIZZLE_128B_ATOM_32B) and one dy
// box per 32-channel chunk of k serve all R*S taps: the tap shift is a K-row
// offset of the A descriptor.  One M = 64 MMA per (tap, 8 positions); the R*S
// accumulators (64 lanes x 64 columns each, an M = 64 result occupying lanes
// 16 x {0..3} + lane0, lane0 in {0, 16}) are packed two per 64-column TMEM
// block.  Each persistent CTA accumulates a contiguous range of bands and
// writes its partial [R*S*C][K] slice; splitk_reduce sums the CTAs' slices
// in a fixed order into dw[K][R][S][C].
namespace sn {
namespace {

struct HaloWgArgs {
  int Wp, TR, R, S, pad, P, Q, bands, units;  // units = N * bands
  uint32_t xbox_bytes, dybox_bytes;           // one TMA box (one 32-channel chunk)
  uint32_t xslot, dyslot;                     // smem bytes per chunk buffer (with zeroed slack rows)
  int ksteps;                                 // ceil(TR*Wp / 8)
  float* partial;                             // [gridDim.x][R*S*Ct][Kt]
  int c0, k0, Ct, Kt;                         // this 64 x 64 sub-problem's channel / k offsets, full C / K
};

constexpr int kWgStages = 2;

template <int RC, int SC>  // compile-time taps (0: runtime a.R x a.S)
__global__ void __launch_bounds__(kHaloThreads, 1)
    tc_conv_halo_wgrad64(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmDY,
                         HaloWgArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const uint32_t stage_bytes = 2 * a.xslot + 2 * a.dyslot;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kWgStages * stage_bytes);
  uint64_t* empty = full + kWgStages;
  uint64_t* done = empty + kWgStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int taps = a.R * a.S;

  // zero every buffer once: the slack rows past each TMA box are read by the
  // shifted descriptors (x) or the last partial k step (dy) and must be finite
  for (uint32_t i = threadIdx.x * 16; i < kWgStages * stage_bytes; i += blockDim.x * 16)
    *reinterpret_cast<float4*>(smem + i) = make_float4(0.f, 0.f, 0.f, 0.f);
  fence_proxy_async();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kWgStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // contiguous range of work units (image, band) for this CTA
  const int per = (a.units + gridDim.x - 1) / gridDim.x;
  const int u0 = min(a.units, blockIdx.x * per), u1 = min(a.units, u0 + per);

  if (warp == 4) {
    uint32_t s = 0, ph = 0;
    bool wrap = false;
    for (int u = u0; u < u1; ++u) {
      const int n = u / a.bands, y0 = (u - n * a.bands) * a.TR;
      if (wrap) mbar_wait(&empty[s], ph ^ 1);
      if (elect_one()) {
        uint8_t* st = smem + s * stage_bytes;
        mbar_arrive_expect_tx(&full[s], 2 * a.xbox_bytes + 2 * a.dybox_bytes);
        for (int c = 0; c < 2; ++c) {
          tma_load_4d(smem_u32(st + c * a.xslot), &tmX, &full[s], a.c0 + c * 32, -a.pad, y0 - a.pad, n);
          tma_load_4d(smem_u32(st + 2 * a.xslot + c * a.dyslot), &tmDY, &full[s], a.k0 + c * 32, 0, y0, n);
        }
      }
      __syncwarp();
      if (++s == kWgStages) {
        s = 0;
        ph ^= 1;
        wrap = true;
      }
    }
  } else if (warp == 5) {
    // M = 64, N = 64, both operands MN-major (SW128_BASE32B): LBO = the other
    // 32-channel chunk's buffer, SBO = 4 K rows (512 B); 8 positions = 1024 B
    constexpr uint32_t idesc = idesc_tf32(64, 64, true, true);
    const uint64_t xd0 = umma_desc(smem_u32(smem), a.xslot, 512, kLayoutSW128Base32);
    const uint64_t dd0 = umma_desc(smem_u32(smem + 2 * a.xslot), a.dyslot, 512, kLayoutSW128Base32);
    const uint32_t sstep = stage_bytes >> 4;
    uint32_t s = 0, ph = 0;
    bool first = true;
    for (int u = u0; u < u1; ++u) {
      mbar_wait(&full[s], ph);
      tc_fence_after();
      if (elect_one()) {
        const uint64_t xd = xd0 + s * sstep, dd = dd0 + s * sstep;
        const uint32_t rowstep = static_cast<uint32_t>(a.Wp) * 8u;  // one padded row, 16-byte units
        for (int kq = 0; kq < a.ksteps; ++kq) {
          const uint64_t xk = xd + static_cast<uint32_t>(kq) * 64u, dk = dd + static_cast<uint32_t>(kq) * 64u;
          const uint32_t acc = (first && kq == 0) ? 0u : 1u;
          if constexpr (RC > 0) {
#pragma unroll
            for (int t = 0; t < RC * SC; ++t) {
              const uint32_t d = tmem + static_cast<uint32_t>((t >> 1) * 64) + (static_cast<uint32_t>((t & 1) * 16) << 16);
              umma_tf32(d, xk + (t / SC) * rowstep + (t % SC) * 8u, dk, idesc, acc);
            }
          } else {
            int r = 0, sx = 0;
            for (int t = 0; t < taps; ++t) {
              const uint32_t d = tmem + static_cast<uint32_t>((t >> 1) * 64) + (static_cast<uint32_t>((t & 1) * 16) << 16);
              umma_tf32(d, xk + r * rowstep + sx * 8u, dk, idesc, acc);
              if (++sx == a.S) {
                sx = 0;
                ++r;
              }
            }
          }
        }
        umma_commit(&empty[s]);
      }
      __syncwarp();
      first = false;
      if (++s == kWgStages) {
        s = 0;
        ph ^= 1;
      }
    }
    if (elect_one()) umma_commit(done);
    __syncwarp();
  } else {
    // epilogue: warp w, lane l -> tap 2b + (l >= 16), channel 16 w + (l & 15)
    const int RSC = taps * a.Ct;
    float* out = a.partial + static_cast<size_t>(blockIdx.x) * RSC * a.Kt;
    if (u0 >= u1) {
      // no work: this CTA's block of the slice is zero
      for (int i = threadIdx.x; i < taps * 64 * 64; i += 128) {
        const int tap = i / 4096, c = (i / 64) % 64, k = i % 64;
        out[(static_cast<size_t>(tap) * a.Ct + a.c0 + c) * a.Kt + a.k0 + k] = 0.f;
      }
    } else {
      mbar_wait(done, 0);
      tc_fence_after();
      for (int b = 0; b < (taps + 1) / 2; ++b) {
        const int tap = 2 * b + (lane >> 4);
        const int c = 16 * warp + (lane & 15);
        for (int k0 = 0; k0 < 64; k0 += 32) {
          float v[32];
          tmem_ld32(tmem + static_cast<uint32_t>(b * 64 + k0) + (static_cast<uint32_t>(warp * 32) << 16), v);
          if (tap < taps) {
            float4* dst =
                reinterpret_cast<float4*>(out + (static_cast<size_t>(tap) * a.Ct + a.c0 + c) * a.Kt + a.k0 + k0);
#pragma unroll
            for (int q = 0; q < 8; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace

int conv_halo_wgrad_splits();

// Applicable: C, K multiples of 64 (run as (C/64) x (K/64) sub-problems of
// 64 x 64, each re-reading its x / dy chunks), stride 1, padded width <= 128
// rows per band; by shape only up to C, K <= 128 (the sub-problems multiply
// the operand traffic; at 256 channels the im2col kernel is as fast).
bool conv_halo_wgrad_ok(int N, int H, int W, int C, int K, int R, int S, int pad, int P, int Q) {
  if (halo_mode() == 0 || C % 64 != 0 || K % 64 != 0 || R * S < 2 || R * S > 10 || !tma_encoders_ok()) return false;
  // by shape only C = K = 64: the sub-problems re-read x / dy and each writes a
  // full partial slice per CTA; at C = K = 128 the im2col kernel is faster
  // (profiles/r01_conv_bench_wgrad_halo.txt: 222 vs 260 us on ResNet stage 2)
  if (halo_mode() == 1 && (C > 64 || K > 64)) return false;
  // one R*S*C*K partial slice per CTA must fit the executor's split-K scratch (64 Mi floats)
  if (static_cast<int64_t>(conv_halo_wgrad_splits()) * R * S * C * K > (64ll << 20)) return false;
  if (P != H + 2 * pad - R + 1 || Q != W + 2 * pad - S + 1 || pad < 0) return false;
  const int Wp = W + 2 * pad;
  if (Wp > kBM) return false;
  const int TR = std::min(kBM / Wp, P);
  // by shape: the padded band must be mostly real positions
  if (halo_mode() == 1 && TR * Q * 4 < 3 * kBM) return false;
  const int xrows = (TR + R - 1) * Wp + 8 + (S - 1);
  const int dyrows = (TR * Wp + 7) / 8 * 8;
  const uint32_t stage = 2 * ((xrows * 128 + 1023) / 1024 * 1024) + 2 * ((dyrows * 128 + 1023) / 1024 * 1024);
  return kWgStages * stage + 1024 + 256 <= 227 * 1024;
}

int conv_halo_wgrad_splits() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

// partial: conv_halo_wgrad_splits() * R*S*C*K floats; dw[K][R][S][C].
cudaError_t conv_halo_wgrad(int N, int H, int W, int C, int K, int R, int S, int pad, int P, int Q, const float* x,
                            const float* dy, float* partial, float* dw, cudaStream_t st) {
  if (!conv_halo_wgrad_ok(N, H, W, C, K, R, S, pad, P, Q)) return cudaErrorInvalidValue;
  HaloWgArgs a{};
  a.Wp = W + 2 * pad;
  a.TR = std::min(kBM / a.Wp, P);
  a.R = R;
  a.S = S;
  a.pad = pad;
  a.P = P;
  a.Q = Q;
  a.bands = (P + a.TR - 1) / a.TR;
  a.units = N * a.bands;
  const int xrows_box = (a.TR + R - 1) * a.Wp;
  a.xbox_bytes = static_cast<uint32_t>(xrows_box) * 128;
  a.dybox_bytes = static_cast<uint32_t>(a.TR * a.Wp) * 128;
  a.xslot = ((xrows_box + 8 + (S - 1)) * 128 + 1023) / 1024 * 1024;
  a.dyslot = (((a.TR * a.Wp + 7) / 8 * 8) * 128 + 1023) / 1024 * 1024;
  a.ksteps = (a.TR * a.Wp + 7) / 8;
  a.partial = partial;
  a.Ct = C;
  a.Kt = K;
  CUtensorMap X, DY;
  if (!tma_map_nhwc(&X, x, N, H, W, C, a.Wp, a.TR + R - 1, 1)) return cudaErrorInvalidValue;
  if (!tma_map_nhwc(&DY, dy, N, P, Q, K, a.Wp, a.TR, 1)) return cudaErrorInvalidValue;
  const int grid = conv_halo_wgrad_splits();
  const int smem = kWgStages * (2 * a.xslot + 2 * a.dyslot) + 1024 + 256;
  auto kern = (R == 3 && S == 3) ? tc_conv_halo_wgrad64<3, 3> : tc_conv_halo_wgrad64<0, 0>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (err != cudaSuccess) return err;
  for (int c0 = 0; c0 < C; c0 += 64)
    for (int k0 = 0; k0 < K; k0 += 64) {
      a.c0 = c0;
      a.k0 = k0;
      if (!xskip(16)) kern<<<grid, kHaloThreads, smem, st>>>(X, DY, a);
      err = cudaGetLastError();
      if (err != cudaSuccess) return err;
    }
  return splitk_reduce(partial, grid, R * S * C, K, dw, nullptr, 0, 1, st);
}

}  // namespace sn

// ---------------------------------------------------------------------------
// Halo weight gradient for C, K multiples of 128 (M = 128, N = 128 MMAs):
//   dW[(r, s, c)][k] = sum_p x[p + r*Wp + s - pad*(Wp+1)][c] dy[p][k]
// A CTA owns one job (filter row r, 128-channel group, 128-k group) and a
// contiguous range of (image, band) work units; per unit it loads, for each of
// its 4 channel chunks, the TR input rows of filter row r (one TMA box, zero
// filled) and the TR rows of dy (one box per k chunk).  The S column taps of
// the row are K-row shifts of the A descriptor; the A operand's four MN atoms
// are the four channel-chunk buffers (uniform LBO).  S accumulators of 128
// columns live in TMEM for the whole range; the CTA then writes its partial
// slice [split][R*S*C][K] for its job's rows (every (split, row) written once:
// the CTAs are split evenly across jobs).
namespace sn {
namespace {

struct HaloWg128Args {
  int Wp, TR, R, S, pad, P, bands, units;  // units = N * bands
  int C, K, jobs_c, jobs_k, per_job;       // per_job = CTAs per job = splits
  uint32_t box_bytes, slot;                // one chunk box; smem per chunk buffer
  int ksteps;
  float* partial;
};

constexpr int kWg128Stages = 2;

__global__ void __launch_bounds__(kHaloThreads, 1)
    tc_conv_halo_wgrad128(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmDY,
                          HaloWg128Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const uint32_t stage_bytes = 8 * a.slot;  // 4 x chunks, 4 dy chunks
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kWg128Stages * stage_bytes);
  uint64_t* empty = full + kWg128Stages;
  uint64_t* done = empty + kWg128Stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (uint32_t i = threadIdx.x * 16; i < kWg128Stages * stage_bytes; i += blockDim.x * 16)
    *reinterpret_cast<float4*>(smem + i) = make_float4(0.f, 0.f, 0.f, 0.f);
  fence_proxy_async();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kWg128Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int jobs = a.R * a.jobs_c * a.jobs_k;
  const int job = blockIdx.x / a.per_job, split = blockIdx.x % a.per_job;
  const bool active = job < jobs;
  const int r = active ? job / (a.jobs_c * a.jobs_k) : 0;
  const int cg = active ? (job / a.jobs_k) % a.jobs_c : 0, kg = active ? job % a.jobs_k : 0;
  const int per = (a.units + a.per_job - 1) / a.per_job;
  const int u0 = active ? min(a.units, split * per) : 0, u1 = active ? min(a.units, u0 + per) : 0;

  if (warp == 4) {
    uint32_t s = 0, ph = 0;
    bool wrap = false;
    for (int u = u0; u < u1; ++u) {
      const int n = u / a.bands, y0 = (u - n * a.bands) * a.TR;
      if (wrap) mbar_wait(&empty[s], ph ^ 1);
      if (elect_one()) {
        uint8_t* st = smem + s * stage_bytes;
        mbar_arrive_expect_tx(&full[s], 8 * a.box_bytes);
        for (int c = 0; c < 4; ++c) {
          tma_load_4d(smem_u32(st + c * a.slot), &tmX, &full[s], cg * 128 + c * 32, -a.pad, y0 + r - a.pad, n);
          tma_load_4d(smem_u32(st + (4 + c) * a.slot), &tmDY, &full[s], kg * 128 + c * 32, 0, y0, n);
        }
      }
      __syncwarp();
      if (++s == kWg128Stages) {
        s = 0;
        ph ^= 1;
        wrap = true;
      }
    }
  } else if (warp == 5) {
    constexpr uint32_t idesc = idesc_tf32(128, 128, true, true);
    const uint64_t xd0 = umma_desc(smem_u32(smem), a.slot, 512, kLayoutSW128Base32);
    const uint64_t dd0 = umma_desc(smem_u32(smem + 4 * a.slot), a.slot, 512, kLayoutSW128Base32);
    const uint32_t sstep = stage_bytes >> 4;
    uint32_t s = 0, ph = 0;
    bool first = true;
    for (int u = u0; u < u1; ++u) {
      mbar_wait(&full[s], ph);
      tc_fence_after();
      if (elect_one()) {
        const uint64_t xd = xd0 + s * sstep, dd = dd0 + s * sstep;
        for (int kq = 0; kq < a.ksteps; ++kq) {
          const uint32_t acc = (first && kq == 0) ? 0u : 1u;
          for (int sx = 0; sx < a.S; ++sx)
            umma_tf32(tmem + static_cast<uint32_t>(sx * 128), xd + static_cast<uint32_t>(sx + 8 * kq) * 8u,
                      dd + static_cast<uint32_t>(kq) * 64u, idesc, acc);
        }
        umma_commit(&empty[s]);
      }
      __syncwarp();
      first = false;
      if (++s == kWg128Stages) {
        s = 0;
        ph ^= 1;
      }
    }
    if (elect_one()) umma_commit(done);
    __syncwarp();
  } else if (active) {
    // epilogue: thread (warp w, lane l) = channel 32 w + l of the group, all 128 k of each tap
    const int c = cg * 128 + warp * 32 + lane;
    float* out = a.partial + static_cast<size_t>(split) * a.R * a.S * a.C * a.K;
    if (u0 >= u1) {
      for (int sx = 0; sx < a.S; ++sx) {
        float4* dst = reinterpret_cast<float4*>(out + (static_cast<size_t>(r * a.S + sx) * a.C + c) * a.K + kg * 128);
        for (int q = 0; q < 32; ++q) dst[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    } else {
      mbar_wait(done, 0);
      tc_fence_after();
      for (int sx = 0; sx < a.S; ++sx) {
        float4* dst = reinterpret_cast<float4*>(out + (static_cast<size_t>(r * a.S + sx) * a.C + c) * a.K + kg * 128);
        for (int k0 = 0; k0 < 128; k0 += 32) {
          float v[32];
          tmem_ld32(tmem + static_cast<uint32_t>(sx * 128 + k0) + (static_cast<uint32_t>(warp * 32) << 16), v);
#pragma unroll
          for (int q = 0; q < 8; ++q) dst[k0 / 4 + q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace

// Rows per band: as many padded rows as keep two stages of 8 chunk buffers
// (with their slack rows) in shared memory.
int wg128_tr(int Wp, int S, int P, uint32_t* slot_out) {
  int best = 0;
  uint32_t best_slot = 0;
  for (int t = 1; t <= P && t * Wp <= kBM; ++t) {
    const int rows = (t * Wp + 7) / 8 * 8 + S + 8;
    const uint32_t slot = (rows * 128 + 1023) / 1024 * 1024;
    if (kWg128Stages * 8 * slot + 1024 + 256 <= 227 * 1024) {
      best = t;
      best_slot = slot;
    }
  }
  if (slot_out) *slot_out = best_slot;
  return best;
}

// C, K multiples of 128, stride 1, S <= 4 taps per row, padded width <= 128.
bool conv_halo_wgrad128_ok(int N, int H, int W, int C, int K, int R, int S, int pad, int P, int Q) {
  if (halo_mode() == 0 || C % 128 != 0 || K % 128 != 0 || S > 4 || R * S < 2 || !tma_encoders_ok()) return false;
  if (P != H + 2 * pad - R + 1 || Q != W + 2 * pad - S + 1 || pad < 0) return false;
  const int Wp = W + 2 * pad;
  if (Wp > kBM) return false;
  const int TR = wg128_tr(Wp, S, P, nullptr);
  if (TR < 1) return false;
  // by shape: most band positions real (junk columns cost MMA work), C = K = 128
  if (halo_mode() == 1 && (TR * Q * 4 < 3 * TR * Wp || C > 128 || K > 128)) return false;
  const int jobs = R * (C / 128) * (K / 128);
  if (jobs > conv_halo_wgrad_splits()) return false;
  const int per_job = conv_halo_wgrad_splits() / jobs;
  return static_cast<int64_t>(per_job) * R * S * C * K <= (64ll << 20);
}

int conv_halo_wgrad128_splits(int C, int K, int R) {
  const int jobs = R * (C / 128) * (K / 128);
  return conv_halo_wgrad_splits() / jobs;
}

cudaError_t conv_halo_wgrad128(int N, int H, int W, int C, int K, int R, int S, int pad, int P, int Q,
                               const float* x, const float* dy, float* partial, float* dw, cudaStream_t st) {
  if (!conv_halo_wgrad128_ok(N, H, W, C, K, R, S, pad, P, Q)) return cudaErrorInvalidValue;
  HaloWg128Args a{};
  a.Wp = W + 2 * pad;
  uint32_t slot = 0;
  a.TR = wg128_tr(a.Wp, S, P, &slot);
  a.R = R;
  a.S = S;
  a.pad = pad;
  a.P = P;
  a.bands = (P + a.TR - 1) / a.TR;
  a.units = N * a.bands;
  a.C = C;
  a.K = K;
  a.jobs_c = C / 128;
  a.jobs_k = K / 128;
  a.per_job = conv_halo_wgrad128_splits(C, K, R);
  a.box_bytes = static_cast<uint32_t>(a.TR * a.Wp) * 128;
  a.slot = slot;
  a.ksteps = (a.TR * a.Wp + 7) / 8;
  a.partial = partial;
  CUtensorMap X, DY;
  // x: TR rows of one filter row; dy: TR rows (columns >= Q read as zero)
  if (!tma_map_nhwc(&X, x, N, H, W, C, a.Wp, a.TR, 1)) return cudaErrorInvalidValue;
  if (!tma_map_nhwc(&DY, dy, N, P, Q, K, a.Wp, a.TR, 1)) return cudaErrorInvalidValue;
  const int smem = kWg128Stages * 8 * a.slot + 1024 + 256;
  cudaError_t err = cudaFuncSetAttribute(tc_conv_halo_wgrad128, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (err != cudaSuccess) return err;
  const int grid = a.per_job * R * a.jobs_c * a.jobs_k;
  tc_conv_halo_wgrad128<<<grid, kHaloThreads, smem, st>>>(X, DY, a);
  err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  return splitk_reduce(partial, a.per_job, R * S * C, K, dw, nullptr, 0, 1, st);
}

}  // namespace sn
