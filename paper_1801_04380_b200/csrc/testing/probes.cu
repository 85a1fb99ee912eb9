// Test-only probes (libsntest.so, never linked into the product libsnexec.so):
// driver acceptance of overlapping TMA windows, and UMMA descriptor start
// addresses shifted inside a SWIZZLE_128B tile (tools/umma_shift_probe.py,
// tests/test_gpu_kernels.py).
#include <cudaTypedefs.h>

#include "../kernels/tc_common.cuh"
#include "../kernels/tma_host.hpp"

namespace sn {
// Probe: does the driver accept a tiled map whose row stride (32 B) is smaller
// than its inner extent (128 B), i.e. overlapping sliding windows?
int tma_probe_overlap(const float* base) {
  if (!tma_encoders_ok()) return -1;
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return -1;
  enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap m;
  cuuint64_t dims[4] = {32, 112, 224, 2};
  cuuint64_t strides[3] = {32, 224 * 16, 224 * 224 * 16};
  cuuint32_t box[4] = {32, 128, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return static_cast<int>(enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
}

// ---------------------------------------------------------------------------
// Probe (tests only): does a UMMA smem descriptor whose start address is
// shifted by `shift` 128-byte rows inside a TMA-written SWIZZLE_128B tile read
// the shifted matrix, with or without the descriptor's base-offset field?
//   mn = 0: A K-major [256 rows][32 k];    D = A[shift : shift+128] . B^T
//   mn = 1: A MN-major [40 k][128 m];      D[m][n] = sum_k A[k + shift][m] B[n][k]
// B: K-major [64][32].  D: [128][64].
namespace {
__global__ void __launch_bounds__(128, 1) umma_shift_probe(const __grid_constant__ CUtensorMap tA,
                                                           const __grid_constant__ CUtensorMap tB, float* D, int mn,
                                                           int shift, int base_off) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                 // 32 KB (K-major) or 4 x 5 KB (MN-major)
  uint8_t* sB = smem + 32768;         // 8 KB
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 32768 + 8192);
  uint64_t* mbar = bar + 1;
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(mbar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(slot, 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    if (!mn) {
      mbar_arrive_expect_tx(bar, 32768 + 8192);
      tma_load_2d(smem_u32(sA), &tA, bar, 0, 0);
    } else {
      mbar_arrive_expect_tx(bar, 4 * 5120 + 8192);
      for (int j = 0; j < 4; ++j) tma_load_2d(smem_u32(sA + j * 5120), &tA, bar, 32 * j, 0);
    }
    tma_load_2d(smem_u32(sB), &tB, bar, 0, 0);
    mbar_wait(bar, 0);
    tc_fence_after();
    const uint32_t idesc = idesc_tf32(128, 64, mn != 0, false);
    for (int kk = 0; kk < 4; ++kk) {
      uint64_t ad;
      uint32_t start;
      if (!mn) {
        start = smem_u32(sA) + shift * 128 + kk * 32;
        ad = umma_desc(start, 16, 1024, kLayoutSW128);
      } else {
        start = smem_u32(sA) + shift * 128 + kk * 1024;
        ad = umma_desc(start, 5120, 512, kLayoutSW128Base32);
      }
      if (base_off) ad |= static_cast<uint64_t>((start >> 7) & 7u) << 49;
      const uint64_t bd = umma_desc(smem_u32(sB) + kk * 32, 16, 1024, kLayoutSW128);
      umma_tf32(tmem, ad, bd, idesc, kk ? 1u : 0u);
    }
    umma_commit(mbar);
  }
  __syncwarp();
  mbar_wait(mbar, 0);
  tc_fence_after();
  for (int c = 0; c < 64; c += 32) {
    float v[32];
    tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, v);
    for (int j = 0; j < 32; ++j) D[(warp * 32 + lane) * 64 + c + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 64);
}
}  // namespace

int umma_shift_probe_run(const float* A, const float* B, float* D, int mn, int shift, int base_off) {
  if (!tma_encoders_ok()) return 1;
  CUtensorMap tA, tB;
  bool ok;
  if (!mn) {
    ok = tma_map_2d(&tA, A, 256, 32, 256, 0);
  } else {
    ok = tma_map_2d(&tA, A, 40, 128, 40, 1);
  }
  ok = ok && tma_map_2d(&tB, B, 64, 32, 64, 0);
  if (!ok) return 2;
  const int smem = 32768 + 8192 + 64 + 1024;
  cudaFuncSetAttribute(umma_shift_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  umma_shift_probe<<<1, 128, smem>>>(tA, tB, D, mn, shift, base_off);
  if (cudaGetLastError() != cudaSuccess) return 3;
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 4;
}
}  // namespace sn
