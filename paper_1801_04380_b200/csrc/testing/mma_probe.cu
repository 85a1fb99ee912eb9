// Probe (tools only): tcgen05.mma issue throughput on this part, operands
// resident in shared memory (no TMA), one CTA per SM, `iters` back-to-back
// MMAs (M = 128, N = n, kind::tf32 or kind::f16) into `accs` interleaved TMEM
// accumulators.  Reports clock64 cycles per MMA (max over CTAs).
#include <cstdint>

#include "../kernels/tc_common.cuh"

namespace sn {
namespace {

__device__ __forceinline__ void umma_f16(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
      : "memory");
}

__global__ void __launch_bounds__(128, 1) mma_rate_kernel(int m, int n, int kind, int iters, int accs,
                                                          long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.001f * (i % 7);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(slot, 512);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 16384);
    const uint32_t idesc = kind == 0 ? idesc_tf32(m, n, false, false)
                           : kind == 2 ? idesc_tf32(m, n, true, true)
                                     : ((1u << 4) | (0u << 7) | (0u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
                                        (static_cast<uint32_t>(m >> 4) << 24));
    uint64_t ad[4], bd[4];
    for (int kk = 0; kk < 4; ++kk) {
      if (kind == 2) {  // MN-major SW128_BASE32B, 32-row boxes (as the wgrad kernels)
        ad[kk] = umma_desc(a0 + kk * 1024, 4096, 512, kLayoutSW128Base32);
        bd[kk] = umma_desc(b0 + kk * 1024, 4096, 512, kLayoutSW128Base32);
      } else {
        ad[kk] = umma_desc(a0 + kk * 32, 16, 1024, kLayoutSW128);
        bd[kk] = umma_desc(b0 + kk * 32, 16, 1024, kLayoutSW128);
      }
    }
    const uint32_t d1 = tmem + static_cast<uint32_t>((accs > 1 ? 1 : 0) * n);
    const long long t0 = clock64();
    // 8 MMAs per iteration, descriptors precomputed: the loop is issue-only
    for (int i = 0; i < iters; i += 8) {
      if (kind != 1) {
#pragma unroll
        for (int u = 0; u < 8; ++u) umma_tf32((u & 1) ? d1 : tmem, ad[u & 3], bd[u & 3], idesc, 1u);
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) umma_f16((u & 1) ? d1 : tmem, ad[u & 3], bd[u & 3], idesc, 1u);
      }
    }
    umma_commit(bar);
    mbar_wait(bar, 0);
    const long long t1 = clock64();
    atomicMax(reinterpret_cast<unsigned long long*>(cycles), static_cast<unsigned long long>(t1 - t0));
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

}  // namespace
}  // namespace sn

extern "C" long long sn_probe_mma_rate_m(int m, int n, int kind, int iters, int accs, int ctas) {
  long long* d = nullptr;
  cudaMalloc(&d, sizeof(long long));
  cudaMemset(d, 0, sizeof(long long));
  const int smem = 65536 + 64 + 1024;
  cudaFuncSetAttribute(sn::mma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  sn::mma_rate_kernel<<<ctas, 128, smem>>>(m, n, kind, iters, accs, d);
  long long h = -1;
  if (cudaDeviceSynchronize() == cudaSuccess) cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return h;
}

extern "C" long long sn_probe_mma_rate(int n, int kind, int iters, int accs, int ctas) {
  return sn_probe_mma_rate_m(128, n, kind, iters, accs, ctas);
}

// TMEM layout of an M = 64 tf32 MMA (cta_group::1): A [64][32] and B [64][32]
// K-major SW128 in smem (written by threads with the absolute-address swizzle),
// D -> TMEM at lane offset `lane0` (0 or 64), column 0; all 128 lanes x 64
// columns are read back into out[128][64] (NaN-initialised TMEM cells stay as
// written by a previous tcgen05.st of NaN).
namespace sn {
namespace {
__global__ void __launch_bounds__(128, 1) m64_layout_kernel(const float* A, const float* B, float* out, int lane0) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;          // 64 rows x 128 B
  uint8_t* sB = smem + 8192;   // 64 rows x 128 B
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) {
    const int r = i / 32, k = i % 32;
    const uint32_t off = sw128_off(r, k / 4) + (k % 4) * 4;
    *reinterpret_cast<float*>(sA + off) = A[i];
    *reinterpret_cast<float*>(sB + off) = B[i];
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(slot, 64);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  // fill TMEM with NaN so untouched cells are recognisable
  {
    uint32_t nanv = 0x7fc00000u;
    for (int c = 0; c < 64; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c),
                   "r"(nanv)
                   : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_tf32(64, 64, false, false);
    for (int kk = 0; kk < 4; ++kk)
      umma_tf32(tmem + (static_cast<uint32_t>(lane0) << 16), umma_desc(smem_u32(sA) + kk * 32, 16, 1024, kLayoutSW128),
                umma_desc(smem_u32(sB) + kk * 32, 16, 1024, kLayoutSW128), idesc, kk ? 1u : 0u);
    umma_commit(bar);
  }
  __syncwarp();
  mbar_wait(bar, 0);
  tc_fence_after();
  for (int c = 0; c < 64; c += 32) {
    float v[32];
    tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, v);
    for (int j = 0; j < 32; ++j) out[(warp * 32 + lane) * 64 + c + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 64);
}
}  // namespace
}  // namespace sn

extern "C" int sn_probe_m64_layout(const float* A, const float* B, float* out, int lane0) {
  const int smem = 16384 + 64 + 1024;
  cudaFuncSetAttribute(sn::m64_layout_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  sn::m64_layout_kernel<<<1, 128, smem>>>(A, B, out, lane0);
  if (cudaGetLastError() != cudaSuccess) return 3;
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 4;
}
