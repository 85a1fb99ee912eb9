// Probe (tools only): tcgen05.mma issue throughput on this part, operands
// resident in shared memory (no TMA), one CTA per SM, `iters` back-to-back
// MMAs (M = 128, N = n, kind::tf32 or kind::f16) into `accs` interleaved TMEM
// accumulators.  Reports clock64 cycles per MMA (max over CTAs).
#include <cstdint>

#include "tc_common.cuh"

namespace sn {
namespace {

__device__ __forceinline__ void umma_f16(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
      : "memory");
}

__global__ void __launch_bounds__(128, 1) mma_rate_kernel(int n, int kind, int iters, int accs, long long* cycles) {
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
    const uint32_t idesc = kind == 0 ? idesc_tf32(128, n, false, false)
                           : kind == 2 ? idesc_tf32(128, n, true, true)
                                     : ((1u << 4) | (0u << 7) | (0u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
                                        (static_cast<uint32_t>(128 >> 4) << 24));
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

extern "C" long long sn_probe_mma_rate(int n, int kind, int iters, int accs, int ctas) {
  long long* d = nullptr;
  cudaMalloc(&d, sizeof(long long));
  cudaMemset(d, 0, sizeof(long long));
  const int smem = 65536 + 64 + 1024;
  cudaFuncSetAttribute(sn::mma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  sn::mma_rate_kernel<<<ctas, 128, smem>>>(n, kind, iters, accs, d);
  long long h = -1;
  if (cudaDeviceSynchronize() == cudaSuccess) cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return h;
}
