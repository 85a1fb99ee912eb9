// BatchNorm element math shared by the layer kernels (layers.cu) and the
// fused stem weight gradient (conv_tma.cu).  Explicit-rounding intrinsics:
// the forward, its replays, the ReLU mask recomputed in the backward and a
// dx recomputed inside another kernel are bit-identical (no compiler FMA
// contraction choices).
#pragma once

namespace sn {

__device__ __forceinline__ float bn_xhat(float x, float m, float is) { return __fmul_rn(__fsub_rn(x, m), is); }
__device__ __forceinline__ float bn_affine(float x, float m, float is, float g, float b) {
  return __fmaf_rn(bn_xhat(x, m, is), g, b);
}
// dx = gamma * invstd * (g - sum(g)/m - xhat * sum(g xhat)/m) with gs = gamma * invstd,
// k1 = sum(g)/m, k2 = sum(g xhat)/m (g already ReLU-masked)
__device__ __forceinline__ float bn_dx_elem(float g, float x, float m, float is, float gs, float k1, float k2) {
  return __fmul_rn(gs, __fsub_rn(__fsub_rn(g, k1), __fmul_rn(bn_xhat(x, m, is), k2)));
}

}  // namespace sn
