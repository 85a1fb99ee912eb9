// Host-side tensor-map encoders shared by the TMA kernels (conv_tma.cu,
// conv_halo.cu).  The driver entry points are fetched at run time (no -lcuda).
#pragma once
#include <cuda.h>

#include <cstdint>

namespace sn {

bool tma_encoders_ok();
// NHWC [N][H][W][C] fp32 as a 4-D tiled map, box {32 channels, box_w, box_h, 1};
// out-of-range coordinates (negative included) read as zeros / are clipped on store.
// swz: 0 = SWIZZLE_128B, 1 = SWIZZLE_128B_ATOM_32B.
// es > 1: element stride es along W and H (box_w x box_h elements land, every es-th pixel).
bool tma_map_nhwc(CUtensorMap* m, const float* base, int N, int H, int W, int C, int box_w, int box_h, int swz,
                  int es = 1);
// Row-major [rows][cols] fp32, box {32 cols, box_rows rows}.
bool tma_map_2d(CUtensorMap* m, const float* base, int64_t rows, int64_t cols, int box_rows, int swz);

}  // namespace sn
