// Bilinear resize arithmetic shared by the tile kernels (K5) and the fused
// correct+tile kernel.  Builder-defined semantics (the reference only crops,
// detect.py:297-300; oracle/camarray_oracle.py: resize_bilinear): half-pixel
// centres, source coordinate (i + 0.5) * (S / out) - 0.5 in float32, clamped
// to [0, S-1]; taps i0 = floor, i1 = min(i0 + 1, S - 1); 8-bit fixed-point
// weights; exact integer blend, round half up.
#pragma once

#include "camx_common.cuh"

namespace camx {

__device__ __forceinline__ void src_coord(int i, float scale, int S, int &i0, int &i1, float &f) {
  float s = __fsub_rn(__fmul_rn(__fadd_rn(static_cast<float>(i), 0.5f), scale), 0.5f);
  s = fminf(fmaxf(s, 0.0f), static_cast<float>(S - 1));
  i0 = static_cast<int>(floorf(s));
  i1 = min(i0 + 1, S - 1);
  f = __fsub_rn(s, static_cast<float>(i0));
}

// 8-bit fixed-point weight of the second tap: rint(256 * f), f in [0, 1)
// (f * 256 is exact; rint is half-even like np.rint).
__device__ __forceinline__ void src_coord_w(int i, float scale, int S, int &i0, int &i1, int &w1) {
  float f;
  src_coord(i, scale, S, i0, i1, f);
  w1 = __float2int_rn(__fmul_rn(f, 256.0f));
}

// h = a*(256-wx) + b*wx per source row, out = (h0*(256-wy) + h1*wy + 2^15) >> 16
// (exact integer arithmetic; round half up; no clamp needed: <= 255).
__device__ __forceinline__ uint32_t bilerp_fx(uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                              uint32_t wx, uint32_t wy) {
  const uint32_t h0 = a * (256u - wx) + b * wx;
  const uint32_t h1 = c * (256u - wx) + d * wx;
  return (h0 * (256u - wy) + h1 * wy + 32768u) >> 16;
}

}  // namespace camx
