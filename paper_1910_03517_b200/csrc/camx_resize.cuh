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

// One output row of a tile from two staged source rows (contiguous mosaic
// bytes: `ra` = first tap row, `rb` = second), lane l producing columns
// l + 32 j: off[j] = byte offset of the column's first tap pixel in a
// staged row (the second tap is the next 3 bytes), wt[j] = dp2a weights
// (256 - w1) | w1 << 16.  Per pixel: 3 aligned words per row + funnel shift
// (the 8 bytes from the tap pair on), channel pairs by PRMT, horizontal
// blend by dp2a, vertical by IMAD (bilerp_fx arithmetic, bit-identical).
template <int J, bool RANGE = false, bool EXACT = false>
__device__ __forceinline__ void resample_row_lanes(const uint8_t *ra, const uint8_t *rb,
                                                   const uint32_t (&off)[J],
                                                   const uint32_t (&wt)[J], uint32_t wy1,
                                                   uint8_t *orow, int out, int lane,
                                                   int ox_lo = 0, int ox_hi = 1 << 30) {
  const uint32_t wy0 = 256u - wy1;
  uint8_t *const ol = orow + 3 * lane;  // column l + 32 j at ol + 96 j (immediate offsets)
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int ox = lane + 32 * j;
    // EXACT: J = ceil(out / 32), so only the last j can run past `out`;
    // RANGE: a camera shard's owned columns [ox_lo, ox_hi)
    if (((EXACT && j < J - 1) || ox < out) && (!RANGE || (ox >= ox_lo && ox < ox_hi))) {
      const uint32_t la = off[j];
      const uint32_t sh = la * 8u;  // funnel shifts use the low 5 bits
      const uint32_t *wa = reinterpret_cast<const uint32_t *>(ra + (la & ~3u));
      const uint32_t *wb = reinterpret_cast<const uint32_t *>(rb + (la & ~3u));
      const uint32_t alo = __funnelshift_r(wa[0], wa[1], sh), ahi = __funnelshift_r(wa[1], wa[2], sh);
      const uint32_t blo = __funnelshift_r(wb[0], wb[1], sh), bhi = __funnelshift_r(wb[1], wb[2], sh);
      uint8_t *o = ol + 96 * j;
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        const uint32_t sel = 0x0030u + 0x0011u * ch;  // bytes (ch, ch + 3)
        const uint32_t v0 = __dp2a_lo(wt[j], __byte_perm(alo, ahi, sel), 0u);
        const uint32_t v1 = __dp2a_lo(wt[j], __byte_perm(blo, bhi, sel), 0u);
        o[ch] = static_cast<uint8_t>((v0 * wy0 + v1 * wy1 + 32768u) >> 16);
      }
    }
  }
}

// Per-lane column taps of resample_row_lanes (lane l: columns l + 32 j).
template <int J>
__device__ __forceinline__ void lane_taps(int lane, int out, float scale, int size, int head,
                                          uint32_t (&off)[J], uint32_t (&wt)[J], int shift = 0) {
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int ox = lane + 32 * j;
    int a = 0, c, w1 = 0;
    if (ox < out) src_coord_w(ox, scale, size, a, c, w1);
    off[j] = static_cast<uint32_t>(head + 3 * (a + shift));  // (unused when not owned)
    wt[j] = static_cast<uint32_t>(256 - w1) | (static_cast<uint32_t>(w1) << 16);
  }
}

}  // namespace camx
