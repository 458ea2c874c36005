// K4: motion mask (mask_diff) and per-window on-pixel counts (stage 4a).
//
// Reference: mask_diff (camarray core.py:191-196): on iff
// max_c |p1 - p2| > t_diff (strict); difference_plan (attention.py:89-103)
// counts on-pixels of each overlap-0 window of the mosaic (:96-100).  The
// mosaic (core.py:102-119, a full np.concatenate copy) is never
// materialised: mosaic column x maps to camera x / W, column x % W.
#include <cstdlib>

#include "camx_common.cuh"

namespace camx {

// 16 pixels (48 bytes = 3 x uint4) per thread when aligned.
__global__ void mask_diff_vec_kernel(const uint4 *a, const uint4 *b, int64_t n16, int t_diff,
                                     uint4 *mask) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n16;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint4 va[3], vb[3];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      va[u] = ld_stream_v4(a + 3 * i + u);
      vb[u] = ld_stream_v4(b + 3 * i + u);
    }
    const uint32_t *wa = reinterpret_cast<const uint32_t *>(va);
    const uint32_t *wb = reinterpret_cast<const uint32_t *>(vb);
    uint32_t dw[12];
#pragma unroll
    for (int u = 0; u < 12; ++u) dw[u] = __vabsdiffu4(wa[u], wb[u]);
    const uint8_t *d = reinterpret_cast<const uint8_t *>(dw);
    uint32_t out[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t w = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int px = q * 4 + e;
        const int m = max(max(d[3 * px], d[3 * px + 1]), d[3 * px + 2]);
        w |= (m > t_diff ? 1u : 0u) << (8 * e);
      }
      out[q] = w;
    }
    st_stream_v4(mask + i, make_uint4(out[0], out[1], out[2], out[3]));
  }
}

__global__ void mask_diff_kernel(const uint8_t *a, const uint8_t *b, int64_t lo, int64_t n,
                                 int t_diff, uint8_t *mask) {
  for (int64_t i = lo + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int m = 0;
#pragma unroll
    for (int c = 0; c < 3; ++c) m = max(m, abs(static_cast<int>(a[3 * i + c]) - b[3 * i + c]));
    mask[i] = m > t_diff ? 1 : 0;
  }
}

// Any channel count (mask_diff's max over axis 2 of an (H, W, C) array).
__global__ void mask_diff_channels_kernel(const uint8_t *a, const uint8_t *b, int64_t n,
                                          int channels, int t_diff, uint8_t *mask) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int m = 0;
    for (int c = 0; c < channels; ++c)
      m = max(m, abs(static_cast<int>(a[channels * i + c]) - b[channels * i + c]));
    mask[i] = m > t_diff ? 1 : 0;
  }
}

// One CTA per (window, row slab).  Counts are exact int64 via one atomic
// per CTA.
struct CountParams {
  const uint8_t *mask, *cur, *prev;
  int32_t t_diff, n_cams, H, W, size, n_windows, slab;
  const int32_t *windows;
  int64_t *counts;
};

template <bool FUSED>
__global__ void __launch_bounds__(256) window_count_kernel(const CountParams p) {
  const int win = blockIdx.y;
  const int x0 = p.windows[2 * win], y0 = p.windows[2 * win + 1];
  const int ys = y0 + blockIdx.x * p.slab;
  const int ye = min(min(y0 + p.size, ys + p.slab), p.H);
  const int total_w = p.n_cams * p.W;
  const int64_t img_px = static_cast<int64_t>(p.H) * p.W;
  unsigned long long local = 0;
  // column-outer: one camera/column split per column, then the slab's rows
  // (consecutive threads still read consecutive columns of a row)
  for (int dx = threadIdx.x; dx < p.size; dx += blockDim.x) {
    const int x = x0 + dx;
    if (x < 0 || x >= total_w) continue;
    const int cam = x / p.W;
    const int col = x - cam * p.W;
    for (int y = ys; y < ye; ++y) {
      const int64_t pix = cam * img_px + static_cast<int64_t>(y) * p.W + col;
      bool on;
      if (FUSED) {
        int m = 0;
#pragma unroll
        for (int c = 0; c < 3; ++c)
          m = max(m, abs(static_cast<int>(p.cur[3 * pix + c]) - p.prev[3 * pix + c]));
        on = m > p.t_diff;
      } else {
        on = p.mask[pix] != 0;
      }
      local += on ? 1 : 0;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  __shared__ unsigned long long part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += part[w];
    atomicAdd(reinterpret_cast<unsigned long long *>(p.counts + win), t);
  }
}

// Quad-vectorised counts (W % 4 == 0, 4-byte aligned frames / mask): a
// thread owns fixed 4-pixel column groups of the window (a group never
// straddles a camera since W % 4 == 0; 12-byte RGB loads as 3 words, the
// per-pixel max |diff| by SIMD byte ops) and walks the slab's rows; the
// window's unaligned first / last pixels go through the scalar test.
__device__ __forceinline__ uint32_t quad_on(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t p0,
                                            uint32_t p1, uint32_t p2, uint32_t tq) {
  const uint32_t d0 = __vabsdiffu4(c0, p0), d1 = __vabsdiffu4(c1, p1), d2 = __vabsdiffu4(c2, p2);
  // channel c of pixels 0..3 (bytes r g b r | g b r g | b r g b)
  const uint32_t x = __byte_perm(__byte_perm(d0, d1, 0x0630u), d2, 0x5210u);
  const uint32_t y = __byte_perm(__byte_perm(d0, d1, 0x0741u), d2, 0x6210u);
  const uint32_t z = __byte_perm(__byte_perm(d0, d1, 0x0052u), d2, 0x7410u);
  const uint32_t m = __vmaxu4(__vmaxu4(x, y), z);
  return __vcmpgtu4(m, tq);  // 0xFF per pixel on
}

template <bool FUSED>
__global__ void __launch_bounds__(256) window_count_quad_kernel(const CountParams p) {
  const int win = blockIdx.y;
  const int x0 = p.windows[2 * win], y0 = p.windows[2 * win + 1];
  const int ys = y0 + blockIdx.x * p.slab;
  const int ye = min(min(y0 + p.size, ys + p.slab), p.H);
  const int total_w = p.n_cams * p.W;
  const int xa = max(x0, 0), xb = min(x0 + p.size, total_w);  // columns on this mosaic
  const int qa = (xa + 3) & ~3, qb = xb & ~3;                  // whole quads [qa, qb)
  const int64_t img_px = static_cast<int64_t>(p.H) * p.W;
  const uint32_t tq = p.t_diff < 0 ? 0u : static_cast<uint32_t>(min(p.t_diff, 255)) * 0x01010101u;
  unsigned long long local = 0;
  if (ys < ye && xa < xb) {
    const int nquads = qb > qa ? (qb - qa) >> 2 : 0;
    for (int q = threadIdx.x; q < nquads; q += blockDim.x) {
      const int x = qa + 4 * q;
      const int cam = x / p.W;
      const int64_t pix0 = cam * img_px + static_cast<int64_t>(ys) * p.W + (x - cam * p.W);
      for (int y = ys; y < ye; ++y) {
        const int64_t pix = pix0 + static_cast<int64_t>(y - ys) * p.W;
        uint32_t on;
        if (FUSED) {
          const uint32_t *c = reinterpret_cast<const uint32_t *>(p.cur + 3 * pix);
          const uint32_t *r = reinterpret_cast<const uint32_t *>(p.prev + 3 * pix);
          on = p.t_diff < 0 ? 0xFFFFFFFFu : quad_on(c[0], c[1], c[2], r[0], r[1], r[2], tq);
        } else {
          on = __vcmpne4(*reinterpret_cast<const uint32_t *>(p.mask + pix), 0u);
        }
        local += __popc(on) >> 3;
      }
    }
    // unaligned edge columns [xa, qa) and [max(qb, qa), xb): scalar
    const int ne0 = min(qa, xb) - xa, ne1 = xb - max(qb, qa);
    const int ne = max(ne0, 0) + max(ne1, 0);
    for (int i = threadIdx.x; i < ne * (ye - ys); i += blockDim.x) {
      const int e = i % ne, y = ys + i / ne;
      const int x = e < ne0 ? xa + e : max(qb, qa) + (e - max(ne0, 0));
      const int cam = x / p.W;
      const int64_t pix = cam * img_px + static_cast<int64_t>(y) * p.W + (x - cam * p.W);
      bool hit;
      if (FUSED) {
        int m = 0;
#pragma unroll
        for (int c = 0; c < 3; ++c)
          m = max(m, abs(static_cast<int>(p.cur[3 * pix + c]) - p.prev[3 * pix + c]));
        hit = m > p.t_diff;
      } else {
        hit = p.mask[pix] != 0;
      }
      local += hit ? 1 : 0;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  __shared__ unsigned long long part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += part[w];
    atomicAdd(reinterpret_cast<unsigned long long *>(p.counts + win), t);
  }
}

// One pass over the mosaic (W % 16 == 0, 16-byte aligned frames / mask): a
// CTA owns a 256-px x 32-row tile, a thread one 16-pixel group of two rows
// (3 x 16-byte loads per frame and row, or 16 mask bytes, all issued before
// the window scan), so every pixel is read once however many windows
// overlap it - the per-window kernels above read the overlap rows of the
// sliding plan twice.  The CTA collects the windows that intersect its tile
// (window list in chunks of 256), and each thread adds popc(on-flags & the
// window's column mask) for every window whose rows contain its row; one
// int64 atomic per (CTA, window).  Config-2 difference plan (36 windows):
// 36.9 us per array-frame vs 53.3 us for the per-window quad kernel.
#ifndef CAMX_K4_TILE_ROWS
#define CAMX_K4_TILE_ROWS 2
#endif
constexpr int kTileRows = CAMX_K4_TILE_ROWS;  // rows per thread
constexpr int kTileW = 256, kTileH = 16 * kTileRows, kTileSlots = 8;

__device__ __forceinline__ uint32_t group16_on(const uint4 *c, const uint4 *r, uint32_t tq) {
  const uint32_t *wc = reinterpret_cast<const uint32_t *>(c);
  const uint32_t *wr = reinterpret_cast<const uint32_t *>(r);
  uint32_t bits = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t on = quad_on(wc[3 * q], wc[3 * q + 1], wc[3 * q + 2], wr[3 * q], wr[3 * q + 1],
                                wr[3 * q + 2], tq);  // 0xFF per pixel
    bits |= ((on & 1u) | ((on >> 7) & 2u) | ((on >> 14) & 4u) | ((on >> 21) & 8u)) << (4 * q);
  }
  return bits;
}

template <bool FUSED>
__global__ void __launch_bounds__(256) window_count_tile_kernel(const CountParams p) {
  __shared__ int2 wins[256];
  __shared__ int widx[256];
  __shared__ int nw;
  __shared__ unsigned long long acc[kTileSlots];
  const int total_w = p.n_cams * p.W;
  const int tx0 = blockIdx.x * kTileW, ty0 = blockIdx.y * kTileH;
  const int g = threadIdx.x & 15, r = threadIdx.x >> 4;
  const int x = tx0 + 16 * g;
  const uint32_t tq = p.t_diff < 0 ? 0u : static_cast<uint32_t>(min(p.t_diff, 255)) * 0x01010101u;
  // the pixels first (every thread: kTileRows rows of its 16-pixel group),
  // so the loads are in flight while the CTA scans the window list
  uint32_t flags[kTileRows];
  {
    uint4 c[kTileRows][3], pv[kTileRows][3];
    uint4 mk[kTileRows];
    const int cam = x / p.W;
    const int64_t base = cam * (static_cast<int64_t>(p.H) * p.W) + (x - cam * p.W);
#pragma unroll
    for (int i = 0; i < kTileRows; ++i) {
      const int y = ty0 + r + 16 * i;
      if (x < total_w && y < p.H) {
        const int64_t pix = base + static_cast<int64_t>(y) * p.W;
        if (FUSED) {
#pragma unroll
          for (int u = 0; u < 3; ++u) {
            c[i][u] = ld_stream_v4(p.cur + 3 * pix + 16 * u);
            pv[i][u] = ld_stream_v4(p.prev + 3 * pix + 16 * u);
          }
        } else {
          mk[i] = ld_stream_v4(p.mask + pix);
        }
      } else {
        if (FUSED) {
#pragma unroll
          for (int u = 0; u < 3; ++u) c[i][u] = pv[i][u] = make_uint4(0, 0, 0, 0);
        } else {
          mk[i] = make_uint4(0, 0, 0, 0);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < kTileRows; ++i) {
      const int y = ty0 + r + 16 * i;
      uint32_t bits = 0;
      if (FUSED) {
        bits = p.t_diff < 0 ? 0xFFFFu : group16_on(c[i], pv[i], tq);
      } else {
        const uint32_t mw[4] = {mk[i].x, mk[i].y, mk[i].z, mk[i].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t on = __vcmpne4(mw[q], 0u);
          bits |= ((on & 1u) | ((on >> 7) & 2u) | ((on >> 14) & 4u) | ((on >> 21) & 8u)) << (4 * q);
        }
      }
      flags[i] = (x < total_w && y < p.H) ? bits : 0u;
    }
  }
  for (int w0 = 0; w0 < p.n_windows; w0 += 256) {
    if (threadIdx.x == 0) nw = 0;
    __syncthreads();
    {
      const int w = w0 + threadIdx.x;
      if (w < p.n_windows) {
        const int wx = p.windows[2 * w], wy = p.windows[2 * w + 1];
        if (wx < tx0 + kTileW && wx + p.size > tx0 && wy < ty0 + kTileH && wy + p.size > ty0) {
          const int k = atomicAdd(&nw, 1);
          wins[k] = make_int2(wx, wy);
          widx[k] = w;
        }
      }
    }
    __syncthreads();
    const int n = nw;  // CTA-uniform
    for (int s0 = 0; s0 < n; s0 += kTileSlots) {
      if (threadIdx.x < kTileSlots) acc[threadIdx.x] = 0;
      __syncthreads();
      const int ns = min(kTileSlots, n - s0);
#pragma unroll
      for (int k = 0; k < kTileSlots; ++k) {
        if (k >= ns) break;
        const int2 wv = wins[s0 + k];
        const int lo = min(max(wv.x - x, 0), 16), hi = min(max(wv.x + p.size - x, 0), 16);
        const uint32_t m = ((1u << hi) - 1u) & ~((1u << lo) - 1u);
        uint32_t cnt = 0;
#pragma unroll
        for (int i = 0; i < kTileRows; ++i) {
          const int y = ty0 + r + 16 * i;
          if (y >= wv.y && y < wv.y + p.size) cnt += __popc(flags[i] & m);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&acc[k], static_cast<unsigned long long>(cnt));
      }
      __syncthreads();
      if (threadIdx.x < ns && acc[threadIdx.x])
        atomicAdd(reinterpret_cast<unsigned long long *>(p.counts + widx[s0 + threadIdx.x]),
                  acc[threadIdx.x]);
      __syncthreads();
    }
  }
}

}  // namespace camx

using namespace camx;

extern "C" int camx_mask_diff(const uint8_t *a, const uint8_t *b, int64_t n_pixels, int32_t t_diff,
                              uint8_t *mask_out, void *stream) {
  if (n_pixels < 0 || !a || !b || !mask_out) return CAMX_EINVAL;
  if (n_pixels == 0) return CAMX_OK;
  cudaStream_t s = as_stream(stream);
  int64_t done = 0;
  const bool aligned = (reinterpret_cast<uintptr_t>(a) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(b) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(mask_out) % 16 == 0);
  if (aligned && n_pixels >= 16) {
    const int64_t n16 = n_pixels / 16;
    int64_t blocks = (n16 + 255) / 256;
    const int64_t cap = static_cast<int64_t>(sm_count()) * 8;
    if (blocks > cap) blocks = cap;
    mask_diff_vec_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(
        reinterpret_cast<const uint4 *>(a), reinterpret_cast<const uint4 *>(b), n16, t_diff,
        reinterpret_cast<uint4 *>(mask_out));
    done = n16 * 16;
  }
  if (done < n_pixels) {
    const int64_t rest = n_pixels - done;
    int64_t blocks = (rest + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    mask_diff_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(a, b, done, n_pixels, t_diff,
                                                                    mask_out);
  }
  return launch_status();
}

extern "C" int camx_mask_diff_channels(const uint8_t *a, const uint8_t *b, int64_t n_pixels,
                                       int32_t channels, int32_t t_diff, uint8_t *mask_out,
                                       void *stream) {
  if (n_pixels < 0 || channels < 1 || !a || !b || !mask_out) return CAMX_EINVAL;
  if (channels == 3) return camx_mask_diff(a, b, n_pixels, t_diff, mask_out, stream);
  if (n_pixels == 0) return CAMX_OK;
  int64_t blocks = (n_pixels + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  mask_diff_channels_kernel<<<static_cast<unsigned>(blocks), 256, 0, as_stream(stream)>>>(
      a, b, n_pixels, channels, t_diff, mask_out);
  return launch_status();
}

extern "C" int camx_window_counts(const uint8_t *mask, const uint8_t *cur, const uint8_t *prev,
                                  int32_t t_diff, int32_t n_cams, int32_t height, int32_t width,
                                  const int32_t *windows, int32_t n_windows, int32_t size,
                                  int64_t *counts_out, void *stream) {
  if (n_cams < 1 || height < 1 || width < 1 || size < 1 || n_windows < 0 || !counts_out)
    return CAMX_EINVAL;
  if ((mask == nullptr) == (cur == nullptr || prev == nullptr)) return CAMX_EINVAL;
  // windows may extend past this (sharded) mosaic: columns outside it are
  // skipped, so a rank counts only its own cameras' share
  if (size > height) return CAMX_EINVAL;
  cudaStream_t s = as_stream(stream);
  if (n_windows == 0) return CAMX_OK;
  if (!windows) return CAMX_EINVAL;
  cudaError_t e = cudaMemsetAsync(counts_out, 0, sizeof(int64_t) * n_windows, s);
  if (e != cudaSuccess) return static_cast<int>(e);
  CountParams p{};
  p.mask = mask;
  p.cur = cur;
  p.prev = prev;
  p.t_diff = t_diff;
  p.n_cams = n_cams;
  p.H = height;
  p.W = width;
  p.size = size;
  p.n_windows = n_windows;
  p.windows = windows;
  p.counts = counts_out;
  p.slab = 32;
  auto al4 = [](const void *x) { return reinterpret_cast<uintptr_t>(x) % 4 == 0; };
  auto al16 = [](const void *x) { return reinterpret_cast<uintptr_t>(x) % 16 == 0; };
  const bool quad = width % 4 == 0 && (mask ? al4(mask) : (al4(cur) && al4(prev)));
  if (width % 16 == 0 && (mask ? al16(mask) : (al16(cur) && al16(prev)))) {
    const int64_t total_w = static_cast<int64_t>(n_cams) * width;
    const dim3 grid(static_cast<unsigned>((total_w + kTileW - 1) / kTileW),
                    static_cast<unsigned>((height + kTileH - 1) / kTileH));
    if (mask)
      window_count_tile_kernel<false><<<grid, 256, 0, s>>>(p);
    else
      window_count_tile_kernel<true><<<grid, 256, 0, s>>>(p);
    return launch_status();
  }
  // windows ride on gridDim.y (<= 65535): chunk longer lists
  for (int32_t w0 = 0; w0 < n_windows; w0 += 65535) {
    CountParams pc = p;
    pc.windows = windows + 2 * static_cast<int64_t>(w0);
    pc.counts = counts_out + w0;
    pc.n_windows = min(65535, n_windows - w0);
    dim3 grid((size + p.slab - 1) / p.slab, pc.n_windows);
    if (quad) {
      if (mask)
        window_count_quad_kernel<false><<<grid, 256, 0, s>>>(pc);
      else
        window_count_quad_kernel<true><<<grid, 256, 0, s>>>(pc);
    } else if (mask) {
      window_count_kernel<false><<<grid, 256, 0, s>>>(pc);
    } else {
      window_count_kernel<true><<<grid, 256, 0, s>>>(pc);
    }
    const int st = launch_status();
    if (st != CAMX_OK) return st;
  }
  return CAMX_OK;
}
