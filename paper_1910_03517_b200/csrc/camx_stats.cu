// K1: seam band statistics (stage 1) + float moments.
//
// Reference: band_stats (camarray exposure.py:152-185) over the band of
// `band_width` columns at each seam edge (LEFT side = last bw columns,
// RIGHT side = first bw columns, :163-168), per row block of block_bounds
// (:123-135), with an optional exclusion mask (:178-180).  OBJECT_REMOVAL
// builds that mask with mask_diff (core.py:191-196) against the previous
// frame (exposure.py:313-316); here it is fused: only band pixels are
// diffed.
//
// Output is exact integer statistics (count, sum, sum of squares per
// channel) from which mean / population std follow; the optional 256-bin
// histograms are an exact sufficient statistic of the same pixel sets.
//
// Decomposition: one warp (a 32-thread CTA) per (image, side, block) unit,
// scheduled dynamically (CAMX_K1_WARPS warps per unit is a build knob).
// When the band is 4-pixel aligned (W % 4 == 0, bw % 4 == 0) a lane reads
// pixel quads as three 32-bit words (12 bytes = r g b r g b r g b r g b,
// so the channel of every byte is fixed), U quads per step so U*3 loads are
// in flight per lane, and the channel sums / sums of squares come from
// dp4a with constant byte masks; otherwise per-pixel byte loads.
// Histograms: one shared-memory atomic per (kept pixel, channel) into the
// warp's 3 x 256 bins.  Reductions: warp shuffles only (32-bit halves when
// a unit cannot overflow them).
#include <algorithm>

#include <cstdlib>

#include "camx_common.cuh"

namespace camx {

struct StatsParams {
  const uint8_t *img;
  const uint8_t *prev;   // mode 2
  int64_t prev_seq;      // mode 2 over a batch: images >= prev_seq diff against
                         // image - prev_seq (the previous array-frame), the
                         // first prev_seq against `prev`; 0 = always `prev`
  const uint8_t *mask;   // mode 1
  int64_t img_bytes;
  int64_t mask_bytes;    // H * W
  int64_t n_units;       // n_images * 2 * K
  int32_t H, W, bw, K, bh, t_diff;
  camx_band_stat *out;
  uint32_t *hist;        // optional
};

#ifndef CAMX_K1_MINB
#define CAMX_K1_MINB 32  // one-warp CTAs: 64 registers, every warp slot of an SM usable
#endif
#ifndef CAMX_K1_WARPS
#define CAMX_K1_WARPS 1
#endif
// warps per (image, side, block) unit = per CTA.  One: every warp streams
// its own band blocks with shuffle-only reductions and no CTA barrier
// (K1 + histograms 49 -> 39 us, OBJECT_REMOVAL 53 -> 46 us per 30 config-2
// frames vs four warps per block; tools/k1_probe.py)
constexpr int kStatsWarps = CAMX_K1_WARPS;
#ifndef CAMX_K1_QB_REMOVAL
#define CAMX_K1_QB_REMOVAL 3
#endif
#ifndef CAMX_K1_QB
#define CAMX_K1_QB 6
#endif
constexpr int kQuadBatchMax = CAMX_K1_QB;
#ifndef CAMX_K1_G16
#define CAMX_K1_G16 2
#endif
#ifndef CAMX_K1_G16_REMOVAL
#define CAMX_K1_G16_REMOVAL 1
#endif
constexpr int kG16Groups = CAMX_K1_G16, kG16GroupsRemoval = CAMX_K1_G16_REMOVAL;
// Histograms: per-warp [3][256] uint32 bins in shared memory, one atomic
// per (kept pixel, channel).  (A band block is only 3,072 pixels: per-lane
// private byte counters - conflict-free, but a 768-word flush and re-zero
// per lane per block - measured ~4x slower; profiles/r01/SUMMARY.md.)
constexpr int kHistWords = 3 * 256;
// dp4a byte selectors of channel c in word k of a 12-byte pixel quad
// (bytes r g b r | g b r g | b r g b)
//   r: w0 b0,b3  w1 b2  w2 b1;  g: w0 b1  w1 b0,b3  w2 b2;  b: w0 b2  w1 b1  w2 b0,b3
__host__ __device__ constexpr uint32_t quad_sel(int c, int k) {
  return ((c + 3 - k) % 3 == 0) ? 0x01000001u : ((c + 3 - k) % 3 == 1) ? 0x00000100u : 0x00010000u;
}  // a standard 32-px x 96-row band unit: one batch

__device__ __forceinline__ uint64_t warp_sum_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct Acc {
  uint64_t raw_s[3], raw_q[3], val_s[3], val_q[3];
  uint32_t nvalid;
};

template <bool HIST>
__device__ __forceinline__ void add_pixel(Acc &a, uint32_t *cnt, int lane, uint32_t r, uint32_t g,
                                          uint32_t b, bool excluded) {
  const uint32_t v[3] = {r, g, b};
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    a.raw_s[c] += v[c];
    a.raw_q[c] += v[c] * v[c];
  }
  if (!excluded) {
    a.nvalid += 1;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      if (HIST) {
        atomicAdd(cnt + c * 256 + v[c], 1u);
      } else {
        a.val_s[c] += v[c];
        a.val_q[c] += v[c] * v[c];
      }
    }
  }
}


// Excluded-pixel flags of a quad (bit e set = pixel e excluded).
template <int MASKMODE>
__device__ __forceinline__ uint32_t quad_exclusion(const StatsParams &p, const uint32_t w[3],
                                                   const uint32_t pw[3], uint32_t mword) {
  if (MASKMODE == 1) {
    // mask bytes nonzero = excluded
    const uint32_t g = __vcmpne4(mword, 0u);  // 0xFF where excluded
    return (g & 0x1u) | ((g >> 7) & 0x2u) | ((g >> 14) & 0x4u) | ((g >> 21) & 0x8u);
  } else if (MASKMODE == 2) {
    const uint32_t d0 = __vabsdiffu4(w[0], pw[0]);
    const uint32_t d1 = __vabsdiffu4(w[1], pw[1]);
    const uint32_t d2 = __vabsdiffu4(w[2], pw[2]);
    // per pixel the three channel diffs: p0 = d0.b0 d0.b1 d0.b2, p1 = d0.b3 d1.b0 d1.b1,
    // p2 = d1.b2 d1.b3 d2.b0, p3 = d2.b1 d2.b2 d2.b3
    const uint32_t x = __byte_perm(__byte_perm(d0, d1, 0x0630u), d2, 0x5210u);  // c0 of p0..p3
    const uint32_t y = __byte_perm(__byte_perm(d0, d1, 0x0741u), d2, 0x6210u);  // c1
    const uint32_t z = __byte_perm(__byte_perm(d0, d1, 0x0052u), d2, 0x7410u);  // c2
    const uint32_t m = __vmaxu4(__vmaxu4(x, y), z);
    if (p.t_diff < 0) return 0xFu;            // every |d| >= 0 > t_diff
    const uint32_t t = static_cast<uint32_t>(min(p.t_diff, 255));
    const uint32_t gt = __vcmpgtu4(m, t * 0x01010101u);  // 0xFF where max > t_diff
    return (gt & 0x1u) | ((gt >> 7) & 0x2u) | ((gt >> 14) & 0x4u) | ((gt >> 21) & 0x8u);
  }
  return 0u;
}

template <bool HIST, int MASKMODE, int QUAD>
__device__ __forceinline__ void stats_unit(const StatsParams &p, const int64_t unit,
                                           uint32_t *smem, uint64_t (*part)[13]) {
  // quads per lane per step: 6 (18 loads in flight; a default 96-row x
  // 32-px band block is 768 quads = exactly 6 per thread of the CTA); the
  // motion-mask path also loads the previous frame's words: 3 (fewer
  // registers, more CTAs per SM).  Measured: tools/k1_probe.py
  // QUAD 2: 16-pixel groups (48 bytes = 3 x 16-byte loads) of 4 quads,
  // kG16Groups per lane per step - 2.7x the bytes in flight per load slot
  constexpr int kQuadBatch = QUAD == 2 ? 4 * (MASKMODE == 2 ? kG16GroupsRemoval : kG16Groups)
                             : MASKMODE == 2 ? CAMX_K1_QB_REMOVAL : kQuadBatchMax;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  constexpr int kStride = 32 * kStatsWarps;  // quads (pixels) per CTA-wide step
  const int k = static_cast<int>(unit % p.K);
  const int side = static_cast<int>((unit / p.K) % 2);
  const int64_t img = unit / (2 * p.K);

  const int r0 = k * p.bh;
  const int r1 = (k == p.K - 1) ? p.H : r0 + p.bh;
  const int col0 = (side == CAMX_SIDE_LEFT) ? p.W - p.bw : 0;
  const int64_t row_bytes = static_cast<int64_t>(p.W) * 3;
  const uint8_t *base = p.img + img * p.img_bytes;
  const uint8_t *pbase =
      (MASKMODE == 2) ? (p.prev_seq > 0 && img >= p.prev_seq
                             ? p.img + (img - p.prev_seq) * p.img_bytes
                             : p.prev + img * p.img_bytes)
                      : nullptr;
  const uint8_t *mbase = (MASKMODE == 1) ? p.mask + img * p.mask_bytes : nullptr;

  uint32_t *cnt = HIST ? smem + warp * kHistWords : nullptr;
  if (HIST) {
    for (int w = lane; w < kHistWords; w += 32) cnt[w] = 0u;
    __syncwarp();
  }
  Acc a;
#pragma unroll
  for (int c = 0; c < 3; ++c) a.raw_s[c] = a.raw_q[c] = a.val_s[c] = a.val_q[c] = 0;
  a.nvalid = 0;

  const int rows = r1 - r0;
  if (QUAD) {
    const int qpr = p.bw >> 2;
    const int nq = rows * qpr;
    const bool pow2 = (qpr & (qpr - 1)) == 0;
    const int qsh = __ffs(qpr) - 1;
    const int gpr = p.bw >> 4;  // QUAD 2: groups per row
    const bool gpow2 = (gpr & (gpr - 1)) == 0;
    const int gsh = __ffs(gpr) - 1;
    const int n_items = QUAD == 2 ? rows * gpr : nq;
    constexpr int kItemBatch = QUAD == 2 ? kQuadBatch / 4 : kQuadBatch;
    for (int i0 = warp * 32; i0 < n_items; i0 += kStride * kItemBatch) {
      uint32_t w[kQuadBatch][3], pw[kQuadBatch][3], mw[kQuadBatch];
      bool live[kQuadBatch];
      if (QUAD == 2) {
#pragma unroll
        for (int ug = 0; ug < kItemBatch; ++ug) {
          const int gi = i0 + ug * kStride + lane;
          const bool lv = gi < n_items;
          const int ii = lv ? gi : 0;
          const int rq = gpow2 ? (ii >> gsh) : ii / gpr;
          const int64_t off = (r0 + rq) * row_bytes +
                              static_cast<int64_t>(col0 + (ii - rq * gpr) * 16) * 3;
          const uint4 *vp = reinterpret_cast<const uint4 *>(base + off);
          const uint4 v0 = __ldg(vp), v1 = __ldg(vp + 1), v2 = __ldg(vp + 2);
          const uint32_t g[12] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y,
                                  v1.z, v1.w, v2.x, v2.y, v2.z, v2.w};
          uint32_t h[12];
          if (MASKMODE == 2) {
            const uint4 *pp = reinterpret_cast<const uint4 *>(pbase + off);
            const uint4 q0 = __ldg(pp), q1 = __ldg(pp + 1), q2 = __ldg(pp + 2);
            h[0] = q0.x; h[1] = q0.y; h[2] = q0.z; h[3] = q0.w;
            h[4] = q1.x; h[5] = q1.y; h[6] = q1.z; h[7] = q1.w;
            h[8] = q2.x; h[9] = q2.y; h[10] = q2.z; h[11] = q2.w;
          }
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            live[4 * ug + t] = lv;
#pragma unroll
            for (int kk = 0; kk < 3; ++kk) {
              w[4 * ug + t][kk] = g[3 * t + kk];
              if (MASKMODE == 2) pw[4 * ug + t][kk] = h[3 * t + kk];
            }
          }
        }
      } else {
#pragma unroll
      for (int u = 0; u < kQuadBatch; ++u) {
        const int i = i0 + u * kStride + lane;
        live[u] = i < nq;
        const int ii = live[u] ? i : 0;
        const int rq = pow2 ? (ii >> qsh) : ii / qpr;
        const int row = r0 + rq;
        const int col = col0 + (ii - rq * qpr) * 4;
        const int64_t off = row * row_bytes + static_cast<int64_t>(col) * 3;
        const uint32_t *wp = reinterpret_cast<const uint32_t *>(base + off);
        w[u][0] = __ldg(wp);
        w[u][1] = __ldg(wp + 1);
        w[u][2] = __ldg(wp + 2);
        if (MASKMODE == 2) {
          const uint32_t *pp = reinterpret_cast<const uint32_t *>(pbase + off);
          pw[u][0] = __ldg(pp);
          pw[u][1] = __ldg(pp + 1);
          pw[u][2] = __ldg(pp + 2);
        }
        if (MASKMODE == 1)
          mw[u] = __ldg(reinterpret_cast<const uint32_t *>(mbase + static_cast<int64_t>(row) * p.W + col));
      }
      }
      if (MASKMODE != 1) {
        // Channel sums / sums of squares with dp4a: in a quad the byte
        // positions of each channel are fixed (r g b r | g b r g | b r g b),
        // so constant byte masks select them.  32-bit per batch (<= 32 px
        // per lane), widened once per batch.  HIST: plus one shared-memory
        // atomic per kept (pixel, channel) - no per-pixel 64-bit moments.
        uint32_t rs[3] = {0, 0, 0}, rq[3] = {0, 0, 0}, vs[3] = {0, 0, 0}, vq[3] = {0, 0, 0};
        uint32_t nv = 0;
#pragma unroll
        for (int u = 0; u < kQuadBatch; ++u) {
          if (!live[u]) continue;
#pragma unroll
          for (int c = 0; c < 3; ++c) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              const uint32_t sel = quad_sel(c, k);
              rs[c] = __dp4a(w[u][k], sel, rs[c]);
              const uint32_t m = w[u][k] & (sel * 0xFFu);
              rq[c] = __dp4a(m, m, rq[c]);
            }
          }
          uint32_t ex = 0u;
          if (MASKMODE == 2) ex = quad_exclusion<MASKMODE>(p, w[u], pw[u], mw[u]);
          if (HIST) {
            // every pixel counted unconditionally (no per-pixel branch), the
            // (rare) excluded ones taken back out
#pragma unroll
            for (int e = 0; e < 4; ++e) {
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                const int byte = 3 * e + c;  // compile-time position in the 12-byte quad
                const uint32_t val = (w[u][byte >> 2] >> ((byte & 3) * 8)) & 0xFFu;
                atomicAdd(cnt + c * 256 + val, 1u);
              }
            }
            if (MASKMODE != 0 && ex != 0u) {
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                if (!((ex >> e) & 1u)) continue;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                  const int byte = 3 * e + c;
                  const uint32_t val = (w[u][byte >> 2] >> ((byte & 3) * 8)) & 0xFFu;
                  atomicSub(cnt + c * 256 + val, 1u);
                }
              }
            }
          }
          if (MASKMODE == 2) {
            nv += 4 - __popc(ex);
            // keep-masks of the 12 bytes: pixel e kept -> its 3 bytes
            const uint32_t kp = (~ex) & 0xFu;
            const uint32_t kb = (kp & 1 ? 0xFFu : 0u) | (kp & 2 ? 0xFF00u : 0u) |
                                (kp & 4 ? 0xFF0000u : 0u) | (kp & 8 ? 0xFF000000u : 0u);
            const uint32_t km0 = __byte_perm(kb, 0, 0x1000);  // px 0 0 0 1
            const uint32_t km1 = __byte_perm(kb, 0, 0x2211);  // px 1 1 2 2
            const uint32_t km2 = __byte_perm(kb, 0, 0x3332);  // px 2 3 3 3
            const uint32_t mw0 = w[u][0] & km0, mw1 = w[u][1] & km1, mw2 = w[u][2] & km2;
            const uint32_t mm[3] = {mw0, mw1, mw2};
#pragma unroll
            for (int c = 0; c < 3; ++c) {
#pragma unroll
              for (int k = 0; k < 3; ++k) {
                const uint32_t sel = quad_sel(c, k);
                vs[c] = __dp4a(mm[k], sel, vs[c]);
                const uint32_t m = mm[k] & (sel * 0xFFu);
                vq[c] = __dp4a(m, m, vq[c]);
              }
            }
          } else {
            nv += 4;
          }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          a.raw_s[c] += rs[c];
          a.raw_q[c] += rq[c];
          if (MASKMODE == 2) {
            a.val_s[c] += vs[c];
            a.val_q[c] += vq[c];
          }
        }
        a.nvalid += nv;
      } else {
#pragma unroll
        for (int u = 0; u < kQuadBatch; ++u) {
          if (!live[u]) continue;
          const uint32_t ex = quad_exclusion<MASKMODE>(p, w[u], pw[u], mw[u]);
          const uint32_t *q = w[u];
          add_pixel<HIST>(a, cnt, lane, q[0] & 0xFF, (q[0] >> 8) & 0xFF, (q[0] >> 16) & 0xFF, ex & 1);
          add_pixel<HIST>(a, cnt, lane, q[0] >> 24, q[1] & 0xFF, (q[1] >> 8) & 0xFF, ex & 2);
          add_pixel<HIST>(a, cnt, lane, (q[1] >> 16) & 0xFF, q[1] >> 24, q[2] & 0xFF, ex & 4);
          add_pixel<HIST>(a, cnt, lane, (q[2] >> 8) & 0xFF, (q[2] >> 16) & 0xFF, q[2] >> 24, ex & 8);
        }
      }
    }
  } else {
    const int npix = rows * p.bw;
    for (int i0 = warp * 32; i0 < npix; i0 += kStride * kQuadBatch) {
      uint32_t v[kQuadBatch][3];
      bool ex[kQuadBatch], live[kQuadBatch];
#pragma unroll
      for (int u = 0; u < kQuadBatch; ++u) {
        const int i = i0 + u * kStride + lane;
        live[u] = i < npix;
        const int ii = live[u] ? i : 0;
        const int row = r0 + ii / p.bw;
        const int col = col0 + (ii - (ii / p.bw) * p.bw);
        const int64_t off = row * row_bytes + static_cast<int64_t>(col) * 3;
        int d = 0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          v[u][c] = __ldg(base + off + c);
          if (MASKMODE == 2) d = max(d, abs(static_cast<int>(v[u][c]) - __ldg(pbase + off + c)));
        }
        ex[u] = (MASKMODE == 2) ? (d > p.t_diff)
                : (MASKMODE == 1) ? (__ldg(mbase + static_cast<int64_t>(row) * p.W + col) != 0)
                                  : false;
      }
#pragma unroll
      for (int u = 0; u < kQuadBatch; ++u)
        if (live[u]) add_pixel<HIST>(a, cnt, lane, v[u][0], v[u][1], v[u][2], ex[u]);
    }
  }

  if (HIST) {
    uint32_t *stage = smem;  // [warp][3][256]
    __syncthreads();  // every warp's bins complete
    // thread t owns bins t, t+128, ... of the 768 (channel, bin) pairs
    if (MASKMODE == 1 || !QUAD) {
#pragma unroll
      for (int c = 0; c < 3; ++c) a.val_s[c] = a.val_q[c] = 0;
    }
    for (int e = threadIdx.x; e < 768; e += kStatsWarps * 32) {
      uint32_t tot = 0;
#pragma unroll
      for (int w2 = 0; w2 < kStatsWarps; ++w2) tot += stage[w2 * kHistWords + e];
      const int c = e >> 8;
      const uint64_t bin = e & 255;
      if (p.hist != nullptr) p.hist[unit * 768 + e] = tot;
      // c is warp-uniform for e in steps of 128 within one channel
      if (MASKMODE == 1 || !QUAD) {  // the dp4a quad path already has the valid sums
        const uint64_t s1 = bin * tot, s2 = bin * bin * tot;
        if (c == 0) { a.val_s[0] += s1; a.val_q[0] += s2; }
        if (c == 1) { a.val_s[1] += s1; a.val_q[1] += s2; }
        if (c == 2) { a.val_s[2] += s1; a.val_q[2] += s2; }
      }
    }
  }
  if (MASKMODE == 0 && (!HIST || QUAD)) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      a.val_s[c] = a.raw_s[c];
      a.val_q[c] = a.raw_q[c];
    }
  }
  // Warp sums.  A unit of <= 66051 pixels has every sum of squares below
  // 2^32, so the shuffles run on 32-bit halves; MASKMODE 0 (no exclusion)
  // reduces only the raw sums (valid == raw, count == area).
  uint64_t r[13];
  const bool narrow = static_cast<int64_t>(rows) * p.bw <= 66051;
  constexpr bool kMasked = HIST || MASKMODE != 0;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    r[6 + c] = narrow ? warp_sum_u32(static_cast<uint32_t>(a.raw_s[c])) : warp_sum_u64(a.raw_s[c]);
    r[9 + c] = narrow ? warp_sum_u32(static_cast<uint32_t>(a.raw_q[c])) : warp_sum_u64(a.raw_q[c]);
    if (kMasked) {
      r[c] = narrow ? warp_sum_u32(static_cast<uint32_t>(a.val_s[c])) : warp_sum_u64(a.val_s[c]);
      r[3 + c] = narrow ? warp_sum_u32(static_cast<uint32_t>(a.val_q[c])) : warp_sum_u64(a.val_q[c]);
    } else {
      r[c] = 0;
      r[3 + c] = 0;
    }
  }
  r[12] = kMasked ? warp_sum_u32(a.nvalid) : 0;
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < 13; ++i) part[warp][i] = r[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < 13; ++i)
      for (int w2 = 1; w2 < kStatsWarps; ++w2) r[i] += part[w2][i];
    camx_band_stat o;
    o.area = static_cast<int64_t>(rows) * p.bw;
    o.valid = kMasked ? static_cast<int64_t>(r[12]) : o.area;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      o.sum[c] = kMasked ? r[c] : r[6 + c];
      o.sumsq[c] = kMasked ? r[3 + c] : r[9 + c];
      o.raw_sum[c] = r[6 + c];
      o.raw_sumsq[c] = r[9 + c];
    }
    p.out[unit] = o;
  }
}

// Persistent: a grid of a few CTAs per SM loops over the (image, side,
// block) units, so the short per-unit load -> reduce phases of resident
// CTAs overlap instead of running as many launch waves.
template <bool HIST, int MASKMODE, int QUAD>
__global__ void __launch_bounds__(kStatsWarps * 32, CAMX_K1_MINB) band_stats_kernel(const StatsParams p) {
  extern __shared__ uint32_t smem[];
  __shared__ uint64_t part[kStatsWarps][13];
  // let a programmatically dependent kernel launch early (K2 waits on
  // griddepcontrol.wait; K3 only prefetches raw pixels before it)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int64_t unit = blockIdx.x; unit < p.n_units; unit += gridDim.x) {
    stats_unit<HIST, MASKMODE, QUAD>(p, unit, smem, part);
    __syncthreads();  // `part` / counters reused by the next unit
  }
}

template <bool HIST, int MASKMODE, int QUAD>
static void launch_stats(const StatsParams &p, cudaStream_t s) {
  const int warps = kStatsWarps;
  const size_t smem = HIST ? static_cast<size_t>(warps) * kHistWords * sizeof(uint32_t) : 0;
  if (HIST) {
    cudaFuncSetAttribute(band_stats_kernel<HIST, MASKMODE, QUAD>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  }
  // 32 CTAs per SM for the plain path (8 resident): units are scheduled
  // dynamically, ~6% faster than a one-wave persistent grid (tools/k1_probe.py)
  const int per_sm = 128 / kStatsWarps;
  const int64_t grid = std::min<int64_t>(p.n_units, static_cast<int64_t>(sm_count()) * per_sm);
  band_stats_kernel<HIST, MASKMODE, QUAD>
      <<<static_cast<unsigned>(grid), warps * 32, smem, s>>>(p);
}

// 16-pixel groups: whole 16-byte-aligned 48-byte runs in every band row
static bool k1_g16(const StatsParams &p) {
  auto al16 = [](const void *x) { return reinterpret_cast<uintptr_t>(x) % 16 == 0; };
  return p.bw % 16 == 0 && (3 * p.W) % 16 == 0 && (3 * (p.W - p.bw)) % 16 == 0 &&
         al16(p.img) && (p.prev == nullptr || al16(p.prev)) && p.mask == nullptr;
}

template <bool HIST, int MASKMODE>
static void launch_stats_q(const StatsParams &p, bool quad, cudaStream_t s) {
  if (quad && MASKMODE != 1 && k1_g16(p))
    launch_stats<HIST, MASKMODE, 2>(p, s);
  else if (quad)
    launch_stats<HIST, MASKMODE, 1>(p, s);
  else
    launch_stats<HIST, MASKMODE, 0>(p, s);
}

// ---- moments --------------------------------------------------------------
// mean = S / n (correctly rounded, = numpy's pairwise mean of integers);
// population variance = (n*Q - S^2) / n^2 with the numerator exact in
// 128-bit integers.
__device__ __forceinline__ void moments_of(uint64_t n, uint64_t s, uint64_t q, double &mean,
                                           double &sd) {
  if (n == 0) {
    mean = 0.0;
    sd = 0.0;
    return;
  }
  const unsigned __int128 nq = static_cast<unsigned __int128>(n) * q;
  const unsigned __int128 ss = static_cast<unsigned __int128>(s) * s;
  const unsigned __int128 d = nq > ss ? nq - ss : 0;
  const double dn = static_cast<double>(n);
  mean = __ddiv_rn(static_cast<double>(s), dn);
  const double var = __ddiv_rn(static_cast<double>(d), __dmul_rn(dn, dn));
  sd = sqrt(var);
}

__global__ void band_moments_kernel(const camx_band_stat *st, int64_t n, int raw, double *mean,
                                    double *sd, int64_t *valid, int64_t *area) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const camx_band_stat r = st[i];
    const uint64_t cnt = raw ? static_cast<uint64_t>(r.area) : static_cast<uint64_t>(r.valid);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double m, s;
      moments_of(cnt, raw ? r.raw_sum[c] : r.sum[c], raw ? r.raw_sumsq[c] : r.sumsq[c], m, s);
      if (mean) mean[i * 3 + c] = m;
      if (sd) sd[i * 3 + c] = s;
    }
    if (valid) valid[i] = raw ? r.area : r.valid;
    if (area) area[i] = r.area;
  }
}

}  // namespace camx

using namespace camx;

namespace camx {
int band_stats_seq(const uint8_t *images, const uint8_t *prev_images, const uint8_t *excl_masks,
                   int64_t n_images, int64_t prev_seq, int32_t height, int32_t width,
                   int32_t band_width, int32_t blocks, int32_t t_diff, camx_band_stat *stats_out,
                   uint32_t *hist_out, void *stream);
}

extern "C" int camx_band_stats(const uint8_t *images, const uint8_t *prev_images,
                               const uint8_t *excl_masks, int64_t n_images, int32_t height,
                               int32_t width, int32_t band_width, int32_t blocks, int32_t t_diff,
                               camx_band_stat *stats_out, uint32_t *hist_out, void *stream) {
  return band_stats_seq(images, prev_images, excl_masks, n_images, 0, height, width, band_width,
                        blocks, t_diff, stats_out, hist_out, stream);
}

// prev_seq > 0 (OBJECT_REMOVAL over a batch of array-frames of prev_seq
// images): image i >= prev_seq is diffed against image i - prev_seq, the
// first prev_seq against prev_images - one launch for the whole batch.
int camx::band_stats_seq(const uint8_t *images, const uint8_t *prev_images,
                         const uint8_t *excl_masks, int64_t n_images, int64_t prev_seq,
                         int32_t height, int32_t width, int32_t band_width, int32_t blocks,
                         int32_t t_diff, camx_band_stat *stats_out, uint32_t *hist_out,
                         void *stream) {
  if (n_images < 0 || height < 1 || width < 1) return CAMX_EINVAL;
  if (band_width < 1 || band_width > width / 2) return CAMX_EINVAL;
  if (blocks < 1 || blocks > height) return CAMX_EINVAL;
  if (prev_images != nullptr && excl_masks != nullptr) return CAMX_EINVAL;
  if (images == nullptr || stats_out == nullptr) return CAMX_EINVAL;
  if (hist_out != nullptr && (reinterpret_cast<uintptr_t>(hist_out) % 16) != 0) return CAMX_EALIGN;
  if (n_images == 0) return CAMX_OK;
  StatsParams p{};
  p.img = images;
  p.prev = prev_images;
  p.prev_seq = prev_images != nullptr ? prev_seq : 0;
  p.mask = excl_masks;
  p.H = height;
  p.W = width;
  p.bw = band_width;
  p.K = blocks;
  p.bh = height / blocks;
  p.t_diff = t_diff;
  p.img_bytes = static_cast<int64_t>(height) * width * 3;
  p.mask_bytes = static_cast<int64_t>(height) * width;
  p.n_units = n_images * 2 * blocks;
  p.out = stats_out;
  p.hist = hist_out;
  cudaStream_t s = as_stream(stream);
  const int mm = prev_images ? 2 : (excl_masks ? 1 : 0);
  auto al4 = [](const void *x) { return reinterpret_cast<uintptr_t>(x) % 4 == 0; };
  const bool quad = (width % 4 == 0) && (band_width % 4 == 0) && al4(images) &&
                    (mm != 2 || al4(prev_images)) && (mm != 1 || al4(excl_masks));
  if (hist_out != nullptr) {
    if (mm == 0) launch_stats_q<true, 0>(p, quad, s);
    if (mm == 1) launch_stats_q<true, 1>(p, quad, s);
    if (mm == 2) launch_stats_q<true, 2>(p, quad, s);
  } else {
    if (mm == 0) launch_stats_q<false, 0>(p, quad, s);
    if (mm == 1) launch_stats_q<false, 1>(p, quad, s);
    if (mm == 2) launch_stats_q<false, 2>(p, quad, s);
  }
  return launch_status();
}

extern "C" int camx_band_moments(const camx_band_stat *stats, int64_t n_records, int32_t use_raw,
                                 double *mean_out, double *std_out, int64_t *valid_out,
                                 int64_t *area_out, void *stream) {
  if (n_records < 0 || stats == nullptr) return CAMX_EINVAL;
  if (n_records == 0) return CAMX_OK;
  const int64_t blocks = (n_records + 127) / 128;
  band_moments_kernel<<<static_cast<unsigned>(blocks > 4096 ? 4096 : blocks), 128, 0,
                        as_stream(stream)>>>(stats, n_records, use_raw, mean_out, std_out,
                                             valid_out, area_out);
  return launch_status();
}
