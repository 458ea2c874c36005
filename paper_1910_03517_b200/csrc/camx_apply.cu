// K3: per-pixel seam exposure correction apply (stage 3).
//
// Reference semantics (camarray exposure.py:347-414):
//   lam(col)  LEFT  = clip((col - c0) / ((W-1) - c0), 0, 1)      c0 = (W-1)/2
//             RIGHT = clip((c0 - col) / c0, 0, 1)
//   M = f32(1 + lam*(g - 1)),  A = f32(lam*b)       (float64, then cast)
//   out = u8(clip(rint(f32(p)*M + A), 0, 255))      (float32 mul, add)
// applied on the lam > 0 columns; everything else is copied.
//
// Bit-exactness without materialising M/A: each thread owns one 16-byte
// column chunk of a row (16 sub-pixels with fixed (column, channel)) and
// evaluates the float64 expressions with explicit _rn intrinsics (no FMA
// contraction) once per block, keeping the float32 results in registers
// while it streams the block's rows.  The per-sub-pixel float32 chain is
// re-expressed exactly:
//   X = 2^23 + p  (PRMT of the byte under exponent 0x4B: exact)
//   fma(X, M/256, -2^15*M) = rn(p*M)/256       (exact: one rounding of p*M)
//   add.sat(., A/256)      = clip(rn(p*M + A), 0, 256)/256   (scaling by 2^-8
//                            commutes with RN in the normal range)
//   fma(., 256, 2^23)      = 2^23 + rint_half_even(clip(y, 0, 256))
//   min(., 255) on the 16-bit lanes (VIMNMX.U16x2), then byte pack.
// Since clamp bounds are integers, clip(rint(y)) == rint(clip(y)).
#include <algorithm>
#include <cstdlib>

#include "camx_resize.cuh"

namespace camx {

struct ApplyParams {
  const uint8_t *src;
  uint8_t *dst;
  int64_t img_bytes;  // H * W * 3
  int32_t H, W, K, bh;
  int32_t row_bytes;
  int32_t n_img;
  int32_t single;  // 0: array maps; 1: one map with role `single_side`
  int32_t single_side;
  int32_t cam_begin, cam_count, n_cams, wrap, S;
  const double *gain;
  const double *offset;
  // fast kernel decomposition
  int32_t chunks_per_row, col_groups, row_splits, rows_per_split;
  int32_t pdl;  // launched as a programmatic dependent of the stats/solve kernel
  // motion counts (K3 with the in-pass K4, apply_tma_kernel<..., MOTION>):
  // previous raw images of array-frame 0 (frames b >= 1 use frame b - 1 of
  // the batch; NULL: no counts for frame 0), per-frame window counts of the
  // overlap-0 tiling of the mosaic (attention.py:66-103), mask_diff threshold
  const uint8_t *prev_first;
  unsigned long long *counts;  // [B][ny][nx]
  int32_t win, nx, ny, nx_reg, ny_reg, mosaic_w, t_motion;
};

// Map pointers (LEFT role = seam at the right edge, RIGHT role = seam at the
// left edge) of image `img`; nullptr when the camera has no such seam.
__device__ __forceinline__ void map_ptrs(const ApplyParams &p, int64_t img, const double *&gl,
                                         const double *&bl, const double *&gr,
                                         const double *&br) {
  gl = bl = gr = br = nullptr;
  const int K3 = p.K * 3;
  if (p.single) {
    if (p.single_side == CAMX_SIDE_LEFT) {
      gl = p.gain;
      bl = p.offset;
    } else {
      gr = p.gain;
      br = p.offset;
    }
    return;
  }
  const int64_t b = img / p.cam_count;
  const int cam = p.cam_begin + static_cast<int>(img % p.cam_count);
  int sl = cam < p.n_cams - 1 ? cam : (p.wrap ? p.n_cams - 1 : -1);
  int sr = cam >= 1 ? cam - 1 : (p.wrap ? p.n_cams - 1 : -1);
  if (sl >= 0 && sl < p.S) {
    const int64_t idx = ((b * p.S + sl) * 2 + 0) * K3;
    gl = p.gain + idx;
    bl = p.offset + idx;
  }
  if (sr >= 0 && sr < p.S) {
    const int64_t idx = ((b * p.S + sr) * 2 + 1) * K3;
    gr = p.gain + idx;
    br = p.offset + idx;
  }
}

// lam of one column (exposure.py:347-355) and which map it uses: 0 = LEFT
// role (seam at the right edge), 1 = RIGHT role, -1 = identity (outside the
// lam > 0 half of every present map).
__device__ __forceinline__ double col_lambda(int col, int W, bool have_l, bool have_r, int &role) {
  const double c0 = (W - 1) * 0.5;
  const double colf = static_cast<double>(col);
  double lam = 0.0;
  role = -1;
  if (have_l && 2 * col > W - 1) {
    lam = __ddiv_rn(__dsub_rn(colf, c0), __dsub_rn(static_cast<double>(W - 1), c0));
    role = 0;
  } else if (have_r && 2 * col < W - 1) {
    lam = __ddiv_rn(__dsub_rn(c0, colf), c0);
    role = 1;
  }
  if (!(lam > 0.0)) role = -1;
  return fmin(lam, 1.0);
}

// Exact float32 (M, A) of one (column, channel, block) given its lam/role.
__device__ __forceinline__ void coef_from_lam(double lam, int role, int k, int ch,
                                              const double *gl, const double *bl,
                                              const double *gr, const double *br, float &m32,
                                              float &a32) {
  if (role < 0) {
    m32 = 1.0f;
    a32 = 0.0f;
    return;
  }
  const double g = role == 0 ? gl[k * 3 + ch] : gr[k * 3 + ch];
  const double b = role == 0 ? bl[k * 3 + ch] : br[k * 3 + ch];
  const double M = __dadd_rn(1.0, __dmul_rn(lam, __dsub_rn(g, 1.0)));
  const double A = __dmul_rn(lam, b);
  m32 = __double2float_rn(M);
  a32 = __double2float_rn(A);
}

__device__ __forceinline__ void coef_f32(int col, int ch, int k, int W, const double *gl,
                                         const double *bl, const double *gr, const double *br,
                                         float &m32, float &a32) {
  int role;
  const double lam = col_lambda(col, W, gl != nullptr, gr != nullptr, role);
  coef_from_lam(lam, role, k, ch, gl, bl, gr, br, m32, a32);
}

// ---------------------------------------------------------------- fast path
// Requires row_bytes % 16 == 0 and 16-byte aligned src/dst.
constexpr int kApplyThreads = 128;

struct Coef16 {
  uint64_t m[8];  // pairs (M/256, M/256) for sub-pixels (2i, 2i+1)
  uint64_t c[8];  // pairs (-2^15*M)
  float a[16];    // A/256
};

__device__ __forceinline__ uint32_t correct_word(uint32_t w, const Coef16 &cf, int base) {
  const uint64_t kScale = pack2(256.0f, 256.0f);
  const uint64_t kMagic = pack2(8388608.0f, 8388608.0f);
  uint32_t z[4];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int i = base + 2 * h;
    const uint32_t x0 = __byte_perm(w, 0x4B00u, 0x5440u + 2 * h);
    const uint32_t x1 = __byte_perm(w, 0x4B00u, 0x5441u + 2 * h);
    const uint64_t y1 = fma2_rn(pack2u(x0, x1), cf.m[i >> 1], cf.c[i >> 1]);
    uint32_t lo, hi;
    unpack2u(y1, lo, hi);
    const float s0 = add_sat_rn(__uint_as_float(lo), cf.a[i]);
    const float s1 = add_sat_rn(__uint_as_float(hi), cf.a[i + 1]);
    const uint64_t q = fma2_rn(pack2(s0, s1), kScale, kMagic);
    unpack2u(q, z[2 * h], z[2 * h + 1]);
  }
  uint32_t p01 = __byte_perm(z[0], z[1], 0x5410u);
  uint32_t p23 = __byte_perm(z[2], z[3], 0x5410u);
  p01 = __vminu2(p01, 0x00FF00FFu);
  p23 = __vminu2(p23, 0x00FF00FFu);
  return __byte_perm(p01, p23, 0x6420u);
}

__device__ __forceinline__ uint4 correct16(uint4 v, const Coef16 &cf) {
  uint4 r;
  r.x = correct_word(v.x, cf, 0);
  r.y = correct_word(v.y, cf, 4);
  r.z = correct_word(v.z, cf, 8);
  r.w = correct_word(v.w, cf, 12);
  return r;
}

// In-range variant (every sub-pixel of the CTA has |M| * 255 + |A| < 32000,
// i.e. |p*M + A| < 2^15 for every byte p - all maps a solver produces): no
// 2^-8 scaling and no saturating adds -
//   fma(X, M, -2^23*M)  = rn(p*M)                 (exact: one rounding)
//   + A                 = rn(rn(p*M) + A)         (the reference's f32 add)
//   + 1.5*2^23          = 1.5*2^23 + rint_half_even(.)   (|.| < 2^22)
// so the low 16 bits of each lane are rint(y) as an int16, and one
// VIMNMX.S16x2.RELU (min 255, then max 0) clamps two sub-pixels: 15 instead
// of 17 instructions per 4 bytes, all paired except the byte permutes.
struct Coef16F {
  uint64_t m[8];  // pairs (M, M)
  uint64_t c[8];  // pairs (-2^23*M)
  uint64_t a[8];  // pairs (A)
};

__device__ __forceinline__ uint32_t min255_relu_s16x2(uint32_t x) {
  uint32_t d;
  asm("min.relu.s16x2 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(0x00FF00FFu));
  return d;
}

__device__ __forceinline__ uint32_t correct_word(uint32_t w, const Coef16F &cf, int base) {
  const uint64_t kMagic = pack2(12582912.0f, 12582912.0f);  // 1.5 * 2^23
  uint32_t z[4];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int i = (base + 2 * h) >> 1;
    const uint32_t x0 = __byte_perm(w, 0x4B00u, 0x5440u + 2 * h);
    const uint32_t x1 = __byte_perm(w, 0x4B00u, 0x5441u + 2 * h);
    const uint64_t y = fma2_rn(pack2u(x0, x1), cf.m[i], cf.c[i]);
    const uint64_t q = add2_rn(add2_rn(y, cf.a[i]), kMagic);
    unpack2u(q, z[2 * h], z[2 * h + 1]);
  }
  const uint32_t p01 = min255_relu_s16x2(__byte_perm(z[0], z[1], 0x5410u));
  const uint32_t p23 = min255_relu_s16x2(__byte_perm(z[2], z[3], 0x5410u));
  return __byte_perm(p01, p23, 0x6420u);
}

__device__ __forceinline__ uint4 correct16(uint4 v, const Coef16F &cf) {
  uint4 r;
  r.x = correct_word(v.x, cf, 0);
  r.y = correct_word(v.y, cf, 4);
  r.z = correct_word(v.z, cf, 8);
  r.w = correct_word(v.w, cf, 12);
  return r;
}

// Coefficients from the per-sub-pixel float32 (M, A); the general form is
// derived from the in-range one (same float32 M and A).
__device__ __forceinline__ void make_coef(const float (&m)[16], const float (&a)[16],
                                          Coef16F &cf) {
#pragma unroll
  for (int i = 0; i < 16; i += 2) {
    cf.m[i >> 1] = pack2(m[i], m[i + 1]);
    cf.c[i >> 1] = pack2(m[i] * -8388608.0f, m[i + 1] * -8388608.0f);
    cf.a[i >> 1] = pack2(a[i], a[i + 1]);
  }
}
__device__ __forceinline__ Coef16 general_coef(const Coef16F &f) {
  Coef16 cf;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t m0, m1, a0, a1;
    unpack2u(f.m[i], m0, m1);
    unpack2u(f.a[i], a0, a1);
    const float mm[2] = {__uint_as_float(m0), __uint_as_float(m1)};
    const float aa[2] = {__uint_as_float(a0), __uint_as_float(a1)};
    cf.m[i] = pack2(mm[0] * 0.00390625f, mm[1] * 0.00390625f);
    cf.c[i] = pack2(mm[0] * -32768.0f, mm[1] * -32768.0f);
#pragma unroll
    for (int h = 0; h < 2; ++h)
      cf.a[2 * i + h] = fabsf(aa[h]) < 7.7037197787136e-34f ? 0.0f : aa[h] * 0.00390625f;
  }
  return cf;
}
__device__ __forceinline__ bool coef_in_range(const float (&m)[16], const float (&a)[16]) {
  bool ok = true;
#pragma unroll
  for (int i = 0; i < 16; ++i) ok &= fabsf(m[i]) * 255.0f + fabsf(a[i]) < 32000.0f;  // NaN: false
  return ok;
}

// ------------------------------------------------- TMA bulk-copy pipeline
// CTA = one 2 KB column group of one row block (split) of one image, thread
// = one 16-byte chunk; the rows stream through a kStages-deep shared-memory
// ring filled by 1-D bulk async copies (cp.async.bulk, the TMA engine)
// completing on mbarriers, so the bytes in flight per SM do not depend on
// registers x occupancy (a plain 128-bit LDG version was long-scoreboard
// bound at 16 warps/SM and ~5% slower: profiles/r01/SUMMARY.md).  Thread 0 issues; every thread
// consumes its 16-byte column chunk of each row from shared memory.
constexpr int kTmaStages = 6;
constexpr int kTmaRows = 2;  // rows per stage

#ifndef CAMX_K3_MINB
#define CAMX_K3_MINB 6  // K3: CTAs per SM the register budget is sized for (78 registers)
#endif

// MINB: CTAs per SM the register budget is sized for (0: CAMX_K3_MINB);
// short-CTA launches use a leaner variant.
// MOTION: the in-pass K4 (attention.py:89-103 counts of mask_diff,
// core.py:191-196): every stage also stages the previous raw frame's rows
// (and 16 bytes past the column group, for the pixel straddling the next
// group) and counts, per window of the overlap-0 tiling that meets the CTA,
// the pixels with max_c |cur - prev| > t_motion.  Per 4 bytes: VABSDIFF4,
// a 3-op SWAR "> t" into the byte MSBs, and one IMAD gathering the 4 MSBs
// into a nibble; a thread's 16 bytes + the next 2 (from the next chunk in
// the ring) give an 18-bit flag mask E, and a pixel is on iff any of its 3
// bytes is: E | E >> 1 | E >> 2 at the thread's pixel starts.
template <bool HI>  // t >= 128
__device__ __forceinline__ uint32_t gt_nibble(uint32_t cur, uint32_t prev, uint32_t k7) {
  const uint32_t d = __vabsdiffu4(cur, prev);
  const uint32_t s = (d & 0x7F7F7F7Fu) + k7;  // bit 7 of a byte: low7(d) > t mod 128
  const uint32_t f = (HI ? (s & d) : (s | d)) & 0x80808080u;
  return (f * 0x00204081u) >> 28;  // byte MSBs 7, 15, 23, 31 -> bits 0..3
}
template <bool HI>
__device__ __forceinline__ uint32_t flags16(uint4 c, uint4 q, uint32_t k7) {
  return gt_nibble<HI>(c.x, q.x, k7) | (gt_nibble<HI>(c.y, q.y, k7) << 4) |
         (gt_nibble<HI>(c.z, q.z, k7) << 8) | (gt_nibble<HI>(c.w, q.w, k7) << 12);
}

template <int ROWS, int STAGES, int MINB = 0, bool MOTION = false, bool MHI = false>
__global__ void __launch_bounds__(kApplyThreads, MINB > 0 ? MINB : CAMX_K3_MINB)
    apply_tma_kernel(const ApplyParams p) {
  // ring row: the 2 KB column group (MOTION: + 16 extra bytes, then the
  // previous frame's same bytes)
  constexpr int RS = MOTION ? 2 * (kApplyThreads + 1) : kApplyThreads;  // uint4 per ring row
  extern __shared__ __align__(128) uint4 ring[];  // [STAGES][ROWS][RS]
  __shared__ __align__(8) uint64_t full[STAGES];
  int64_t item = blockIdx.x;
  const int cg = static_cast<int>(item % p.col_groups);
  item /= p.col_groups;
  const int rs = static_cast<int>(item % p.row_splits);
  item /= p.row_splits;
  const int k = static_cast<int>(item % p.K);
  const int64_t img = item / p.K;

  const int blk_r0 = k * p.bh;
  const int blk_r1 = (k == p.K - 1) ? p.H : blk_r0 + p.bh;
  const int r0 = blk_r0 + rs * p.rows_per_split;
  const int r1 = min(blk_r1, r0 + p.rows_per_split);
  if (r0 >= r1) return;  // CTA-uniform
  const int chunks = min(kApplyThreads, p.chunks_per_row - cg * kApplyThreads);
  const uint32_t seg = static_cast<uint32_t>(chunks) * 16u;
  const int j = cg * kApplyThreads + threadIdx.x;
  const int64_t rb = p.row_bytes;
  const uint8_t *src0 = p.src + img * p.img_bytes + static_cast<int64_t>(r0) * rb +
                        static_cast<int64_t>(cg) * kApplyThreads * 16;
  const int nrows = r1 - r0;
  const int nst = (nrows + ROWS - 1) / ROWS;

  // MOTION: previous raw image rows (CTA-uniform; none -> plain K3)
  const uint8_t *prev0 = nullptr;
  bool extra = false;
  if (MOTION) {
    const int64_t bb = img / p.cam_count;
    const int64_t cc = img - bb * p.cam_count;
    const uint8_t *pimg = bb > 0 ? p.src + (img - p.cam_count) * p.img_bytes
                                 : (p.prev_first ? p.prev_first + cc * p.img_bytes : nullptr);
    if (pimg != nullptr)
      prev0 = pimg + static_cast<int64_t>(r0) * rb + static_cast<int64_t>(cg) * kApplyThreads * 16;
    extra = static_cast<int64_t>(cg) * kApplyThreads * 16 + seg < rb;
  }
  const uint32_t cseg = seg + (prev0 != nullptr && extra ? 16u : 0u);

  auto issue = [&](int st) {
    const int slot = st % STAGES;
    const int rr = min(ROWS, nrows - st * ROWS);
    mbar_expect_tx(&full[slot], (prev0 != nullptr ? 2 * cseg : seg) * rr);
    for (int i = 0; i < rr; ++i) {
      const int64_t ro = static_cast<int64_t>(st * ROWS + i) * rb;
      bulk_g2s(ring + (slot * ROWS + i) * RS, src0 + ro, cseg, &full[slot]);
      if (MOTION && prev0 != nullptr)
        bulk_g2s(ring + (slot * ROWS + i) * RS + kApplyThreads + 1, prev0 + ro, cseg, &full[slot]);
    }
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int st = 0; st < min(STAGES, nst); ++st) issue(st);
  }

  __syncthreads();
  // maps come from the preceding stats/solve grid (programmatic dependent
  // launch): only the raw-pixel prefetch above may run before it completes
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // a programmatic dependent (the tile kernel of config 5) may launch once
  // every K3 CTA has started: its prologue overlaps K3's last wave
  // (config 5: 1.1664 -> 1.1632 ms per 30 frames)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  const bool active = threadIdx.x < chunks;
  const double *gl, *bl, *gr, *br;
  map_ptrs(p, img, gl, bl, gr, br);
  // per sub-pixel (a per-column lambda cache measured ~6% slower end to
  // end on B200: tools/ab_k3.py)
  Coef16F cff;
  bool in_range = true;
  if (active) {
    float m[16], a[16];
    const int q0 = j * 16;
    int col = q0 / 3;
    int ch = q0 - col * 3;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      coef_f32(col, ch, k, p.W, gl, bl, gr, br, m[i], a[i]);
      if (++ch == 3) {
        ch = 0;
        ++col;
      }
    }
    in_range = coef_in_range(m, a);
    make_coef(m, a, cff);
  }
  // CTA-uniform choice of the arithmetic (Coef16F unless some sub-pixel's
  // map is extreme); the two row loops below never hold both coefficient sets.
  // Only where the register budget holds it without spilling: the MOTION and
  // 7-CTA/SM variants keep the general chain (measured: tools/ab_sustain.py,
  // tools/ab_k3.sh - K3 under the power cap 0.786 -> 0.755 ms per 30 frames,
  // config 4 step 7.32-7.37 -> 7.18-7.21 ms; MOTION with it 4% slower)
  constexpr bool kInRangeChain = !MOTION && (MINB == 0 ? CAMX_K3_MINB : MINB) <= 6;
  const bool fast = kInRangeChain && __syncthreads_and(in_range) != 0;

  // MOTION: the windows of the overlap-0 tiling meeting the CTA (<= 3 window
  // columns x 3 window rows: camx_motion_supported), this thread's
  // pixel-start bits per window column; per-window-column counts `acc` of
  // the rows since the last change of the set of window rows containing the
  // row, flushed (warp sum + one atomic per window) when that set changes
  constexpr int XW = MOTION ? 3 : 1;
  uint32_t xmask[XW], acc[XW];
  int xwin[XW], ywin[XW], ylo[XW];
  int nxs = 0, nys = 0, yset = 0, ynext = 0;
  const int lane = threadIdx.x & 31;
  uint32_t k7 = 0;
  auto yset_at = [&](int R, int &next) {  // window rows containing row R; next change
    int m = 0;
    next = r1;
#pragma unroll
    for (int b2 = 0; b2 < XW; ++b2)
      if (b2 < nys) {
        if (R >= ylo[b2] && R < ylo[b2] + p.win) {
          m |= 1 << b2;
          next = min(next, ylo[b2] + p.win);
        } else if (ylo[b2] > R) {
          next = min(next, ylo[b2]);
        }
      }
    return m;
  };
  auto flush = [&]() {
    const int64_t bb = img / p.cam_count;
#pragma unroll
    for (int a = 0; a < XW; ++a)
      if (a < nxs) {
        const uint32_t c = __reduce_add_sync(0xffffffffu, acc[a]);
        if (lane == 0 && c != 0) {
#pragma unroll
          for (int b2 = 0; b2 < XW; ++b2)
            if (yset & (1 << b2))
              atomicAdd(p.counts + (bb * p.ny + ywin[b2]) * p.nx + xwin[a],
                        static_cast<unsigned long long>(c));
        }
        acc[a] = 0;
      }
  };
  if (MOTION && prev0 != nullptr) {
    const int cam = p.cam_begin + static_cast<int>(img % p.cam_count);
    const int cb0 = cg * kApplyThreads * 16;
    const int X0 = cam * p.W + (cb0 + 2) / 3;
    const int X1 = cam * p.W + (cb0 + static_cast<int>(seg) + 2) / 3;
    auto wins = [](int a0, int a1, int S, int n, int nreg, int len, int *out) {
      // <= XW by the host's geometry check (camx_motion_supported)
      int m = 0;
      for (int i = a0 / S; i <= (a1 - 1) / S && i < nreg && m < XW; ++i) out[m++] = i;
      if (n > nreg && len - S < a1 && m < XW) out[m++] = n - 1;  // the clamped last window
      return m;
    };
    nxs = wins(X0, X1, p.win, p.nx, p.nx_reg, p.mosaic_w, xwin);
    nys = wins(r0, r1, p.win, p.ny, p.ny_reg, p.H, ywin);
#pragma unroll
    for (int a = 0; a < XW; ++a) {
      xmask[a] = 0;
      acc[a] = 0;
      ylo[a] = a < nys ? (ywin[a] < p.ny_reg ? ywin[a] * p.win : p.H - p.win) : 0;
    }
    const int ph = (3 - j % 3) % 3;  // first pixel start in the chunk (16 j + ph = 0 mod 3)
    for (int a = 0; a < nxs && active; ++a) {  // inactive threads count nothing
      const int wx0 = xwin[a] < p.nx_reg ? xwin[a] * p.win : p.mosaic_w - p.win;
      for (int sb = ph; sb < 16; sb += 3) {
        const int x = cam * p.W + (j * 16 + sb) / 3;
        if (x >= wx0 && x < wx0 + p.win) xmask[a] |= 1u << sb;
      }
    }
    yset = yset_at(r0, ynext);
    k7 = static_cast<uint32_t>(127 - (p.t_motion & 127)) * 0x01010101u;  // MHI: t >= 128
  }
  // the next chunk's first 2 bytes: the next thread's chunk, or the 16
  // extra bytes past the group; none at the row end
  const uint32_t next_mask = (threadIdx.x + 1 < chunks || extra) ? 3u : 0u;

  uint8_t *const dst0 = p.dst + img * p.img_bytes + static_cast<int64_t>(r0) * rb + j * 16;
  auto stream_rows = [&](const auto cf) {
  uint8_t *dst = dst0;  // row st * ROWS of the split
  for (int st = 0; st < nst; ++st, dst += ROWS * rb) {
    const int slot = st % STAGES;
    mbar_wait(&full[slot], (st / STAGES) & 1);
    const int rr = min(ROWS, nrows - st * ROWS);
    uint4 v[ROWS];
#pragma unroll
    for (int i = 0; i < ROWS; ++i)  // (inactive threads read ring bytes they never use)
      if (i < rr) v[i] = ring[(slot * ROWS + i) * RS + threadIdx.x];
    if (active) {
#pragma unroll
      for (int i = 0; i < ROWS; ++i)
        if (i < rr) {
          const uint4 o = correct16(v[i], cf);
          st_stream_v4(dst + i * rb, o);
        }
    }
    if (MOTION && prev0 != nullptr) {
#pragma unroll
      for (int i = 0; i < ROWS; ++i)
        if (i < rr) {  // CTA-uniform
          // branch-free: inactive threads have no pixel bits (xmask 0); the
          // next chunk's word is always in the ring (the row has a spare 16
          // bytes, the ring a spare 16 at its end), masked at the row end
          const uint4 *row = ring + (slot * ROWS + i) * RS;
          const uint32_t nc = reinterpret_cast<const uint32_t *>(row + threadIdx.x + 1)[0];
          const uint32_t np =
              reinterpret_cast<const uint32_t *>(row + kApplyThreads + 2 + threadIdx.x)[0];
          const uint32_t E = flags16<MHI>(v[i], row[kApplyThreads + 1 + threadIdx.x], k7) |
                             ((gt_nibble<MHI>(nc, np, k7) & next_mask) << 16);
          const uint32_t on = E | (E >> 1) | (E >> 2);
#pragma unroll
          for (int a = 0; a < XW; ++a) acc[a] += __popc(on & xmask[a]);  // 0 past nxs
          const int R1 = r0 + st * ROWS + i + 1;  // the set of window rows changes after row i?
          if (R1 == ynext) {
            flush();
            yset = yset_at(R1, ynext);
          }
        }
    }
    __syncthreads();  // slot consumed
    if (threadIdx.x == 0 && st + STAGES < nst) issue(st + STAGES);
  }
  };
  if (fast)
    stream_rows(cff);
  else
    stream_rows(general_coef(cff));
  if (MOTION && prev0 != nullptr) flush();
}

// ------------------------------------------------------------- generic path
// Any width / alignment (rows not 16-byte multiples): thread = one pixel
// column of one row block (split) of one image; the three channels' float32
// (M, A) are made once and the block's rows are streamed with byte loads and
// stores (a warp covers 96 contiguous bytes of a row).  Same float32 chain
// as the reference: rn(p * M), + A, rint, clip.
constexpr int kColThreads = 128;
__global__ void __launch_bounds__(kColThreads) apply_cols_kernel(const ApplyParams p,
                                                                 int64_t img0) {
  const int col = blockIdx.x * kColThreads + threadIdx.x;
  if (col >= p.W) return;
  const int k = static_cast<int>(blockIdx.y) / p.row_splits;
  const int rs = static_cast<int>(blockIdx.y) - k * p.row_splits;
  const int64_t img = img0 + blockIdx.z;
  const int blk_r0 = k * p.bh;
  const int blk_r1 = (k == p.K - 1) ? p.H : blk_r0 + p.bh;
  const int r0 = blk_r0 + rs * p.rows_per_split;
  const int r1 = min(blk_r1, r0 + p.rows_per_split);
  if (r0 >= r1) return;
  const double *gl, *bl, *gr, *br;
  map_ptrs(p, img, gl, bl, gr, br);
  float m[3], a[3];
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) coef_f32(col, ch, k, p.W, gl, bl, gr, br, m[ch], a[ch]);
  const int64_t off = img * p.img_bytes + static_cast<int64_t>(r0) * p.row_bytes + col * 3;
  const uint8_t *s = p.src + off;
  uint8_t *d = p.dst + off;
  for (int r = r0; r < r1; ++r, s += p.row_bytes, d += p.row_bytes) {
    const uint32_t v0 = s[0], v1 = s[1], v2 = s[2];
    const uint32_t v[3] = {v0, v1, v2};
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      float y = __fadd_rn(__fmul_rn(static_cast<float>(v[ch]), m[ch]), a[ch]);
      y = fminf(fmaxf(rintf(y), 0.0f), 255.0f);
      d[ch] = static_cast<uint8_t>(y);
    }
  }
}

// Decomposition of the fast path (shared by K3 and the tile fix-up).
static bool plan_fast(ApplyParams &p) {
  const bool aligned = (p.row_bytes % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(p.src) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(p.dst) % 16 == 0);
  if (!aligned) return false;
  p.chunks_per_row = p.row_bytes / 16;
  p.col_groups = (p.chunks_per_row + kApplyThreads - 1) / kApplyThreads;
  // Whole block rows per CTA unless the grid would under-fill the GPU.
  const int max_rows = p.H - (p.K - 1) * p.bh;  // last block is the tallest
  const int64_t base = static_cast<int64_t>(p.n_img) * p.K * p.col_groups;
  int splits = 1;
  const int64_t target = static_cast<int64_t>(sm_count()) * 8;
  while (base * splits < target && (max_rows + splits) / (splits + 1) >= 16) ++splits;
  // under ~4 waves of 96-row CTAs (a camera shard's group): halve the CTAs,
  // which then run 7 per SM - the partial last wave and the ramp/drain
  // shrink (one camera x 30 frames: 103.8 -> 96.9 us; profiles/r02)
  if (splits == 1 && base < 4 * static_cast<int64_t>(sm_count()) * CAMX_K3_MINB &&
      (max_rows + 1) / 2 >= 16)
    splits = 2;
  p.row_splits = splits;
  p.rows_per_split = (max_rows + splits - 1) / splits;
  return true;
}

template <int ROWS = kTmaRows, int STAGES = kTmaStages, int MINB = 0, bool MOTION = false,
          bool MHI = false>
static int launch_tma(const ApplyParams &p, cudaStream_t stream) {
  const int64_t grid = static_cast<int64_t>(p.n_img) * p.K * p.col_groups * p.row_splits;
  const size_t smem = STAGES * ROWS * (MOTION ? 2 * (kApplyThreads + 1) : kApplyThreads) * 16 +
                      (MOTION ? 16 : 0);  // MOTION: the last row's next-word read
  cudaError_t e = cudaFuncSetAttribute(apply_tma_kernel<ROWS, STAGES, MINB, MOTION, MHI>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return static_cast<int>(e);
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(static_cast<unsigned>(grid));
  lc.blockDim = dim3(kApplyThreads);
  lc.dynamicSmemBytes = smem;
  lc.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = p.pdl ? 1 : 0;
  e = cudaLaunchKernelEx(&lc, apply_tma_kernel<ROWS, STAGES, MINB, MOTION, MHI>, p);
  return e == cudaSuccess ? launch_status() : static_cast<int>(e);
}

static int launch_apply(ApplyParams &p, cudaStream_t stream) {
  if (p.n_img <= 0 || p.H <= 0 || p.W <= 0) return CAMX_OK;
  if (plan_fast(p)) {
    // short CTAs (<= 48 rows, e.g. 640x480 frames: 30-row blocks) spend more
    // of their life in the prologue / first fills: one more resident CTA per
    // SM (72 registers) hides it (config 1 K3 56.8 -> 51.3 us); whole 96-row
    // blocks run best at 6 (config 2: 0.7275 vs 0.7302 ms per step)
    if (p.rows_per_split <= 48) return launch_tma<kTmaRows, kTmaStages, 7>(p, stream);
    return launch_tma<>(p, stream);
  }
  // unaligned rows: column-per-thread kernel, rows split until the grid has
  // ~8 CTAs per SM
  const int max_rows = p.H - (p.K - 1) * p.bh;
  const int64_t gx = (p.W + kColThreads - 1) / kColThreads;
  const int64_t base = static_cast<int64_t>(p.n_img) * p.K * gx;
  int splits = 1;
  while (base * splits < static_cast<int64_t>(sm_count()) * 8 &&
         (max_rows + splits) / (splits + 1) >= 8)
    ++splits;
  p.row_splits = splits;
  p.rows_per_split = (max_rows + splits - 1) / splits;
  for (int64_t i0 = 0; i0 < p.n_img; i0 += 65535) {  // images ride on gridDim.z
    const int64_t n = std::min<int64_t>(65535, p.n_img - i0);
    const dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(p.K * splits),
                    static_cast<unsigned>(n));
    apply_cols_kernel<<<grid, kColThreads, 0, stream>>>(p, i0);
    const int st = launch_status();
    if (st != CAMX_OK) return st;
  }
  return CAMX_OK;
}

}  // namespace camx

using namespace camx;

namespace camx {
int launch_seam_solve(const camx_band_stat *stats, int32_t n_batch, int32_t n_cams, int32_t wrap,
                      const camx_solve_config *cfg, const double *prev_gain,
                      const double *prev_offset, double *gain_out, double *offset_out,
                      uint8_t *fit_ok_out, cudaStream_t stream, bool pdl, int32_t world = 1,
                      int32_t cmax = 0);
}

extern "C" int camx_apply_array(const uint8_t *images, uint8_t *out, int32_t n_batch,
                                int32_t cam_begin, int32_t cam_count, int32_t n_cams_total,
                                int32_t wrap, int32_t height, int32_t width, int32_t blocks,
                                const double *gain, const double *offset, void *stream) {
  if (n_batch < 0 || cam_count < 0 || cam_begin < 0 || cam_begin + cam_count > n_cams_total)
    return CAMX_EINVAL;
  if (height < 1 || width < 1 || blocks < 1 || blocks > height) return CAMX_EINVAL;
  if (wrap && n_cams_total < 2) return CAMX_EINVAL;
  if (images == nullptr || out == nullptr) return CAMX_EINVAL;
  const int S = wrap ? n_cams_total : n_cams_total - 1;
  if (S > 0 && (gain == nullptr || offset == nullptr)) return CAMX_EINVAL;
  ApplyParams p{};
  p.src = images;
  p.dst = out;
  p.H = height;
  p.W = width;
  p.K = blocks;
  p.bh = height / blocks;
  p.row_bytes = width * 3;
  p.img_bytes = static_cast<int64_t>(height) * width * 3;
  p.n_img = n_batch * cam_count;
  p.single = 0;
  p.cam_begin = cam_begin;
  p.cam_count = cam_count;
  p.n_cams = n_cams_total;
  p.wrap = wrap;
  p.S = S;
  p.gain = gain;
  p.offset = offset;
  return launch_apply(p, as_stream(stream));
}

extern "C" int camx_apply_map(const uint8_t *images, uint8_t *out, int64_t n_images,
                              int32_t height, int32_t width, int32_t side, int32_t blocks,
                              const double *gain, const double *offset, void *stream) {
  if (n_images < 0 || height < 1 || width < 1 || blocks < 1 || blocks > height) return CAMX_EINVAL;
  if (side != CAMX_SIDE_LEFT && side != CAMX_SIDE_RIGHT) return CAMX_EINVAL;
  if (images == nullptr || out == nullptr || gain == nullptr || offset == nullptr)
    return CAMX_EINVAL;
  ApplyParams p{};
  p.src = images;
  p.dst = out;
  p.H = height;
  p.W = width;
  p.K = blocks;
  p.bh = height / blocks;
  p.row_bytes = width * 3;
  p.img_bytes = static_cast<int64_t>(height) * width * 3;
  p.n_img = static_cast<int32_t>(n_images);
  p.single = 1;
  p.single_side = side;
  p.cam_count = 1;
  p.n_cams = 1;
  p.gain = gain;
  p.offset = offset;
  return launch_apply(p, as_stream(stream));
}

namespace camx {

// K1 (+ K2 as a programmatic dependent) for a whole batch.
int band_stats_seq(const uint8_t *images, const uint8_t *prev_images, const uint8_t *excl_masks,
                   int64_t n_images, int64_t prev_seq, int32_t height, int32_t width,
                   int32_t band_width, int32_t blocks, int32_t t_diff, camx_band_stat *stats_out,
                   uint32_t *hist_out, void *stream);

// K1 over a batch: n_batch frames of `per_frame` images, frames 1.. against
// their predecessors and frame 0 against prev_frame when `removal`.
int band_stats_frames(const uint8_t *images, const uint8_t *prev_frame, int32_t n_batch,
                             int32_t per_frame, int32_t height, int32_t width, int32_t band_width,
                             int32_t blocks, int32_t t_diff, bool removal, camx_band_stat *stats,
                             uint32_t *hist, void *stream) {
  const int64_t frame_bytes = static_cast<int64_t>(height) * width * 3 * per_frame;
  const int64_t rec_frame = static_cast<int64_t>(per_frame) * 2 * blocks;
  int st;
  if (removal && n_batch > 1 && prev_frame != nullptr)  // one launch for the whole batch
    return band_stats_seq(images, prev_frame, nullptr, int64_t(n_batch) * per_frame, per_frame,
                          height, width, band_width, blocks, t_diff, stats, hist, stream);
  if (removal && n_batch > 1) {  // no previous frame: array-frame 0 unmasked
    st = camx_band_stats(images + frame_bytes, images, nullptr, (n_batch - 1) * int64_t(per_frame),
                         height, width, band_width, blocks, t_diff, stats + rec_frame,
                         hist == nullptr ? nullptr : hist + rec_frame * 768, stream);
    if (st != CAMX_OK) return st;
    return camx_band_stats(images, prev_frame, nullptr, per_frame, height, width, band_width,
                           blocks, t_diff, stats, hist, stream);
  }
  return camx_band_stats(images, removal ? prev_frame : nullptr, nullptr,
                         int64_t(n_batch) * per_frame, height, width, band_width, blocks, t_diff,
                         stats, hist, stream);
}

static int stats_and_solve(const uint8_t *images, const uint8_t *prev_frame, int32_t n_batch,
                           int32_t n_cams, int32_t wrap, int32_t height, int32_t width,
                           int32_t band_width, int32_t t_diff, const camx_solve_config *cfg,
                           const double *prev_gain, const double *prev_offset,
                           camx_band_stat *stats, uint32_t *hist, double *gain_out,
                           double *offset_out, uint8_t *fit_ok_out, void *stream) {
  if (cfg == nullptr || images == nullptr || stats == nullptr) return CAMX_EINVAL;
  if (gain_out == nullptr || offset_out == nullptr) return CAMX_EINVAL;
  if (n_batch < 1 || n_cams < 2 || cfg->blocks < 1 || cfg->blocks > height) return CAMX_EINVAL;
  if (cfg->mode < CAMX_MODE_STANDARD || cfg->mode > CAMX_MODE_SMOOTHING) return CAMX_EINVAL;
  if (cfg->have_prev_maps && (prev_gain == nullptr || prev_offset == nullptr)) return CAMX_EINVAL;
  const bool removal = cfg->mode == CAMX_MODE_OBJECT_REMOVAL;
  const int st = band_stats_frames(images, prev_frame, n_batch, n_cams, height, width, band_width,
                                   cfg->blocks, t_diff, removal, stats, hist, stream);
  if (st != CAMX_OK) return st;
  return launch_seam_solve(stats, n_batch, n_cams, wrap, cfg, prev_gain, prev_offset, gain_out,
                           offset_out, fit_ok_out, as_stream(stream), true);
}

static ApplyParams array_params(const uint8_t *images, uint8_t *out, int32_t n_batch,
                                int32_t n_cams, int32_t wrap, int32_t height, int32_t width,
                                int32_t blocks, const double *gain, const double *offset) {
  ApplyParams p{};
  p.src = images;
  p.dst = out;
  p.H = height;
  p.W = width;
  p.K = blocks;
  p.bh = height / blocks;
  p.row_bytes = width * 3;
  p.img_bytes = static_cast<int64_t>(height) * width * 3;
  p.n_img = n_batch * n_cams;
  p.cam_begin = 0;
  p.cam_count = n_cams;
  p.n_cams = n_cams;
  p.wrap = wrap;
  p.S = wrap ? n_cams : n_cams - 1;
  p.gain = gain;
  p.offset = offset;
  return p;
}

extern "C" int camx_tiles(const uint8_t *images, int32_t n_cams, int32_t height, int32_t width,
                          const int32_t *windows, int32_t n_tiles, int32_t size, int32_t out_size,
                          uint8_t *tiles_out, void *stream);
int tiles_after_apply(const uint8_t *images, int32_t n_cams, int32_t height, int32_t width,
                      const int32_t *windows, int32_t n_tiles, int32_t size, int32_t out_size,
                      uint8_t *tiles_out, void *stream);

// K3 then K5 (camx_tiles' TMA-staged resample reading the corrected frames).
// windows are (b, x, y) triples; frame_off / max_tiles_per_frame describe
// their grouping by array-frame (ABI v1; not needed by this schedule).
static int apply_and_tile(ApplyParams &p, const int32_t *windows, const int32_t *frame_off,
                          int32_t n_tiles, int32_t max_tiles_per_frame, int32_t size,
                          int32_t out_size, uint8_t *tiles_out, void *stream) {
  (void)frame_off;
  (void)max_tiles_per_frame;
  if (n_tiles < 0 || size < 1 || out_size < 1 || size > p.H || size > p.n_cams * p.W)
    return CAMX_EINVAL;
  if (n_tiles > 0 && (windows == nullptr || tiles_out == nullptr)) return CAMX_EINVAL;
  int st = launch_apply(p, as_stream(stream));
  if (st != CAMX_OK || n_tiles == 0) return st;
  return tiles_after_apply(p.dst, p.n_cams, p.H, p.W, windows, n_tiles, size, out_size,
                           tiles_out, stream);
}

}  // namespace camx
using namespace camx;

extern "C" int camx_correct_batch(const uint8_t *images, uint8_t *out, const uint8_t *prev_frame,
                                  int32_t n_batch, int32_t n_cams, int32_t wrap, int32_t height,
                                  int32_t width, int32_t band_width, int32_t t_diff,
                                  const camx_solve_config *cfg, const double *prev_gain,
                                  const double *prev_offset, camx_band_stat *stats,
                                  uint32_t *hist, double *gain_out, double *offset_out,
                                  uint8_t *fit_ok_out, int32_t *counters, void *stream) {
  (void)counters;  // reserved (ABI v1 slot; may be NULL)
  if (out == nullptr) return CAMX_EINVAL;
  int st = stats_and_solve(images, prev_frame, n_batch, n_cams, wrap, height, width, band_width,
                           t_diff, cfg, prev_gain, prev_offset, stats, hist, gain_out, offset_out,
                           fit_ok_out, stream);
  if (st != CAMX_OK) return st;
  ApplyParams p = array_params(images, out, n_batch, n_cams, wrap, height, width, cfg->blocks,
                               gain_out, offset_out);
  p.pdl = 1;  // K3 is a programmatic dependent of K2
  return launch_apply(p, as_stream(stream));
}

// Origins of the overlap-0 tiling along one axis (attention.py:53-63 with
// stride == size): `nreg` regular windows at i * size (i * size + size <
// len), then the clamped last window at len - size (never a duplicate).
static void tiling_axis(int len, int size, int &n, int &nreg) {
  nreg = len > size ? (len - size + size - 1) / size : 0;
  n = nreg + 1;
}

extern "C" int camx_tiling_size(int32_t mosaic_w, int32_t mosaic_h, int32_t size, int32_t *nx,
                                int32_t *ny) {
  if (size < 1 || size > mosaic_w || size > mosaic_h || nx == nullptr || ny == nullptr)
    return CAMX_EINVAL;
  int a, b;
  tiling_axis(mosaic_w, size, a, b);
  *nx = a;
  tiling_axis(mosaic_h, size, a, b);
  *ny = a;
  return CAMX_OK;
}

// Windows of the overlap-0 tiling meeting [a0, a1) (regular + clamped).
static int windows_meeting(int a0, int a1, int S, int n, int nreg, int len) {
  int m = 0;
  for (int i = a0 / S; i <= (a1 - 1) / S && i < nreg; ++i) ++m;
  return m + ((n > nreg && len - S < a1) ? 1 : 0);
}

// The fused motion counts keep <= 3 x 3 windows per K3 CTA in registers:
// the largest number of windows any CTA's columns / rows meet.
static bool motion_fits(const ApplyParams &p, int size) {
  int nx, nxr, ny, nyr;
  tiling_axis(p.n_cams * p.W, size, nx, nxr);
  tiling_axis(p.H, size, ny, nyr);
  const int cgb = kApplyThreads * 16;
  for (int cam = 0; cam < p.n_cams; ++cam)
    for (int cg = 0; cg < p.col_groups; ++cg) {
      const int cb0 = cg * cgb, seg = std::min(cgb, p.row_bytes - cb0);
      const int X0 = cam * p.W + (cb0 + 2) / 3, X1 = cam * p.W + (cb0 + seg + 2) / 3;
      if (windows_meeting(X0, X1, size, nx, nxr, p.n_cams * p.W) > 3) return false;
    }
  for (int k = 0; k < p.K; ++k)
    for (int rs = 0; rs < p.row_splits; ++rs) {
      const int r0 = k * p.bh + rs * p.rows_per_split;
      const int r1 = std::min(k == p.K - 1 ? p.H : (k + 1) * p.bh, r0 + p.rows_per_split);
      if (r0 < r1 && windows_meeting(r0, r1, size, ny, nyr, p.H) > 3) return false;
    }
  return true;
}

// K3 with the motion counts needs 16-byte aligned rows and <= 3 x 3 windows
// per CTA for this launch's decomposition.
static bool motion_plan(ApplyParams &p, int size) { return plan_fast(p) && motion_fits(p, size); }

extern "C" int camx_motion_supported(int32_t n_batch, int32_t n_cams, int32_t cam_count,
                                     int32_t height, int32_t width, int32_t blocks,
                                     int32_t size) {
  if (n_batch < 1 || n_cams < 2 || height < 1 || width < 1 || blocks < 1 || blocks > height)
    return 0;
  if (cam_count < 1 || cam_count > n_cams) return 0;
  if (size < 1 || size > n_cams * width || size > height) return 0;
  alignas(16) uint8_t dummy[16];
  ApplyParams p = array_params(dummy, dummy, n_batch, cam_count, 0, height, width, blocks,
                               nullptr, nullptr);
  p.n_cams = n_cams;
  return motion_plan(p, size) ? 1 : 0;
}

#ifndef CAMX_K3M_STAGES
#define CAMX_K3M_STAGES 5
#endif
#ifndef CAMX_K3M_MINB
#define CAMX_K3M_MINB 5
#endif

namespace camx {
// Motion fields of p (planned by motion_plan) and the K3 <MOTION> launch:
// 5 stages x 2 rows x (2 KB + 16 B) x 2 frames = 41 KB per CTA, 5 CTAs/SM
// (96 registers): 1.12 ms per 30 config-2 frames incl. K1 + K2, vs 1.19 at 4
// stages, 1.26 at 6 x 4 CTAs, 1.23-1.31 at 6 CTAs/SM (80 registers, spills);
// profiles/r02/SUMMARY.md.  Counts accumulate (atomics) into `counts`.
int launch_motion_apply(ApplyParams &p, const uint8_t *motion_prev, int32_t win_size,
                        int32_t t_motion, int64_t *counts, cudaStream_t stream) {
  const int32_t mw = p.n_cams * p.W;
  tiling_axis(mw, win_size, p.nx, p.nx_reg);
  tiling_axis(p.H, win_size, p.ny, p.ny_reg);
  p.win = win_size;
  p.mosaic_w = mw;
  p.t_motion = t_motion;
  p.prev_first = motion_prev;
  p.counts = reinterpret_cast<unsigned long long *>(counts);
  constexpr int kS = CAMX_K3M_STAGES, kB = CAMX_K3M_MINB;
  if (t_motion >= 128) return launch_tma<kTmaRows, kS, kB, true, true>(p, stream);
  return launch_tma<kTmaRows, kS, kB, true, false>(p, stream);
}

// The sharded K3 with counts (camx_shard.cu): this rank's cameras, counts of
// its pixels only (the ranks' counts sum to the array's).
int apply_camera_group_motion(const uint8_t *images, uint8_t *out, int nb, int cam_begin,
                              int cam_count, int n_cams, int wrap, int height, int width,
                              int blocks, const double *gain, const double *offset,
                              const uint8_t *motion_prev, int32_t win_size, int32_t t_motion,
                              int64_t *counts, cudaStream_t s) {
  ApplyParams p = array_params(images, out, nb, cam_count, wrap, height, width, blocks, gain,
                               offset);
  p.cam_begin = cam_begin;
  p.n_cams = n_cams;
  p.S = wrap ? n_cams : n_cams - 1;
  if (!motion_plan(p, win_size)) return CAMX_EINVAL;
  return launch_motion_apply(p, motion_prev, win_size, t_motion, counts, s);
}
}  // namespace camx

extern "C" int camx_correct_batch_motion(
    const uint8_t *images, uint8_t *out, const uint8_t *prev_frame, int32_t n_batch,
    int32_t n_cams, int32_t wrap, int32_t height, int32_t width, int32_t band_width,
    int32_t t_diff, const camx_solve_config *cfg, const double *prev_gain,
    const double *prev_offset, camx_band_stat *stats, uint32_t *hist, double *gain_out,
    double *offset_out, uint8_t *fit_ok_out, const uint8_t *motion_prev, int32_t win_size,
    int32_t t_motion, int64_t *counts_out, void *stream) {
  if (out == nullptr || counts_out == nullptr || cfg == nullptr) return CAMX_EINVAL;
  if (n_batch < 1 || n_cams < 2 || height < 1 || width < 1) return CAMX_EINVAL;
  if (cfg->blocks < 1 || cfg->blocks > height) return CAMX_EINVAL;
  if (t_motion < 0 || t_motion > 255) return CAMX_EINVAL;
  const int32_t mw = n_cams * width;
  if (win_size < 1 || win_size > mw || win_size > height) return CAMX_EINVAL;
  ApplyParams p = array_params(images, out, n_batch, n_cams, wrap, height, width, cfg->blocks,
                               gain_out, offset_out);
  // 16-byte aligned rows and <= 3 x 3 windows per CTA (camx_motion_supported)
  if (!motion_plan(p, win_size)) return CAMX_EINVAL;
  int nx, nxr, ny, nyr;
  tiling_axis(mw, win_size, nx, nxr);
  tiling_axis(height, win_size, ny, nyr);
  // zeroed before K1, so that K2 -> K3 stay programmatically chained
  cudaError_t e = cudaMemsetAsync(counts_out, 0,
                                  sizeof(int64_t) * static_cast<size_t>(n_batch) * nx * ny,
                                  as_stream(stream));
  if (e != cudaSuccess) return static_cast<int>(e);
  int st = stats_and_solve(images, prev_frame, n_batch, n_cams, wrap, height, width, band_width,
                           t_diff, cfg, prev_gain, prev_offset, stats, hist, gain_out, offset_out,
                           fit_ok_out, stream);
  if (st != CAMX_OK) return st;
  p.pdl = 1;
  return launch_motion_apply(p, motion_prev, win_size, t_motion, counts_out, as_stream(stream));
}

namespace camx {
// K3 over this rank's cameras of nb frames (camx_shard.cu).
int apply_camera_group(const uint8_t *images, uint8_t *out, int nb, int cam_begin, int cam_count,
                       int n_cams, int wrap, int height, int width, int blocks,
                       const double *gain, const double *offset, bool pdl, cudaStream_t s) {
  ApplyParams p = array_params(images, out, nb, cam_count, wrap, height, width, blocks, gain,
                               offset);
  p.cam_begin = cam_begin;
  p.n_cams = n_cams;
  p.S = wrap ? n_cams : n_cams - 1;
  p.pdl = pdl ? 1 : 0;
  return launch_apply(p, s);
}
}  // namespace camx

extern "C" int camx_correct_batch_tiles(
    const uint8_t *images, uint8_t *out, const uint8_t *prev_frame, int32_t n_batch,
    int32_t n_cams, int32_t wrap, int32_t height, int32_t width, int32_t band_width,
    int32_t t_diff, const camx_solve_config *cfg, const double *prev_gain,
    const double *prev_offset, camx_band_stat *stats, uint32_t *hist, double *gain_out,
    double *offset_out, uint8_t *fit_ok_out, const int32_t *windows, const int32_t *frame_off,
    int32_t n_tiles, int32_t max_tiles_per_frame, int32_t size, int32_t out_size,
    uint8_t *tiles_out, void *stream) {
  if (out == nullptr) return CAMX_EINVAL;
  int st = stats_and_solve(images, prev_frame, n_batch, n_cams, wrap, height, width, band_width,
                           t_diff, cfg, prev_gain, prev_offset, stats, hist, gain_out, offset_out,
                           fit_ok_out, stream);
  if (st != CAMX_OK) return st;
  ApplyParams p = array_params(images, out, n_batch, n_cams, wrap, height, width, cfg->blocks,
                               gain_out, offset_out);
  p.pdl = 1;
  return apply_and_tile(p, windows, frame_off, n_tiles, max_tiles_per_frame, size, out_size,
                        tiles_out, stream);
}

extern "C" int camx_correct_and_tile(const uint8_t *images, uint8_t *out, int32_t n_batch,
                                     int32_t n_cams, int32_t wrap, int32_t height, int32_t width,
                                     int32_t blocks, const double *gain, const double *offset,
                                     const int32_t *windows, const int32_t *frame_off,
                                     int32_t n_tiles, int32_t max_tiles_per_frame, int32_t size,
                                     int32_t out_size, uint8_t *tiles_out, void *stream) {
  if (images == nullptr || out == nullptr || n_batch < 0 || n_cams < 1) return CAMX_EINVAL;
  if (height < 1 || width < 1 || blocks < 1 || blocks > height) return CAMX_EINVAL;
  if (wrap && n_cams < 2) return CAMX_EINVAL;
  const int S = wrap ? n_cams : n_cams - 1;
  if (S > 0 && (gain == nullptr || offset == nullptr)) return CAMX_EINVAL;
  if (n_batch == 0) return CAMX_OK;
  ApplyParams p = array_params(images, out, n_batch, n_cams, wrap, height, width, blocks, gain,
                               offset);
  return apply_and_tile(p, windows, frame_off, n_tiles, max_tiles_per_frame, size, out_size,
                        tiles_out, stream);
}
