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

// Same arithmetic with 16 fewer live registers (for the fused tile kernel,
// which is occupancy-bound): X - 2^23 = p exactly, then p * (M/256) =
// rn(p*M)/256 (power-of-two scale) - one more instruction per sub-pixel pair.
__device__ __forceinline__ uint32_t correct_word_lean(uint32_t w, const Coef16 &cf, int base) {
  const uint64_t kScale = pack2(256.0f, 256.0f);
  const uint64_t kMagic = pack2(8388608.0f, 8388608.0f);
  const uint64_t kUnmagic = pack2(-8388608.0f, -8388608.0f);
  uint32_t z[4];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int i = base + 2 * h;
    const uint32_t x0 = __byte_perm(w, 0x4B00u, 0x5440u + 2 * h);
    const uint32_t x1 = __byte_perm(w, 0x4B00u, 0x5441u + 2 * h);
    const uint64_t y1 = mul2_rn(add2_rn(pack2u(x0, x1), kUnmagic), cf.m[i >> 1]);
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

template <bool LEAN>
__device__ __forceinline__ uint4 correct16_t(uint4 v, const Coef16 &cf) {
  if (!LEAN) {
    uint4 r;
    r.x = correct_word(v.x, cf, 0);
    r.y = correct_word(v.y, cf, 4);
    r.z = correct_word(v.z, cf, 8);
    r.w = correct_word(v.w, cf, 12);
    return r;
  }
  uint4 r;
  r.x = correct_word_lean(v.x, cf, 0);
  r.y = correct_word_lean(v.y, cf, 4);
  r.z = correct_word_lean(v.z, cf, 8);
  r.w = correct_word_lean(v.w, cf, 12);
  return r;
}

__device__ __forceinline__ uint4 correct16(uint4 v, const Coef16 &cf) {
  uint4 r;
  r.x = correct_word(v.x, cf, 0);
  r.y = correct_word(v.y, cf, 4);
  r.z = correct_word(v.z, cf, 8);
  r.w = correct_word(v.w, cf, 12);
  return r;
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

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Tile fusion (config 5): the corrected rows of every stage are written back
// into their ring slot; each output row of each attention tile whose two
// source rows the CTA holds (the previous stage stays resident: a slot is
// refilled two stages late) is resampled from shared memory for
// the output columns whose two column taps are whole pixels of the CTA's
// byte range.  Outputs whose taps straddle CTAs are produced afterwards by
// tile_fixup_kernel from the corrected frame.
struct TileFuse {
  const int32_t *wins;       // [T][3] (batch, x, y), grouped by batch
  const int32_t *frame_off;  // [B+1] first tile of each array-frame
  uint8_t *tiles;            // [T][out][out][3]
  int32_t size, out;
  float scale;
};
constexpr int kFuseMaxWin = 48;  // windows per array-frame the fused path accepts
// strict downscale only (out < size): i0 is strictly increasing and i1 =
// i0 + 1, so a source row is the second tap of at most one output row per
// window (orow[] is well defined)
// ring of the fused kernel: 4-row stages (one CTA barrier and one hit
// enumeration per stage); refill lags two stages (previous row resident)
#ifndef CAMX_K3_MINB
#define CAMX_K3_MINB 6  // K3 (no tiles): CTAs per SM the register budget is sized for (78 registers)
#endif
#ifndef CAMX_FUSE_ROWS
#define CAMX_FUSE_ROWS 4
#endif
#ifndef CAMX_FUSE_STAGES
#define CAMX_FUSE_STAGES 4
#endif
#ifndef CAMX_FUSE_SPLIT
#define CAMX_FUSE_SPLIT 1  // resample work unit: 0 hit per CTA, 1 hit per warp, 2 half hit per warp
#endif
#ifndef CAMX_FUSE_MINB
#define CAMX_FUSE_MINB 5  // CTAs per SM the register budget is sized for
#endif
constexpr int kFuseRows = CAMX_FUSE_ROWS;
constexpr int kFuseStages = CAMX_FUSE_STAGES;
static_assert(kFuseRows == 4, "hit enumeration uses e >> 2 / e & 3");
// a slot is refilled two stages after it was consumed (the previous stage
// stays resident for the resample): two stages would never be issued
static_assert(kFuseStages >= 3, "the fused ring needs at least 3 stages");

struct FuseSmem {  // carved from dynamic shared memory after the ring
  uint2 *tap;              // [out] (3 * i0, dp2a weights (256 - w1) | w1 << 16);
                           // i1 = i0 + 1 (strict downscale)
  int16_t *orow;           // [size] output row whose second tap is window row lr, or -1
  int4 *win;               // intersecting windows: (tile, x0, y0, lo | hi << 16)
  int32_t *counts;         // [0] n_win
};

__device__ __forceinline__ int tap_i0(uint2 tv) { return static_cast<int>(tv.x) / 3; }

// Shared-memory carve of the fusion state after the ring; every region
// starts 16-byte aligned (int4 records).  fuse_smem_bytes() == the total.
__host__ __device__ __forceinline__ size_t r16(size_t v) { return (v + 15) & ~static_cast<size_t>(15); }
__host__ __device__ __forceinline__ size_t fuse_layout(int out, int size, size_t *off) {
  size_t o = 0;
  off[0] = o; o += r16(8 * static_cast<size_t>(out));   // tap
  off[1] = o; o += r16(2 * static_cast<size_t>(size));  // orow
  off[2] = o; o += sizeof(int4) * kFuseMaxWin;           // win
  off[3] = o; o += 16;                                   // counts
  return o;
}
__device__ __forceinline__ FuseSmem carve_fuse(uint8_t *base, int out, int size) {
  size_t off[4];
  fuse_layout(out, size, off);
  FuseSmem fs;
  fs.tap = reinterpret_cast<uint2 *>(base + off[0]);
  fs.orow = reinterpret_cast<int16_t *>(base + off[1]);
  fs.win = reinterpret_cast<int4 *>(base + off[2]);
  fs.counts = reinterpret_cast<int32_t *>(base + off[3]);
  return fs;
}

// Resample one hit (an output row segment [lo, hi) of one tile) from the
// corrected source rows ra (first tap row) and rb (second tap row) in shared
// memory; threads t, t + nt, ... of the group.  Per pixel: the 6 bytes
// of the two column taps (adjacent pixels) of each row via 3 aligned words
// + funnel shift, channel pairs by PRMT, horizontal blend by dp2a, vertical
// by IMAD, round half up (camx_resize.cuh: bilerp_fx).
__device__ __forceinline__ void resample_hit(const uint8_t *ringb, uint32_t offa, uint32_t offb,
                                             uint32_t wyp, int xc3, uint8_t *trow, int lo, int hi,
                                             int t, int nt, const FuseSmem &fs) {
  const uint32_t wy0 = wyp & 0xFFFFu, wy1 = wyp >> 16;
  // byte offsets into the ring (128-byte aligned), so (offset & 3) is the
  // word shift and the loads stay in shared memory
  const uint32_t a0off = offa + static_cast<uint32_t>(xc3);
  const uint32_t db = offb - offa;
  uint8_t *o = trow + 3 * (lo + t);
  for (int ox = lo + t; ox < hi; ox += nt, o += 3 * nt) {
    const uint2 tv = fs.tap[ox];
    const uint32_t la = a0off + tv.x;
    const uint32_t sh = la * 8u;  // funnel shifts use the low 5 bits
    const uint32_t *wa = reinterpret_cast<const uint32_t *>(ringb + (la & ~3u));
    const uint32_t *wb = reinterpret_cast<const uint32_t *>(ringb + (la & ~3u) + db);
    const uint32_t a0 = wa[0], a1 = wa[1], a2 = wa[2];
    const uint32_t b0 = wb[0], b1 = wb[1], b2 = wb[2];
    const uint32_t alo = __funnelshift_r(a0, a1, sh), ahi = __funnelshift_r(a1, a2, sh);
    const uint32_t blo = __funnelshift_r(b0, b1, sh), bhi = __funnelshift_r(b1, b2, sh);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      const uint32_t sel = 0x0030u + 0x0011u * ch;  // bytes (ch, ch + 3)
      const uint32_t v0 = __dp2a_lo(tv.y, __byte_perm(alo, ahi, sel), 0u);
      const uint32_t v1 = __dp2a_lo(tv.y, __byte_perm(blo, bhi, sel), 0u);
      o[ch] = static_cast<uint8_t>((v0 * wy0 + v1 * wy1 + 32768u) >> 16);
    }
  }
}

// MINB: CTAs per SM the register budget is sized for (0: the default of the
// TILES / plain variant); short-CTA launches use a leaner plain variant.
template <bool TILES, int ROWS, int STAGES, int MINB = 0>
__global__ void __launch_bounds__(kApplyThreads,
                                  MINB > 0 ? MINB : (TILES ? CAMX_FUSE_MINB : CAMX_K3_MINB))
    apply_tma_kernel(const ApplyParams p, const TileFuse q) {
  extern __shared__ __align__(128) uint4 ring[];  // [STAGES][ROWS][kApplyThreads]
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

  auto issue = [&](int st) {
    const int slot = st % STAGES;
    const int rr = min(ROWS, nrows - st * ROWS);
    mbar_expect_tx(&full[slot], seg * rr);
    for (int i = 0; i < rr; ++i)
      bulk_g2s(ring + (slot * ROWS + i) * kApplyThreads,
               src0 + static_cast<int64_t>(st * ROWS + i) * rb, seg, &full[slot]);
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int st = 0; st < min(STAGES, nst); ++st) issue(st);
  }

  // ---- tile fusion prologue (independent of the maps: overlaps the PDL wait)
  FuseSmem fs{};
  int cam = 0, cb0 = 0, px_lo = 0, px_hi = 0;
  int64_t bfr = 0;
  if (TILES) {
    fs = carve_fuse(reinterpret_cast<uint8_t *>(ring + STAGES * ROWS * kApplyThreads),
                    q.out, q.size);
    bfr = img / p.cam_count;
    cam = p.cam_begin + static_cast<int>(img % p.cam_count);
    cb0 = cg * kApplyThreads * 16;
    px_lo = (cb0 + 2) / 3;                       // first whole pixel of the byte range
    px_hi = (cb0 + static_cast<int>(seg)) / 3;   // one past the last whole pixel
    for (int i = threadIdx.x; i < q.out; i += blockDim.x) {
      int a, b, w1;
      src_coord_w(i, q.scale, q.size, a, b, w1);
      fs.tap[i] = make_uint2(3u * static_cast<uint32_t>(a),
                             static_cast<uint32_t>(256 - w1) | (static_cast<uint32_t>(w1) << 16));
      (void)b;  // = a + 1 (strict downscale)
    }
    for (int i = threadIdx.x; i < q.size; i += blockDim.x) fs.orow[i] = -1;
    if (threadIdx.x == 0) fs.counts[0] = 0;
    __syncthreads();  // tap tables complete before the window scan reads them
    for (int i = threadIdx.x; i < q.out; i += blockDim.x) fs.orow[tap_i0(fs.tap[i]) + 1] = static_cast<int16_t>(i);
    // windows of this array-frame that overlap the CTA region (mosaic coords),
    // with the contiguous range [lo, hi) of output columns whose two column
    // taps are whole pixels of this CTA (i0, i1 are nondecreasing in ox)
    const int w_lo = q.frame_off[bfr], w_hi = q.frame_off[bfr + 1];
    const int mx0 = cam * p.W + px_lo, mx1 = cam * p.W + px_hi;
    for (int t = w_lo + threadIdx.x; t < w_hi; t += blockDim.x) {
      const int x0 = q.wins[3 * t + 1], y0 = q.wins[3 * t + 2];
      if (x0 < mx1 && x0 + q.size > mx0 && y0 < r1 && y0 + q.size > r0) {
        const int xc = x0 - cam * p.W;
        int lo = 0, hi = q.out;  // first ox with xc + i0 >= px_lo
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (xc + tap_i0(fs.tap[mid]) >= px_lo) hi = mid; else lo = mid + 1;
        }
        int lo2 = lo, hi2 = q.out;  // first ox with xc + i1 >= px_hi
        while (lo2 < hi2) {
          const int mid = (lo2 + hi2) >> 1;
          if (xc + tap_i0(fs.tap[mid]) + 1 >= px_hi) hi2 = mid; else lo2 = mid + 1;
        }
        if (lo2 > lo) {
          // bounded: the host caps max_tiles_per_frame at kFuseMaxWin, but
          // frame_off is caller data - never write past the shared array
          const int slot = atomicAdd(&fs.counts[0], 1);
          if (slot < kFuseMaxWin) fs.win[slot] = make_int4(t, x0, y0, lo | (lo2 << 16));
        }
      }
    }
  }
  __syncthreads();
  const int nwin = TILES ? min(fs.counts[0], kFuseMaxWin) : 0;
  const int xbase = 3 * cam * p.W + cb0;  // window column -> CTA byte offset
  // maps come from the preceding stats/solve grid (programmatic dependent
  // launch): only the raw-pixel prefetch above may run before it completes
  asm volatile("griddepcontrol.wait;" ::: "memory");

  const bool active = threadIdx.x < chunks;
  const double *gl, *bl, *gr, *br;
  map_ptrs(p, img, gl, bl, gr, br);
  Coef16 cf;
  if (active) {
    // per sub-pixel (a per-column lambda cache measured ~6% slower end to
    // end on B200: tools/ab_k3.py)
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
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      cf.m[i >> 1] = pack2(m[i] * 0.00390625f, m[i + 1] * 0.00390625f);
      if (!TILES) cf.c[i >> 1] = pack2(m[i] * -32768.0f, m[i + 1] * -32768.0f);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i)
      cf.a[i] = fabsf(a[i]) < 7.7037197787136e-34f ? 0.0f : a[i] * 0.00390625f;
  }

  uint8_t *dst = p.dst + img * p.img_bytes + static_cast<int64_t>(r0) * rb + j * 16;
  for (int st = 0; st < nst; ++st) {
    const int slot = st % STAGES;
    mbar_wait(&full[slot], (st / STAGES) & 1);
    const int rr = min(ROWS, nrows - st * ROWS);
    if (active) {
      uint4 v[ROWS];
#pragma unroll
      for (int i = 0; i < ROWS; ++i)
        if (i < rr) v[i] = ring[(slot * ROWS + i) * kApplyThreads + threadIdx.x];
#pragma unroll
      for (int i = 0; i < ROWS; ++i)
        if (i < rr) {
          const uint4 o = correct16_t<TILES>(v[i], cf);
          st_stream_v4(dst + static_cast<int64_t>(st * ROWS + i) * rb, o);
          if (TILES) ring[(slot * ROWS + i) * kApplyThreads + threadIdx.x] = o;
        }
    }
    // TILES: the corrected rows were written into the slot through the
    // generic proxy and the slot is refilled by cp.async.bulk (async proxy)
    // two stages later: order the writes before that refill (PTX memory
    // model: fence.proxy.async between the proxies)
    if (TILES) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();  // slot consumed (and, with TILES, corrected rows visible)
    if (TILES) {
      // every thread has finished the previous stage's resample (it came
      // before this barrier): the slot of stage st-2 is free
      if (threadIdx.x == 0 && st >= 2 && st - 2 + STAGES < nst) issue(st - 2 + STAGES);
      // Hits of this stage (one output-row segment of one tile each): every
      // warp enumerates the same (window, row) pairs in the same order in
      // registers, so the 128 threads split each hit's columns consistently
      // with no shared hit list and no second barrier.
      const uint8_t *ringb = reinterpret_cast<const uint8_t *>(ring);
      const int lane = threadIdx.x & 31;
#if CAMX_FUSE_SPLIT != 0
      const int warp = threadIdx.x >> 5;
      int hit_seq = st;  // rotates which warp takes a stage's first hit
#endif
      const int rs0 = st * ROWS;  // CTA-relative first row of the stage
      for (int e0 = 0; e0 < 4 * nwin; e0 += 32) {
        const int e = e0 + lane;
        const int ri = e & 3;
        bool ok = false;
        uint32_t offs = 0, wpk = 0;
        int xc3 = 0, lohi = 0;
        uint64_t trow = 0;
        if (e < 4 * nwin && ri < rr) {
          const int4 w = fs.win[e >> 2];
          const int R = r0 + rs0 + ri;
          const int lr = R - w.z;
          const int oy = (lr >= 0 && lr < q.size) ? fs.orow[lr] : -1;
          if (oy >= 0) {
            const uint2 tv = fs.tap[oy];
            const int ra = w.z + tap_i0(tv) - r0;  // first tap row, CTA-relative
            if (ra >= 0) {  // else it belongs to the previous CTA (fix-up kernel)
              ok = true;
              const int rb = rs0 + ri;
              offs = static_cast<uint32_t>(((ra / ROWS) % STAGES * ROWS + ra % ROWS) *
                                           kApplyThreads * 16) |
                     (static_cast<uint32_t>(((rb / ROWS) % STAGES * ROWS + ri) * kApplyThreads * 16)
                      << 16);
              wpk = tv.y;
              xc3 = 3 * w.y - xbase;
              lohi = w.w;
              trow = reinterpret_cast<uint64_t>(
                  q.tiles + (static_cast<int64_t>(w.x) * q.out + oy) * q.out * 3);
            }
          }
        }
        unsigned bal = __ballot_sync(0xffffffffu, ok);
        while (bal) {
          const int src = __ffs(bal) - 1;
          bal &= bal - 1u;
#if CAMX_FUSE_SPLIT == 0
          // every hit split over the CTA's 128 threads
          const int t0 = threadIdx.x, nt = kApplyThreads;
#else
          // hits (CAMX_FUSE_SPLIT 1) or half hits (2) dealt round-robin to the
          // warps: the per-hit broadcast and set-up run once per hit instead
          // of once per warp; the sequence is identical in every warp
          const int j = hit_seq++;
          const int t0 = lane, nt = 32;
#if CAMX_FUSE_SPLIT == 1
          if ((j & 3) != warp) continue;
#else
          const int half = (warp - 2 * j) & 3;
          if (half > 1) continue;
#endif
#endif
          const uint32_t o = __shfl_sync(0xffffffffu, offs, src);
          const uint32_t wp = __shfl_sync(0xffffffffu, wpk, src);
          const int x3 = __shfl_sync(0xffffffffu, xc3, src);
          const int lh = __shfl_sync(0xffffffffu, lohi, src);
          const uint32_t tl = __shfl_sync(0xffffffffu, static_cast<uint32_t>(trow), src);
          const uint32_t th = __shfl_sync(0xffffffffu, static_cast<uint32_t>(trow >> 32), src);
          int hlo = lh & 0xFFFF, hhi = lh >> 16;
#if CAMX_FUSE_SPLIT == 2
          const int mid = hlo + ((hhi - hlo + 1) >> 1);
          if (half == 0) hhi = mid; else hlo = mid;
#endif
          resample_hit(ringb, o & 0xFFFFu, o >> 16, wp, x3,
                          reinterpret_cast<uint8_t *>((static_cast<uint64_t>(th) << 32) | tl),
                          hlo, hhi, t0, nt, fs);
        }
      }
    } else {
      if (threadIdx.x == 0 && st + STAGES < nst) issue(st + STAGES);
    }
  }
}

// Tile outputs the fused kernel could not produce (taps straddling CTA rows
// or column groups), resampled from the corrected frame.  One CTA per tile.
__device__ __forceinline__ int row_cta(const ApplyParams &p, int r) {
  const int k = min(r / p.bh, p.K - 1);
  return k * p.row_splits + (r - k * p.bh) / p.rows_per_split;
}
__device__ __forceinline__ int col_cta(const ApplyParams &p, int mx) {
  // whole-pixel column group of mosaic column mx, or -1 if the pixel's bytes
  // straddle two groups
  const int camc = mx / p.W, px = mx - camc * p.W;
  const int g0 = (3 * px) / (kApplyThreads * 16), g1 = (3 * px + 2) / (kApplyThreads * 16);
  return g0 == g1 ? camc * p.col_groups + g0 : -1 - camc;
}

// Per-tile tables (dynamic shared memory, fixup_smem_bytes()): for every
// output column the byte offsets of its two column taps inside an image row
// (camera image + pixel) and its weight; for every output row the byte
// offsets of its two tap rows and its weight; then the bad-column / bad-row
// lists.  Source bytes come through the read-only path (the corrected frame
// is not written by this kernel), so the loads of several outputs overlap.
struct FixupSmem {
  int64_t *cola, *colb;  // [out] image-relative byte offset of column taps a, b
  int32_t *rowa, *rowb;  // [out] row byte offset of row taps a, b
  int32_t *colw, *roww;  // [out] fixed-point weights
  int32_t *colbad, *rowbad;
};
__host__ __device__ __forceinline__ size_t fixup_smem_bytes(int out) {
  return static_cast<size_t>(out) * (2 * sizeof(int64_t) + 6 * sizeof(int32_t));
}

__global__ void __launch_bounds__(256) tile_fixup_kernel(const ApplyParams p, const TileFuse q) {
  extern __shared__ __align__(16) uint8_t fx_raw[];
  FixupSmem fs;
  fs.cola = reinterpret_cast<int64_t *>(fx_raw);
  fs.colb = fs.cola + q.out;
  fs.rowa = reinterpret_cast<int32_t *>(fs.colb + q.out);
  fs.rowb = fs.rowa + q.out;
  fs.colw = fs.rowb + q.out;
  fs.roww = fs.colw + q.out;
  fs.colbad = fs.roww + q.out;
  fs.rowbad = fs.colbad + q.out;
  __shared__ int ncol, nrow;
  const int t = blockIdx.x;
  const int64_t b = q.wins[3 * t];
  const int x0 = q.wins[3 * t + 1], y0 = q.wins[3 * t + 2];
  if (threadIdx.x == 0) ncol = nrow = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < q.out; i += blockDim.x) {
    int a, c, w;
    src_coord_w(i, q.scale, q.size, a, c, w);
    const int ga = col_cta(p, x0 + a), gb = col_cta(p, x0 + c);
    if (ga < 0 || ga != gb) fs.colbad[atomicAdd(&ncol, 1)] = i;
    if (row_cta(p, y0 + a) != row_cta(p, y0 + c)) fs.rowbad[atomicAdd(&nrow, 1)] = i;
    const int ma = x0 + a, mc = x0 + c;
    const int ca = ma / p.W, cc = mc / p.W;
    fs.cola[i] = ca * p.img_bytes + static_cast<int64_t>(ma - ca * p.W) * 3;
    fs.colb[i] = cc * p.img_bytes + static_cast<int64_t>(mc - cc * p.W) * 3;
    fs.colw[i] = w;
    fs.rowa[i] = (y0 + a) * p.row_bytes;
    fs.rowb[i] = (y0 + c) * p.row_bytes;
    fs.roww[i] = w;
  }
  __syncthreads();
  const int nc = ncol, nr = nrow;
  // work items: every ox of a bad row, then the bad columns of every row
  // (bad rows included twice would only rewrite identical bytes; skip them)
  const uint8_t *frame = p.dst + b * p.cam_count * p.img_bytes;
  uint8_t *tile = q.tiles + static_cast<int64_t>(t) * q.out * q.out * 3;
  auto emit = [&](int oy, int ox) {
    const uint8_t *ra = frame + fs.rowa[oy], *rb = frame + fs.rowb[oy];
    const int64_t xa = fs.cola[ox], xb = fs.colb[ox];
    const uint32_t wx = static_cast<uint32_t>(fs.colw[ox]), wy = static_cast<uint32_t>(fs.roww[oy]);
    uint32_t A[3], B[3], C[3], D[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      A[ch] = __ldg(ra + xa + ch);
      B[ch] = __ldg(ra + xb + ch);
      C[ch] = __ldg(rb + xa + ch);
      D[ch] = __ldg(rb + xb + ch);
    }
    uint8_t *o = tile + (static_cast<int64_t>(oy) * q.out + ox) * 3;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch)
      o[ch] = static_cast<uint8_t>(bilerp_fx(A[ch], B[ch], C[ch], D[ch], wx, wy));
  };
  const int nrow_items = nr * q.out;  // (bad row j, ox), ox fastest
#pragma unroll 4
  for (int it = threadIdx.x; it < nrow_items; it += blockDim.x) {
    const int j = it / q.out;
    emit(fs.rowbad[j], it - j * q.out);
  }
  if (nc > 0) {  // bad columns of every row: (row, column) stepped without divisions
    int oy = threadIdx.x / nc, j = threadIdx.x - oy * nc;
    const int step_y = blockDim.x / nc, step_j = blockDim.x - step_y * nc;
#pragma unroll 4
    while (oy < q.out) {
      emit(oy, fs.colbad[j]);
      oy += step_y;
      j += step_j;
      if (j >= nc) {
        j -= nc;
        ++oy;
      }
    }
  }
}

// ------------------------------------------------------------- generic path
// Any width / alignment: one thread per pixel, coefficients per pixel.
__global__ void apply_generic_kernel(const ApplyParams p) {
  const int64_t npx = static_cast<int64_t>(p.n_img) * p.H * p.W;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < npx;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int col = static_cast<int>(t % p.W);
    const int64_t rest = t / p.W;
    const int row = static_cast<int>(rest % p.H);
    const int64_t img = rest / p.H;
    const int k = min(row / p.bh, p.K - 1);
    const double *gl, *bl, *gr, *br;
    map_ptrs(p, img, gl, bl, gr, br);
    const int64_t off = img * p.img_bytes + static_cast<int64_t>(row) * p.row_bytes + col * 3;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      float m, a;
      coef_f32(col, ch, k, p.W, gl, bl, gr, br, m, a);
      float y = __fadd_rn(__fmul_rn(static_cast<float>(p.src[off + ch]), m), a);
      y = rintf(y);
      y = fminf(fmaxf(y, 0.0f), 255.0f);
      p.dst[off + ch] = static_cast<uint8_t>(y);
    }
  }
}

static size_t fuse_smem_bytes(const TileFuse &q) {
  size_t off[8];
  return fuse_layout(q.out, q.size, off);
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
  p.row_splits = splits;
  p.rows_per_split = (max_rows + splits - 1) / splits;
  return true;
}

template <bool TILES, int ROWS = kTmaRows, int STAGES = kTmaStages, int MINB = 0>
static int launch_tma(const ApplyParams &p, const TileFuse &q, cudaStream_t stream) {
  const int64_t grid = static_cast<int64_t>(p.n_img) * p.K * p.col_groups * p.row_splits;
  const size_t smem = STAGES * ROWS * kApplyThreads * 16 + (TILES ? fuse_smem_bytes(q) : 0);
  cudaError_t e = cudaFuncSetAttribute(apply_tma_kernel<TILES, ROWS, STAGES, MINB>,
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
  e = cudaLaunchKernelEx(&lc, apply_tma_kernel<TILES, ROWS, STAGES, MINB>, p, q);
  return e == cudaSuccess ? launch_status() : static_cast<int>(e);
}

static int launch_apply(ApplyParams &p, cudaStream_t stream) {
  if (p.n_img <= 0 || p.H <= 0 || p.W <= 0) return CAMX_OK;
  if (plan_fast(p)) {
    // short CTAs (<= 48 rows, e.g. 640x480 frames: 30-row blocks) spend more
    // of their life in the prologue / first fills: one more resident CTA per
    // SM (72 registers) hides it (config 1 K3 56.8 -> 51.3 us); whole 96-row
    // blocks run best at 6 (config 2: 0.7275 vs 0.7302 ms per step)
    if (p.rows_per_split <= 48) return launch_tma<false, kTmaRows, kTmaStages, 7>(p, TileFuse{}, stream);
    return launch_tma<false>(p, TileFuse{}, stream);
  }
  const int64_t npx = static_cast<int64_t>(p.n_img) * p.H * p.W;
  int64_t blocks = (npx + 255) / 256;
  const int64_t cap = static_cast<int64_t>(sm_count()) * 16;
  if (blocks > cap) blocks = cap;
  apply_generic_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(p);
  return launch_status();
}

// Fused K3 + K5 (+ fix-up).  Returns CAMX_EINVAL if the geometry is not
// fusable (caller falls back to apply + tiles).
static int launch_apply_tiles(ApplyParams &p, TileFuse &q, int32_t n_tiles,
                              int32_t max_tiles_per_frame, cudaStream_t stream) {
  if (!plan_fast(p)) return CAMX_EINVAL;
  // strict downscale: no clamped taps, each source row is the second tap of <= 1 output row
  if (max_tiles_per_frame > kFuseMaxWin || q.out >= q.size || q.size > 4096) return CAMX_EINVAL;
  int st = launch_tma<true, kFuseRows, kFuseStages>(p, q, stream);
  if (st != CAMX_OK || n_tiles == 0) return st;
  const size_t smem = fixup_smem_bytes(q.out);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(tile_fixup_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  tile_fixup_kernel<<<n_tiles, 256, smem, stream>>>(p, q);
  return launch_status();
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

// K3 + K5: fused when the geometry allows (one pass over the raw frames),
// else apply followed by the row-staged tile kernel on the corrected frames.
static int apply_and_tile(ApplyParams &p, const int32_t *windows, const int32_t *frame_off,
                          int32_t n_tiles, int32_t max_tiles_per_frame, int32_t size,
                          int32_t out_size, uint8_t *tiles_out, void *stream) {
  if (n_tiles < 0 || size < 1 || out_size < 1 || size > p.H || size > p.n_cams * p.W)
    return CAMX_EINVAL;
  if (n_tiles > 0 && (windows == nullptr || tiles_out == nullptr)) return CAMX_EINVAL;
  if (n_tiles > 0 && frame_off != nullptr && max_tiles_per_frame > 0 &&
      p.cam_count == p.n_cams) {
    TileFuse q{};
    q.wins = windows;
    q.frame_off = frame_off;
    q.tiles = tiles_out;
    q.size = size;
    q.out = out_size;
    q.scale = static_cast<float>(size) / static_cast<float>(out_size);
    ApplyParams pf = p;
    const int st = launch_apply_tiles(pf, q, n_tiles, max_tiles_per_frame, as_stream(stream));
    if (st != CAMX_EINVAL) return st;
  }
  int st = launch_apply(p, as_stream(stream));
  if (st != CAMX_OK || n_tiles == 0) return st;
  return camx_tiles(p.dst, p.n_cams, p.H, p.W, windows, n_tiles, size, out_size, tiles_out,
                    stream);
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
