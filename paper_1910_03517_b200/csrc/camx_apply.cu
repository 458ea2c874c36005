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

#include "camx_common.cuh"

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

// Exact float32 (M, A) of one (column, channel, block); identity outside
// the lam > 0 half of each present map.
__device__ __forceinline__ void coef_f32(int col, int ch, int k, int W, const double *gl,
                                         const double *bl, const double *gr, const double *br,
                                         float &m32, float &a32) {
  const double c0 = (W - 1) * 0.5;
  const double colf = static_cast<double>(col);
  double lam = 0.0, g = 1.0, b = 0.0;
  bool have = false;
  if (gl != nullptr && 2 * col > W - 1) {
    lam = __ddiv_rn(__dsub_rn(colf, c0), __dsub_rn(static_cast<double>(W - 1), c0));
    g = gl[k * 3 + ch];
    b = bl[k * 3 + ch];
    have = true;
  } else if (gr != nullptr && 2 * col < W - 1) {
    lam = __ddiv_rn(__dsub_rn(c0, colf), c0);
    g = gr[k * 3 + ch];
    b = br[k * 3 + ch];
    have = true;
  }
  if (!have || !(lam > 0.0)) {
    m32 = 1.0f;
    a32 = 0.0f;
    return;
  }
  lam = fmin(lam, 1.0);
  const double M = __dadd_rn(1.0, __dmul_rn(lam, __dsub_rn(g, 1.0)));
  const double A = __dmul_rn(lam, b);
  m32 = __double2float_rn(M);
  a32 = __double2float_rn(A);
}

// ---------------------------------------------------------------- fast path
// Requires row_bytes % 16 == 0 and 16-byte aligned src/dst.
constexpr int kApplyThreads = 128;
constexpr int kUnroll = 4;

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

__global__ void __launch_bounds__(kApplyThreads, 4) apply_fast_kernel(const ApplyParams p) {
  int64_t item = blockIdx.x;
  const int cg = static_cast<int>(item % p.col_groups);
  item /= p.col_groups;
  const int rs = static_cast<int>(item % p.row_splits);
  item /= p.row_splits;
  const int k = static_cast<int>(item % p.K);
  const int64_t img = item / p.K;

  const int j = cg * kApplyThreads + threadIdx.x;  // 16-byte chunk in the row
  if (j >= p.chunks_per_row) return;

  const int blk_r0 = k * p.bh;
  const int blk_r1 = (k == p.K - 1) ? p.H : blk_r0 + p.bh;
  const int r0 = blk_r0 + rs * p.rows_per_split;
  const int r1 = min(blk_r1, r0 + p.rows_per_split);
  if (r0 >= r1) return;

  const double *gl, *bl, *gr, *br;
  map_ptrs(p, img, gl, bl, gr, br);

  Coef16 cf;
  {
    const int q0 = j * 16;
    int col = q0 / 3;
    int ch = q0 - col * 3;
    float m[16], a[16];
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
      cf.c[i >> 1] = pack2(m[i] * -32768.0f, m[i + 1] * -32768.0f);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      // |A| < 2^-110 cannot change rn(p*M + A) (see header); zero it so the
      // 2^-8 scaling stays exact (no subnormal).
      cf.a[i] = fabsf(a[i]) < 7.7037197787136e-34f ? 0.0f : a[i] * 0.00390625f;
    }
  }

  const uint8_t *src = p.src + img * p.img_bytes + static_cast<int64_t>(r0) * p.row_bytes + j * 16;
  uint8_t *dst = p.dst + img * p.img_bytes + static_cast<int64_t>(r0) * p.row_bytes + j * 16;
  const int64_t rb = p.row_bytes;
  int r = r0;
  for (; r + kUnroll <= r1; r += kUnroll) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) v[u] = ld_stream_v4(src + u * rb);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) st_stream_v4(dst + u * rb, correct16(v[u], cf));
    src += kUnroll * rb;
    dst += kUnroll * rb;
  }
  for (; r < r1; ++r) {
    st_stream_v4(dst, correct16(ld_stream_v4(src), cf));
    src += rb;
    dst += rb;
  }
}

// ------------------------------------------------- TMA bulk-copy pipeline
// Same work decomposition as apply_fast_kernel, but the rows stream through
// a kStages-deep shared-memory ring filled by 1-D bulk async copies
// (cp.async.bulk, the TMA engine) completing on mbarriers, so the bytes in
// flight per SM no longer depend on registers x occupancy (the LDG version
// is long-scoreboard bound at 16 warps/SM).  Thread 0 issues; every thread
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

__global__ void __launch_bounds__(kApplyThreads, 4) apply_tma_kernel(const ApplyParams p) {
  extern __shared__ __align__(128) uint4 ring[];  // [kTmaStages][kTmaRows][kApplyThreads]
  __shared__ __align__(8) uint64_t full[kTmaStages];
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
  const int nst = (nrows + kTmaRows - 1) / kTmaRows;

  auto issue = [&](int st) {
    const int slot = st % kTmaStages;
    const int rr = min(kTmaRows, nrows - st * kTmaRows);
    mbar_expect_tx(&full[slot], seg * rr);
    for (int i = 0; i < rr; ++i)
      bulk_g2s(ring + (slot * kTmaRows + i) * kApplyThreads,
               src0 + static_cast<int64_t>(st * kTmaRows + i) * rb, seg, &full[slot]);
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < kTmaStages; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int st = 0; st < min(kTmaStages, nst); ++st) issue(st);
  }
  __syncthreads();
  // maps come from the preceding stats/solve grid (programmatic dependent
  // launch): only the raw-pixel prefetch above may run before it completes
  asm volatile("griddepcontrol.wait;" ::: "memory");

  const bool active = threadIdx.x < chunks;
  const double *gl, *bl, *gr, *br;
  map_ptrs(p, img, gl, bl, gr, br);
  Coef16 cf;
  if (active) {
    const int q0 = j * 16;
    int col = q0 / 3;
    int ch = q0 - col * 3;
    float m[16], a[16];
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
      cf.c[i >> 1] = pack2(m[i] * -32768.0f, m[i + 1] * -32768.0f);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i)
      cf.a[i] = fabsf(a[i]) < 7.7037197787136e-34f ? 0.0f : a[i] * 0.00390625f;
  }

  uint8_t *dst = p.dst + img * p.img_bytes + static_cast<int64_t>(r0) * rb + j * 16;
  for (int st = 0; st < nst; ++st) {
    const int slot = st % kTmaStages;
    mbar_wait(&full[slot], (st / kTmaStages) & 1);
    const int rr = min(kTmaRows, nrows - st * kTmaRows);
    if (active) {
      uint4 v[kTmaRows];
#pragma unroll
      for (int i = 0; i < kTmaRows; ++i)
        if (i < rr) v[i] = ring[(slot * kTmaRows + i) * kApplyThreads + threadIdx.x];
#pragma unroll
      for (int i = 0; i < kTmaRows; ++i)
        if (i < rr) st_stream_v4(dst + static_cast<int64_t>(st * kTmaRows + i) * rb, correct16(v[i], cf));
    }
    __syncthreads();  // slot fully consumed
    if (threadIdx.x == 0 && st + kTmaStages < nst) issue(st + kTmaStages);
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

static int launch_apply(ApplyParams &p, cudaStream_t stream) {
  if (p.n_img <= 0 || p.H <= 0 || p.W <= 0) return CAMX_OK;
  const bool aligned = (p.row_bytes % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(p.src) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(p.dst) % 16 == 0);
  if (aligned) {
    p.chunks_per_row = p.row_bytes / 16;
    p.col_groups = (p.chunks_per_row + kApplyThreads - 1) / kApplyThreads;
    // Whole block rows per CTA unless the grid would under-fill the GPU.
    const int max_rows = p.H - (p.K - 1) * p.bh;  // last block is the tallest
    int64_t base = static_cast<int64_t>(p.n_img) * p.K * p.col_groups;
    int splits = 1;
    const int64_t target = static_cast<int64_t>(sm_count()) * 8;
    while (base * splits < target && (max_rows + splits) / (splits + 1) >= 16) ++splits;
    p.row_splits = splits;
    p.rows_per_split = (max_rows + splits - 1) / splits;
    const int64_t grid = base * splits;
    static const int use_ldg = [] {
      const char *e = getenv("CAMX_APPLY_KERNEL");
      return (e != nullptr && e[0] == 'l') ? 1 : 0;
    }();
    if (use_ldg) {
      apply_fast_kernel<<<static_cast<unsigned>(grid), kApplyThreads, 0, stream>>>(p);
    } else {
      const int smem = kTmaStages * kTmaRows * kApplyThreads * 16;
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(apply_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
      }
      if (p.pdl) {
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(static_cast<unsigned>(grid));
        lc.blockDim = dim3(kApplyThreads);
        lc.dynamicSmemBytes = smem;
        lc.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&lc, apply_tma_kernel, p);
        if (e != cudaSuccess) return static_cast<int>(e);
      } else {
        apply_tma_kernel<<<static_cast<unsigned>(grid), kApplyThreads, smem, stream>>>(p);
      }
    }
  } else {
    const int64_t npx = static_cast<int64_t>(p.n_img) * p.H * p.W;
    int64_t blocks = (npx + 255) / 256;
    const int64_t cap = static_cast<int64_t>(sm_count()) * 16;
    if (blocks > cap) blocks = cap;
    apply_generic_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(p);
  }
  return launch_status();
}

}  // namespace camx

using namespace camx;

namespace camx {
int launch_seam_solve(const camx_band_stat *stats, int32_t n_batch, int32_t n_cams, int32_t wrap,
                      const camx_solve_config *cfg, const double *prev_gain,
                      const double *prev_offset, double *gain_out, double *offset_out,
                      uint8_t *fit_ok_out, cudaStream_t stream, bool pdl);
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

extern "C" int camx_correct_batch(const uint8_t *images, uint8_t *out, const uint8_t *prev_frame,
                                  int32_t n_batch, int32_t n_cams, int32_t wrap, int32_t height,
                                  int32_t width, int32_t band_width, int32_t t_diff,
                                  const camx_solve_config *cfg, const double *prev_gain,
                                  const double *prev_offset, camx_band_stat *stats,
                                  uint32_t *hist, double *gain_out, double *offset_out,
                                  uint8_t *fit_ok_out, int32_t *counters, void *stream) {
  if (cfg == nullptr || images == nullptr || out == nullptr || stats == nullptr) return CAMX_EINVAL;
  if (gain_out == nullptr || offset_out == nullptr) return CAMX_EINVAL;
  if (n_batch < 1 || n_cams < 2 || cfg->blocks < 1 || cfg->blocks > height) return CAMX_EINVAL;
  if (cfg->mode < CAMX_MODE_STANDARD || cfg->mode > CAMX_MODE_SMOOTHING) return CAMX_EINVAL;
  if (cfg->have_prev_maps && (prev_gain == nullptr || prev_offset == nullptr)) return CAMX_EINVAL;
  (void)counters;  // used by the fused variant (camx_band_stats_solve)
  const int64_t img_bytes = static_cast<int64_t>(height) * width * 3;
  const int64_t frame_bytes = img_bytes * n_cams;
  const int64_t rec_frame = static_cast<int64_t>(n_cams) * 2 * cfg->blocks;
  const bool removal = cfg->mode == CAMX_MODE_OBJECT_REMOVAL;
  int st;
  // K1: band statistics (frames 1.. against their predecessors, frame 0
  // against prev_frame, for OBJECT_REMOVAL)
  if (removal && n_batch > 1) {
    st = camx_band_stats(images + frame_bytes, images, nullptr, (n_batch - 1) * int64_t(n_cams),
                         height, width, band_width, cfg->blocks, t_diff, stats + rec_frame,
                         hist == nullptr ? nullptr : hist + rec_frame * 768, stream);
    if (st != CAMX_OK) return st;
    st = camx_band_stats(images, prev_frame, nullptr, n_cams, height, width, band_width,
                         cfg->blocks, t_diff, stats, hist, stream);
  } else {
    st = camx_band_stats(images, removal ? prev_frame : nullptr, nullptr,
                         int64_t(n_batch) * n_cams, height, width, band_width, cfg->blocks,
                         t_diff, stats, hist, stream);
  }
  if (st != CAMX_OK) return st;
  // K2 as a programmatic dependent of K1, K3 as one of K2
  st = launch_seam_solve(stats, n_batch, n_cams, wrap, cfg, prev_gain, prev_offset, gain_out,
                         offset_out, fit_ok_out, as_stream(stream), true);
  if (st != CAMX_OK) return st;
  ApplyParams p{};
  p.src = images;
  p.dst = out;
  p.H = height;
  p.W = width;
  p.K = cfg->blocks;
  p.bh = height / cfg->blocks;
  p.row_bytes = width * 3;
  p.img_bytes = img_bytes;
  p.n_img = n_batch * n_cams;
  p.cam_begin = 0;
  p.cam_count = n_cams;
  p.n_cams = n_cams;
  p.wrap = wrap;
  p.S = wrap ? n_cams : n_cams - 1;
  p.gain = gain_out;
  p.offset = offset_out;
  p.pdl = 1;
  return launch_apply(p, as_stream(stream));
}
