// K5: attention-tile crop / resize (stage 4b) and the seam quality metric.
//
// Crop: ExternalDetector.detect (camarray detect.py:297-300) slices
// mosaic.pixels[y:y+S, x:x+S] of the concatenated mosaic (core.py:102-119);
// here the mosaic is virtual (column x -> camera x / W).  Resize to the
// detector input size is builder-defined (the reference has none):
// bilinear, half-pixel centres, source coordinate in float32, 8-bit
// fixed-point weights and an exact integer blend rounded half up
// (camx_resize.cuh; oracle/camarray_oracle.py: resize_bilinear).
// Kernels: exact crop (two-segment row copies), band-staged downscale
// (the default resize path), row-staged resize (any geometry with <= 2
// cameras per window row), per-pixel gather (windows wider than a camera),
// camera-sharded band-staged kernel and gather fallback (multi-GPU).
//
// seam_cost: exposure.py:417-445 (box downsample, Eq. 1 of the paper).
#include <cstdlib>

#include <algorithm>

#include "camx_resize.cuh"

namespace camx {

struct TileParams {
  const uint8_t *img;
  int32_t n_cams, H, W, size, out;
  const int32_t *wins;  // [n][3] (batch, x, y)
  uint8_t *tiles;
  float scale;
};

__device__ __forceinline__ const uint8_t *mosaic_px(const TileParams &p, int64_t b, int row,
                                                     int mx) {
  const int cam = mx / p.W;
  const int col = mx - cam * p.W;
  return p.img + (((b * p.n_cams + cam) * p.H + row) * static_cast<int64_t>(p.W) + col) * 3;
}

__global__ void tiles_kernel(const TileParams p) {
  const int t = blockIdx.y;
  const int64_t b = p.wins[3 * t];
  const int x0 = p.wins[3 * t + 1], y0 = p.wins[3 * t + 2];
  const int64_t npx = static_cast<int64_t>(p.out) * p.out;
  uint8_t *dst = p.tiles + static_cast<int64_t>(t) * npx * 3;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < npx;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int oy = static_cast<int>(q / p.out);
    const int ox = static_cast<int>(q - static_cast<int64_t>(oy) * p.out);
    if (p.out == p.size) {
      const uint8_t *s = mosaic_px(p, b, y0 + oy, x0 + ox);
      dst[3 * q] = s[0];
      dst[3 * q + 1] = s[1];
      dst[3 * q + 2] = s[2];
      continue;
    }
    int y_0, y_1, x_0, x_1, wy, wx;
    src_coord_w(oy, p.scale, p.size, y_0, y_1, wy);
    src_coord_w(ox, p.scale, p.size, x_0, x_1, wx);
    const uint8_t *a = mosaic_px(p, b, y0 + y_0, x0 + x_0);
    const uint8_t *bb = mosaic_px(p, b, y0 + y_0, x0 + x_1);
    const uint8_t *c = mosaic_px(p, b, y0 + y_1, x0 + x_0);
    const uint8_t *d = mosaic_px(p, b, y0 + y_1, x0 + x_1);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch)
      dst[3 * q + ch] = static_cast<uint8_t>(bilerp_fx(a[ch], bb[ch], c[ch], d[ch], wx, wy));
  }
}

// Exact crop (out == size <= W): each window row is at most two camera
// segments; CTA = (tile, band of 8 rows), coalesced byte copies, no
// per-pixel index arithmetic.
__global__ void __launch_bounds__(256) tiles_crop_kernel(const TileParams p) {
  const int t = blockIdx.y;
  const int64_t b = p.wins[3 * t];
  const int x0 = p.wins[3 * t + 1], y0 = p.wins[3 * t + 2];
  const int S3 = p.size * 3;
  const int cam0 = x0 / p.W;
  const int n0 = min(p.size, (cam0 + 1) * p.W - x0) * 3;  // bytes from camera cam0
  const int64_t img_bytes = static_cast<int64_t>(p.H) * p.W * 3;
  const uint8_t *c0 = p.img + (b * p.n_cams + cam0) * img_bytes + static_cast<int64_t>(x0 - cam0 * p.W) * 3;
  const uint8_t *c1 = p.img + (b * p.n_cams + min(cam0 + 1, p.n_cams - 1)) * img_bytes;
  const int oy_end = min(p.size, (blockIdx.x + 1) * 8);
  for (int oy = blockIdx.x * 8; oy < oy_end; ++oy) {
    const int64_t roff = static_cast<int64_t>(y0 + oy) * p.W * 3;
    uint8_t *dst = p.tiles + (static_cast<int64_t>(t) * p.size + oy) * S3;
    for (int i = threadIdx.x; i < S3; i += blockDim.x)
      dst[i] = i < n0 ? c0[roff + i] : c1[roff + (i - n0)];
  }
}

// Row-staged version: CTA = (tile, band of kTileRowsPerCta output rows).  For
// each output row the two source rows' window segments (one per camera the
// window covers) are staged in shared memory as their 16-byte-aligned
// supersets (plain vector copies; `head` = offset of the first wanted byte),
// then every output pixel is resampled from shared memory with the fixed-point
// funnel/dp2a path (taps straddling two cameras: byte path), and the output
// row is stored with 16-byte stores when aligned.  Arithmetic: camx_resize.cuh.
constexpr int kTileThreads = 256;
constexpr int kTileRowsPerCta = 8;

struct RowSeg {   // one camera's part of a staged window row
  int off;        // smem byte offset of the aligned superset
  int head;       // first wanted byte within it
  int x0;         // window-local pixel index where the segment starts
};

__device__ __forceinline__ int stage_row(const TileParams &p, int64_t b, int row, int x0,
                                         uint8_t *buf, RowSeg &s0, RowSeg &s1) {
  int x = x0, nseg = 0, off = 0;
  const int xe = x0 + p.size;
  while (x < xe) {  // CTA-uniform: at most two camera segments when S <= W
    const int cam = x / p.W;
    const int seg_end = min(xe, (cam + 1) * p.W);
    const int nbytes = (seg_end - x) * 3;
    const uint8_t *src = p.img + (((b * p.n_cams + cam) * p.H + row) * static_cast<int64_t>(p.W) +
                                  (x - cam * p.W)) * 3;
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(src);
    const uint4 *base = reinterpret_cast<const uint4 *>(a0 & ~static_cast<uintptr_t>(15));
    const int head = static_cast<int>(a0 & 15);
    const int nvec = (head + nbytes + 15) >> 4;
    uint4 *dst = reinterpret_cast<uint4 *>(buf + off);
    for (int v = threadIdx.x; v < nvec; v += blockDim.x) dst[v] = __ldg(base + v);
    if (nseg == 0) s0 = RowSeg{off, head, x - x0};
    else s1 = RowSeg{off, head, x - x0};
    ++nseg;
    off += nvec * 16 + 16;  // +16: slack for the 12-byte tap window reads
    x = seg_end;
  }
  return nseg;
}

__device__ __forceinline__ int tap_addr(const RowSeg &s0, const RowSeg &s1, int nseg, int x) {
  return (nseg > 1 && x >= s1.x0) ? s1.off + s1.head + 3 * (x - s1.x0)
                                  : s0.off + s0.head + 3 * (x - s0.x0);
}

__global__ void __launch_bounds__(kTileThreads) tiles_rows_kernel(const TileParams p) {
  extern __shared__ __align__(16) uint8_t tsm[];
  const int S3p = ((p.size * 3 + 15) & ~15) + 64;  // two segments + slack
  uint8_t *rowA = tsm;
  uint8_t *rowB = tsm + S3p;
  uint8_t *orow = rowB + S3p;
  const int t = blockIdx.y;
  const int64_t b = p.wins[3 * t];
  const int x0 = p.wins[3 * t + 1], y0 = p.wins[3 * t + 2];
  const int O3 = p.out * 3;
  uint8_t *tile = p.tiles + static_cast<int64_t>(t) * p.out * O3;
  const int oy_end = min(p.out, (blockIdx.x + 1) * kTileRowsPerCta);
  for (int oy = blockIdx.x * kTileRowsPerCta; oy < oy_end; ++oy) {
    int y_0, y_1, wy;
    src_coord_w(oy, p.scale, p.size, y_0, y_1, wy);
    RowSeg sa0{0, 0, 0}, sa1{0, 0, 0}, sb0{0, 0, 0}, sb1{0, 0, 0};
    const int na = stage_row(p, b, y0 + y_0, x0, rowA, sa0, sa1);
    stage_row(p, b, y0 + y_1, x0, rowB, sb0, sb1);
    __syncthreads();
    const uint32_t wy1 = static_cast<uint32_t>(wy), wy0 = 256u - wy1;
    for (int ox = threadIdx.x; ox < p.out; ox += blockDim.x) {
      int x_0, x_1, wx;
      src_coord_w(ox, p.scale, p.size, x_0, x_1, wx);
      const uint32_t wpk = static_cast<uint32_t>(256 - wx) | (static_cast<uint32_t>(wx) << 16);
      uint8_t *o = orow + 3 * ox;
      const bool same = (na == 1) || ((x_0 >= sa1.x0) == (x_1 >= sa1.x0));
      if (same && x_1 == x_0 + 1) {  // two adjacent pixels of one segment: 6 contiguous bytes
        const int la = tap_addr(sa0, sa1, na, x_0);
        const int lb = tap_addr(sb0, sb1, na, x_0);
        const uint32_t *pa = reinterpret_cast<const uint32_t *>(rowA + (la & ~3));
        const uint32_t *pb = reinterpret_cast<const uint32_t *>(rowB + (lb & ~3));
        const uint32_t sha = (la & 3) * 8, shb = (lb & 3) * 8;
        const uint32_t alo = __funnelshift_r(pa[0], pa[1], sha), ahi = __funnelshift_r(pa[1], pa[2], sha);
        const uint32_t blo = __funnelshift_r(pb[0], pb[1], shb), bhi = __funnelshift_r(pb[1], pb[2], shb);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          const uint32_t sel = 0x0030u + 0x0011u * ch;
          const uint32_t v0 = __dp2a_lo(wpk, __byte_perm(alo, ahi, sel), 0u);
          const uint32_t v1 = __dp2a_lo(wpk, __byte_perm(blo, bhi, sel), 0u);
          o[ch] = static_cast<uint8_t>((v0 * wy0 + v1 * wy1 + 32768u) >> 16);
        }
      } else {  // clamped edge or taps in two cameras
        const int a0 = tap_addr(sa0, sa1, na, x_0), a1 = tap_addr(sa0, sa1, na, x_1);
        const int b0 = tap_addr(sb0, sb1, na, x_0), b1 = tap_addr(sb0, sb1, na, x_1);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch)
          o[ch] = static_cast<uint8_t>(bilerp_fx(rowA[a0 + ch], rowA[a1 + ch], rowB[b0 + ch],
                                                 rowB[b1 + ch], wx, wy));
      }
    }
    __syncthreads();
    uint8_t *dst = tile + static_cast<int64_t>(oy) * O3;
    if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0 && (O3 & 15) == 0) {
      for (int v = threadIdx.x; v < O3 / 16; v += blockDim.x)
        reinterpret_cast<uint4 *>(dst)[v] = reinterpret_cast<const uint4 *>(orow)[v];
    } else {
      for (int j = threadIdx.x; j < O3; j += blockDim.x) dst[j] = orow[j];
    }
    __syncthreads();
  }
}

// ---- TMA-staged resize (the default resize path) ---------------------------
// CTA = (tile, band of output rows), 4 warps; warp w resamples output rows
// w, w + 4, ... of the band, one whole row at a time: lane l owns output
// columns l + 32 j (j < J), whose tap byte offsets and dp2a weights sit in
// registers for the CTA's life.  Per output row, lane 0 stages the two tap
// source rows of the window with 1-D bulk copies (TMA engine, completion on
// a per-slot mbarrier; kTmaTileSlots rows in flight per warp): a window row
// spanning several cameras is one segment per camera, and the segments land
// back to back - the first ends at its camera's row end and the next starts
// at its camera's row start, both 16-byte aligned - so the staged row is the
// contiguous mosaic byte range from `head` on and a tap pair straddling two
// cameras needs no special case.  The output row is assembled in shared
// memory and leaves with one bulk store.  Per output pixel: 6 LDS, 4 funnel
// shifts, 6 PRMT, 6 dp2a, 6 IMAD/IMUL, 3 shifts, 3 byte STS (camx_resize.cuh
// bilerp_fx arithmetic: bit-identical to the other tile paths).
constexpr int kTmaTileWarps = 4;
constexpr int kTmaTileSlots = 2;

struct TmaTileGeom {
  int pitch;         // staged source row bytes (16-multiple, with read slack)
  int opitch;        // output row buffer bytes (16-multiple)
  int rows_per_cta;  // output rows per CTA
  int bulk_out;      // output rows leave by bulk store (3 * out % 16 == 0, aligned tiles)
};

__host__ __device__ __forceinline__ int tma_tile_pitch(int size) {
  return (size * 3 + 32 + 15) & ~15;
}
__host__ __device__ __forceinline__ size_t tma_tile_smem(const TmaTileGeom &g) {
  return static_cast<size_t>(kTmaTileWarps) * kTmaTileSlots * (2 * g.pitch + g.opitch);
}

// Camera shard (camx_tiles_shard): this GPU holds mosaic columns
// [col_begin, col_begin + local_cols); it stages the window's local columns
// (+ the halo pixel: the next rank's first column) and writes the output
// columns whose first tap is local, leaving the others untouched.
struct TileShard {
  int32_t col_begin, local_cols;
  const uint8_t *halo;  // [B][H][3] or nullptr
};

template <int J, bool EXACT>
__global__ void __launch_bounds__(kTmaTileWarps * 32) tiles_tma_kernel(const TileParams p,
                                                                       const TmaTileGeom g,
                                                                       const TileShard sd) {
  extern __shared__ __align__(128) uint8_t tts[];
  __shared__ __align__(8) uint64_t full[kTmaTileWarps][kTmaTileSlots];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.y;
  const int64_t b = p.wins[3 * t];
  const int x0 = p.wins[3 * t + 1], y0 = p.wins[3 * t + 2];
  const int out = p.out, O3 = out * 3;
  // the window's local pixels [ps, pe) (the whole window without a shard)
  const int lx0 = x0 - sd.col_begin;
  const int ps = max(lx0, 0), pe = min(lx0 + p.size, sd.local_cols);
  if (ps >= pe) return;  // no local column (CTA-uniform)
  const bool halo = sd.halo != nullptr && lx0 + p.size > sd.local_cols;
  const int64_t rowbytes = static_cast<int64_t>(p.W) * 3;
  const int64_t img_bytes = static_cast<int64_t>(p.H) * rowbytes;
  const int cam0 = ps / p.W, cam1 = (pe - 1) / p.W;
  const int sb = (ps - cam0 * p.W) * 3;                          // first wanted byte (cam0 row)
  const int head = sb & 15;
  const int eb = ((pe - cam1 * p.W) * 3 + 15) & ~15;             // staged end (cam1 row)
  const uint32_t n_first = static_cast<uint32_t>((cam0 == cam1 ? eb : rowbytes) - (sb - head));
  const uint32_t row_tx = cam0 == cam1 ? n_first
      : n_first + static_cast<uint32_t>((cam1 - cam0 - 1) * rowbytes + eb);
  const uint8_t *frame = p.img + b * p.n_cams * img_bytes;
  const int slot_bytes = 2 * g.pitch + g.opitch;
  uint8_t *wbase = tts + warp * kTmaTileSlots * slot_bytes;
  // owned output columns: first tap lx0 + i0(ox) in [0, local_cols)
  // (a contiguous range: i0 is nondecreasing)
  int ox_lo = 0, ox_hi = out;
  if (lx0 < 0 || lx0 + p.size > sd.local_cols) {
    auto first = [&](int lim) {  // first ox with lx0 + i0(ox) >= lim
      int lo = 0, hi = out;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        int a, c, w;
        src_coord_w(mid, p.scale, p.size, a, c, w);
        if (lx0 + a >= lim) hi = mid; else lo = mid + 1;
      }
      return lo;
    };
    ox_lo = first(0);
    ox_hi = first(sd.local_cols);
  }
  const bool bulk = g.bulk_out && ox_lo == 0 && ox_hi == out;  // whole rows are ours

  uint32_t off[J], wt[J];
  lane_taps<J>(lane, out, p.scale, p.size, head, off, wt, lx0 - ps);
  const int oy0 = blockIdx.x * g.rows_per_cta;
  const int oy1 = min(out, oy0 + g.rows_per_cta);
  const int n_rows = oy1 - oy0 > warp ? (oy1 - oy0 - warp + kTmaTileWarps - 1) / kTmaTileWarps : 0;
  if (lane == 0) {
    for (int s = 0; s < kTmaTileSlots; ++s) mbar_init(&full[warp][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  auto issue = [&](int i) {  // lane 0: the two tap rows of this warp's i-th output row
    const int oy = oy0 + warp + i * kTmaTileWarps;
    int ya, yb, w;
    src_coord_w(oy, p.scale, p.size, ya, yb, w);
    uint8_t *dst = wbase + (i % kTmaTileSlots) * slot_bytes;
    uint64_t *bar = &full[warp][i % kTmaTileSlots];
    mbar_expect_tx(bar, 2 * row_tx);
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int64_t y = y0 + (r ? yb : ya);
      uint8_t *d = dst + r * g.pitch;
      bulk_g2s(d, frame + cam0 * img_bytes + y * rowbytes + (sb - head), n_first, bar);
      if (cam1 > cam0) {
        d += n_first;
        for (int c = cam0 + 1; c < cam1; ++c, d += rowbytes)
          bulk_g2s(d, frame + c * img_bytes + y * rowbytes, static_cast<uint32_t>(rowbytes), bar);
        bulk_g2s(d, frame + cam1 * img_bytes + y * rowbytes, static_cast<uint32_t>(eb), bar);
      }
    }
  };
  // launched as a programmatic dependent of K3 (config 5): the corrected
  // frames are complete only past this point (a no-op otherwise)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (lane == 0)
    for (int i = 0; i < min(kTmaTileSlots, n_rows); ++i) issue(i);

  uint8_t *tile = p.tiles + static_cast<int64_t>(t) * out * O3;
  // the halo pixel sits right after the shard's last pixel (the staged
  // bytes end at that camera's row end, 16-byte aligned)
  const int halo_off = head + 3 * (sd.local_cols - ps);
  for (int i = 0; i < n_rows; ++i) {
    const int slot = i % kTmaTileSlots;
    const int oy = oy0 + warp + i * kTmaTileWarps;
    int ya, yb, w1y;
    src_coord_w(oy, p.scale, p.size, ya, yb, w1y);
    uint8_t *ra = wbase + slot * slot_bytes;
    uint8_t *ob = wbase + slot * slot_bytes + 2 * g.pitch;
    uint8_t *orow = bulk ? ob : tile + static_cast<int64_t>(oy) * O3;
    mbar_wait(&full[warp][slot], (i / kTmaTileSlots) & 1);
    if (halo) {
      if (lane < 6) {
        const int r = lane / 3, ch = lane - 3 * r;
        ra[r * g.pitch + halo_off + ch] = sd.halo[(b * p.H + y0 + (r ? yb : ya)) * 3 + ch];
      }
      __syncwarp();
    }
    // (the output row buffer is shared memory on the bulk path: 32-bit
    // addresses, byte stores at immediate offsets; a shard's partial row
    // goes straight to global memory)
    if (bulk)
      resample_row_lanes<J, false, EXACT>(ra, ra + g.pitch, off, wt, static_cast<uint32_t>(w1y), ob,
                                          out, lane);
    else
      resample_row_lanes<J, true>(ra, ra + g.pitch, off, wt, static_cast<uint32_t>(w1y), orow, out,
                                  lane, ox_lo, ox_hi);
    if (bulk) {
      fence_proxy_async_smem();  // this lane's row bytes before the bulk store reads them
      __syncwarp();
      if (lane == 0) {
        bulk_s2g(tile + static_cast<int64_t>(oy) * O3, ob, static_cast<uint32_t>(O3));
        bulk_commit();
      }
    }
    __syncwarp();  // every lane is done with the slot's source rows
    if (lane == 0) {
      if (i + kTmaTileSlots < n_rows) {
        if (halo) fence_proxy_async_smem();  // the halo bytes (generic) before the refill
        issue(i + kTmaTileSlots);
      }
      // the next row writes the output buffer last read by row i + 1 - slots
      if (bulk) bulk_wait_read<kTmaTileSlots - 1>();
    }
    __syncwarp();
  }
  if (bulk && lane == 0) bulk_wait<0>();
}

static int launch_tiles_tma(const TileParams &p, int32_t n_tiles, cudaStream_t s,
                            const TileShard &sd, bool pdl = false) {
  const int J = (p.out + 31) / 32;
  TmaTileGeom g{};
  g.pitch = tma_tile_pitch(p.size);
  g.opitch = (p.out * 3 + 15) & ~15;
  g.bulk_out = ((p.out * 3) % 16 == 0 && reinterpret_cast<uintptr_t>(p.tiles) % 16 == 0) ? 1 : 0;
  // enough CTAs for ~3 waves of 4 CTAs per SM, bands of >= 8 output rows
  const int64_t want = static_cast<int64_t>(sm_count()) * 12;
  int64_t per_tile = (want + n_tiles - 1) / n_tiles;
  per_tile = std::max<int64_t>(1, std::min<int64_t>(per_tile, (p.out + 7) / 8));
  g.rows_per_cta = static_cast<int>((p.out + per_tile - 1) / per_tile);
  const size_t smem = tma_tile_smem(g);
  const dim3 grid(static_cast<unsigned>((p.out + g.rows_per_cta - 1) / g.rows_per_cta),
                  static_cast<unsigned>(n_tiles));
  auto go = [&](auto kern) -> int {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return static_cast<int>(e);
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid;
    lc.blockDim = dim3(kTmaTileWarps * 32);
    lc.dynamicSmemBytes = smem;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = pdl ? 1 : 0;
    e = cudaLaunchKernelEx(&lc, kern, p, g, sd);
    return e == cudaSuccess ? launch_status() : static_cast<int>(e);
  };
  // EXACT instantiations where J = ceil(out / 32) (416 -> 13)
  if (J == 2) return go(tiles_tma_kernel<2, true>);
  if (J <= 4) return J == 4 ? go(tiles_tma_kernel<4, true>) : go(tiles_tma_kernel<4, false>);
  if (J <= 8) return J == 8 ? go(tiles_tma_kernel<8, true>) : go(tiles_tma_kernel<8, false>);
  if (J <= 13) return J == 13 ? go(tiles_tma_kernel<13, true>) : go(tiles_tma_kernel<13, false>);
  return J == 16 ? go(tiles_tma_kernel<16, true>) : go(tiles_tma_kernel<16, false>);
}

static bool tiles_tma_ok(const TileParams &p) {
  const TmaTileGeom g{tma_tile_pitch(p.size), (p.out * 3 + 15) & ~15, 1, 0};
  return p.out <= 16 * 32 && (p.W * 3) % 16 == 0 &&
         reinterpret_cast<uintptr_t>(p.img) % 16 == 0 && tma_tile_smem(g) <= 200 * 1024;
}

// ---- camera-sharded tiles ---------------------------------------
// Rank g holds cameras [c0, c0 + n_cams) of the array, i.e. mosaic columns
// [col_begin, col_begin + n_cams * W).  Output column ox of a window belongs
// to the rank that holds its first column tap (x0 + i0(ox)); its second tap
// may be the first column of the next rank, supplied as `halo` (B, H, 3) -
// the 1-pixel corrected halo column.  Output pixels of other ranks' columns
// are left untouched (the caller zero-fills and sums the partials).
// The TMA-staged kernel (tiles_tma_kernel with a TileShard) serves aligned
// geometries; this per-pixel gather the rest.
struct ShardTileParams {
  TileParams t;
  int32_t col_begin;    // global mosaic column of local column 0
  int32_t local_cols;   // n_cams * W
  const uint8_t *halo;  // (B, H, 3) or nullptr
};

__device__ __forceinline__ const uint8_t *shard_px(const ShardTileParams &p, int64_t b, int row,
                                                   int gx) {
  const int lx = gx - p.col_begin;
  if (lx == p.local_cols) return p.halo + (b * p.t.H + row) * 3;
  return mosaic_px(p.t, b, row, lx);
}

__global__ void tiles_shard_kernel(const ShardTileParams p) {
  const int t = blockIdx.y;
  const int64_t b = p.t.wins[3 * t];
  const int x0 = p.t.wins[3 * t + 1], y0 = p.t.wins[3 * t + 2];
  const int out = p.t.out;
  const int64_t npx = static_cast<int64_t>(out) * out;
  uint8_t *dst = p.t.tiles + static_cast<int64_t>(t) * npx * 3;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < npx;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int oy = static_cast<int>(q / out);
    const int ox = static_cast<int>(q - static_cast<int64_t>(oy) * out);
    int x_0 = ox, x_1 = ox, wx = 0, y_0 = oy, y_1 = oy, wy = 0;
    if (out != p.t.size) {
      src_coord_w(ox, p.t.scale, p.t.size, x_0, x_1, wx);
      src_coord_w(oy, p.t.scale, p.t.size, y_0, y_1, wy);
    }
    const int g0 = x0 + x_0;
    if (g0 < p.col_begin || g0 >= p.col_begin + p.local_cols) continue;  // another rank's column
    const uint8_t *a = shard_px(p, b, y0 + y_0, g0);
    const uint8_t *bb = shard_px(p, b, y0 + y_0, x0 + x_1);
    const uint8_t *c = shard_px(p, b, y0 + y_1, g0);
    const uint8_t *d = shard_px(p, b, y0 + y_1, x0 + x_1);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch)
      dst[3 * q + ch] = static_cast<uint8_t>(bilerp_fx(a[ch], bb[ch], c[ch], d[ch], wx, wy));
  }
}

// ---- seam cost ------------------------------------------------------------
__device__ __forceinline__ void box_mean(const uint8_t *img, int W, int f, int row2, int col2,
                                         double out[3]) {
  uint64_t s[3] = {0, 0, 0};
  for (int r = row2 * f; r < row2 * f + f; ++r)
    for (int c = col2 * f; c < col2 * f + f; ++c)
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) s[ch] += img[(static_cast<int64_t>(r) * W + c) * 3 + ch];
  const double n = static_cast<double>(f) * f;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) out[ch] = __ddiv_rn(static_cast<double>(s[ch]), n);
}

// One CTA per pair; thread = one (downsampled row, box) of the four boxes a
// row needs (left columns w2-2, w2-1; right columns 0, 1), so all the box
// loads of a pair are in flight at once (the four boxes of a row sit in four
// consecutive lanes and meet by shuffles).  Row costs are summed in a fixed
// order (lane tree, then warps in order, then passes): deterministic.
// f == 8 with 8-byte aligned rows: a box row is 24 bytes = 3 x 8-byte loads
// = 6 words whose channel pattern repeats every 3 words (r g b r | g b r g |
// b r g b), so per-channel byte sums are dp4a with constant masks.
__device__ __forceinline__ void box_mean8(const uint8_t *img, int W, int row2, int col2,
                                          double out[3]) {
  uint32_t s[3] = {0, 0, 0};
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const uint2 *q = reinterpret_cast<const uint2 *>(
        img + (static_cast<int64_t>(row2 * 8 + r) * W + col2 * 8) * 3);
    const uint2 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
    const uint32_t w[6] = {a.x, a.y, b.x, b.y, c.x, c.y};
#pragma unroll
    for (int k = 0; k < 6; ++k)
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        const int sh = (ch + 3 - k % 3) % 3;  // byte positions of channel ch in word k
        const uint32_t sel = sh == 0 ? 0x01000001u : sh == 1 ? 0x00000100u : 0x00010000u;
        s[ch] = __dp4a(w[k], sel, s[ch]);
      }
  }
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) out[ch] = __ddiv_rn(static_cast<double>(s[ch]), 64.0);
}

__global__ void __launch_bounds__(1024) seam_cost_kernel(const uint8_t *left, const uint8_t *right,
                                                         int H, int WL, int WR, int f,
                                                         double *cost) {
  const bool vec8 = f == 8 && (3 * WL) % 8 == 0 && (3 * WR) % 8 == 0 &&
                    reinterpret_cast<uintptr_t>(left) % 8 == 0 &&
                    reinterpret_cast<uintptr_t>(right) % 8 == 0;
  const int64_t pair = blockIdx.x;
  const uint8_t *L = left + pair * static_cast<int64_t>(H) * WL * 3;
  const uint8_t *R = right + pair * static_cast<int64_t>(H) * WR * 3;
  const int h2 = H / f, wl2 = WL / f;
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  for (int i0 = 0; i0 < 4 * h2; i0 += blockDim.x) {  // CTA-uniform trip count
    const int i = i0 + threadIdx.x;
    const int row = i >> 2, box = i & 3;
    double m[3] = {0.0, 0.0, 0.0};
    if (row < h2) {
      const uint8_t *img = box < 2 ? L : R;
      const int W = box < 2 ? WL : WR;
      const int col2 = box == 0 ? wl2 - 2 : box == 1 ? wl2 - 1 : box - 2;
      if (vec8) {
        box_mean8(img, W, row, col2, m);
      } else {
        box_mean(img, W, f, row, col2, m);
      }
    }
    // lanes 4q .. 4q+3: lm1, l0, r0, r1 of one row
    double v[4][3];
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) v[b][ch] = __shfl_sync(0xffffffffu, m[ch], (lane & ~3) | b);
    if (box == 0 && row < h2) {
      double dp = 0.0, dm = 0.0;
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        const double a = __dsub_rn(__dsub_rn(v[3][ch], v[2][ch]), __dsub_rn(v[2][ch], v[1][ch]));
        const double b = __dsub_rn(__dsub_rn(v[0][ch], v[1][ch]), __dsub_rn(v[1][ch], v[2][ch]));
        dp = __dadd_rn(dp, __dmul_rn(a, a));
        dm = __dadd_rn(dm, __dmul_rn(b, b));
      }
      acc += __ddiv_rn(__dadd_rn(sqrt(dp), sqrt(dm)), 2.0);
    }
  }
  __shared__ double part[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += part[w];
    cost[pair] = t / h2;
  }
}

static int launch_tiles(const uint8_t *images, int32_t n_cams, int32_t height, int32_t width,
                        const int32_t *windows, int32_t n_tiles, int32_t size, int32_t out_size,
                        uint8_t *tiles_out, cudaStream_t s) {
  TileParams p{};
  p.img = images;
  p.n_cams = n_cams;
  p.H = height;
  p.W = width;
  p.size = size;
  p.out = out_size;
  p.wins = windows;
  p.tiles = tiles_out;
  // host SSE float division is IEEE round-to-nearest, = np.float32(S) / np.float32(out)
  p.scale = static_cast<float>(size) / static_cast<float>(out_size);
  if (out_size == size && size <= width) {  // exact crop, <= 2 camera segments per row
    dim3 grid((size + 7) / 8, n_tiles);
    tiles_crop_kernel<<<grid, 256, 0, s>>>(p);
    return launch_status();
  }
  if (out_size == size) {  // exact crop over > 2 cameras: per-pixel gather kernel
    const int64_t npx = static_cast<int64_t>(out_size) * out_size;
    int64_t bx = (npx + 255) / 256;
    if (bx > 64) bx = 64;
    tiles_kernel<<<dim3(static_cast<unsigned>(bx), n_tiles), 256, 0, s>>>(p);
    return launch_status();
  }
  if (tiles_tma_ok(p)) return launch_tiles_tma(p, n_tiles, s, TileShard{0, n_cams * width, nullptr});
  if (size > width) {  // a window row spans > 2 cameras: per-pixel gather kernel
    const int64_t npx = static_cast<int64_t>(out_size) * out_size;
    int64_t bx = (npx + 255) / 256;
    if (bx > 64) bx = 64;
    tiles_kernel<<<dim3(static_cast<unsigned>(bx), n_tiles), 256, 0, s>>>(p);
    return launch_status();
  }
  const int S3p = ((size * 3 + 15) & ~15) + 64;
  const int smem = 2 * S3p + ((out_size * 3 + 15) & ~15);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(tiles_rows_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  dim3 grid((out_size + kTileRowsPerCta - 1) / kTileRowsPerCta, n_tiles);
  tiles_rows_kernel<<<grid, kTileThreads, smem, s>>>(p);
  return launch_status();
}

}  // namespace camx

using namespace camx;

static bool tiles_args_ok(int32_t n_cams, int32_t height, int32_t width, const int32_t *windows,
                          int32_t n_tiles, int32_t size, int32_t out_size, uint8_t *tiles_out) {
  if (n_cams < 1 || height < 1 || width < 1 || size < 1 || out_size < 1 || n_tiles < 0)
    return false;
  if (size > height || size > n_cams * width) return false;
  if (n_tiles > 0 && (windows == nullptr || tiles_out == nullptr)) return false;
  return true;
}

extern "C" int camx_tiles(const uint8_t *images, int32_t n_cams, int32_t height, int32_t width,
                          const int32_t *windows, int32_t n_tiles, int32_t size, int32_t out_size,
                          uint8_t *tiles_out, void *stream) {
  if (!images || !tiles_args_ok(n_cams, height, width, windows, n_tiles, size, out_size, tiles_out))
    return CAMX_EINVAL;
  if (n_tiles == 0) return CAMX_OK;
  // tiles ride on gridDim.y (<= 65535): chunk larger batches
  constexpr int32_t kChunk = 65535;
  const int64_t tile_bytes = static_cast<int64_t>(out_size) * out_size * 3;
  for (int32_t t0 = 0; t0 < n_tiles; t0 += kChunk) {
    const int32_t n = n_tiles - t0 < kChunk ? n_tiles - t0 : kChunk;
    const int st = launch_tiles(images, n_cams, height, width, windows + 3 * static_cast<int64_t>(t0),
                                n, size, out_size, tiles_out + t0 * tile_bytes, as_stream(stream));
    if (st != CAMX_OK) return st;
  }
  return CAMX_OK;
}

namespace camx {
// camx_tiles right behind K3 (config 5): the TMA tile kernel as a
// programmatic dependent, so its prologue overlaps K3's last wave.
int tiles_after_apply(const uint8_t *images, int32_t n_cams, int32_t height, int32_t width,
                      const int32_t *windows, int32_t n_tiles, int32_t size, int32_t out_size,
                      uint8_t *tiles_out, void *stream) {
  TileParams p{};
  p.img = images;
  p.n_cams = n_cams;
  p.H = height;
  p.W = width;
  p.size = size;
  p.out = out_size;
  p.wins = windows;
  p.tiles = tiles_out;
  p.scale = static_cast<float>(size) / static_cast<float>(out_size);
  if (out_size == size || n_tiles > 65535 || !tiles_tma_ok(p))
    return camx_tiles(images, n_cams, height, width, windows, n_tiles, size, out_size, tiles_out,
                      stream);
  return launch_tiles_tma(p, n_tiles, as_stream(stream), TileShard{0, n_cams * width, nullptr},
                          true);
}
}  // namespace camx

extern "C" int camx_seam_cost(const uint8_t *left, const uint8_t *right, int64_t n_pairs,
                              int32_t height, int32_t left_width, int32_t right_width,
                              int32_t factor, double *cost_out, void *stream) {
  if (n_pairs < 0 || !left || !right || !cost_out || factor < 1) return CAMX_EINVAL;
  if (height / factor < 1 || left_width / factor < 2 || right_width / factor < 2) return CAMX_EINVAL;
  if (n_pairs == 0) return CAMX_OK;
  const int items = 4 * (height / factor);
  const int threads = std::min(1024, (items + 31) & ~31);
  seam_cost_kernel<<<static_cast<unsigned>(n_pairs), threads, 0, as_stream(stream)>>>(
      left, right, height, left_width, right_width, factor, cost_out);
  return launch_status();
}

static int tiles_shard_launch(const uint8_t *images, int32_t n_cams, int32_t height,
                                int32_t width, int32_t col_begin, const uint8_t *halo,
                                const int32_t *windows, int32_t n_tiles, int32_t size,
                                int32_t out_size, uint8_t *tiles_out, void *stream) {
  if (!images || col_begin < 0 || n_cams < 1 || height < 1 || width < 1 || size < 1 ||
      out_size < 1 || n_tiles < 0 || size > height)
    return CAMX_EINVAL;
  if (n_tiles > 0 && (windows == nullptr || tiles_out == nullptr)) return CAMX_EINVAL;
  if (n_tiles == 0) return CAMX_OK;
  ShardTileParams p{};
  p.t.img = images;
  p.t.n_cams = n_cams;
  p.t.H = height;
  p.t.W = width;
  p.t.size = size;
  p.t.out = out_size;
  p.t.wins = windows;
  p.t.tiles = tiles_out;
  p.t.scale = static_cast<float>(size) / static_cast<float>(out_size);
  p.col_begin = col_begin;
  p.local_cols = n_cams * width;
  p.halo = halo;
  if (out_size != size && tiles_tma_ok(p.t))  // TMA-staged, warp per output row
    return launch_tiles_tma(p.t, n_tiles, as_stream(stream),
                            TileShard{col_begin, n_cams * width, halo});
  const int64_t npx = static_cast<int64_t>(out_size) * out_size;
  int64_t bx = (npx + 255) / 256;
  if (bx > 128) bx = 128;
  tiles_shard_kernel<<<dim3(static_cast<unsigned>(bx), static_cast<unsigned>(n_tiles)), 256, 0,
                       as_stream(stream)>>>(p);
  return launch_status();
}


extern "C" int camx_tiles_shard(const uint8_t *images, int32_t n_cams, int32_t height,
                                int32_t width, int32_t col_begin, const uint8_t *halo,
                                const int32_t *windows, int32_t n_tiles, int32_t size,
                                int32_t out_size, uint8_t *tiles_out, void *stream) {
  if (n_tiles < 0) return CAMX_EINVAL;
  if (n_tiles == 0)
    return tiles_shard_launch(images, n_cams, height, width, col_begin, halo, windows, 0, size,
                              out_size, tiles_out, stream);
  constexpr int32_t kChunk = 65535;  // tiles ride on gridDim.y
  const int64_t tile_bytes = static_cast<int64_t>(out_size) * out_size * 3;
  for (int32_t t0 = 0; t0 < n_tiles; t0 += kChunk) {
    const int32_t n = n_tiles - t0 < kChunk ? n_tiles - t0 : kChunk;
    const int st = tiles_shard_launch(images, n_cams, height, width, col_begin, halo,
                                      windows + 3 * static_cast<int64_t>(t0), n, size, out_size,
                                      tiles_out + t0 * tile_bytes, stream);
    if (st != CAMX_OK) return st;
  }
  return CAMX_OK;
}
