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
// Decomposition: one CTA of 3 warps per (image, side, block); warp w owns
// colour channel w, so every lane counts only one channel.  Histograms use
// per-lane private 8-bit counters in shared memory (4 bins per 32-bit word,
// word (bin/4, lane) at bank `lane`, so increments never conflict and need
// no atomics), flushed every 255 pixels per lane into per-lane registers
// by a SWAR (2 x 16-bit lanes) column sum.
#include "camx_common.cuh"

namespace camx {

struct StatsParams {
  const uint8_t *img;
  const uint8_t *prev;   // mode 2
  const uint8_t *mask;   // mode 1
  int64_t img_bytes;
  int64_t mask_bytes;    // H * W
  int32_t H, W, bw, K, bh, t_diff;
  camx_band_stat *out;
  uint32_t *hist;        // optional
};

constexpr int kStatsWarps = 3;
constexpr int kCounterWords = 64 * 32;  // per warp: 64 bin-quads x 32 lanes

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <bool HIST, int MASKMODE>
__global__ void __launch_bounds__(96) band_stats_kernel(const StatsParams p) {
  extern __shared__ uint32_t smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ch = warp;
  const int64_t unit = blockIdx.x;
  const int k = static_cast<int>(unit % p.K);
  const int side = static_cast<int>((unit / p.K) % 2);
  const int64_t img = unit / (2 * p.K);

  const int r0 = k * p.bh;
  const int r1 = (k == p.K - 1) ? p.H : r0 + p.bh;
  const int col0 = (side == CAMX_SIDE_LEFT) ? p.W - p.bw : 0;
  const int64_t npix = static_cast<int64_t>(r1 - r0) * p.bw;
  const int64_t row_bytes = static_cast<int64_t>(p.W) * 3;
  const uint8_t *base = p.img + img * p.img_bytes;
  const uint8_t *pbase = (MASKMODE == 2) ? p.prev + img * p.img_bytes : nullptr;
  const uint8_t *mbase = (MASKMODE == 1) ? p.mask + img * p.mask_bytes : nullptr;

  uint32_t *cnt = smem + warp * kCounterWords;
  if (HIST) {
    for (int w = 0; w < 64; ++w) cnt[w * 32 + lane] = 0u;
    __syncwarp();
  }
  uint32_t bins[8];  // this lane's bins 4*lane..4*lane+3 and 128+4*lane..+3
#pragma unroll
  for (int i = 0; i < 8; ++i) bins[i] = 0u;

  uint64_t raw_s = 0, raw_q = 0, val_s = 0, val_q = 0, nvalid = 0;
  // (row, col) of pixel index p = lane + 32 t, stepped incrementally
  int rr = r0 + lane / p.bw;
  int cc = lane % p.bw;
  int64_t pidx = lane;
  int round_left = 255;
  const int64_t iters = (npix + 31) / 32;
  for (int64_t t = 0; t < iters; ++t) {
    if (pidx < npix) {
      const int64_t off = static_cast<int64_t>(rr) * row_bytes + static_cast<int64_t>(col0 + cc) * 3;
      const uint32_t v = base[off + ch];
      bool excluded = false;
      if (MASKMODE == 1) {
        excluded = mbase[static_cast<int64_t>(rr) * p.W + col0 + cc] != 0;
      } else if (MASKMODE == 2) {
        int d = 0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int a = base[off + c], b = pbase[off + c];
          d = max(d, abs(a - b));
        }
        excluded = d > p.t_diff;
      }
      raw_s += v;
      raw_q += v * v;
      if (!excluded) {
        nvalid += 1;
        if (HIST) {
          uint32_t *wp = cnt + (v >> 2) * 32 + lane;
          *wp += 1u << ((v & 3u) * 8u);
        } else {
          val_s += v;
          val_q += v * v;
        }
      }
    }
    pidx += 32;
    cc += 32;
    while (cc >= p.bw) {
      cc -= p.bw;
      ++rr;
    }
    if (HIST && (--round_left == 0 || t == iters - 1)) {
      round_left = 255;
      __syncwarp();
      // lane owns bin-quads w = lane and lane + 32; sum them over 32 lanes
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int w = lane + 32 * h;
        uint32_t lo = 0, hi = 0;
#pragma unroll 8
        for (int l = 0; l < 32; ++l) {
          const uint32_t x = cnt[w * 32 + ((l + lane) & 31)];
          lo += x & 0x00FF00FFu;
          hi += (x >> 8) & 0x00FF00FFu;
        }
        bins[4 * h + 0] += lo & 0xFFFFu;
        bins[4 * h + 1] += hi & 0xFFFFu;
        bins[4 * h + 2] += lo >> 16;
        bins[4 * h + 3] += hi >> 16;
      }
      __syncwarp();
      for (int w = 0; w < 64; ++w) cnt[w * 32 + lane] = 0u;
      __syncwarp();
    }
  }

  if (HIST) {
    val_s = 0;
    val_q = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint64_t bin = 4 * (lane + 32 * h) + i;
        val_s += bin * bins[4 * h + i];
        val_q += bin * bin * bins[4 * h + i];
      }
    }
    if (p.hist != nullptr) {
      uint32_t *hp = p.hist + ((img * 2 + side) * p.K + k) * 768 + ch * 256;
      reinterpret_cast<uint4 *>(hp)[lane] = make_uint4(bins[0], bins[1], bins[2], bins[3]);
      reinterpret_cast<uint4 *>(hp + 128)[lane] = make_uint4(bins[4], bins[5], bins[6], bins[7]);
    }
  }
  raw_s = warp_sum_u64(raw_s);
  raw_q = warp_sum_u64(raw_q);
  val_s = warp_sum_u64(val_s);
  val_q = warp_sum_u64(val_q);
  nvalid = warp_sum_u64(nvalid);
  if (lane == 0) {
    camx_band_stat *o = p.out + (img * 2 + side) * p.K + k;
    o->sum[ch] = val_s;
    o->sumsq[ch] = val_q;
    o->raw_sum[ch] = raw_s;
    o->raw_sumsq[ch] = raw_q;
    if (ch == 0) {
      o->area = npix;
      o->valid = static_cast<int64_t>(nvalid);
    }
  }
}

template <bool HIST, int MASKMODE>
static void launch_stats(const StatsParams &p, int64_t n_units, cudaStream_t s) {
  const size_t smem = HIST ? kStatsWarps * kCounterWords * sizeof(uint32_t) : 0;
  if (HIST) {
    cudaFuncSetAttribute(band_stats_kernel<HIST, MASKMODE>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  }
  band_stats_kernel<HIST, MASKMODE>
      <<<static_cast<unsigned>(n_units), kStatsWarps * 32, smem, s>>>(p);
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

extern "C" int camx_band_stats(const uint8_t *images, const uint8_t *prev_images,
                               const uint8_t *excl_masks, int64_t n_images, int32_t height,
                               int32_t width, int32_t band_width, int32_t blocks, int32_t t_diff,
                               camx_band_stat *stats_out, uint32_t *hist_out, void *stream) {
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
  p.mask = excl_masks;
  p.H = height;
  p.W = width;
  p.bw = band_width;
  p.K = blocks;
  p.bh = height / blocks;
  p.t_diff = t_diff;
  p.img_bytes = static_cast<int64_t>(height) * width * 3;
  p.mask_bytes = static_cast<int64_t>(height) * width;
  p.out = stats_out;
  p.hist = hist_out;
  const int64_t units = n_images * 2 * blocks;
  cudaStream_t s = as_stream(stream);
  const int mm = prev_images ? 2 : (excl_masks ? 1 : 0);
  const bool h = hist_out != nullptr;
  if (h) {
    if (mm == 0) launch_stats<true, 0>(p, units, s);
    if (mm == 1) launch_stats<true, 1>(p, units, s);
    if (mm == 2) launch_stats<true, 2>(p, units, s);
  } else {
    if (mm == 0) launch_stats<false, 0>(p, units, s);
    if (mm == 1) launch_stats<false, 1>(p, units, s);
    if (mm == 2) launch_stats<false, 2>(p, units, s);
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
