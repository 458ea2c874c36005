// K2: per-seam affine gain solve (stage 2), float64.
//
// Reference: fit_affine (camarray exposure.py:188-229), smooth_exposure
// (:232-242) and the per-mode driver update_exposure (:245-344) with its
// `resolve` fallback (:275-293).  One thread per (seam, block, channel)
// walks the batch's array-frames in order (tick loop: frame b's maps are
// frame b+1's prev_maps).  Every float64 operation uses an explicit _rn
// intrinsic in the reference's evaluation order, so there is no FMA
// contraction and results follow numpy's rounding.
#include "camx_common.cuh"

namespace camx {

struct Mom {
  double mean, sd;
  int64_t valid, area;
};

__device__ __forceinline__ Mom mom_of(const camx_band_stat &r, int ch, bool raw) {
  Mom m;
  m.area = r.area;
  m.valid = raw ? r.area : r.valid;
  const uint64_t n = static_cast<uint64_t>(m.valid);
  const uint64_t s = raw ? r.raw_sum[ch] : r.sum[ch];
  const uint64_t q = raw ? r.raw_sumsq[ch] : r.sumsq[ch];
  if (n == 0) {
    m.mean = 0.0;
    m.sd = 0.0;
    return m;
  }
  const unsigned __int128 nq = static_cast<unsigned __int128>(n) * q;
  const unsigned __int128 ss = static_cast<unsigned __int128>(s) * s;
  const unsigned __int128 d = nq > ss ? nq - ss : 0;
  const double dn = static_cast<double>(n);
  m.mean = __ddiv_rn(static_cast<double>(s), dn);
  m.sd = sqrt(__ddiv_rn(static_cast<double>(d), __dmul_rn(dn, dn)));
  return m;
}

struct Pair {
  double gl, ol, gr, orr;
};

// exposure.py:205-229 for one (block, channel).
__device__ __forceinline__ void side_coeffs(bool ok, double mu_s, double sd_s, double mean,
                                            double sd, double sigma_min, double &g, double &o) {
  const bool usable = ok && (sd >= sigma_min);
  g = usable ? __ddiv_rn(sd_s, sd) : 1.0;
  o = ok ? __dsub_rn(mu_s, __dmul_rn(g, mean)) : 0.0;
  if (ok && !usable) o = __dsub_rn(mu_s, mean);
  g = fmax(g, 1e-12);
}

__device__ __forceinline__ Pair fit_pair(double lmean, double lsd, int64_t lvalid, double rmean,
                                         double rsd, int64_t rvalid, double sigma_min,
                                         int64_t min_px, bool &ok) {
  ok = (lvalid > min_px) && (rvalid > min_px);
  const double mu_s = __ddiv_rn(__dadd_rn(lmean, rmean), 2.0);
  const double sd_s = __ddiv_rn(__dadd_rn(lsd, rsd), 2.0);
  Pair p;
  side_coeffs(ok, mu_s, sd_s, lmean, lsd, sigma_min, p.gl, p.ol);
  side_coeffs(ok, mu_s, sd_s, rmean, rsd, sigma_min, p.gr, p.orr);
  return p;
}

__device__ __forceinline__ double blend(double prev, double nw, double alpha) {
  // (1 - alpha) * prev + alpha * new   (exposure.py:240-241)
  return __dadd_rn(__dmul_rn(__dsub_rn(1.0, alpha), prev), __dmul_rn(alpha, nw));
}

__device__ __forceinline__ Pair blend_pair(const Pair &a, const Pair &b, double alpha) {
  return Pair{blend(a.gl, b.gl, alpha), blend(a.ol, b.ol, alpha), blend(a.gr, b.gr, alpha),
              blend(a.orr, b.orr, alpha)};
}

struct SolveParams {
  const camx_band_stat *stats;  // [B][N][2][K]
  int32_t B, N, S, K, wrap;
  camx_solve_config cfg;
  const double *prev_gain, *prev_offset;  // [S][2][K][3]
  double *gain, *offset;                  // [B][S][2][K][3]
  uint8_t *fit_ok;                        // [B][S][K]
};

__global__ void seam_solve_kernel(const SolveParams p) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= p.S * p.K * 3) return;
  const int ch = t % 3;
  const int k = (t / 3) % p.K;
  const int s = t / (3 * p.K);
  const int camL = s;
  const int camR = (s + 1) % p.N;
  const camx_solve_config &cfg = p.cfg;
  const int K3 = p.K * 3;
  const int iL = k * 3 + ch;                 // offset inside a [K][3] map
  const int64_t prev_base = static_cast<int64_t>(s) * 2 * K3;

  bool have_prev = cfg.have_prev_maps != 0;
  Pair prev{1.0, 0.0, 1.0, 0.0};
  if (have_prev) {
    prev.gl = p.prev_gain[prev_base + iL];
    prev.ol = p.prev_offset[prev_base + iL];
    prev.gr = p.prev_gain[prev_base + K3 + iL];
    prev.orr = p.prev_offset[prev_base + K3 + iL];
  }
  for (int b = 0; b < p.B; ++b) {
    const camx_band_stat &L =
        p.stats[((static_cast<int64_t>(b) * p.N + camL) * 2 + CAMX_SIDE_LEFT) * p.K + k];
    const camx_band_stat &R =
        p.stats[((static_cast<int64_t>(b) * p.N + camR) * 2 + CAMX_SIDE_RIGHT) * p.K + k];
    const Mom Lr = mom_of(L, ch, true), Rr = mom_of(R, ch, true);
    bool ok_raw;
    const Pair raw = fit_pair(Lr.mean, Lr.sd, Lr.valid, Rr.mean, Rr.sd, Rr.valid, cfg.sigma_min,
                              cfg.min_band_pixels, ok_raw);
    // resolve(): unfittable blocks keep the previous maps, else identity
    const Pair fallback = have_prev ? prev : Pair{1.0, 0.0, 1.0, 0.0};
    const Pair fresh = ok_raw ? raw : fallback;
    Pair out;
    const bool prev_frames = (b > 0) || (cfg.have_prev_frames != 0);
    if (cfg.mode == CAMX_MODE_SMOOTHING) {
      out = have_prev ? blend_pair(prev, fresh, cfg.alpha) : fresh;
    } else if (cfg.mode == CAMX_MODE_OBJECT_REMOVAL && prev_frames) {
      const Mom Lm = mom_of(L, ch, false), Rm = mom_of(R, ch, false);
      bool ok_m;
      const Pair masked = fit_pair(Lm.mean, Lm.sd, Lm.valid, Rm.mean, Rm.sd, Rm.valid,
                                   cfg.sigma_min, cfg.min_band_pixels, ok_m);
      const double fl = __ddiv_rn(static_cast<double>(Lm.valid),
                                  static_cast<double>(Lm.area > 1 ? Lm.area : 1));
      const double fr = __ddiv_rn(static_cast<double>(Rm.valid),
                                  static_cast<double>(Rm.area > 1 ? Rm.area : 1));
      const bool keep = ok_m && (fmin(fl, fr) >= cfg.min_valid_fraction);
      const Pair smoothed = have_prev ? blend_pair(prev, fresh, cfg.alpha) : fresh;
      out = keep ? masked : smoothed;
    } else {  // STANDARD, or OBJECT_REMOVAL without previous frames
      out = fresh;
    }
    const int64_t ob = (static_cast<int64_t>(b) * p.S + s) * 2 * K3;
    p.gain[ob + iL] = out.gl;
    p.offset[ob + iL] = out.ol;
    p.gain[ob + K3 + iL] = out.gr;
    p.offset[ob + K3 + iL] = out.orr;
    if (p.fit_ok != nullptr && ch == 0)
      p.fit_ok[(static_cast<int64_t>(b) * p.S + s) * p.K + k] = ok_raw ? 1 : 0;
    prev = out;
    have_prev = true;
  }
}

__global__ void fit_affine_kernel(const double *lm, const double *ls, const int64_t *lv,
                                  const double *rm, const double *rs, const int64_t *rv, int K,
                                  double sigma_min, int64_t min_px, double *gain, double *offset,
                                  uint8_t *fit_ok) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K * 3) return;
  const int k = t / 3;
  bool ok;
  const Pair p = fit_pair(lm[t], ls[t], lv[k], rm[t], rs[t], rv[k], sigma_min, min_px, ok);
  gain[t] = p.gl;
  offset[t] = p.ol;
  gain[K * 3 + t] = p.gr;
  offset[K * 3 + t] = p.orr;
  if (fit_ok != nullptr && t % 3 == 0) fit_ok[k] = ok ? 1 : 0;
}

__global__ void smooth_kernel(const double *pg, const double *po, const double *ng,
                              const double *no, int64_t n, double alpha, double *g, double *o) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    g[i] = blend(pg[i], ng[i], alpha);
    o[i] = blend(po[i], no[i], alpha);
  }
}

}  // namespace camx

using namespace camx;

extern "C" int camx_seam_solve(const camx_band_stat *stats, int32_t n_batch, int32_t n_cams,
                               int32_t wrap, const camx_solve_config *cfg,
                               const double *prev_gain, const double *prev_offset,
                               double *gain_out, double *offset_out, uint8_t *fit_ok_out,
                               void *stream) {
  if (cfg == nullptr || stats == nullptr || gain_out == nullptr || offset_out == nullptr)
    return CAMX_EINVAL;
  if (n_batch < 0 || n_cams < 1 || cfg->blocks < 1) return CAMX_EINVAL;
  if (wrap && n_cams < 2) return CAMX_EINVAL;
  if (cfg->mode < CAMX_MODE_STANDARD || cfg->mode > CAMX_MODE_SMOOTHING) return CAMX_EINVAL;
  if (cfg->have_prev_maps && (prev_gain == nullptr || prev_offset == nullptr)) return CAMX_EINVAL;
  SolveParams p{};
  p.stats = stats;
  p.B = n_batch;
  p.N = n_cams;
  p.S = wrap ? n_cams : n_cams - 1;
  p.K = cfg->blocks;
  p.wrap = wrap;
  p.cfg = *cfg;
  p.prev_gain = prev_gain;
  p.prev_offset = prev_offset;
  p.gain = gain_out;
  p.offset = offset_out;
  p.fit_ok = fit_ok_out;
  const int threads = p.S * p.K * 3;
  if (threads == 0 || n_batch == 0) return CAMX_OK;
  seam_solve_kernel<<<(threads + 63) / 64, 64, 0, as_stream(stream)>>>(p);
  return launch_status();
}

extern "C" int camx_fit_affine(const double *l_mean, const double *l_std, const int64_t *l_valid,
                               const double *r_mean, const double *r_std, const int64_t *r_valid,
                               int32_t blocks, double sigma_min, int64_t min_band_pixels,
                               double *gain_out, double *offset_out, uint8_t *fit_ok_out,
                               void *stream) {
  if (blocks < 1 || !l_mean || !l_std || !l_valid || !r_mean || !r_std || !r_valid || !gain_out ||
      !offset_out)
    return CAMX_EINVAL;
  const int n = blocks * 3;
  fit_affine_kernel<<<(n + 127) / 128, 128, 0, as_stream(stream)>>>(
      l_mean, l_std, l_valid, r_mean, r_std, r_valid, blocks, sigma_min, min_band_pixels,
      gain_out, offset_out, fit_ok_out);
  return launch_status();
}

extern "C" int camx_smooth_maps(const double *prev_gain, const double *prev_offset,
                                const double *new_gain, const double *new_offset, int64_t n,
                                double alpha, double *gain_out, double *offset_out,
                                void *stream) {
  if (n < 0 || !prev_gain || !prev_offset || !new_gain || !new_offset || !gain_out || !offset_out)
    return CAMX_EINVAL;
  if (n == 0) return CAMX_OK;
  const int64_t blocks = (n + 127) / 128;
  smooth_kernel<<<static_cast<unsigned>(blocks > 1024 ? 1024 : blocks), 128, 0,
                  as_stream(stream)>>>(prev_gain, prev_offset, new_gain, new_offset, n, alpha,
                                       gain_out, offset_out);
  return launch_status();
}
