// Shared float64 seam-solve device code (K2), used by the standalone solve
// kernel and by the fused stats+solve kernel.
//
// Reference: fit_affine (camarray exposure.py:188-229), smooth_exposure
// (:232-242) and the per-mode driver update_exposure (:245-344) with its
// `resolve` fallback (:275-293), for every seam of a batch of array-frames
// processed as a tick loop (frame b's maps are frame b+1's prev_maps).
// Every float64 operation uses an explicit _rn intrinsic in the reference's
// evaluation order, so there is no FMA contraction and results follow
// numpy's rounding.
#pragma once

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
  const camx_band_stat *stats;  // [B][N][2][K], or rank-major (world > 1, see rec_index)
  int32_t B, N, S, K, wrap;
  int32_t world, cmax;          // camera shards: world ranks, <= cmax cameras each
  camx_solve_config cfg;
  const double *prev_gain, *prev_offset;  // [S][2][K][3]
  double *gain, *offset;                  // [B][S][2][K][3]
  uint8_t *fit_ok;                        // [B][S][K]
};

// Two phases per CTA = one (seam, block):
//  A (parallel over frames x channels): raw fit, fit_ok, masked fit and the
//    keep flag of every frame -> shared memory.  All global loads of the
//    batch are independent, so they overlap.
//  B (one thread per channel): the cheap loop-carried part of the tick loop
//    (resolve fallback / smoothing / selection) over the candidates.
constexpr int kSolveFrames = 64;  // frames per shared-memory chunk

struct Cand {
  Pair raw, masked;
  int ok_raw, keep;
};

// One (seam s, block k) over the whole batch, by the calling CTA (any
// blockDim >= 3).  `load_rec` must see records written by other CTAs of a
// still-running grid (fused path), hence the L1-bypassing loads.
__device__ __forceinline__ camx_band_stat load_rec(const camx_band_stat *r) {
  camx_band_stat o;
  const uint64_t *src = reinterpret_cast<const uint64_t *>(r);
  uint64_t *dst = reinterpret_cast<uint64_t *>(&o);
#pragma unroll
  for (int i = 0; i < 14; ++i) dst[i] = __ldcg(src + i);
  return o;
}

// Record of (frame b, camera cam, side, block k).  world <= 1: the dense
// [B][N][2][K] layout.  world > 1: the NCCL all-gather of the camera shards
// (dist.camera_partition: contiguous groups, sizes differing by <= 1), rank
// g's block [B][cmax][2][K] at g * B * cmax records, camera cam at local
// index cam - begin(g).
__device__ __forceinline__ int64_t rec_index(const SolveParams &p, int b, int cam, int side,
                                             int k) {
  int64_t slot;
  if (p.world <= 1) {
    slot = static_cast<int64_t>(b) * p.N + cam;
  } else {
    const int q = p.N / p.world, r = p.N % p.world;
    const int g = cam < (q + 1) * r ? cam / (q + 1) : r + (cam - (q + 1) * r) / q;
    const int beg = g * q + min(g, r);
    slot = (static_cast<int64_t>(g) * p.B + b) * p.cmax + (cam - beg);
  }
  return (slot * 2 + side) * p.K + k;
}

__device__ __forceinline__ void solve_seam_block(const SolveParams &p, int s, int k,
                                                 Cand (*cand)[3]) {
  const int camL = s;
  const int camR = (s + 1) % p.N;
  const camx_solve_config &cfg = p.cfg;
  const int K3 = p.K * 3;
  const bool removal = cfg.mode == CAMX_MODE_OBJECT_REMOVAL;
  const int chB = threadIdx.x;
  bool have_prev = cfg.have_prev_maps != 0;
  Pair prev{1.0, 0.0, 1.0, 0.0};
  __shared__ Pair prev_s[3], next_s[3];
  if (chB < 3 && have_prev) {
    const int64_t pb = static_cast<int64_t>(s) * 2 * K3 + k * 3 + chB;
    prev.gl = p.prev_gain[pb];
    prev.ol = p.prev_offset[pb];
    prev.gr = p.prev_gain[pb + K3];
    prev.orr = p.prev_offset[pb + K3];
  }
  for (int b0 = 0; b0 < p.B; b0 += kSolveFrames) {
    const int nb = min(kSolveFrames, p.B - b0);
    bool any_blend = false;
    // ---- phase A: independent per (frame, channel)
    for (int idx = threadIdx.x; idx < nb * 3; idx += blockDim.x) {
      const int bl = idx / 3;
      const int ch = idx % 3;
      const int b = b0 + bl;
      const camx_band_stat L = load_rec(&p.stats[rec_index(p, b, camL, CAMX_SIDE_LEFT, k)]);
      const camx_band_stat R = load_rec(&p.stats[rec_index(p, b, camR, CAMX_SIDE_RIGHT, k)]);
      Cand c;
      const Mom Lr = mom_of(L, ch, true), Rr = mom_of(R, ch, true);
      bool ok;
      c.raw = fit_pair(Lr.mean, Lr.sd, Lr.valid, Rr.mean, Rr.sd, Rr.valid, cfg.sigma_min,
                       cfg.min_band_pixels, ok);
      c.ok_raw = ok;
      c.keep = 0;
      c.masked = c.raw;
      if (removal && ((b > 0) || (cfg.have_prev_frames != 0))) {
        const Mom Lm = mom_of(L, ch, false), Rm = mom_of(R, ch, false);
        bool ok_m;
        c.masked = fit_pair(Lm.mean, Lm.sd, Lm.valid, Rm.mean, Rm.sd, Rm.valid, cfg.sigma_min,
                            cfg.min_band_pixels, ok_m);
        const double fl = __ddiv_rn(static_cast<double>(Lm.valid),
                                    static_cast<double>(Lm.area > 1 ? Lm.area : 1));
        const double fr = __ddiv_rn(static_cast<double>(Rm.valid),
                                    static_cast<double>(Rm.area > 1 ? Rm.area : 1));
        c.keep = (ok_m && (fmin(fl, fr) >= cfg.min_valid_fraction)) ? 1 : 2;  // 2: smooth
      }
      cand[bl][ch] = c;
      any_blend |= (c.keep == 2);
    }
    // Without a blend (SMOOTHING, or OBJECT_REMOVAL's smoothing fallback)
    // the tick loop only carries the previous output through unfittable
    // frames: out[b] = value of the last "defined" frame j <= b (masked fit
    // kept, or raw fit ok), else the chunk's incoming maps - every frame is
    // independent given that, so phase B runs in parallel.
    const bool parallel =
        !__syncthreads_or(any_blend) && cfg.mode != CAMX_MODE_SMOOTHING;
    if (parallel) {
      if (chB < 3) prev_s[chB] = have_prev ? prev : Pair{1.0, 0.0, 1.0, 0.0};
      __syncthreads();
      for (int idx = threadIdx.x; idx < nb * 3; idx += blockDim.x) {
        const int bl = idx / 3;
        const int ch = idx % 3;
        int j = bl;
        while (j >= 0 && !(cand[j][ch].keep == 1 || cand[j][ch].ok_raw)) --j;
        const Pair out = j < 0 ? prev_s[ch] : (cand[j][ch].keep == 1 ? cand[j][ch].masked
                                                                       : cand[j][ch].raw);
        const int b = b0 + bl;
        const int64_t ob = (static_cast<int64_t>(b) * p.S + s) * 2 * K3 + k * 3 + ch;
        p.gain[ob] = out.gl;
        p.offset[ob] = out.ol;
        p.gain[ob + K3] = out.gr;
        p.offset[ob + K3] = out.orr;
        if (p.fit_ok != nullptr && ch == 0)
          p.fit_ok[(static_cast<int64_t>(b) * p.S + s) * p.K + k] = cand[bl][0].ok_raw ? 1 : 0;
        if (bl == nb - 1) next_s[ch] = out;  // carried into the next chunk
      }
      __syncthreads();
      if (chB < 3) {
        prev = next_s[chB];
        have_prev = true;
      }
    }
    // ---- phase B: the tick loop (exposure.py:295-342)
    if (!parallel && chB < 3) {
      for (int bl = 0; bl < nb; ++bl) {
        const int b = b0 + bl;
        const Cand &c = cand[bl][chB];
        const Pair fallback = have_prev ? prev : Pair{1.0, 0.0, 1.0, 0.0};
        const Pair fresh = c.ok_raw ? c.raw : fallback;  // resolve()
        Pair out;
        if (cfg.mode == CAMX_MODE_SMOOTHING) {
          out = have_prev ? blend_pair(prev, fresh, cfg.alpha) : fresh;
        } else if (c.keep == 1) {
          out = c.masked;
        } else if (c.keep == 2) {
          out = have_prev ? blend_pair(prev, fresh, cfg.alpha) : fresh;
        } else {  // STANDARD, or OBJECT_REMOVAL without previous frames
          out = fresh;
        }
        const int64_t ob = (static_cast<int64_t>(b) * p.S + s) * 2 * K3 + k * 3 + chB;
        p.gain[ob] = out.gl;
        p.offset[ob] = out.ol;
        p.gain[ob + K3] = out.gr;
        p.offset[ob + K3] = out.orr;
        if (p.fit_ok != nullptr && chB == 0)
          p.fit_ok[(static_cast<int64_t>(b) * p.S + s) * p.K + k] = c.ok_raw ? 1 : 0;
        prev = out;
        have_prev = true;
      }
    }
    __syncthreads();
  }
}

}  // namespace camx
