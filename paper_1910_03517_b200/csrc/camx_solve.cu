// K2: per-seam affine gain solve (stage 2), float64 - standalone kernels
// (array solve, fit_affine, smooth_exposure).  Device code: camx_solve.cuh.
#include "camx_solve.cuh"

namespace camx {

__global__ void __launch_bounds__(3 * kSolveFrames) seam_solve_kernel(const SolveParams p) {
  __shared__ Cand cand[kSolveFrames][3];
  // programmatic dependent launch (camx_correct_batch): the records come
  // from the preceding K1 grid; let K3 start its pixel prefetch right away
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  solve_seam_block(p, blockIdx.x / p.K, blockIdx.x % p.K, cand);
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

namespace camx {
// Launch helper shared with camx_correct_batch (pdl = programmatic dependent).
int launch_seam_solve(const camx_band_stat *stats, int32_t n_batch, int32_t n_cams, int32_t wrap,
                      const camx_solve_config *cfg, const double *prev_gain,
                      const double *prev_offset, double *gain_out, double *offset_out,
                      uint8_t *fit_ok_out, cudaStream_t stream, bool pdl, int32_t world,
                      int32_t cmax) {
  SolveParams p{};
  p.stats = stats;
  p.world = world;
  p.cmax = cmax;
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
  if (p.S * p.K == 0 || n_batch == 0) return CAMX_OK;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(p.S * p.K);
  lc.blockDim = dim3(3 * kSolveFrames);
  lc.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = pdl ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&lc, seam_solve_kernel, p);
  return e == cudaSuccess ? launch_status() : static_cast<int>(e);
}
}  // namespace camx

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
  return launch_seam_solve(stats, n_batch, n_cams, wrap, cfg, prev_gain, prev_offset, gain_out,
                           offset_out, fit_ok_out, as_stream(stream), false, 1, n_cams);
}

extern "C" int camx_seam_solve_sharded(const camx_band_stat *stats_all, int32_t n_batch,
                                       int32_t n_cams, int32_t world, int32_t wrap,
                                       const camx_solve_config *cfg, const double *prev_gain,
                                       const double *prev_offset, double *gain_out,
                                       double *offset_out, uint8_t *fit_ok_out, void *stream) {
  if (cfg == nullptr || stats_all == nullptr || gain_out == nullptr || offset_out == nullptr)
    return CAMX_EINVAL;
  if (n_batch < 0 || n_cams < 1 || cfg->blocks < 1 || world < 1 || world > n_cams)
    return CAMX_EINVAL;
  if (wrap && n_cams < 2) return CAMX_EINVAL;
  if (cfg->mode < CAMX_MODE_STANDARD || cfg->mode > CAMX_MODE_SMOOTHING) return CAMX_EINVAL;
  if (cfg->have_prev_maps && (prev_gain == nullptr || prev_offset == nullptr)) return CAMX_EINVAL;
  const int32_t cmax = (n_cams + world - 1) / world;
  return launch_seam_solve(stats_all, n_batch, n_cams, wrap, cfg, prev_gain, prev_offset,
                           gain_out, offset_out, fit_ok_out, as_stream(stream), false, world, cmax);
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
