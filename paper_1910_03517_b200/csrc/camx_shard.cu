// Camera-sharded arrays: one process per GPU, rank g owns the
// contiguous camera group of dist.camera_partition.  Per batch: K1 on the
// rank's cameras -> one ncclAllGather of the fixed-size seam records
// (camx_comm.cu) -> K2 for every seam on the rank-major gathered records
// (camx_solve.cuh: rec_index) -> K3 on the rank's cameras.  Corrected
// pixels are byte-identical to the one-GPU path.
//   camx_correct_batch_sharded       one batch (optionally chunked: the
//                                    front half of chunk c+1 on a side
//                                    stream under K3 of chunk c)
//   camx_correct_batch_sharded_step  one step of a pipelined stream: the
//                                    front half of batch k under K3 of
//                                    batch k-1 (ArrayCorrector.submit)
#include <map>
#include <mutex>
#include <utility>

#include <algorithm>

#include "camx_common.cuh"

namespace camx {
int comm_all_gather(const void *send, void *recv, size_t bytes, void *comm, cudaStream_t s);
int band_stats_frames(const uint8_t *images, const uint8_t *prev_frame, int32_t n_batch,
                      int32_t per_frame, int32_t height, int32_t width, int32_t band_width,
                      int32_t blocks, int32_t t_diff, bool removal, camx_band_stat *stats,
                      uint32_t *hist, void *stream);
int launch_seam_solve(const camx_band_stat *stats, int32_t n_batch, int32_t n_cams, int32_t wrap,
                      const camx_solve_config *cfg, const double *prev_gain,
                      const double *prev_offset, double *gain_out, double *offset_out,
                      uint8_t *fit_ok_out, cudaStream_t stream, bool pdl, int32_t world,
                      int32_t cmax);
int apply_camera_group_motion(const uint8_t *images, uint8_t *out, int nb, int cam_begin,
                              int cam_count, int n_cams, int wrap, int height, int width,
                              int blocks, const double *gain, const double *offset,
                              const uint8_t *motion_prev, int32_t win_size, int32_t t_motion,
                              int64_t *counts, cudaStream_t s);
int apply_camera_group(const uint8_t *images, uint8_t *out, int nb, int cam_begin, int cam_count,
                       int n_cams, int wrap, int height, int width, int blocks,
                       const double *gain, const double *offset, bool pdl, cudaStream_t s);

constexpr int kMaxShardChunks = 8;

// Library-owned side stream + events of the sharded pipelines, one set per
// (device, communicator) - several ranks of a loopback group share a device
// but never a pipeline (capture-safe: only event record / wait).  ev[0]
// fork, ev[1..] per chunk, step[0] the join of camx_correct_batch_sharded_step.
struct SidePipe {
  cudaStream_t side = nullptr;
  cudaEvent_t ev[kMaxShardChunks + 1] = {};
  cudaEvent_t step[1] = {};
};
static std::mutex g_pipe_mu;
static int side_pipe(SidePipe *&out, void *comm) {
  static std::map<std::pair<int, void *>, SidePipe> pipes;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return static_cast<int>(e);
  std::lock_guard<std::mutex> lock(g_pipe_mu);
  SidePipe &sp = pipes[std::make_pair(dev, comm)];  // std::map: stable addresses
  if (sp.side == nullptr) {
    e = cudaStreamCreateWithFlags(&sp.side, cudaStreamNonBlocking);
    for (int i = 0; e == cudaSuccess && i < kMaxShardChunks + 1; ++i)
      e = cudaEventCreateWithFlags(&sp.ev[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sp.step[0], cudaEventDisableTiming);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  out = &sp;
  return CAMX_OK;
}

// Geometry of one rank's shard, validated against camera_partition.
struct ShardGeom {
  int n_cams, cam_begin, cam_count, world, rank, cmax, wrap, S, H, W, bw, t_diff;
  bool removal;
  int64_t frame_bytes;  // one frame of this rank's cameras
  size_t rec;           // one camera-frame of records (2 sides x K)
  int64_t map_frame;    // one frame of maps (S x 2 x K x 3 doubles)
};
static int shard_geom(ShardGeom &g, int32_t n_cams, int32_t cam_begin, int32_t cam_count,
                      int32_t world, int32_t wrap, int32_t height, int32_t width,
                      int32_t band_width, int32_t t_diff, const camx_solve_config *cfg,
                      const double *prev_gain, const double *prev_offset, void *comm) {
  if (cfg == nullptr || n_cams < 2 || world < 1 || world > n_cams) return CAMX_EINVAL;
  if (cfg->blocks < 1 || cfg->blocks > height) return CAMX_EINVAL;
  if (cfg->mode < CAMX_MODE_STANDARD || cfg->mode > CAMX_MODE_SMOOTHING) return CAMX_EINVAL;
  if (cfg->have_prev_maps && (prev_gain == nullptr || prev_offset == nullptr)) return CAMX_EINVAL;
  // this rank's group must be one of camera_partition(n_cams, world)
  const int q = n_cams / world, r = n_cams % world;
  g.rank = -1;
  for (int k = 0; k < world; ++k)
    if (k * q + (k < r ? k : r) == cam_begin && q + (k < r ? 1 : 0) == cam_count) g.rank = k;
  if (g.rank < 0) return CAMX_EINVAL;
  if (world > 1 && comm == nullptr) return CAMX_EINVAL;
  g.n_cams = n_cams;
  g.cam_begin = cam_begin;
  g.cam_count = cam_count;
  g.world = world;
  g.cmax = (n_cams + world - 1) / world;
  g.wrap = wrap;
  g.S = wrap ? n_cams : n_cams - 1;
  g.H = height;
  g.W = width;
  g.bw = band_width;
  g.t_diff = t_diff;
  g.removal = cfg->mode == CAMX_MODE_OBJECT_REMOVAL;
  g.frame_bytes = static_cast<int64_t>(height) * width * 3 * cam_count;
  g.rec = sizeof(camx_band_stat) * 2 * cfg->blocks;
  g.map_frame = static_cast<int64_t>(g.S) * 2 * cfg->blocks * 3;
  return CAMX_OK;
}

// Front half for nb frames on stream s: K1 on this rank's cameras -> pad +
// ncclAllGather -> K2 (all seams, rank-major records).  stats_local is
// dense [nb][cam_count], stats_all [world][nb][cmax].
static int shard_front(const ShardGeom &g, const uint8_t *images, const uint8_t *prev_frame,
                       int nb, const camx_solve_config *cfg, const double *prev_gain,
                       const double *prev_offset, camx_band_stat *stats_local,
                       camx_band_stat *stats_all, uint32_t *hist, double *gain, double *offset,
                       uint8_t *fit_ok, void *comm, cudaStream_t s) {
  int st = band_stats_frames(images, prev_frame, nb, g.cam_count, g.H, g.W, g.bw, cfg->blocks,
                             g.t_diff, g.removal, stats_local, hist, s);
  if (st != CAMX_OK) return st;
  const size_t block = g.rec * g.cmax * nb;  // one rank's block
  uint8_t *sa = reinterpret_cast<uint8_t *>(stats_all);
  if (g.world > 1 || comm != nullptr) {  // (a one-rank comm still goes through NCCL)
    const void *send = stats_local;
    if (g.cam_count < g.cmax) {  // pad each frame to cmax cameras, in this rank's slot
      uint8_t *slot = sa + block * g.rank;
      cudaError_t e = cudaMemcpy2DAsync(slot, g.rec * g.cmax, stats_local, g.rec * g.cam_count,
                                        g.rec * g.cam_count, nb, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) return static_cast<int>(e);
      send = slot;  // in-place all-gather
    }
    st = comm_all_gather(send, sa, block, comm, s);
    if (st != CAMX_OK) return st;
  } else if (reinterpret_cast<void *>(sa) != reinterpret_cast<void *>(stats_local)) {
    cudaError_t e = cudaMemcpyAsync(sa, stats_local, block, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  return launch_seam_solve(stats_all, nb, g.n_cams, g.wrap, cfg, prev_gain, prev_offset, gain,
                           offset, fit_ok, s, false, g.world, g.cmax);
}

// Back half: K3 on this rank's cameras of nb frames.
static int shard_apply(const ShardGeom &g, const uint8_t *images, uint8_t *out, int nb, int blocks,
                       const double *gain, const double *offset, bool pdl, cudaStream_t s) {
  return apply_camera_group(images, out, nb, g.cam_begin, g.cam_count, g.n_cams, g.wrap, g.H,
                            g.W, blocks, gain, offset, pdl, s);
}

extern "C" int camx_correct_batch_sharded(
    const uint8_t *images, uint8_t *out, const uint8_t *prev_frame, int32_t n_batch,
    int32_t n_cams, int32_t cam_begin, int32_t cam_count, int32_t world, int32_t wrap,
    int32_t height, int32_t width, int32_t band_width, int32_t t_diff, const camx_solve_config *cfg,
    const double *prev_gain, const double *prev_offset, camx_band_stat *stats_local,
    camx_band_stat *stats_all, uint32_t *hist, double *gain_out, double *offset_out,
    uint8_t *fit_ok_out, int32_t n_chunks, void *comm, void *stream) {
  if (!images || !out || !stats_local || !stats_all || !gain_out || !offset_out || !fit_ok_out)
    return CAMX_EINVAL;
  if (n_batch < 1 || n_chunks < 1 || n_chunks > kMaxShardChunks) return CAMX_EINVAL;
  ShardGeom g;
  int st = shard_geom(g, n_cams, cam_begin, cam_count, world, wrap, height, width, band_width,
                      t_diff, cfg, prev_gain, prev_offset, comm);
  if (st != CAMX_OK) return st;
  n_chunks = n_chunks > n_batch ? n_batch : n_chunks;
  cudaStream_t main = as_stream(stream);
  SidePipe *sp = nullptr;
  cudaStream_t side = main;
  if (n_chunks > 1) {
    st = side_pipe(sp, comm);
    if (st != CAMX_OK) return st;
    side = sp->side;
    cudaError_t e = cudaEventRecord(sp->ev[0], main);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(side, sp->ev[0], 0);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  // Chunk c: front half on `side`, K3 on `main`; the front half of chunk c+1
  // overlaps K3 of chunk c.  The tick-loop state flows between chunks
  // through gain_out (previous frame's maps) and the raw frames.
  for (int c = 0; c < n_chunks; ++c) {
    const int lo = static_cast<int>(static_cast<int64_t>(n_batch) * c / n_chunks);
    const int hi = static_cast<int>(static_cast<int64_t>(n_batch) * (c + 1) / n_chunks);
    const int nb = hi - lo;
    if (nb <= 0) continue;
    const uint8_t *img = images + lo * g.frame_bytes;
    camx_solve_config cc = *cfg;
    const double *pg = prev_gain, *po = prev_offset;
    if (lo > 0) {  // the previous chunk's last frame seeds this one
      cc.have_prev_maps = 1;
      cc.have_prev_frames = g.removal ? 1 : cc.have_prev_frames;
      pg = gain_out + (lo - 1) * g.map_frame;
      po = offset_out + (lo - 1) * g.map_frame;
    }
    st = shard_front(g, img, lo == 0 ? prev_frame : img - g.frame_bytes, nb, &cc, pg, po,
                     stats_local + static_cast<int64_t>(lo) * cam_count * 2 * cfg->blocks,
                     reinterpret_cast<camx_band_stat *>(reinterpret_cast<uint8_t *>(stats_all) +
                                                        g.rec * g.cmax * world * lo),
                     hist == nullptr ? nullptr
                                     : hist + static_cast<int64_t>(lo) * cam_count * 2 *
                                                  cfg->blocks * 768,
                     gain_out + lo * g.map_frame, offset_out + lo * g.map_frame,
                     fit_ok_out + static_cast<int64_t>(lo) * g.S * cfg->blocks, comm, side);
    if (st != CAMX_OK) return st;
    if (side != main) {
      cudaError_t e = cudaEventRecord(sp->ev[1 + c], side);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(main, sp->ev[1 + c], 0);
      if (e != cudaSuccess) return static_cast<int>(e);
    }
    st = shard_apply(g, img, out + lo * g.frame_bytes, nb, cfg->blocks,
                     gain_out + lo * g.map_frame, offset_out + lo * g.map_frame, side == main,
                     main);
    if (st != CAMX_OK) return st;
  }
  return CAMX_OK;
}

// counts_out[i] = sum over ranks of counts_all[w][i]
__global__ void sum_ranks_kernel(const int64_t *all, int64_t *out, int64_t n, int world) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t v = 0;
    for (int w = 0; w < world; ++w) v += all[w * n + i];
    out[i] = v;
  }
}

extern "C" int camx_correct_batch_sharded_motion(
    const uint8_t *images, uint8_t *out, const uint8_t *prev_frame, int32_t n_batch,
    int32_t n_cams, int32_t cam_begin, int32_t cam_count, int32_t world, int32_t wrap,
    int32_t height, int32_t width, int32_t band_width, int32_t t_diff, const camx_solve_config *cfg,
    const double *prev_gain, const double *prev_offset, camx_band_stat *stats_local,
    camx_band_stat *stats_all, uint32_t *hist, double *gain_out, double *offset_out,
    uint8_t *fit_ok_out, const uint8_t *motion_prev, int32_t win_size, int32_t t_motion,
    int64_t *counts_all, int64_t *counts_out, void *comm, void *stream) {
  if (!images || !out || !stats_local || !stats_all || !gain_out || !offset_out || !fit_ok_out ||
      !counts_all || !counts_out)
    return CAMX_EINVAL;
  if (n_batch < 1 || t_motion < 0 || t_motion > 255) return CAMX_EINVAL;
  if (win_size < 1 || win_size > n_cams * width || win_size > height) return CAMX_EINVAL;
  ShardGeom g;
  int st = shard_geom(g, n_cams, cam_begin, cam_count, world, wrap, height, width, band_width,
                      t_diff, cfg, prev_gain, prev_offset, comm);
  if (st != CAMX_OK) return st;
  int32_t nx = 0, ny = 0;
  st = camx_tiling_size(n_cams * width, height, win_size, &nx, &ny);
  if (st != CAMX_OK) return st;
  const int64_t n = static_cast<int64_t>(n_batch) * nx * ny;
  int64_t *mine = counts_all + g.rank * n;  // this rank's slot (in-place all-gather)
  cudaStream_t s = as_stream(stream);
  cudaError_t e = cudaMemsetAsync(mine, 0, sizeof(int64_t) * n, s);
  if (e != cudaSuccess) return static_cast<int>(e);
  st = shard_front(g, images, prev_frame, n_batch, cfg, prev_gain, prev_offset, stats_local,
                   stats_all, hist, gain_out, offset_out, fit_ok_out, comm, s);
  if (st != CAMX_OK) return st;
  st = apply_camera_group_motion(images, out, n_batch, g.cam_begin, g.cam_count, g.n_cams,
                                 g.wrap, g.H, g.W, cfg->blocks, gain_out, offset_out, motion_prev,
                                 win_size, t_motion, mine, s);
  if (st != CAMX_OK) return st;
  if (g.world > 1 || comm != nullptr) {
    st = comm_all_gather(mine, counts_all, sizeof(int64_t) * n, comm, s);
    if (st != CAMX_OK) return st;
  }
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((n + threads - 1) / threads, 1024);
  sum_ranks_kernel<<<static_cast<unsigned>(std::max<int64_t>(blocks, 1)), threads, 0, s>>>(
      counts_all, counts_out, n, g.world);
  return launch_status();
}

extern "C" int camx_correct_batch_sharded_step(
    const uint8_t *images, const uint8_t *prev_frame, int32_t n_batch, int32_t n_cams,
    int32_t cam_begin, int32_t cam_count, int32_t world, int32_t wrap, int32_t height,
    int32_t width, int32_t band_width, int32_t t_diff, const camx_solve_config *cfg,
    const double *prev_gain, const double *prev_offset, camx_band_stat *stats_local,
    camx_band_stat *stats_all, uint32_t *hist, double *gain_out, double *offset_out,
    uint8_t *fit_ok_out, const uint8_t *apply_images, uint8_t *apply_out, int32_t apply_batch,
    const double *apply_gain, const double *apply_offset, void *comm, void *stream) {
  ShardGeom g;
  int st = shard_geom(g, n_cams, cam_begin, cam_count, world, wrap, height, width, band_width,
                      t_diff, cfg, prev_gain, prev_offset, comm);
  if (st != CAMX_OK) return st;
  const bool front = images != nullptr && n_batch > 0;
  const bool back = apply_images != nullptr && apply_batch > 0;
  if (front && (!stats_local || !stats_all || !gain_out || !offset_out || !fit_ok_out))
    return CAMX_EINVAL;
  if (back && (!apply_out || !apply_gain || !apply_offset)) return CAMX_EINVAL;
  SidePipe *sp = nullptr;
  st = side_pipe(sp, comm);
  if (st != CAMX_OK) return st;
  cudaStream_t main = as_stream(stream);
  cudaError_t e = cudaSuccess;
  if (front) {
    // the side stream sees everything issued on main so far: the frames,
    // and K3 of two steps back (the last reader of the maps buffer K2 fills)
    e = cudaEventRecord(sp->ev[0], main);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sp->side, sp->ev[0], 0);
    if (e != cudaSuccess) return static_cast<int>(e);
    st = shard_front(g, images, prev_frame, n_batch, cfg, prev_gain, prev_offset, stats_local,
                     stats_all, hist, gain_out, offset_out, fit_ok_out, comm, sp->side);
    if (st != CAMX_OK) return st;
  }
  if (back) {  // K3 of the previous batch: its front half is already joined into main
    st = shard_apply(g, apply_images, apply_out, apply_batch, cfg->blocks, apply_gain,
                     apply_offset, false, main);
    if (st != CAMX_OK) return st;
  }
  if (front) {
    // join: work the caller issues on main after this call (refilling the
    // frames, the next step's K3) runs after this front half
    e = cudaEventRecord(sp->step[0], sp->side);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(main, sp->step[0], 0);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  return CAMX_OK;
}


}  // namespace camx
