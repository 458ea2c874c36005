/*
 * camx.h — C ABI of the B200-native seam-exposure + attention-tile path.
 *
 * This is the drop-in boundary for the data-parallel video path of the
 * `camarray` reference (arXiv 1910.03517 remote-tower pipeline).  The
 * reference is pure Python/numpy; each entry point below replaces one
 * reference function (cited file:line, relative to the reference's
 * pkg/src/camarray/) and is what a ctypes/cffi binding of that function
 * binds to.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Pixel/mask/statistics/map buffers are
 *    caller-owned DEVICE pointers (cudaMalloc / torch storage) unless the
 *    parameter name says `host_`.  `stream` is a cudaStream_t passed as
 *    void* (NULL = legacy default stream).  All calls are asynchronous on
 *    `stream` unless stated otherwise.
 *  - Images are (H, W, 3) uint8 row-major RGB, packed back to back
 *    (image i starts at i*H*W*3).  An "array" of B array-frames x N cameras
 *    is B*N images, camera-major inside each array-frame.
 *  - Return value: CAMX_OK (0); negative = invalid argument (the Python
 *    boundary raises ValueError, like the reference); positive = CUDA error
 *    code (RuntimeError).  No exception crosses the ABI.
 *  - Sides: CAMX_SIDE_LEFT = frame sits left of the seam (band/correction at
 *    its RIGHT edge), CAMX_SIDE_RIGHT = frame sits right of the seam
 *    (exposure.py:41-45).
 *  - Seams of an N-camera array: seam s joins camera s (LEFT side) and
 *    camera s+1 (RIGHT side), s = 0..N-2; with `wrap` a 360-degree array
 *    has an extra seam N-1 joining camera N-1 and camera 0.
 *  - Maps: gain/offset are float64 [n_maps][K][3]; an array solve writes
 *    map index ((b*S + s)*2 + side).
 */
#ifndef CAMX_H
#define CAMX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CAMX_ABI_VERSION 1

#define CAMX_OK 0
#define CAMX_EINVAL (-1)      /* bad shape / size / config -> ValueError  */
#define CAMX_EALIGN (-2)      /* pointer alignment not met                 */
#define CAMX_ENOMEM (-3)      /* scratch allocation failed                 */
/* positive, like CUDA errors (RuntimeError): */
#define CAMX_ENCCL_BASE 100000 /* + ncclResult_t of a failed NCCL call       */
#define CAMX_ENONCCL 199999    /* libnccl.so.2 could not be loaded           */

#define CAMX_SIDE_LEFT 0
#define CAMX_SIDE_RIGHT 1

#define CAMX_MODE_STANDARD 0
#define CAMX_MODE_OBJECT_REMOVAL 1
#define CAMX_MODE_SMOOTHING 2

/* Exact integer statistics of one (image, side, block) band segment.
 * Replaces the float moments of BandStats (exposure.py:138-149): mean/std
 * follow exactly from (valid, sum, sumsq).  `sum/sumsq` cover the pixels
 * that survive the exclusion mask; `raw_*` cover all band pixels (the
 * unmasked fit of OBJECT_REMOVAL, exposure.py:327).  112 bytes. */
typedef struct camx_band_stat {
  int64_t area;           /* band pixels in the block  (band_area)   */
  int64_t valid;          /* pixels not excluded       (valid_count) */
  uint64_t sum[3];
  uint64_t sumsq[3];
  uint64_t raw_sum[3];
  uint64_t raw_sumsq[3];
} camx_band_stat;

/* ExposureConfig (exposure.py:54-63) fields the solve needs. */
typedef struct camx_solve_config {
  int32_t mode;                 /* CAMX_MODE_*                               */
  int32_t blocks;               /* K                                         */
  int64_t min_band_pixels;      /* strict: valid > min_band_pixels           */
  double sigma_min;
  double alpha;
  double min_valid_fraction;
  int32_t have_prev_maps;       /* prev_gain/prev_offset valid for frame 0   */
  int32_t have_prev_frames;     /* OBJECT_REMOVAL: stats carry masked sums   */
} camx_solve_config;

/* ---- library ---------------------------------------------------------- */
int camx_abi_version(void);
const char *camx_status_string(int status);
/* Number of SMs of the current device (grid sizing); host-synchronous. */
int camx_device_sm_count(int32_t *sm_count_out);

/* ---- stage 1: seam band statistics (K1) ---------------------------------
 * Replaces band_stats (exposure.py:152-185) for BOTH sides of every image,
 * plus the in-band part of mask_diff (core.py:191-196) when `prev_images`
 * is given (OBJECT_REMOVAL, exposure.py:313-316): a band pixel is excluded
 * iff max_c |cur - prev| > t_diff.  `excl_masks` (optional, (n,H,W) bytes,
 * nonzero = excluded) is the explicit exclusion_mask argument; at most one
 * of prev_images / excl_masks may be non-NULL.
 * stats_out: [n_images][2 sides][blocks] records.
 * hist_out (optional): uint32 [n_images][2][blocks][3][256] histograms of
 * the non-excluded band pixels (builder-defined product; moments derive
 * from it exactly).  Errors: band_width > W/2, blocks < 1, blocks > H. */
int camx_band_stats(const uint8_t *images, const uint8_t *prev_images,
                    const uint8_t *excl_masks, int64_t n_images,
                    int32_t height, int32_t width, int32_t band_width,
                    int32_t blocks, int32_t t_diff,
                    camx_band_stat *stats_out, uint32_t *hist_out,
                    void *stream);

/* Float moments of records: mean/std (K,3) float64 per record as in
 * BandStats (population std), valid/area int64.  use_raw selects raw_*.
 * mean_out/std_out: [n_records][3]; valid_out/area_out: [n_records]. */
int camx_band_moments(const camx_band_stat *stats, int64_t n_records,
                      int32_t use_raw, double *mean_out, double *std_out,
                      int64_t *valid_out, int64_t *area_out, void *stream);

/* ---- stage 2: seam gain solve (K2) --------------------------------------
 * Replaces update_exposure (exposure.py:245-344) = fit_affine :188-229 +
 * resolve :275-293 + smooth_exposure :232-242 for every seam of a batch of
 * n_batch consecutive array-frames.  Frame b uses frame b-1's output maps
 * as prev_maps (frame 0 uses prev_gain/prev_offset when
 * cfg->have_prev_maps), i.e. the batch is a tick loop.
 * stats: [n_batch][n_cams][2][blocks] from camx_band_stats.
 * prev_gain/prev_offset: [S][2][K][3]; gain_out/offset_out:
 * [n_batch][S][2][K][3]; fit_ok_out (optional): [n_batch][S][K] bytes
 * (the raw fit's fit_ok).  S = n_cams-1 (+1 with wrap). */
int camx_seam_solve(const camx_band_stat *stats, int32_t n_batch,
                    int32_t n_cams, int32_t wrap,
                    const camx_solve_config *cfg, const double *prev_gain,
                    const double *prev_offset, double *gain_out,
                    double *offset_out, uint8_t *fit_ok_out, void *stream);

/* fit_affine (exposure.py:188-229) on float moments (BandStats fields).
 * l_mean/l_std/r_mean/r_std: [K][3]; l_valid/r_valid: [K].
 * gain_out/offset_out: [2 sides][K][3]; fit_ok_out: [K] bytes. */
int camx_fit_affine(const double *l_mean, const double *l_std,
                    const int64_t *l_valid, const double *r_mean,
                    const double *r_std, const int64_t *r_valid,
                    int32_t blocks, double sigma_min,
                    int64_t min_band_pixels, double *gain_out,
                    double *offset_out, uint8_t *fit_ok_out, void *stream);

/* smooth_exposure (exposure.py:232-242): out = (1-alpha)*prev + alpha*new,
 * coefficient-wise over n doubles (gain and offset each). */
int camx_smooth_maps(const double *prev_gain, const double *prev_offset,
                     const double *new_gain, const double *new_offset,
                     int64_t n, double alpha, double *gain_out,
                     double *offset_out, void *stream);

/* ---- stage 3: per-pixel correction apply (K3) ---------------------------
 * Replaces _lambda_profile + _apply_arrays + apply_exposure
 * (exposure.py:347-414): out = clip(rint(f32(p)*M + A), 0, 255) on the
 * near half of each seam side, M = f32(1 + lam*(g-1)), A = f32(lam*b)
 * evaluated in float64 per (block, column, channel) without materialising
 * the (H, W/2, 3) tables; the far half is copied.  Bit-exact with numpy.
 * Array form: images [n_batch][cam_count][H][W][3] are cameras
 * cam_begin..cam_begin+cam_count-1 of an n_cams_total array; camera c uses
 * the LEFT map of seam c and the RIGHT map of seam c-1 (wrap: seam N-1 for
 * camera 0 / N-1).  maps: [n_batch][S][2][K][3].  `out` may equal
 * `images` (apply_exposure_inplace, exposure.py:404-414). */
int camx_apply_array(const uint8_t *images, uint8_t *out, int32_t n_batch,
                     int32_t cam_begin, int32_t cam_count,
                     int32_t n_cams_total, int32_t wrap, int32_t height,
                     int32_t width, int32_t blocks, const double *gain,
                     const double *offset, void *stream);

/* The whole hot path for a batch of n_batch array-frames x n_cams cameras
 * on one GPU: K1 band statistics, K2 seam solve and K3 apply, K2 and K3 as
 * programmatic dependent launches (K3's TMA pixel prefetch overlaps the
 * solve).  `counters` is unused (reserved; may be NULL).  = update_exposure for every seam + apply of
 * both seam sides of every camera, tick loop over the batch.  prev_frame
 * (n_cams images, OBJECT_REMOVAL only, may be NULL) is the array-frame
 * before frame 0.  stats [n_batch][n_cams][2][K] records; hist (optional)
 * [n_batch][n_cams][2][K][3][256]; gain/offset [n_batch][S][2][K][3];
 * fit_ok [n_batch][S][K]. */
int camx_correct_batch(const uint8_t *images, uint8_t *out,
                       const uint8_t *prev_frame, int32_t n_batch,
                       int32_t n_cams, int32_t wrap, int32_t height,
                       int32_t width, int32_t band_width, int32_t t_diff,
                       const camx_solve_config *cfg, const double *prev_gain,
                       const double *prev_offset, camx_band_stat *stats,
                       uint32_t *hist, double *gain_out, double *offset_out,
                       uint8_t *fit_ok_out, int32_t *counters, void *stream);

/* camx_correct_batch with the motion counts of the attention tick fused
 * into K3 (replaces difference_plan's per-window count_nonzero of
 * mask_diff, attention.py:89-103 / core.py:191-196, for every array-frame):
 * K3 also reads the previous raw array-frame (frame b - 1 of the batch;
 * `motion_prev` (n_cams images, may be NULL: no counts for frame 0) before
 * frame 0) and counts, per window of the overlap-0 tiling of the
 * (n_cams * width) x height mosaic with side win_size (row-major, nx * ny
 * windows: camx_tiling_size), the pixels with max_c |cur - prev| > t_motion
 * (0..255).  counts_out [n_batch][ny][nx] int64 (zeroed here).  Needs
 * width * 3 % 16 == 0 (else CAMX_EINVAL: use camx_correct_batch +
 * camx_window_counts). */
int camx_correct_batch_motion(
    const uint8_t *images, uint8_t *out, const uint8_t *prev_frame,
    int32_t n_batch, int32_t n_cams, int32_t wrap, int32_t height,
    int32_t width, int32_t band_width, int32_t t_diff,
    const camx_solve_config *cfg, const double *prev_gain,
    const double *prev_offset, camx_band_stat *stats, uint32_t *hist,
    double *gain_out, double *offset_out, uint8_t *fit_ok_out,
    const uint8_t *motion_prev, int32_t win_size, int32_t t_motion,
    int64_t *counts_out, void *stream);
/* 1 when camx_correct_batch_motion (cam_count = n_cams) or
 * camx_correct_batch_sharded_motion (this rank's cam_count cameras) can run
 * this geometry (16-byte aligned rows; every K3 CTA meets <= 3 x 3 windows,
 * e.g. size >= ~700 px at 2048-px frames), else 0 (count with
 * camx_window_counts instead). */
int camx_motion_supported(int32_t n_batch, int32_t n_cams, int32_t cam_count,
                          int32_t height, int32_t width, int32_t blocks,
                          int32_t size);
/* Window grid of the overlap-0 tiling (attention.py:53-86): nx, ny. */
int camx_tiling_size(int32_t mosaic_w, int32_t mosaic_h, int32_t size,
                     int32_t *nx, int32_t *ny);

/* ---- camera-sharded arrays (multi-GPU) ------------------------
 * One process per GPU; rank g owns the contiguous camera group
 * [begin(g), begin(g) + count(g)) of dist.camera_partition (counts differ by
 * at most one; cmax = ceil(n_cams / world)).  The seam statistics are
 * exchanged with one NCCL all-gather; NCCL is resolved at run time from the
 * process's libnccl.so.2 (PyTorch's).  The 128-byte unique id is created on
 * one rank (camx_comm_unique_id) and broadcast by the caller. */
int camx_comm_available(void);
int camx_comm_unique_id(uint8_t *id_out /* 128 bytes */);
int camx_comm_init(void **comm_out, const uint8_t *id, int32_t n_ranks, int32_t rank);
int camx_comm_destroy(void *comm);
/* Test-only loopback group: `world` communicator handles (comms_out[rank])
 * for ranks that live in ONE process on one GPU, each driven from its own
 * host thread and stream (NCCL refuses two ranks per device).  The
 * all-gather stages the bytes through a shared device buffer with event
 * waits and host barriers, so the world > 1 code of the sharded entry
 * points runs exactly as under NCCL.  Release each handle with
 * camx_comm_destroy. */
int camx_comm_loopback_create(int32_t world, void **comms_out);

/* K2 on the all-gathered records: stats_all = [world][n_batch][cmax][2][K]
 * (rank-major, each rank's block padded to cmax cameras).  Otherwise as
 * camx_seam_solve (update_exposure for every seam, exposure.py:245-344). */
int camx_seam_solve_sharded(const camx_band_stat *stats_all, int32_t n_batch,
                            int32_t n_cams, int32_t world, int32_t wrap,
                            const camx_solve_config *cfg,
                            const double *prev_gain, const double *prev_offset,
                            double *gain_out, double *offset_out,
                            uint8_t *fit_ok_out, void *stream);

/* camx_correct_batch for this rank's cameras: K1 on images [n_batch]
 * [cam_count][H][W][3] -> stats_local [n_batch][cmax][2][K] (dense over
 * cam_count), ncclAllGather into stats_all [world][n_batch][cmax][2][K],
 * K2 for every seam of the whole array (redundant on every rank, tiny),
 * K3 on this rank's cameras.  Corrected pixels are byte-identical to the
 * one-GPU camx_correct_batch.  comm = camx_comm_init handle (NULL only when
 * world == 1); prev_frame = this rank's cameras of the previous frame
 * (OBJECT_REMOVAL); hist (optional) [n_batch][cam_count][2][K][3][256];
 * gain/offset/fit_ok for all seams as camx_correct_batch.  n_chunks (1..8)
 * > 1 splits the batch: K1 + all-gather + K2 of chunk c+1 run on a
 * library-owned side stream under K3 of chunk c; stats_all then holds the
 * chunks' [world][n_c][cmax][2][K] blocks one after another. */
int camx_correct_batch_sharded(const uint8_t *images, uint8_t *out,
                               const uint8_t *prev_frame, int32_t n_batch,
                               int32_t n_cams, int32_t cam_begin,
                               int32_t cam_count, int32_t world, int32_t wrap,
                               int32_t height, int32_t width,
                               int32_t band_width, int32_t t_diff,
                               const camx_solve_config *cfg,
                               const double *prev_gain,
                               const double *prev_offset,
                               camx_band_stat *stats_local,
                               camx_band_stat *stats_all, uint32_t *hist,
                               double *gain_out, double *offset_out,
                               uint8_t *fit_ok_out, int32_t n_chunks,
                               void *comm, void *stream);

/* Software-pipelined step of the sharded path: the front half (K1 ->
 * all-gather -> K2) of batch k runs on a library-owned side stream while K3
 * of batch k-1 (apply_images / apply_out / apply_gain / apply_offset: the
 * previous step's batch and maps) runs on `stream`; `stream` then joins the
 * side stream, so work issued on it afterwards (refilling `images`, the next
 * step) is ordered after both.  images == NULL: no front half (flush);
 * apply_images == NULL: no back half (first step).  The caller double-buffers
 * the maps / records between consecutive steps.  One pipelined sequence per
 * (device, communicator) at a time. */
/* camx_correct_batch_sharded with the attention tick's motion counts fused
 * into this rank's K3 (as camx_correct_batch_motion; n_chunks = 1):
 * motion_prev = this rank's cameras of the array-frame before frame 0 (may
 * be NULL).  Each rank counts the pixels of its cameras into its slot of
 * counts_all [world][n_batch][ny][nx] int64, the slots are all-gathered
 * through `comm` and summed: counts_out [n_batch][ny][nx] holds the whole
 * array's counts on every rank. */
int camx_correct_batch_sharded_motion(
    const uint8_t *images, uint8_t *out, const uint8_t *prev_frame,
    int32_t n_batch, int32_t n_cams, int32_t cam_begin, int32_t cam_count,
    int32_t world, int32_t wrap, int32_t height, int32_t width,
    int32_t band_width, int32_t t_diff, const camx_solve_config *cfg,
    const double *prev_gain, const double *prev_offset,
    camx_band_stat *stats_local, camx_band_stat *stats_all, uint32_t *hist,
    double *gain_out, double *offset_out, uint8_t *fit_ok_out,
    const uint8_t *motion_prev, int32_t win_size, int32_t t_motion,
    int64_t *counts_all, int64_t *counts_out, void *comm, void *stream);

int camx_correct_batch_sharded_step(
    const uint8_t *images, const uint8_t *prev_frame, int32_t n_batch,
    int32_t n_cams, int32_t cam_begin, int32_t cam_count, int32_t world,
    int32_t wrap, int32_t height, int32_t width, int32_t band_width,
    int32_t t_diff, const camx_solve_config *cfg, const double *prev_gain,
    const double *prev_offset, camx_band_stat *stats_local,
    camx_band_stat *stats_all, uint32_t *hist, double *gain_out,
    double *offset_out, uint8_t *fit_ok_out, const uint8_t *apply_images,
    uint8_t *apply_out, int32_t apply_batch, const double *apply_gain,
    const double *apply_offset, void *comm, void *stream);

/* One map on n_images images (apply_exposure / apply_exposure_inplace):
 * gain/offset [K][3], side CAMX_SIDE_*. */
int camx_apply_map(const uint8_t *images, uint8_t *out, int64_t n_images,
                   int32_t height, int32_t width, int32_t side,
                   int32_t blocks, const double *gain, const double *offset,
                   void *stream);

/* ---- stage 4a: motion mask + window counts (K4) -------------------------
 * mask_diff (core.py:191-196): mask[i] = max_c |a - b| > t_diff over
 * n_pixels RGB pixels; mask_out bytes 0/1. */
int camx_mask_diff(const uint8_t *a, const uint8_t *b, int64_t n_pixels,
                   int32_t t_diff, uint8_t *mask_out, void *stream);

/* mask_diff over n_pixels pixels of `channels` interleaved uint8 channels
 * (the reference takes the max over axis 2 of any (H, W, C) array). */
int camx_mask_diff_channels(const uint8_t *a, const uint8_t *b, int64_t n_pixels,
                            int32_t channels, int32_t t_diff, uint8_t *mask_out,
                            void *stream);

/* Per-window on-pixel counts of difference_plan (attention.py:96-100) on
 * the mosaic of n_cams images (mosaic col x -> camera x / width), without
 * materialising the mosaic.  Either `mask` ((n_cams,H,W) bytes, nonzero =
 * on) or (`cur`, `prev`, t_diff) frames (fused mask_diff).  Windows are
 * [n_windows][2] int32 (x, y) origins of size x size squares, device
 * memory.  counts_out: int64 [n_windows]. */
int camx_window_counts(const uint8_t *mask, const uint8_t *cur,
                       const uint8_t *prev, int32_t t_diff, int32_t n_cams,
                       int32_t height, int32_t width, const int32_t *windows,
                       int32_t n_windows, int32_t size, int64_t *counts_out,
                       void *stream);

/* ---- stage 4b: attention tile crop / resize (K5) ------------------------
 * Crop of ExternalDetector.detect (detect.py:297-300) of window (x, y, S)
 * from the (virtual) mosaic of n_cams images, then bilinear resize to
 * out_size x out_size (half-pixel centres; source coordinate in float32,
 * 8-bit fixed-point weights round(256 f), exact integer blend
 * (h0*(256-wy) + h1*wy + 2^15) >> 16; the resize is builder-defined - the
 * reference only crops).  out_size == S is
 * the exact crop.  images: [n_batch][n_cams][H][W][3]; windows: device
 * int32 [n_tiles][3] = (batch index, x, y); tiles_out: uint8
 * [n_tiles][out_size][out_size][3]. */
int camx_tiles(const uint8_t *images, int32_t n_cams, int32_t height,
               int32_t width, const int32_t *windows, int32_t n_tiles,
               int32_t size, int32_t out_size, uint8_t *tiles_out,
               void *stream);

/* Tiles over a camera shard (multi-GPU).  images: this rank's
 * cameras [n_batch][n_cams][H][W][3], holding mosaic columns
 * [col_begin, col_begin + n_cams*W); windows: (batch, x, y) in GLOBAL mosaic
 * coordinates.  Writes exactly the output columns whose first column tap
 * lies on this shard (every output pixel has one owner); the second tap may
 * be the next shard's first column, passed as halo [n_batch][H][3] (NULL
 * only for the last shard).  Other pixels of tiles_out are not written:
 * zero-fill and sum the ranks' partials (dist.sharded_tiles).  Replaces the
 * crop of ExternalDetector.detect (detect.py:297-300) on a sharded mosaic. */
int camx_tiles_shard(const uint8_t *images, int32_t n_cams, int32_t height,
                     int32_t width, int32_t col_begin, const uint8_t *halo,
                     const int32_t *windows, int32_t n_tiles, int32_t size,
                     int32_t out_size, uint8_t *tiles_out, void *stream);

/* Stage 3 + 4b (config 5): apply the array correction, then cut the tiles
 * from the corrected frames with camx_tiles' TMA-staged resample (the tile
 * kernel reads each output row's two tap rows of `out`).  windows: device
 * int32 [n_tiles][3] (batch index, x, y); frame_off (device int32
 * [n_batch+1], first tile of each array-frame) and max_tiles_per_frame
 * describe their grouping by array-frame (ABI v1 arguments, may be NULL /
 * 0).  Maps as camx_apply_array (cam_begin = 0, cam_count = n_cams). */
int camx_correct_and_tile(const uint8_t *images, uint8_t *out,
                          int32_t n_batch, int32_t n_cams, int32_t wrap,
                          int32_t height, int32_t width, int32_t blocks,
                          const double *gain, const double *offset,
                          const int32_t *windows, const int32_t *frame_off,
                          int32_t n_tiles, int32_t max_tiles_per_frame,
                          int32_t size, int32_t out_size, uint8_t *tiles_out,
                          void *stream);

/* camx_correct_batch + tiles: K1, K2 (PDL), K3 (PDL), tiles (camx_tiles). */
int camx_correct_batch_tiles(
    const uint8_t *images, uint8_t *out, const uint8_t *prev_frame,
    int32_t n_batch, int32_t n_cams, int32_t wrap, int32_t height,
    int32_t width, int32_t band_width, int32_t t_diff,
    const camx_solve_config *cfg, const double *prev_gain,
    const double *prev_offset, camx_band_stat *stats, uint32_t *hist,
    double *gain_out, double *offset_out, uint8_t *fit_ok_out,
    const int32_t *windows, const int32_t *frame_off, int32_t n_tiles,
    int32_t max_tiles_per_frame, int32_t size, int32_t out_size,
    uint8_t *tiles_out, void *stream);

/* ---- next: motion-blob components -------------------------
 * BlobDetector.detect (detect.py:192-249): 8-connected components of the
 * motion mask inside the window (x0, y0, size) of the virtual mosaic of
 * n_cams (H, W) masks (nonzero = on), as scipy.ndimage.label with a 3x3
 * structure.  comp_out: int32 [max_comp][6] = (raster index of the
 * component's first pixel, xmin, ymin, xmax, ymax (window coordinates,
 * inclusive), on-pixels of ANY component inside that box (detect.py:241)),
 * in scipy label order; *n_comp_out = number of components (may exceed
 * max_comp).  scratch: 16-byte aligned int32 [6 * size * size + 2 * size + 1 +
 * (size * size + 1023) / 1024]
 * device memory. */
int camx_blob_components(const uint8_t *mask, int32_t n_cams, int32_t height,
                         int32_t width, int32_t x0, int32_t y0, int32_t size,
                         int32_t *scratch, int32_t *comp_out, int32_t max_comp,
                         int32_t *n_comp_out, void *stream);

/* ---- next: seam quality metric ------------------------------
 * seam_cost (exposure.py:417-445) of n_pairs (left, right) image pairs of
 * equal height: box-downsample by `factor`, per-row trend discrepancy,
 * mean over rows.  left/right: [n_pairs][H][W][3] (widths may differ:
 * left_width / right_width).  cost_out: float64 [n_pairs]. */
int camx_seam_cost(const uint8_t *left, const uint8_t *right,
                   int64_t n_pairs, int32_t height, int32_t left_width,
                   int32_t right_width, int32_t factor, double *cost_out,
                   void *stream);

#ifdef __cplusplus
}
#endif

#endif /* CAMX_H */
