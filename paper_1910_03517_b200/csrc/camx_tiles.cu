// K5: attention-tile crop / resize (stage 4b) and the seam quality metric.
//
// Crop: ExternalDetector.detect (camarray detect.py:297-300) slices
// mosaic.pixels[y:y+S, x:x+S] of the concatenated mosaic (core.py:102-119);
// here the mosaic is virtual (column x -> camera x / W).  Resize to the
// detector input size is builder-defined (the reference has none):
// bilinear, half-pixel centres, float32 weights/blend in a fixed operation
// order, round-half-even (oracle/camarray_oracle.py: resize_bilinear).
//
// seam_cost: exposure.py:417-445 (box downsample, Eq. 1 of the paper).
#include "camx_common.cuh"

namespace camx {

struct TileParams {
  const uint8_t *img;
  int32_t n_cams, H, W, size, out;
  const int32_t *wins;  // [n][3] (batch, x, y)
  uint8_t *tiles;
  float scale;
};

__device__ __forceinline__ void src_coord(int i, float scale, int S, int &i0, int &i1, float &f) {
  float s = __fsub_rn(__fmul_rn(__fadd_rn(static_cast<float>(i), 0.5f), scale), 0.5f);
  s = fminf(fmaxf(s, 0.0f), static_cast<float>(S - 1));
  i0 = static_cast<int>(floorf(s));
  i1 = min(i0 + 1, S - 1);
  f = __fsub_rn(s, static_cast<float>(i0));
}

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
    int y_0, y_1, x_0, x_1;
    float fy, fx;
    src_coord(oy, p.scale, p.size, y_0, y_1, fy);
    src_coord(ox, p.scale, p.size, x_0, x_1, fx);
    const uint8_t *a = mosaic_px(p, b, y0 + y_0, x0 + x_0);
    const uint8_t *bb = mosaic_px(p, b, y0 + y_0, x0 + x_1);
    const uint8_t *c = mosaic_px(p, b, y0 + y_1, x0 + x_0);
    const uint8_t *d = mosaic_px(p, b, y0 + y_1, x0 + x_1);
    const float gx = __fsub_rn(1.0f, fx), gy = __fsub_rn(1.0f, fy);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      const float top = __fadd_rn(__fmul_rn(static_cast<float>(a[ch]), gx),
                                  __fmul_rn(static_cast<float>(bb[ch]), fx));
      const float bot = __fadd_rn(__fmul_rn(static_cast<float>(c[ch]), gx),
                                  __fmul_rn(static_cast<float>(d[ch]), fx));
      float v = __fadd_rn(__fmul_rn(top, gy), __fmul_rn(bot, fy));
      v = fminf(fmaxf(rintf(v), 0.0f), 255.0f);
      dst[3 * q + ch] = static_cast<uint8_t>(v);
    }
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

__global__ void seam_cost_kernel(const uint8_t *left, const uint8_t *right, int H, int WL, int WR,
                                 int f, double *cost) {
  const int64_t pair = blockIdx.x;
  const uint8_t *L = left + pair * static_cast<int64_t>(H) * WL * 3;
  const uint8_t *R = right + pair * static_cast<int64_t>(H) * WR * 3;
  const int h2 = H / f, wl2 = WL / f;
  double acc = 0.0;
  for (int r = threadIdx.x; r < h2; r += blockDim.x) {
    double lm1[3], l0[3], r0[3], r1[3];
    box_mean(L, WL, f, r, wl2 - 2, lm1);
    box_mean(L, WL, f, r, wl2 - 1, l0);
    box_mean(R, WR, f, r, 0, r0);
    box_mean(R, WR, f, r, 1, r1);
    double dp = 0.0, dm = 0.0;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      const double a = __dsub_rn(__dsub_rn(r1[ch], r0[ch]), __dsub_rn(r0[ch], l0[ch]));
      const double b = __dsub_rn(__dsub_rn(lm1[ch], l0[ch]), __dsub_rn(l0[ch], r0[ch]));
      dp = __dadd_rn(dp, __dmul_rn(a, a));
      dm = __dadd_rn(dm, __dmul_rn(b, b));
    }
    acc += __ddiv_rn(__dadd_rn(sqrt(dp), sqrt(dm)), 2.0);
  }
  __shared__ double part[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
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
  const int64_t npx = static_cast<int64_t>(out_size) * out_size;
  int64_t bx = (npx + 255) / 256;
  if (bx > 64) bx = 64;
  dim3 grid(static_cast<unsigned>(bx), n_tiles);
  tiles_kernel<<<grid, 256, 0, s>>>(p);
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
  return launch_tiles(images, n_cams, height, width, windows, n_tiles, size, out_size, tiles_out,
                      as_stream(stream));
}

extern "C" int camx_correct_and_tile(const uint8_t *images, uint8_t *out, int32_t n_batch,
                                     int32_t n_cams, int32_t wrap, int32_t height, int32_t width,
                                     int32_t blocks, const double *gain, const double *offset,
                                     const int32_t *windows, int32_t n_tiles, int32_t size,
                                     int32_t out_size, uint8_t *tiles_out, void *stream) {
  if (!images || !out || !tiles_args_ok(n_cams, height, width, windows, n_tiles, size, out_size,
                                        tiles_out))
    return CAMX_EINVAL;
  int st = camx_apply_array(images, out, n_batch, 0, n_cams, n_cams, wrap, height, width, blocks,
                            gain, offset, stream);
  if (st != CAMX_OK || n_tiles == 0) return st;
  return launch_tiles(out, n_cams, height, width, windows, n_tiles, size, out_size, tiles_out,
                      as_stream(stream));
}

extern "C" int camx_seam_cost(const uint8_t *left, const uint8_t *right, int64_t n_pairs,
                              int32_t height, int32_t left_width, int32_t right_width,
                              int32_t factor, double *cost_out, void *stream) {
  if (n_pairs < 0 || !left || !right || !cost_out || factor < 1) return CAMX_EINVAL;
  if (height / factor < 1 || left_width / factor < 2 || right_width / factor < 2) return CAMX_EINVAL;
  if (n_pairs == 0) return CAMX_OK;
  seam_cost_kernel<<<static_cast<unsigned>(n_pairs), 128, 0, as_stream(stream)>>>(
      left, right, height, left_width, right_width, factor, cost_out);
  return launch_status();
}
