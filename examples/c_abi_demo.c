/* Plain-C use of the camx C ABI (include/camx.h): the hot path driven with
 * raw device pointers, no Python and no torch.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/c_abi_demo.c \
 *       -L paper_1910_03517_b200 -lcamx -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,paper_1910_03517_b200 -o c_abi_demo && ./c_abi_demo
 *
 * A 3-camera array of 2 frames: camera 1 sees the same scene as camera 0
 * with an exposure/white-balance distortion (gain, offset per channel);
 * camera 2 is an exact copy of camera 0.  After camx_correct_batch:
 *   - the seam 0|1 band means move towards each other (the correction),
 *   - camera 2 only gets the seam 1|2 right-half correction, and the
 *     reference semantics hold: gains are finite and positive,
 *   - invalid arguments come back as CAMX_EINVAL (negative), not a crash.
 * Exit status 0 on success. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "camx.h"

#define CHECK_CUDA(x)                                                         \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, \
              __LINE__);                                                      \
      return 2;                                                               \
    }                                                                         \
  } while (0)
#define CHECK_CAMX(x)                                                         \
  do {                                                                        \
    int s_ = (x);                                                             \
    if (s_ != CAMX_OK) {                                                      \
      fprintf(stderr, "camx %d (%s) at %s:%d\n", s_, camx_status_string(s_), \
              __FILE__, __LINE__);                                            \
      return 3;                                                               \
    }                                                                         \
  } while (0)

enum { NB = 2, NC = 3, H = 96, W = 128, BW = 16, K = 4 };

static double band_mean(const uint8_t *img, int left_band, int ch) {
  /* mean of one channel over a seam band of one image (H x W x 3) */
  double s = 0;
  int c0 = left_band ? W - BW : 0;
  for (int r = 0; r < H; ++r)
    for (int c = c0; c < c0 + BW; ++c) s += img[((size_t)r * W + c) * 3 + ch];
  return s / (H * BW);
}

int main(void) {
  const size_t img = (size_t)H * W * 3, n = img * NC * NB;
  uint8_t *h_in = (uint8_t *)malloc(n), *h_out = (uint8_t *)malloc(n);
  const double g1[3] = {1.4, 0.8, 1.1}, o1[3] = {-12.0, 9.0, 3.0};
  for (int b = 0; b < NB; ++b)
    for (int r = 0; r < H; ++r)
      for (int c = 0; c < W; ++c)
        for (int ch = 0; ch < 3; ++ch) {
          /* a smooth scene continuing across the seams, plus texture */
          int x = c;
          double v = 60 + 0.5 * x + 0.4 * r + 20 * sin(0.3 * r + 0.2 * x + ch + b);
          uint8_t *f = h_in + (size_t)b * NC * img;
          size_t o = ((size_t)r * W + c) * 3 + ch;
          f[o] = (uint8_t)fmin(255, fmax(0, v));
          double d = g1[ch] * v + o1[ch];
          f[img + o] = (uint8_t)fmin(255, fmax(0, d));
          f[2 * img + o] = f[o];
        }
  uint8_t *d_in, *d_out;
  camx_band_stat *d_stats;
  double *d_gain, *d_off;
  uint8_t *d_ok;
  const int S = NC - 1;
  CHECK_CUDA(cudaMalloc((void **)&d_in, n));
  CHECK_CUDA(cudaMalloc((void **)&d_out, n));
  CHECK_CUDA(cudaMalloc((void **)&d_stats, sizeof(camx_band_stat) * NB * NC * 2 * K));
  CHECK_CUDA(cudaMalloc((void **)&d_gain, sizeof(double) * NB * S * 2 * K * 3));
  CHECK_CUDA(cudaMalloc((void **)&d_off, sizeof(double) * NB * S * 2 * K * 3));
  CHECK_CUDA(cudaMalloc((void **)&d_ok, NB * S * K));
  CHECK_CUDA(cudaMemcpy(d_in, h_in, n, cudaMemcpyHostToDevice));

  camx_solve_config cfg;
  memset(&cfg, 0, sizeof cfg);
  cfg.mode = CAMX_MODE_STANDARD;
  cfg.blocks = K;
  cfg.min_band_pixels = 64;
  cfg.sigma_min = 1e-3;
  cfg.alpha = 0.05;
  cfg.min_valid_fraction = 0.25;
  printf("camx ABI %d\n", camx_abi_version());
  CHECK_CAMX(camx_correct_batch(d_in, d_out, NULL, NB, NC, 0, H, W, BW, 20, &cfg, NULL, NULL,
                                d_stats, NULL, d_gain, d_off, d_ok, NULL, NULL));
  CHECK_CUDA(cudaDeviceSynchronize());
  CHECK_CUDA(cudaMemcpy(h_out, d_out, n, cudaMemcpyDeviceToHost));
  double gain[NB * S * 2 * K * 3];
  CHECK_CUDA(cudaMemcpy(gain, d_gain, sizeof gain, cudaMemcpyDeviceToHost));

  int fail = 0;
  for (size_t i = 0; i < sizeof gain / sizeof gain[0]; ++i)
    if (!(gain[i] > 0) || !isfinite(gain[i])) fail = 1;
  for (int ch = 0; ch < 3; ++ch) {
    double before = fabs(band_mean(h_in, 1, ch) - band_mean(h_in + img, 0, ch));
    double after = fabs(band_mean(h_out, 1, ch) - band_mean(h_out + img, 0, ch));
    printf("seam 0|1 channel %d: |band mean difference| %.2f -> %.2f\n", ch, before, after);
    if (!(after < 0.5 * before)) fail = 1;
  }
  /* invalid argument -> negative status, nothing launched */
  int st = camx_correct_batch(d_in, d_out, NULL, NB, 1, 0, H, W, BW, 20, &cfg, NULL, NULL,
                              d_stats, NULL, d_gain, d_off, d_ok, NULL, NULL);
  printf("one-camera array -> status %d (%s)\n", st, camx_status_string(st));
  if (st >= 0) fail = 1;
  cudaFree(d_in);
  cudaFree(d_out);
  cudaFree(d_stats);
  cudaFree(d_gain);
  cudaFree(d_off);
  cudaFree(d_ok);
  free(h_in);
  free(h_out);
  printf(fail ? "FAIL\n" : "OK\n");
  return fail;
}
