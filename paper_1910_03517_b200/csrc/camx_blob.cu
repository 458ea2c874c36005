// Motion-blob components: BlobDetector.detect
// (camarray detect.py:192-249) labels the 8-connected components of the
// frame-difference mask inside a detector window (scipy.ndimage.label with a
// 3x3 structure, :238) and reports each component's bounding box and the
// number of mask-on pixels inside that box (`np.count_nonzero(labels[sl])`,
// :241 - it counts every component's pixels in the box).
//
// GPU: union-find connected components over the window of the virtual mosaic
// (column x -> camera x / W):
//   1. init     parent[i] = i for on-pixels, -1 otherwise
//   2. union    each on-pixel links to its on-neighbours W, NW, N, NE with an
//               atomicMin-based union (roots = smallest index of the set)
//   3. flatten  parent[i] = root(i); the root is the component's raster-first
//               pixel, so sorting roots reproduces scipy's label order
//   4. boxes    per-root atomic min/max of (x, y); roots compacted in
//               raster order (per-block counts, one scan, ballot ranks)
//   5. counts   summed-area table of the window mask (row scan + column
//               scan), 4 lookups per box
#include <algorithm>

#include "camx_common.cuh"

namespace camx {

struct BlobParams {
  const uint8_t *mask;  // (n_cams, H, W) bytes, nonzero = on
  int32_t n_cams, H, W, x0, y0, size;
  int32_t *parent;      // [size*size]
  int32_t *box;         // [size*size][4] per-root xmin, ymin, xmax, ymax
  int32_t *sat;         // [(size+1)*(size+1)] summed-area table
};

__device__ __forceinline__ bool mask_on(const BlobParams &p, int wx, int wy) {
  const int x = p.x0 + wx, y = p.y0 + wy;
  const int cam = x / p.W;
  return p.mask[(static_cast<int64_t>(cam) * p.H + y) * p.W + (x - cam * p.W)] != 0;
}

__device__ __forceinline__ int find_root(int32_t *parent, int i) {
  int r = parent[i];
  while (r != parent[r]) r = parent[r];
  return r;
}

// Lock-free union: hook the larger root under the smaller one.
__device__ __forceinline__ void unite(int32_t *parent, int a, int b) {
  while (true) {
    a = find_root(parent, a);
    b = find_root(parent, b);
    if (a == b) return;
    if (a > b) {
      const int t = a;
      a = b;
      b = t;
    }
    const int old = atomicMin(&parent[b], a);
    if (old == b) return;  // b was a root and now points at a
    b = old;               // b was re-hooked concurrently: retry from there
  }
}

__global__ void blob_init_kernel(const BlobParams p) {
  const int n = p.size * p.size;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int wx = i % p.size, wy = i / p.size;
    p.parent[i] = mask_on(p, wx, wy) ? i : -1;
    int4 *bx = reinterpret_cast<int4 *>(p.box) + i;
    *bx = make_int4(0x7FFFFFFF, 0x7FFFFFFF, -1, -1);
  }
}

__global__ void blob_union_kernel(const BlobParams p) {
  const int n = p.size * p.size;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (p.parent[i] < 0) continue;
    const int wx = i % p.size, wy = i / p.size;
    if (wx > 0 && p.parent[i - 1] >= 0) unite(p.parent, i, i - 1);
    if (wy > 0) {
      const int up = i - p.size;
      if (p.parent[up] >= 0) unite(p.parent, i, up);
      if (wx > 0 && p.parent[up - 1] >= 0) unite(p.parent, i, up - 1);
      if (wx + 1 < p.size && p.parent[up + 1] >= 0) unite(p.parent, i, up + 1);
    }
  }
}

__global__ void blob_flatten_kernel(const BlobParams p) {
  const int n = p.size * p.size;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (p.parent[i] < 0) continue;
    const int r = find_root(p.parent, i);
    p.parent[i] = r;
    const int wx = i % p.size, wy = i / p.size;
    atomicMin(&p.box[4 * r + 0], wx);
    atomicMin(&p.box[4 * r + 1], wy);
    atomicMax(&p.box[4 * r + 2], wx);
    atomicMax(&p.box[4 * r + 3], wy);
  }
}

// Summed-area table: sat[(y+1)*(S+1) + (x+1)] = on-pixels in [0,x] x [0,y].
__global__ void blob_sat_rows_kernel(const BlobParams p) {
  const int S1 = p.size + 1;
  for (int y = blockIdx.x; y < p.size; y += gridDim.x) {  // one warp per row
    if (threadIdx.x >= 32) return;
    int carry = 0;
    for (int x0 = 0; x0 < p.size; x0 += 32) {
      const int x = x0 + threadIdx.x;
      int v = (x < p.size && p.parent[y * p.size + x] >= 0) ? 1 : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (threadIdx.x >= o) v += u;
      }
      if (x < p.size) p.sat[(y + 1) * S1 + x + 1] = carry + v;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
    if (threadIdx.x == 0) p.sat[(y + 1) * S1] = 0;
  }
}

// Column prefix of the row-scanned table: CTA = 32 columns x 32 row chunks;
// thread (column, chunk) keeps its chunk's values in registers, the 32 chunk
// sums of a column are scanned in shared memory, then the chunk is written
// back with its offset (31 CTAs x 1024 threads for a 960 window, where one
// thread per column walked 960 dependent rows).
constexpr int kSatChunkMax = 32;  // rows per chunk: size <= 32 * 32 = 1024 (else the serial kernel)
__global__ void __launch_bounds__(1024) blob_sat_cols_kernel(const BlobParams p) {
  __shared__ int tot[32][33];
  const int S1 = p.size + 1;
  const int cx = threadIdx.x & 31, ry = threadIdx.x >> 5;
  const int x = blockIdx.x * 32 + cx;
  const int R = (p.size + 31) / 32;  // rows per chunk (rows 1..size)
  const int y0 = 1 + ry * R, y1 = min(p.size + 1, y0 + R);
  int v[kSatChunkMax];
  int sum = 0;
#pragma unroll
  for (int k = 0; k < kSatChunkMax; ++k) {
    const int y = y0 + k;
    v[k] = (k < R && y < y1 && x < S1) ? p.sat[y * S1 + x] : 0;
    sum += v[k];
  }
  tot[ry][cx] = sum;
  __syncthreads();
  int off = 0;
  for (int j = 0; j < ry; ++j) off += tot[j][cx];
  if (x < S1) {
    if (ry == 0) p.sat[x] = 0;
#pragma unroll
    for (int k = 0; k < kSatChunkMax; ++k) {
      const int y = y0 + k;
      if (k < R && y < y1) {
        off += v[k];
        p.sat[y * S1 + x] = off;
      }
    }
  }
}
__global__ void blob_sat_cols_serial_kernel(const BlobParams p) {  // size > 1024
  const int S1 = p.size + 1;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < S1; x += gridDim.x * blockDim.x) {
    p.sat[x] = 0;
    int acc = 0;
    for (int y = 1; y <= p.size; ++y) {
      acc += p.sat[y * S1 + x];
      p.sat[y * S1 + x] = acc;
    }
  }
}

// Roots in raster order over many CTAs: (1) roots per 1024-pixel block,
// (2) one CTA scans the block counts, (3) every block writes its roots at
// its offset in raster order (ballot ranks), with the box's on-pixel count
// from the summed-area table.
__global__ void __launch_bounds__(1024) blob_root_count_kernel(const BlobParams p, int32_t *cnt) {
  __shared__ int wt[32];
  const int n = p.size * p.size;
  const int i = blockIdx.x * 1024 + threadIdx.x;
  const bool root = i < n && p.parent[i] == i;
  const unsigned bal = __ballot_sync(0xffffffffu, root);
  if ((threadIdx.x & 31) == 0) wt[threadIdx.x >> 5] = __popc(bal);
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < 32; ++w) t += wt[w];
    cnt[blockIdx.x] = t;
  }
}
__global__ void __launch_bounds__(1024) blob_scan_kernel(int32_t *cnt, int nb, int32_t *n_comp) {
  __shared__ int carry;
  __shared__ int wt[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int b0 = 0; b0 < nb; b0 += 1024) {
    const int b = b0 + threadIdx.x;
    const int c = b < nb ? cnt[b] : 0;
    int v = c;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    if (lane == 31) wt[warp] = v;
    __syncthreads();
    int before = carry;
    for (int w = 0; w < warp; ++w) before += wt[w];
    if (b < nb) cnt[b] = before + v - c;  // exclusive offset
    __syncthreads();
    if (threadIdx.x == 1023) carry = before + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_comp = carry;
}
__global__ void __launch_bounds__(1024) blob_emit_kernel(const BlobParams p, const int32_t *off,
                                                         int32_t *comp, int32_t max_comp) {
  __shared__ int wt[32];
  const int n = p.size * p.size;
  const int S1 = p.size + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = blockIdx.x * 1024 + threadIdx.x;
  const bool root = i < n && p.parent[i] == i;
  const unsigned bal = __ballot_sync(0xffffffffu, root);
  if (lane == 0) wt[warp] = __popc(bal);
  __syncthreads();
  if (!root) return;
  int before = off[blockIdx.x];
  for (int w = 0; w < warp; ++w) before += wt[w];
  const int k = before + __popc(bal & ((1u << lane) - 1u));
  if (k >= max_comp) return;
  const int4 b = reinterpret_cast<const int4 *>(p.box)[i];
  const int c = p.sat[(b.w + 1) * S1 + b.z + 1] - p.sat[b.y * S1 + b.z + 1] -
                p.sat[(b.w + 1) * S1 + b.x] + p.sat[b.y * S1 + b.x];
  int32_t *o = comp + 6 * k;
  o[0] = i;
  o[1] = b.x;
  o[2] = b.y;
  o[3] = b.z;
  o[4] = b.w;
  o[5] = c;
}

}  // namespace camx

using namespace camx;

extern "C" int camx_blob_components(const uint8_t *mask, int32_t n_cams, int32_t height,
                                    int32_t width, int32_t x0, int32_t y0, int32_t size,
                                    int32_t *scratch, int32_t *comp_out, int32_t max_comp,
                                    int32_t *n_comp_out, void *stream) {
  if (!mask || !scratch || !comp_out || !n_comp_out || n_cams < 1 || height < 1 || width < 1)
    return CAMX_EINVAL;
  if (size < 1 || x0 < 0 || y0 < 0 || x0 + size > n_cams * width || y0 + size > height)
    return CAMX_EINVAL;
  if (max_comp < 0) return CAMX_EINVAL;
  if (reinterpret_cast<uintptr_t>(scratch) % 16 != 0) return CAMX_EALIGN;
  BlobParams p{};
  p.mask = mask;
  p.n_cams = n_cams;
  p.H = height;
  p.W = width;
  p.x0 = x0;
  p.y0 = y0;
  p.size = size;
  const int64_t n = static_cast<int64_t>(size) * size;
  p.box = scratch;                       // n int4 (16-byte aligned)
  p.parent = scratch + 4 * n;
  p.sat = p.parent + n;
  cudaStream_t s = as_stream(stream);
  const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, sm_count() * 8));
  blob_init_kernel<<<blocks, 256, 0, s>>>(p);
  blob_union_kernel<<<blocks, 256, 0, s>>>(p);
  blob_flatten_kernel<<<blocks, 256, 0, s>>>(p);
  blob_sat_rows_kernel<<<std::min(size, sm_count() * 16), 32, 0, s>>>(p);
  if (size <= 32 * kSatChunkMax)
    blob_sat_cols_kernel<<<(size + 1 + 31) / 32, 1024, 0, s>>>(p);
  else
    blob_sat_cols_serial_kernel<<<(size + 1 + 127) / 128, 128, 0, s>>>(p);
  const int nb = static_cast<int>((n + 1023) / 1024);
  int32_t *cnt = p.sat + static_cast<int64_t>(size + 1) * (size + 1);  // [nb] block offsets
  blob_root_count_kernel<<<nb, 1024, 0, s>>>(p, cnt);
  blob_scan_kernel<<<1, 1024, 0, s>>>(cnt, nb, n_comp_out);
  blob_emit_kernel<<<nb, 1024, 0, s>>>(p, cnt, comp_out, max_comp);
  return launch_status();
}
