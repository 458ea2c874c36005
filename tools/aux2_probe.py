"""Device time of the remaining per-call kernels at config-2 sizes:
camx_mask_diff (one 8-camera array-frame pair), camx_apply_map (one camera,
one map), camx_band_moments (a 30-frame batch of records), camx_fit_affine
and camx_smooth_maps (one seam)."""
import torch

from paper_1910_03517_b200 import _lib
from paper_1910_03517_b200.synth import synthetic_batch

N, H, W, K = 8, 1536, 2048, 16
fr = synthetic_batch(2, N, H, W, seed=5)
mask = torch.empty((N, H, W), dtype=torch.uint8, device="cuda")


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


npx = N * H * W
us = timeit(lambda: _lib.call("camx_mask_diff", fr[1].data_ptr(), fr[0].data_ptr(), npx, 20,
                              mask.data_ptr(), None))
print(f"mask_diff, 8 x 2048x1536: {us:.1f} us = {npx * 7 / us / 1e3:.0f} GB/s (7 B/px)", flush=True)

img = fr[0, 0].contiguous()
out = torch.empty_like(img)
g = torch.full((K, 3), 1.1, dtype=torch.float64, device="cuda")
o = torch.full((K, 3), 3.0, dtype=torch.float64, device="cuda")
us = timeit(lambda: _lib.call("camx_apply_map", img.data_ptr(), out.data_ptr(), 1, H, W, 0, K,
                              g.data_ptr(), o.data_ptr(), None))
print(f"apply_map, one 2048x1536 camera: {us:.1f} us = {H * W * 6 / us / 1e3:.0f} GB/s", flush=True)
