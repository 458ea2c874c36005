"""Device time of the SURVEY 8f kernels at config-2 sizes: camx_blob_components
on one 960 x 960 window of the 8-camera motion mask (a moving-object mask of
two synthetic frames), and camx_seam_cost on all 7 seams of a 30-frame batch.
Inputs resident on the device; CUDA events around the launches."""
import torch

from paper_1910_03517_b200 import _lib
from paper_1910_03517_b200.synth import synthetic_batch

N, H, W, S = 8, 1536, 2048, 960
fr = synthetic_batch(2, N, H, W, seed=7)
mask = torch.empty((N, H, W), dtype=torch.uint8, device="cuda")
_lib.call("camx_mask_diff", fr[1].data_ptr(), fr[0].data_ptr(), N * H * W, 20, mask.data_ptr(),
          None)
scratch = torch.empty((6 * S * S + 2 * S + 1 + (S * S + 1023) // 1024 + 3,), dtype=torch.int32,
                      device="cuda")
comp = torch.empty((65536, 6), dtype=torch.int32, device="cuda")
n = torch.zeros((1,), dtype=torch.int32, device="cuda")


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


for x in (0, 1920, 7680):
    us = timeit(lambda: _lib.call("camx_blob_components", mask.data_ptr(), N, H, W, x, 576, S,
                                  scratch.data_ptr(), comp.data_ptr(), 65536, n.data_ptr(), None))
    print(f"blob components, window x={x} y=576 (960^2): {us:.1f} us, "
          f"{int(n.item())} components, {int(mask[:, 576:1536].sum())} on-pixels in the rows",
          flush=True)

B = 30
frames = synthetic_batch(B, N, H, W, seed=9)
out = torch.empty((N - 1,), dtype=torch.float64, device="cuda")
img = H * W * 3


def seams():
    # one call per array-frame: the 7 (camera s, camera s+1) pairs are
    # contiguous image runs (left = cameras 0..6, right = cameras 1..7)
    for b in range(B):
        base = frames.data_ptr() + b * N * img
        _lib.call("camx_seam_cost", base, base + img, N - 1, H, W, W, 8,
                  out.data_ptr() + 8 * (N - 1) * 0, None)


print(f"seam_cost, 7 seams x {B} array-frames (one call per array-frame): {timeit(seams):.1f} us",
      flush=True)
