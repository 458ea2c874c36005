"""Config 1 (2 x 640x480, 64-frame batches): where the step goes.  Graph
step vs K1 / K3 alone (CUDA events, device-resident, L2 not flushed: the
whole batch is 59 MB in + 59 MB out)."""
import torch

from paper_1910_03517_b200 import _lib
from paper_1910_03517_b200.array import ArrayCorrector
from paper_1910_03517_b200.synth import synthetic_batch

N, H, W, B, K = 2, 480, 640, 64, 16
frames = synthetic_batch(B, N, H, W, seed=1)
out = torch.empty_like(frames)


def timeit(fn, steps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps * 1e3


ac = ArrayCorrector(N, H, W, histograms=True)
print(f"graph step {timeit(lambda: ac.correct_graphed(frames, out)):.1f} us")
print(f"eager step {timeit(lambda: ac.correct(frames, out)):.1f} us")
g = torch.ones((B, N - 1, 2, K, 3), dtype=torch.float64, device="cuda") * 1.1
o = torch.ones_like(g)
s = torch.cuda.current_stream().cuda_stream
k3 = timeit(lambda: _lib.call("camx_apply_array", frames.data_ptr(), out.data_ptr(), B, 0, N, N, 0,
                              H, W, K, g.data_ptr(), o.data_ptr(), s))
print(f"K3 alone {k3:.1f} us = {2 * frames.numel() / k3 / 1e3:.0f} GB/s")
stats = torch.empty((B, N, 2, K, _lib.STAT_BYTES), dtype=torch.uint8, device="cuda")
hist = torch.empty((B, N, 2, K, 3, 256), dtype=torch.int32, device="cuda")
k1 = timeit(lambda: _lib.call("camx_band_stats", frames.data_ptr(), None, None, B * N, H, W, 32,
                              K, 20, stats.data_ptr(), hist.data_ptr(), s))
print(f"K1 (+hist) alone {k1:.1f} us")
