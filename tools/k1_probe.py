"""K1 (camx_band_stats) time for the config-2 batch (30 frames x 8 cameras),
plain and with histograms, L2 flushed between runs."""
import os

import torch

from paper_1910_03517_b200 import _lib
from paper_1910_03517_b200.synth import synthetic_batch

N, H, W, B, K = 8, 1536, 2048, 30, 16
frames = synthetic_batch(B, N, H, W, seed=1)
stats = torch.empty((B, N, 2, K, 112), dtype=torch.uint8, device="cuda")
hist = torch.empty((B, N, 2, K, 3, 256), dtype=torch.int32, device="cuda")
for h in (None, hist):
    ts = []
    for i in range(23):
        frames[:2].add_(0)  # evicts the bands from L2
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("camx_band_stats", frames.data_ptr(), None, None, B * N, H, W, 32, K, 20,
                  stats.data_ptr(), None if h is None else h.data_ptr(), None)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts = sorted(ts[3:])
    print(os.environ.get("CAMX_LIB", "in-tree"), "hist" if h is not None else "plain",
          "K1 us", round(ts[len(ts) // 2], 2), flush=True)

# OBJECT_REMOVAL: frames 1.. against their predecessors (fused in-band motion mask)
fb = N * H * W * 3
for h in (None, hist):
    ts = []
    for i in range(23):
        frames[:2].add_(0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("camx_band_stats", frames.data_ptr() + fb, frames.data_ptr(), None,
                  (B - 1) * N, H, W, 32, K, 20, stats.data_ptr(),
                  None if h is None else h.data_ptr(), None)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts = sorted(ts[3:])
    print(os.environ.get("CAMX_LIB", "in-tree"), "removal", "hist" if h is not None else "plain",
          "K1 us", round(ts[len(ts) // 2], 2), flush=True)
