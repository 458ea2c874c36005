"""K1 (camx_band_stats) time for the config-2 batch: 30 frames x 8 cameras."""
import os
import sys

import torch

from paper_1910_03517_b200 import _lib
from paper_1910_03517_b200.synth import synthetic_batch

N, H, W, B, K = 8, 1536, 2048, 30, 16
frames = synthetic_batch(B, N, H, W, seed=1)
stats = torch.empty((B, N, 2, K, 112), dtype=torch.uint8, device="cuda")
for _ in range(3):
    _lib.call("camx_band_stats", frames.data_ptr(), None, None, B * N, H, W, 32, K, 20,
              stats.data_ptr(), None, None)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # flush L2 between runs (inputs of K1 alone would otherwise stay resident)
    frames[:2].add_(0)
    e0.record()
    _lib.call("camx_band_stats", frames.data_ptr(), None, None, B * N, H, W, 32, K, 20,
              stats.data_ptr(), None, None)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
ts.sort()
print(os.environ.get("CAMX_K1_PER_SM", "default"), "K1 us median", round(ts[len(ts) // 2], 2))
