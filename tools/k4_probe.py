"""K4 (camx_window_counts with the fused mask_diff of two frames) for the
config-2 difference plan: 36 windows of 960 over the 16384x1536 mosaic;
prints us per array-frame and the effective read bandwidth."""
import numpy as np
import torch

from paper_1910_03517_b200 import _lib
from paper_1910_03517_b200.attention import window_origins
from paper_1910_03517_b200.synth import synthetic_batch

N, H, W, S = 8, 1536, 2048, 960
fr = synthetic_batch(2, N, H, W, seed=3)
cur, prev = fr[1].contiguous(), fr[0].contiguous()
org = window_origins((N * W, H), S, 0.0)
wd = torch.as_tensor(np.asarray(org, np.int32), device="cuda")
counts = torch.empty(len(org), dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def run():
    _lib.call("camx_window_counts", None, cur.data_ptr(), prev.data_ptr(), 20, N, H, W,
              wd.data_ptr(), len(org), S, counts.data_ptr(), None)


for _ in range(3):
    run()
ts = []
for _ in range(20):
    flush.add_(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
ts.sort()
us = ts[len(ts) // 2]
covered = len(org) * S * S * 2 * 3  # bytes read (both frames) counting window overlaps
print(f"K4 {len(org)} windows: {us:.1f} us per array-frame, "
      f"{covered / us / 1e3:.0f} GB/s over the windows' bytes")
