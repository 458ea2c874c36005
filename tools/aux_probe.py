"""One launch each of K1 (+ histograms), K4 (window counts) and the
band-staged tile kernel on config-2 data, for a single ncu capture."""
import numpy as np
import torch

from paper_1910_03517_b200 import _lib
from paper_1910_03517_b200.array import ArrayCorrector
from paper_1910_03517_b200.attention import window_origins
from paper_1910_03517_b200.synth import synthetic_batch

N, H, W, B, K = 8, 1536, 2048, 30, 16
frames = synthetic_batch(B, N, H, W, seed=1)
stats = torch.empty((B, N, 2, K, 112), dtype=torch.uint8, device="cuda")
hist = torch.empty((B, N, 2, K, 3, 256), dtype=torch.int32, device="cuda")
_lib.call("camx_band_stats", frames.data_ptr(), None, None, B * N, H, W, 32, K, 20,
          stats.data_ptr(), hist.data_ptr(), None)
org = window_origins((N * W, H), 960, 0.0)
wd = torch.as_tensor(np.asarray(org, np.int32), device="cuda")
counts = torch.empty(len(org), dtype=torch.int64, device="cuda")
_lib.call("camx_window_counts", None, frames[1].data_ptr(), frames[0].data_ptr(), 20, N, H, W,
          wd.data_ptr(), len(org), 960, counts.data_ptr(), None)
out = ArrayCorrector(N, H, W).correct(frames).out
wins = [(b, x, y) for b in range(B) for (x, y) in org]
wt = torch.as_tensor(np.asarray(wins, np.int32), device="cuda")
tiles = torch.empty((len(wins), 416, 416, 3), dtype=torch.uint8, device="cuda")
_lib.call("camx_tiles", out.data_ptr(), N, H, W, wt.data_ptr(), len(wins), 960, 416,
          tiles.data_ptr(), None)
torch.cuda.synchronize()
print("ok")
