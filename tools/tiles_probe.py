"""camx_tiles alone on a corrected config-2 batch: 1080 tiles (30 frames x 36
windows, 960 -> 416); prints ms per call."""
import numpy as np
import torch

from paper_1910_03517_b200 import _lib
from paper_1910_03517_b200.array import ArrayCorrector
from paper_1910_03517_b200.synth import synthetic_batch

N, H, W, B = 8, 1536, 2048, 30
frames = synthetic_batch(B, N, H, W, seed=1)
ac = ArrayCorrector(N, H, W)
out = ac.correct(frames).out
wins = [(b, x, y) for b in range(B) for (x, y) in ac.tile_windows(960)]
wd = torch.as_tensor(np.asarray(wins, np.int32), device="cuda")
tiles = torch.empty((len(wins), 416, 416, 3), dtype=torch.uint8, device="cuda")
for _ in range(3):
    _lib.call("camx_tiles", out.data_ptr(), N, H, W, wd.data_ptr(), len(wins), 960, 416,
              tiles.data_ptr(), None)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    _lib.call("camx_tiles", out.data_ptr(), N, H, W, wd.data_ptr(), len(wins), 960, 416,
              tiles.data_ptr(), None)
e1.record()
torch.cuda.synchronize()
print("camx_tiles ms", round(e0.elapsed_time(e1) / 10, 3))

# the camera-sharded kernel on the whole array (one "rank", no halo)
zero = torch.zeros_like(tiles)
for _ in range(2):
    _lib.call("camx_tiles_shard", out.data_ptr(), N, H, W, 0, None, wd.data_ptr(), len(wins), 960,
              416, zero.data_ptr(), None)
torch.cuda.synchronize()
e0.record()
for _ in range(5):
    _lib.call("camx_tiles_shard", out.data_ptr(), N, H, W, 0, None, wd.data_ptr(), len(wins), 960,
              416, zero.data_ptr(), None)
e1.record()
torch.cuda.synchronize()
print("camx_tiles_shard ms", round(e0.elapsed_time(e1) / 5, 3), "equal:", torch.equal(zero, tiles))
