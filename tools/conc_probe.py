"""Probe: K3 (apply, HBM-bound) concurrently with the standalone tile kernel
(camx_tiles on an already corrected batch) on two streams - is the sum
hidden?  Config-5 geometry, 30-frame batches."""
import numpy as np
import torch

from paper_1910_03517_b200 import _lib
from paper_1910_03517_b200.array import ArrayCorrector
from paper_1910_03517_b200.synth import synthetic_batch

N, H, W, B = 8, 1536, 2048, 30
frames = synthetic_batch(B, N, H, W, seed=1)
out = torch.empty_like(frames)
out2 = torch.empty_like(frames)
ac = ArrayCorrector(N, H, W)
res = ac.correct(frames, out)
wins = [(b, x, y) for b in range(B) for (x, y) in ac.tile_windows(960)]
wd = torch.as_tensor(np.asarray(wins, np.int32), device="cuda")
tiles = torch.empty((len(wins), 416, 416, 3), dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def k3(s):
    _lib.call("camx_apply_array", frames.data_ptr(), out2.data_ptr(), B, 0, N, N, 0, H, W, 16,
              res.gain.data_ptr(), res.offset.data_ptr(), s.cuda_stream)


def tl(s):
    _lib.call("camx_tiles", out.data_ptr(), N, H, W, wd.data_ptr(), len(wins), 960, 416,
              tiles.data_ptr(), s.cuda_stream)


def t(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


print("K3 alone      ", round(t(lambda: k3(torch.cuda.current_stream())), 3), "ms")
print("tiles alone   ", round(t(lambda: tl(torch.cuda.current_stream())), 3), "ms")


def both():
    k3(s1)
    tl(s2)


print("K3 || tiles   ", round(t(both), 3), "ms")
