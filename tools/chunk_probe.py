"""Config 5 with K3 and the tile kernel interleaved per chunk of array-frames
(tiles of chunk c read corrected rows that may still be in L2) vs batched.
    CAMX_LIB=... python tools/chunk_probe.py"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1910_03517_b200 import _lib
from paper_1910_03517_b200.array import ArrayCorrector
from paper_1910_03517_b200.synth import synthetic_batch

N, H, W, B = 8, 1536, 2048, 30
frames = synthetic_batch(B, N, H, W, seed=1)
ac = ArrayCorrector(N, H, W)
res = ac.correct(frames)
gain, off = res.gain.contiguous(), res.offset.contiguous()
org = ac.tile_windows(960)
out = torch.empty_like(frames)
tiles = torch.empty((B * len(org), 416, 416, 3), dtype=torch.uint8, device="cuda")
fb = N * H * W * 3
gb = gain[0].numel() * 8


def run(chunk):
    for c0 in range(0, B, chunk):
        n = min(chunk, B - c0)
        wins = [(b, x, y) for b in range(n) for (x, y) in org]
        wd = WD[n]
        _lib.call("camx_apply_array", frames.data_ptr() + c0 * fb, out.data_ptr() + c0 * fb, n, 0,
                  N, N, 0, H, W, 16, gain.data_ptr() + c0 * gb, off.data_ptr() + c0 * gb, None)
        _lib.call("camx_tiles", out.data_ptr() + c0 * fb, N, H, W, wd.data_ptr(), len(wins), 960,
                  416, tiles.data_ptr() + c0 * len(org) * 416 * 416 * 3, None)


WD = {n: torch.as_tensor(np.asarray([(b, x, y) for b in range(n) for (x, y) in org], np.int32),
                         device="cuda") for n in (1, 2, 3, 5, 6, 10, 15, 30)}
ref = None
for chunk in (30, 1, 2, 3, 5, 6, 10, 15):
    run(chunk)
    torch.cuda.synchronize()
    if ref is None:
        ref = tiles.clone()
    ok = torch.equal(ref, tiles)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        run(chunk)
    e1.record()
    torch.cuda.synchronize()
    print(f"chunk {chunk:2d}: {e0.elapsed_time(e1) / 5:.4f} ms per 30 frames, tiles equal {ok}")
