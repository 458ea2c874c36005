"""Config 5 as a two-stream frame pipeline: K3 of chunk c+1 (stream A)
alongside the tile kernel of chunk c (stream B, after an event), so the tile
kernel reads corrected rows K3 wrote moments earlier - from L2 if they are
still there - instead of after the whole 30-frame batch.  Same kernels as the
shipping path (camx_apply_array, camx_tiles), per-chunk launches.

    python tools/pipe5_probe.py [chunk ...]      # default 1 2 3 5 30
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1910_03517_b200 import _lib  # noqa: E402
from paper_1910_03517_b200.array import ArrayCorrector  # noqa: E402
from paper_1910_03517_b200.synth import synthetic_batch  # noqa: E402

N, H, W, B, K = 8, 1536, 2048, 30, 16
S = N - 1
frames = synthetic_batch(B, N, H, W, seed=1)
ac = ArrayCorrector(N, H, W)
res = ac.correct(frames)
gain, off = res.gain.contiguous(), res.offset.contiguous()
wins_f = ac.tile_windows(960)
per = len(wins_f)
tiles = torch.empty((B * per, 416, 416, 3), dtype=torch.uint8, device="cuda")
out = torch.empty_like(frames)
img_bytes = N * H * W * 3
map_bytes = S * 2 * K * 3 * 8
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
wd = {}


def win_dev(c):
    if c not in wd:
        w = [(b, x, y) for b in range(c) for (x, y) in wins_f]
        wd[c] = torch.as_tensor(np.asarray(w, np.int32), device="cuda")
    return wd[c]


def run(chunk):
    evs = []
    for f0 in range(0, B, chunk):
        c = min(chunk, B - f0)
        _lib.call("camx_apply_array", frames.data_ptr() + f0 * img_bytes,
                  out.data_ptr() + f0 * img_bytes, c, 0, N, N, 0, H, W, K,
                  gain.data_ptr() + f0 * map_bytes, off.data_ptr() + f0 * map_bytes,
                  sa.cuda_stream)
        e = torch.cuda.Event()
        e.record(sa)
        evs.append((f0, c, e))
    for f0, c, e in evs:
        sb.wait_event(e)
        _lib.call("camx_tiles", out.data_ptr() + f0 * img_bytes, N, H, W, win_dev(c).data_ptr(),
                  c * per, 960, 416, tiles.data_ptr() + f0 * per * 416 * 416 * 3, sb.cuda_stream)


def timed(chunk, reps=10):
    for _ in range(2):
        run(chunk)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(sa)
    sb.wait_stream(sa)
    for _ in range(reps):
        run(chunk)
        sa.wait_stream(sb)  # next rep's K3 rewrites `out`
    e1.record(sa)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ref_tiles = None
for chunk in [int(a) for a in sys.argv[1:]] or [1, 2, 3, 5, 30]:
    ms = timed(chunk)
    if ref_tiles is None:
        ref_tiles = tiles.clone()
    same = torch.equal(tiles, ref_tiles)
    print(f"chunk {chunk:2d}: {ms:.4f} ms per 30 frames ({B / ms * 1e3:.0f} array-fps), "
          f"tiles identical to the first variant: {same}", flush=True)
