"""Config-5 K3 + K5 alone (maps given; camx_correct_and_tile: K3 then the tile kernel) over a
config-2 batch with the 36-window sliding plan per array-frame.

    python tools/fused_probe.py [B] [reps]      # ms per call, GB/s on algorithmic bytes
    CHECK=1 python tools/fused_probe.py 2       # bit-exact vs apply + camx_tiles
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1910_03517_b200 import _lib  # noqa: E402
from paper_1910_03517_b200.array import ArrayCorrector  # noqa: E402
from paper_1910_03517_b200.synth import synthetic_batch  # noqa: E402

N, H, W = 8, 1536, 2048
B = int(sys.argv[1]) if len(sys.argv) > 1 else 30
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
frames = synthetic_batch(B, N, H, W, seed=1)
ac = ArrayCorrector(N, H, W)
res = ac.correct(frames)
gain, off = res.gain.contiguous(), res.offset.contiguous()
wins = [(b, x, y) for b in range(B) for (x, y) in ac.tile_windows(960)]
per = len(wins) // B
wd = torch.as_tensor(np.asarray(wins, np.int32), device="cuda")
fo = torch.as_tensor(np.arange(B + 1, dtype=np.int32) * per, device="cuda")
tiles = torch.empty((len(wins), 416, 416, 3), dtype=torch.uint8, device="cuda")
out = torch.empty_like(frames)


def call():
    _lib.call("camx_correct_and_tile", frames.data_ptr(), out.data_ptr(), B, N, 0, H, W, 16,
              gain.data_ptr(), off.data_ptr(), wd.data_ptr(), fo.data_ptr(), len(wins), per, 960,
              416, tiles.data_ptr(), None)


for _ in range(2):
    call()
torch.cuda.synchronize()
if os.environ.get("NCU"):
    sys.exit(0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    call()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
alg = B * (N * H * W * 6 + per * 416 * 416 * 3)
print(f"fused K3+K5 B={B}: {ms:.4f} ms/call = {alg / ms / 1e6:.1f} GB/s algorithmic, "
      f"{B / ms * 1e3:.0f} array-fps")
if os.environ.get("CHECK"):
    ref_out = torch.empty_like(frames)
    _lib.call("camx_apply_array", frames.data_ptr(), ref_out.data_ptr(), B, 0, N, N, 0, H, W, 16,
              gain.data_ptr(), off.data_ptr(), None)
    ref_t = torch.empty_like(tiles)
    _lib.call("camx_tiles", ref_out.data_ptr(), N, H, W, wd.data_ptr(), len(wins), 960, 416,
              ref_t.data_ptr(), None)
    torch.cuda.synchronize()
    print("frames equal:", torch.equal(out, ref_out), " tiles equal:", torch.equal(tiles, ref_t),
          " tile bytes differing:", int((tiles != ref_t).sum()))
