"""The bench's roofline kernels alone, on the bench's own frames and batch,
for ncu captures (profiles/traffic.json):

    python tools/roofline_probe.py config2|config4|config5 [batch]

Runs the workload's corrector once (K1, K2, K3: the kernels to
--launch-skip), then the roofline leg once: camx_apply_array (K3) and, for
config5, camx_tiles - exactly the launches bench.py's roofline leg times."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1910_03517_b200 import _lib  # noqa: E402
from paper_1910_03517_b200.array import ArrayCorrector  # noqa: E402
from paper_1910_03517_b200.exposure import ExposureConfig  # noqa: E402

name = sys.argv[1]
n_cams, H, W, B0, _ = bench.WORKLOADS[name]
B = int(sys.argv[2]) if len(sys.argv) > 2 else B0
wrap = name == "config4"
frames = bench.bench_frames(name, B, "cuda")
ac = ArrayCorrector(n_cams, H, W, ExposureConfig(), wrap=wrap, histograms=True)
out = torch.empty_like(frames)
res = ac.correct(frames, out)
torch.cuda.synchronize()
if name == "config5m":  # K1 + K2 + K3 with the in-pass motion counts (frame 0's previous = frame B-1)
    sys.argv = ["bench"]
    args = bench.parse()
    wl = bench.Workload(name, B, args, 1, 0, torch)
    wl.res = res
    wl.motion_call()()
    torch.cuda.synchronize()
    print(f"{name} batch {B}: motion call done")
    sys.exit(0)
_lib.call("camx_apply_array", frames.data_ptr(), out.data_ptr(), B, 0, n_cams, n_cams, int(wrap),
          H, W, 16, res.gain.data_ptr(), res.offset.data_ptr(), None)
nbytes = 6 * B * n_cams * H * W
if name == "config5":
    wins = [(b, x, y) for b in range(B) for (x, y) in ac.tile_windows(960)]
    wd = torch.as_tensor(np.asarray(wins, np.int32), device="cuda")
    tiles = torch.empty((len(wins), 416, 416, 3), dtype=torch.uint8, device="cuda")
    _lib.call("camx_tiles", out.data_ptr(), n_cams, H, W, wd.data_ptr(), len(wins), 960, 416,
              tiles.data_ptr(), None)
    nbytes += tiles.numel()
torch.cuda.synchronize()
print(f"{name} batch {B}: algorithmic bytes per roofline launch {nbytes}")
