"""cProfile of the host side of one sharded rank's correct() (see shard_probe)."""
import cProfile
import pstats

import torch

from paper_1910_03517_b200.array import ArrayCorrector
from paper_1910_03517_b200.synth import synthetic_batch

N, H, W, B, c = 8, 1536, 2048, 30, 1
frames = synthetic_batch(B, c, H, W, seed=1)
out = torch.empty_like(frames)
ac = ArrayCorrector(N, H, W, cam_begin=0, cam_count=c,
                    exchange=lambda st: st.repeat(1, N, 1, 1, 1))
for _ in range(5):
    ac.correct(frames, out)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    ac.correct(frames, out)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
