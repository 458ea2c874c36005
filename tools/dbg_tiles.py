import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.getcwd() + "/tests")
import numpy as np, torch
from oracle import camarray_oracle as O
from paper_1910_03517_b200 import detect, exposure as xp
from paper_1910_03517_b200.array import ArrayCorrector
rng = np.random.default_rng(0)
N, H, W, B = 3, 180, 1024, 2
frames = np.stack([O.synthetic_array(N, H, W, seed=80, objects=3, frame_index=t) for t in range(B)])
S = int(rng.choice([64, 100, 150])); out_size = int(rng.integers(8, S))
wins = [(int(rng.integers(0, B)), int(rng.integers(0, N * W - S + 1)), int(rng.integers(0, H - S + 1))) for _ in range(int(rng.integers(5, 40)))]
print("S", S, "out", out_size, "nwin", len(wins), flush=True)
ac = ArrayCorrector(N, H, W, xp.ExposureConfig(band_width=16, blocks=3))
d = torch.from_numpy(frames).cuda()
res = ac.correct(d); torch.cuda.synchronize(); print("correct ok", flush=True)
t = detect.tiles(res.out, sorted(wins, key=lambda w: w[0]), S, out_size); torch.cuda.synchronize(); print("tiles ok", flush=True)

res, tl = ac.correct_and_tile(d, wins, size=S, out_size=out_size); torch.cuda.synchronize(); print("fused ok", flush=True)
