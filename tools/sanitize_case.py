"""Small workload exercising the shared-memory kernels for compute-sanitizer:
K1 with histograms (+ fused mask), K2, fused apply+tile, fix-up, standalone
tiles (band-staged, exact crop), window counts, the one-GPU pipelined stream."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1910_03517_b200 import detect  # noqa: E402
from paper_1910_03517_b200.array import ArrayCorrector  # noqa: E402
from paper_1910_03517_b200.exposure import ExposureConfig, ExposureMode  # noqa: E402
from paper_1910_03517_b200.synth import synthetic_batch  # noqa: E402

N, H, W, B = 3, 200, 1024, 2
frames = synthetic_batch(B, N, H, W, seed=3)
ac = ArrayCorrector(N, H, W, ExposureConfig(band_width=16, blocks=5), ExposureMode.OBJECT_REMOVAL,
                    histograms=True)
ac.correct(frames)
ac.correct(frames)
res, tiles = ac.correct_and_tile(frames, size=128, out_size=52)
t2 = detect.tiles(res.out, [(0, 10, 5), (1, 900, 60)], 128, 52)
t3 = detect.tiles(res.out, [(0, 10, 5), (1, 1000, 60)], 128, 128)   # exact crop
from paper_1910_03517_b200 import attention  # noqa: E402
cnt = attention.window_counts([(3, 0), (901, 50), (2900, 70)], 128, cur=frames[1], prev=frames[0],
                              n_cams=N)
pipe = ArrayCorrector(N, H, W, ExposureConfig(band_width=16, blocks=5), histograms=True)
for _ in range(3):
    pipe.submit(frames)
pipe.flush()
torch.cuda.synchronize()
print("ok", tiles.shape, t2.shape, t3.shape, list(cnt))
