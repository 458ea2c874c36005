"""A camera source streamed through the B200 path end to end: frames are
written into the library's pinned frame ring, corrected on the GPU, and the
attention tick (Scheduler on the host, motion counts from the apply pass)
picks the detector windows whose 416x416 tiles are returned.

    python examples/attention_stream.py [n_batches]

Synthetic 8 x 2048x1536 array (synth.synthetic_batch: a panorama with
per-camera exposure distortion and moving objects), 4 array-frames per batch.
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1910_03517_b200.array import ArrayCorrector, AttendPipeline  # noqa: E402
from paper_1910_03517_b200.attention import AttentionConfig, Scheduler  # noqa: E402
from paper_1910_03517_b200.ring import FrameRing  # noqa: E402
from paper_1910_03517_b200.synth import synthetic_batch  # noqa: E402

N, H, W, B = 8, 1536, 2048, 4
n_batches = int(sys.argv[1]) if len(sys.argv) > 1 else 6

# 1. correction only, host frames in / host frames out (the pinned ring)
ring = FrameRing(ArrayCorrector(N, H, W), slots=4, batch=B)
for k in range(n_batches):
    view = ring.acquire()                     # producer: a free pinned slot
    view[...] = synthetic_batch(B, N, H, W, seed=7, first=k * B, device="cpu").numpy()  # decode
    ring.publish(tag=k * B)
    while ring.pending() >= 3:                # consumer: oldest finished batch
        r = ring.get()
        print(f"ring: frames {r.tag}..{r.tag + B - 1} corrected, "
              f"seam 0 gains (block 0) {np.round(r.gain[-1, 0, 0, 0], 3)}")
        ring.release(r)
for r in ring.drain():
    print(f"ring: frames {r.tag}..{r.tag + B - 1} corrected")
    ring.release(r)

# 2. the attention tick on device-resident batches (motion counts from K3,
#    host Scheduler of batch k-1 while the GPU corrects batch k)
sched = Scheduler((N * W, H), AttentionConfig(budget=4, window_size=960, diff_threshold=50))
pipe = AttendPipeline(ArrayCorrector(N, H, W), sched)
for k in range(n_batches + 1):
    res = (pipe.submit(synthetic_batch(B, N, H, W, seed=7, first=k * B), frame_index=k * B)
           if k < n_batches else pipe.flush())
    if res is None:
        continue
    torch.cuda.synchronize()
    for b, reqs in enumerate(res.requests):
        wins = ", ".join(f"{r.mechanism.value}@({r.window.x},{r.window.y})" for r in reqs)
        print(f"tick {res.frame_index + b}: {wins}")
    print(f"  -> {res.tiles.shape[0]} tiles {tuple(res.tiles.shape[1:])} uint8 on the GPU")
