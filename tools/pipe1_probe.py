"""One GPU, config 2, 30-frame batches with histograms: CUDA-graph step
(K1 -> K2 -> K3, PDL) vs the pipelined stream (ArrayCorrector.submit: front
half of batch k on a side stream under K3 of batch k-1), ms per batch."""
import torch

from paper_1910_03517_b200.array import ArrayCorrector
from paper_1910_03517_b200.synth import synthetic_batch

N, H, W, B = 8, 1536, 2048, 30
frames = synthetic_batch(B, N, H, W, seed=1)
out = torch.empty_like(frames)


def timeit(fn, steps=40, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


for hist in (True, False):
    a = ArrayCorrector(N, H, W, histograms=hist)
    g = timeit(lambda: a.correct_graphed(frames, out))
    b = ArrayCorrector(N, H, W, histograms=hist)
    p = timeit(lambda: b.submit(frames, out))
    b.flush()
    print(f"hist={hist}: graph {g:.4f} ms, pipelined {p:.4f} ms per batch")
