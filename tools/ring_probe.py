"""PCIe ceiling vs the FrameRing end-to-end path (config-2 geometry) for a
few ring shapes; wall clock over many steps."""
import sys
import time

import torch

from paper_1910_03517_b200.array import ArrayCorrector
from paper_1910_03517_b200.ring import FrameRing
from paper_1910_03517_b200.synth import synthetic_batch

N, H, W = 8, 1536, 2048
dev = synthetic_batch(8, N, H, W)
host_in = dev.cpu().pin_memory()
host_out = torch.empty_like(host_in).pin_memory()
nbytes = host_in.numel()


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / reps


t = timed(lambda: dev.copy_(host_in, non_blocking=True))
print(f"H2D alone: {nbytes / t / 1e6:.1f} GB/s")
t = timed(lambda: host_out.copy_(dev, non_blocking=True))
print(f"D2H alone: {nbytes / t / 1e6:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
dev2 = torch.empty_like(dev)


def both():
    with torch.cuda.stream(s1):
        dev.copy_(host_in, non_blocking=True)
    with torch.cuda.stream(s2):
        host_out.copy_(dev2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


t = timed(both)
print(f"H2D || D2H: {nbytes / t / 1e6:.1f} GB/s each")

shapes = [(3, 8, 2, 10), (3, 8, 2, 40), (4, 8, 2, 40), (4, 4, 2, 80), (6, 4, 3, 80), (4, 16, 2, 20),
          (8, 2, 3, 160)]
for slots, B, D, steps in shapes:
    ac = ArrayCorrector(N, H, W, histograms=True)
    ring = FrameRing(ac, slots=slots, batch=B, device_buffers=D)
    for j in range(slots):
        v = ring.acquire(block=False)
        v[...] = host_in.numpy()[[i % 8 for i in range(B)]]
        ring.publish(j)
    for r in ring.drain():
        ring.release(r)

    def run(n):
        for k in range(n):
            ring.acquire(block=False)
            ring.publish(k)
            if ring.pending() >= slots:
                ring.release(ring.get())
        for r in ring.drain():
            ring.release(r)

    run(3)
    t0 = time.perf_counter()
    run(steps)
    ms = (time.perf_counter() - t0) * 1e3 / steps
    px = B * N * H * W
    print(f"ring slots={slots} B={B} D={D} steps={steps}: {ms:.2f} ms/step = "
          f"{px / 1e6 / (ms / 1e3):.0f} MP/s, {px * 3 / (ms / 1e3) / 1e9:.1f} GB/s each way")
    del ring, ac
    torch.cuda.empty_cache()
sys.stdout.flush()
