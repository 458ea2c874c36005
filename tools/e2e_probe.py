"""PCIe ceiling vs the end-to-end correct_host path (config-2 geometry)."""
import torch

from paper_1910_03517_b200.array import ArrayCorrector
from paper_1910_03517_b200.synth import synthetic_batch

N, H, W, B = 8, 1536, 2048, 8
dev = synthetic_batch(B, N, H, W)
host_in = dev.cpu().pin_memory()
host_out = torch.empty_like(host_in).pin_memory()
nbytes = host_in.numel()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


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
for chunk in (1, 2, 4):
    ac = ArrayCorrector(N, H, W)
    t = timed(lambda: ac.correct_host(host_in, host_out, chunk=chunk))
    print(f"correct_host chunk={chunk}: {t:.2f} ms/8 frames = {B * N * H * W / 1e6 / (t / 1e3):.0f} MP/s,"
          f" {nbytes / t / 1e6:.1f} GB/s each way")
