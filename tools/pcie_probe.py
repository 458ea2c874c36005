"""PCIe ceiling: H2D || D2H of one FrameRing slot (4 config-2 array-frames,
302 MB each way) split over 1, 2 or 4 copy streams per direction, and a
one-direction baseline.  Does splitting a slot across copy engines beat one
cudaMemcpyAsync per direction?

    python tools/pcie_probe.py
"""
import time

import torch

nbytes = 4 * 8 * 1536 * 2048 * 3
h_in = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
h_out = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
h_in.fill_(3)
d_in = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
d_out = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]


def run(n_split, h2d=True, d2h=True, reps=10):
    chunk = (nbytes + n_split - 1) // n_split

    def once():
        for i in range(n_split):
            lo, hi = i * chunk, min(nbytes, (i + 1) * chunk)
            if h2d:
                with torch.cuda.stream(streams[i]):
                    d_in[lo:hi].copy_(h_in[lo:hi], non_blocking=True)
            if d2h:
                with torch.cuda.stream(streams[4 + i]):
                    h_out[lo:hi].copy_(d_out[lo:hi], non_blocking=True)
    once()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        once()
    torch.cuda.synchronize()
    return nbytes * reps / (time.perf_counter() - t0) / 1e9


for rnd in range(2):
    for n in (1, 2, 4):
        print(f"round {rnd} split {n}: H2D alone {run(n, d2h=False):5.1f} GB/s, "
              f"D2H alone {run(n, h2d=False):5.1f} GB/s, "
              f"H2D || D2H {run(n):5.1f} GB/s each way", flush=True)
