"""Probe the per-step cost of one rank of the camera-sharded path at N GPUs,
on one GPU: cameras [0, 8/N) with a stand-in exchange (the local records
tiled to the whole array - a device copy where NCCL would all-gather).
Prints GPU ms per step and host enqueue ms per step, to see whether the
N>1 step is host-bound."""
import sys
import time

import torch

from paper_1910_03517_b200.array import ArrayCorrector
from paper_1910_03517_b200.synth import synthetic_batch

N, H, W = 8, 1536, 2048
for world in (1, 2, 4, 8):
    for B in (30, 60):
        c = N // world
        frames = synthetic_batch(B, c, H, W, seed=1)
        out = torch.empty_like(frames)
        if world == 1:
            ac = ArrayCorrector(N, H, W)
        else:
            rep = N // c
            holder = {}

            def exchange(st, rep=rep, holder=holder):
                # stand-in for the NCCL all-gather: one device copy into a
                # persistent (B, N, ...) buffer
                full = holder.get("full")
                if full is None:
                    full = holder["full"] = torch.empty((st.shape[0], rep * st.shape[1],
                                                         *st.shape[2:]), dtype=st.dtype,
                                                        device=st.device)
                full.view(st.shape[0], rep, *st.shape[1:]).copy_(st[:, None])
                return full

            ac = ArrayCorrector(N, H, W, cam_begin=0, cam_count=c, exchange=exchange)
        for _ in range(5):
            ac.correct(frames, out)
        torch.cuda.synchronize()
        steps = 30
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(steps):
            ac.correct(frames, out)
        e1.record()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        print(f"world {world} B {B}: gpu {e0.elapsed_time(e1) / steps:.3f} ms/step, "
              f"host enqueue {(t1 - t0) / steps * 1e3:.3f} ms/step, "
              f"{B / (e0.elapsed_time(e1) / steps / 1e3):.0f} array-fps per rank", flush=True)
        del frames, out, ac
        torch.cuda.empty_cache()
