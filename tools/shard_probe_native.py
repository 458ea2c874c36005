"""Per-step cost of rank 0 of the native sharded path (camx_correct_batch_sharded)
at N GPUs, on one GPU: a one-rank NCCL communicator stands in for the
N-rank one (the all-gather then moves only this rank's block, so the NVLink
transfer is missing; the records of the other ranks are stale - timing only)."""
import ctypes
import os
import time

import torch

from paper_1910_03517_b200 import _lib
from paper_1910_03517_b200.array import ArrayCorrector
from paper_1910_03517_b200.dist import camera_partition
from paper_1910_03517_b200.synth import synthetic_batch

uid = torch.zeros(128, dtype=torch.uint8)
_lib.call("camx_comm_unique_id", uid.data_ptr())
h = ctypes.c_void_p()
_lib.call("camx_comm_init", ctypes.byref(h), uid.data_ptr(), 1, 0)

N, H, W = 8, 1536, 2048
for world, B, ch in [(1, 30, 1), (2, 30, 1), (2, 30, 2), (4, 30, 1), (4, 30, 2), (4, 30, 3),
                     (8, 30, 1), (8, 30, 2), (8, 30, 3), (8, 30, 5), (8, 60, 1), (8, 60, 3)]:
    if True:
        b0, c = camera_partition(N, world)[0]

        class Comm:
            rank = 0
            handle = h.value
        Comm.world = world
        frames = synthetic_batch(B, c, H, W, seed=1)
        out = torch.empty_like(frames)
        ac = ArrayCorrector(N, H, W, cam_begin=b0, cam_count=c, comm=Comm())
        ac.shard_chunk_count = ch
        for _ in range(5):
            ac.correct(frames, out)
        torch.cuda.synchronize()
        steps = 40
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(steps):
            ac.correct(frames, out)
        e1.record()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        print(f"world {world} B {B} chunks {ch}: gpu {ms:.3f} ms/step, host enqueue "
              f"{(t1 - t0) / steps * 1e3:.3f} ms/step, {B / (ms / 1e3):.0f} array-fps per rank "
              f"(ideal {40300 * world:.0f})", flush=True)
        del frames, out, ac
        torch.cuda.empty_cache()

print("-- pipelined (ArrayCorrector.submit: front half of batch k under K3 of batch k-1)")
for world, B in [(1, 30), (2, 30), (4, 30), (8, 30), (8, 60)]:
    b0, c = camera_partition(N, world)[0]

    class Comm:
        rank = 0
        handle = h.value
    Comm.world = world
    frames = synthetic_batch(B, c, H, W, seed=1)
    out = torch.empty_like(frames)
    ac = ArrayCorrector(N, H, W, cam_begin=b0, cam_count=c, comm=Comm())
    for _ in range(5):
        ac.submit(frames, out)
    torch.cuda.synchronize()
    steps = 40
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(steps):
        ac.submit(frames, out)
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    ac.flush()
    ms = e0.elapsed_time(e1) / steps
    print(f"world {world} B {B} pipelined: gpu {ms:.3f} ms/step, host enqueue "
          f"{(t1 - t0) / steps * 1e3:.3f} ms/step, {B / (ms / 1e3):.0f} array-fps per rank "
          f"(ideal {40300 * world:.0f})", flush=True)
    del frames, out, ac
    torch.cuda.empty_cache()
