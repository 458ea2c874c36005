"""Where the N=8 sharded step loses time (one GPU, stand-in one-rank comm):
K3 alone on one camera vs the pipelined submit() step, at B = 30 (WEAK=1: B = 30 N)."""
import ctypes
import os
import sys

import torch

from paper_1910_03517_b200 import _lib
from paper_1910_03517_b200.array import ArrayCorrector
from paper_1910_03517_b200.dist import camera_partition
from paper_1910_03517_b200.synth import synthetic_batch

uid = torch.zeros(128, dtype=torch.uint8)
_lib.call("camx_comm_unique_id", uid.data_ptr())
h = ctypes.c_void_p()
_lib.call("camx_comm_init", ctypes.byref(h), uid.data_ptr(), 1, 0)
N, H, W, K = 8, 1536, 2048, 16
B = int(sys.argv[1]) if len(sys.argv) > 1 else 30


def timeit(fn, steps=40):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


B0 = B
for world in (1, 2, 4, 8):
    # WEAK=1: 30 N array-frames per step (bench.py config 3), else a fixed batch
    B = B0 * world if os.environ.get("WEAK") else B0
    b0, c = camera_partition(N, world)[0]
    frames = synthetic_batch(B, c, H, W, seed=1)
    out = torch.empty_like(frames)
    g = torch.ones((B, N - 1, 2, K, 3), dtype=torch.float64, device="cuda") * 1.1
    o = torch.ones((B, N - 1, 2, K, 3), dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    k3 = timeit(lambda: _lib.call("camx_apply_array", frames.data_ptr(), out.data_ptr(), B, b0, c,
                                  N, 0, H, W, K, g.data_ptr(), o.data_ptr(), s))

    class Comm:
        rank = 0
        handle = h.value
    Comm.world = world
    ac = ArrayCorrector(N, H, W, cam_begin=b0, cam_count=c, comm=Comm())
    step = timeit(lambda: ac.submit(frames, out))
    ac.flush()
    ac2 = ArrayCorrector(N, H, W, cam_begin=b0, cam_count=c, comm=Comm())
    seq = timeit(lambda: ac2.correct(frames, out))
    byt = 2 * frames.numel()
    print(f"world {world} B {B}: K3 alone {k3 * 1e3:.1f} us ({byt / k3 / 1e6:.0f} GB/s), "
          f"pipelined step {step * 1e3:.1f} us, unpipelined {seq * 1e3:.1f} us; "
          f"whole-job array-fps {B / (step / 1e3):.0f} (every rank holds 1/N of each "
          f"array-frame) = {B / (step / 1e3) / (world * 40700):.1%} of N x 40.7K", flush=True)
    del frames, out, ac, ac2
    torch.cuda.empty_cache()
