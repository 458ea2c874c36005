"""Host cost of one pipelined sharded step (ArrayCorrector.submit) at
N = 8 on one GPU (one-rank NCCL stand-in): wall time of 40 submits with no
sync (host enqueue rate) vs the GPU time of the same 40 steps."""
import ctypes
import time
import torch
import sys
sys.path.insert(0, ".")
from paper_1910_03517_b200 import _lib
from paper_1910_03517_b200.array import ArrayCorrector
from paper_1910_03517_b200.dist import camera_partition
from paper_1910_03517_b200.synth import synthetic_batch

uid = torch.zeros(128, dtype=torch.uint8)
_lib.call("camx_comm_unique_id", uid.data_ptr())
h = ctypes.c_void_p()
_lib.call("camx_comm_init", ctypes.byref(h), uid.data_ptr(), 1, 0)
N, H, W, B = 8, 1536, 2048, 30
for world in (4, 8):
    b0, c = camera_partition(N, world)[0]
    frames = synthetic_batch(B, c, H, W, seed=1)
    out = torch.empty_like(frames)

    class Comm:
        rank = 0
        handle = h.value
    Comm.world = world
    ac = ArrayCorrector(N, H, W, cam_begin=b0, cam_count=c, comm=Comm())
    for _ in range(5):
        ac.submit(frames, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(40):
        ac.submit(frames, out)
    t_host = (time.perf_counter() - t0) / 40 * 1e6
    e1.record()
    torch.cuda.synchronize()
    t_gpu = e0.elapsed_time(e1) / 40 * 1e3
    print(f"world {world}: host enqueue {t_host:.1f} us per submit, GPU {t_gpu:.1f} us per step")
    ac.flush()
