"""Bidirectional PCIe with a write-combined pinned H2D source vs a default
pinned one (cudaHostAlloc flags), one FrameRing slot's size."""
import ctypes
import time

import numpy as np
import torch

rt = ctypes.CDLL("/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/cuda_runtime/lib/"
                 "libcudart.so.12")
nbytes = 4 * 8 * 1536 * 2048 * 3
torch.cuda.init()


def host_alloc(flags):
    p = ctypes.c_void_p()
    assert rt.cudaHostAlloc(ctypes.byref(p), ctypes.c_size_t(nbytes), ctypes.c_uint(flags)) == 0
    arr = np.ctypeslib.as_array((ctypes.c_uint8 * nbytes).from_address(p.value))
    return torch.from_numpy(arr), p


dev_a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
dev_b = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
out_h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, flags in (("default", 0), ("write-combined", 4), ("portable", 1)):
    src, _ = host_alloc(flags)
    src.fill_(7)
    print(name, "pinned:", src.is_pinned())

    def both():
        with torch.cuda.stream(s1):
            dev_a.copy_(src, non_blocking=True)
        with torch.cuda.stream(s2):
            out_h.copy_(dev_b, non_blocking=True)

    def h2d():
        with torch.cuda.stream(s1):
            dev_a.copy_(src, non_blocking=True)

    for fn, lbl in ((h2d, "H2D alone"), (both, "H2D || D2H")):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 10
        print(f"  {lbl}: {nbytes / dt / 1e9:.1f} GB/s")
