"""Sustained A/B of K3 between builds of libcamx.so: the libraries take turns
running `chunk` back-to-back camx_apply_array launches (config-2 geometry,
batch 30) for `rounds` rounds, so both see the same power / clock state once
the GPU sits at its power cap.  One event pair per chunk; prints ms per launch.

    python tools/ab_sustain.py variants/libcamx_old.so variants/libcamx_new.so [--rounds 12]
"""
import argparse
import ctypes
import statistics

import torch

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--batch", type=int, default=30)
ap.add_argument("--chunk", type=int, default=150)
ap.add_argument("--rounds", type=int, default=12)
a = ap.parse_args()
N, H, W, K = 8, 1536, 2048, 16
B = a.batch
P, I = ctypes.c_void_p, ctypes.c_int32
frames = torch.randint(0, 256, (B, N, H, W, 3), dtype=torch.uint8, device="cuda")
out = torch.empty_like(frames)
g = torch.rand((B, N - 1, 2, K, 3), dtype=torch.float64, device="cuda") * 1.5 + 0.5
o = torch.rand((B, N - 1, 2, K, 3), dtype=torch.float64, device="cuda") * 80 - 40
libs = []
for path in a.libs:
    lib = ctypes.CDLL(path)
    fn = lib.camx_apply_array
    fn.argtypes = [P, P, I, I, I, I, I, I, I, I, P, P, P]
    fn.restype = ctypes.c_int
    libs.append((path, fn))
s = torch.cuda.current_stream()
res = {p: [] for p, _ in libs}
for rnd in range(a.rounds):
    for path, fn in (libs if rnd % 2 == 0 else libs[::-1]):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.chunk):
            fn(frames.data_ptr(), out.data_ptr(), B, 0, N, N, 0, H, W, K, g.data_ptr(),
               o.data_ptr(), s.cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        res[path].append(e0.elapsed_time(e1) / a.chunk)
    print(f"round {rnd}: " + "  ".join(f"{p.split('/')[-1]} {res[p][-1]:.4f}" for p, _ in libs),
          flush=True)
for path, ts in res.items():
    print(f"{path}: median {statistics.median(ts):.4f} ms (rounds 4+: "
          f"{statistics.median(ts[4:]):.4f})")
