"""A/B timing of the K3 apply kernel between two builds of libcamx.so.

    python tools/ab_k3.py LIB_A LIB_B [--batch 8] [--reps 20]
Both libraries are driven through camx_apply_array with identical buffers
(config-2 geometry); CUDA events around each launch; prints GB/s."""
import argparse
import ctypes

import torch

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--reps", type=int, default=20)
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
bytes_ = 6 * B * N * H * W
res = {p: [] for p, _ in libs}
for rnd in range(3):
    for path, fn in libs:
        for _ in range(3):
            fn(frames.data_ptr(), out.data_ptr(), B, 0, N, N, 0, H, W, K, g.data_ptr(), o.data_ptr(), s.cuda_stream)
        torch.cuda.synchronize()
        for _ in range(a.reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            st = fn(frames.data_ptr(), out.data_ptr(), B, 0, N, N, 0, H, W, K, g.data_ptr(), o.data_ptr(), s.cuda_stream)
            e1.record()
            assert st == 0, st
            torch.cuda.synchronize()
            res[path].append(e0.elapsed_time(e1))
for path, ts in res.items():
    ts = sorted(ts)
    med = ts[len(ts) // 2]
    print(f"{path}: median {med*1e3:.1f} us  min {ts[0]*1e3:.1f} us  -> {bytes_/med/1e6:.1f} GB/s (min-time {bytes_/ts[0]/1e6:.1f})")
