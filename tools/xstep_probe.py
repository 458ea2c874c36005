"""Config 2: does running K1 of the NEXT batch concurrently with K2 + K3 of
the current one (two streams, captured in one CUDA graph; double-buffered
records) shorten the per-batch step vs the sequential K1 -> K2 -> K3 graph?
Separate launches (camx_band_stats, camx_seam_solve, camx_apply_array),
STANDARD mode, histograms on.

    python tools/xstep_probe.py
"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1910_03517_b200 import _lib  # noqa: E402

N, H, W, B, K, BW = 8, 1536, 2048, 30, 16, 32
frames = bench.bench_frames("config2", B, "cuda")
out = torch.empty_like(frames)
R = _lib.STAT_BYTES
stats = [torch.empty((B, N, 2, K, R), dtype=torch.uint8, device="cuda") for _ in range(2)]
hist = [torch.empty((B, N, 2, K, 3, 256), dtype=torch.int32, device="cuda") for _ in range(2)]
gain = torch.empty((B, N - 1, 2, K, 3), dtype=torch.float64, device="cuda")
off = torch.empty_like(gain)
ok = torch.empty((B, N - 1, K), dtype=torch.uint8, device="cuda")
sc = _lib.SolveConfig(0, K, 64, 1e-3, 0.05, 0.5, 0, 0)


def k1(i, s):
    _lib.call("camx_band_stats", frames.data_ptr(), None, None, B * N, H, W, BW, K, 20,
              stats[i].data_ptr(), hist[i].data_ptr(), s.cuda_stream)


def k2k3(i, s):
    _lib.call("camx_seam_solve", stats[i].data_ptr(), B, N, 0, ctypes.byref(sc), None, None,
              gain.data_ptr(), off.data_ptr(), ok.data_ptr(), s.cuda_stream)
    _lib.call("camx_apply_array", frames.data_ptr(), out.data_ptr(), B, 0, N, N, 0, H, W, K,
              gain.data_ptr(), off.data_ptr(), s.cuda_stream)


main, side = torch.cuda.Stream(), torch.cuda.Stream()


def seq_step():
    k1(0, main)
    k2k3(0, main)


def pipe_step(i):
    # K1 of the next batch on the side stream while K2 + K3 of this one run
    ev = torch.cuda.Event()
    ev.record(main)
    side.wait_event(ev)
    k1(1 - i, side)
    k2k3(i, main)
    ev2 = torch.cuda.Event()
    ev2.record(side)
    main.wait_event(ev2)


def graph_of(fn):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(main):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=main):
            fn()
    return g


def timed(replay, steps=60):
    for _ in range(5):
        replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(steps):
        replay()
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


gs = graph_of(seq_step)
g0 = graph_of(lambda: pipe_step(0))
g1 = graph_of(lambda: pipe_step(1))
flip = [0]


def pipe_replay():
    (g0 if flip[0] == 0 else g1).replay()
    flip[0] ^= 1


for r in range(3):
    with torch.cuda.stream(main):
        t_seq = timed(gs.replay)
        t_pipe = timed(pipe_replay)
    print(f"run {r}: sequential {t_seq * 1e3:.1f} us, K1(next) || K2+K3 {t_pipe * 1e3:.1f} us "
          f"per 30-frame step")
