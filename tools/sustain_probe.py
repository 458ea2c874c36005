"""Burst vs sustained: a plain torch copy (the MEASURED_PEAKS hbm recipe) and
the config-5 K3 + tile call, each timed over 20 and over 400 back-to-back
reps, with SM / memory clocks, power and temperatures sampled (NVML) during
the long run. Explains why a leg timed late in a long bench reads slower
than the same call timed cold.

    python tools/sustain_probe.py [--split]   # --split: K3 alone, tile kernel alone
"""
import statistics
import sys
import threading

import numpy as np
import pynvml
import torch

sys.path.insert(0, ".")
from paper_1910_03517_b200 import _lib  # noqa: E402
from paper_1910_03517_b200.array import ArrayCorrector  # noqa: E402
from paper_1910_03517_b200.synth import synthetic_batch  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())


def sampled(fn):
    smp, stop = [], threading.Event()

    def run():
        while not stop.is_set():
            try:
                smp.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1e3,
                            pynvml.nvmlDeviceGetTemperature(h, pynvml.NVML_TEMPERATURE_GPU),
                            pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except pynvml.NVMLError:
                pass
            stop.wait(0.005)
    th = threading.Thread(target=run, daemon=True)
    th.start()
    r = fn()
    stop.set()
    th.join()
    if not smp:
        return r, {}
    cols = list(zip(*smp))
    reasons = 0
    for x in cols[4]:
        reasons |= x
    return r, {"sm": statistics.median(cols[0]), "mem": statistics.median(cols[1]),
               "w_max": max(cols[2]), "temp_max": max(cols[3]), "reasons": hex(reasons)}


def timed(call, reps):
    for _ in range(2):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


n = 1 << 30
a = torch.empty(n, dtype=torch.bfloat16, device="cuda").fill_(1)
b = torch.empty_like(a)
copy_bytes = 4 * n

N, H, W, B = 8, 1536, 2048, 30
frames = synthetic_batch(B, N, H, W, seed=1)
ac = ArrayCorrector(N, H, W)
res = ac.correct(frames)
gain, off = res.gain.contiguous(), res.offset.contiguous()
wins = [(bb, x, y) for bb in range(B) for (x, y) in ac.tile_windows(960)]
per = len(wins) // B
wd = torch.as_tensor(np.asarray(wins, np.int32), device="cuda")
fo = torch.as_tensor(np.arange(B + 1, dtype=np.int32) * per, device="cuda")
tiles = torch.empty((len(wins), 416, 416, 3), dtype=torch.uint8, device="cuda")
out = torch.empty_like(frames)
alg = B * (N * H * W * 6 + per * 416 * 416 * 3)


def k3k5():
    _lib.call("camx_correct_and_tile", frames.data_ptr(), out.data_ptr(), B, N, 0, H, W, 16,
              gain.data_ptr(), off.data_ptr(), wd.data_ptr(), fo.data_ptr(), len(wins), per, 960,
              416, tiles.data_ptr(), None)


def k3():
    _lib.call("camx_apply_array", frames.data_ptr(), out.data_ptr(), B, 0, N, N, 0, H, W, 16,
              gain.data_ptr(), off.data_ptr(), None)


def k5():
    _lib.call("camx_tiles", out.data_ptr(), N, H, W, wd.data_ptr(), len(wins), 960, 416,
              tiles.data_ptr(), None)


k3_bytes = B * N * H * W * 6
k5_bytes = B * per * 416 * 416 * 3
legs = [("torch copy 2 GiB", lambda: b.copy_(a), copy_bytes), ("K3 + tiles config5", k3k5, alg)]
if "--split" in sys.argv:
    legs = [("K3 alone", k3, k3_bytes), ("tiles alone (out bytes)", k5, k5_bytes)]
for rnd in range(2):
    for lbl, call, nb in legs:
        for reps in (20, 400 if nb != copy_bytes else 150):
            ms, clk = sampled(lambda: timed(call, reps))
            print(f"round {rnd} {lbl:20s} reps {reps:3d}: {ms:.4f} ms = {nb / ms / 1e6:7.1f} GB/s "
                  f"{clk}", flush=True)
