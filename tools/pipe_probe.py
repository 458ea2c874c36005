"""Probe: does overlapping K1+K2 of batch i+1 (side stream) with K3 of batch
i (main stream) shorten the config-2 step?  Prints ms per 30-frame batch for
the plain eager path, the graph path and the cross-batch pipelined path."""
import torch

from paper_1910_03517_b200 import _dev
from paper_1910_03517_b200.array import ArrayCorrector
from paper_1910_03517_b200.synth import synthetic_batch

N, H, W, B, STEPS = 8, 1536, 2048, 30, 40
frames = synthetic_batch(B, N, H, W, seed=1)
out = torch.empty_like(frames)


def timeit(fn, steps=STEPS, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


ac = ArrayCorrector(N, H, W)
print("eager   ms/step", round(timeit(lambda: ac.correct(frames, out)), 4))
ac2 = ArrayCorrector(N, H, W)
print("graph   ms/step", round(timeit(lambda: ac2.correct_graphed(frames, out)), 4))

ac3 = ArrayCorrector(N, H, W)
ac3.fused = False
b0 = ac3._buffers(B)
bufs = [b0] + [{k: (v.clone() if v is not None else None) for k, v in b0.items()}
               for _ in range(2)]
main = torch.cuda.current_stream()
side = torch.cuda.Stream()
state = {"k": 0, "ev": None, "k3": {}}


def pipelined():
    # step k: K1+K2 of batch k into bufs[k % 3] (side), K3 of batch k-1 from
    # bufs[(k-1) % 3] (main); K2 of step k overwrites what K3 of step k-3
    # read, so the side stream waits for that K3's event
    k = state["k"]
    cur = bufs[k % 3]
    prev = bufs[(k - 1) % 3]
    old = state["k3"].pop(k - 3 + 1, None)  # K3 of step k-2 read bufs[(k-3) % 3]
    if old is not None:
        side.wait_event(old)
    pm = (prev["gain"][B - 1], prev["offset"][B - 1]) if k > 0 else None
    ac3._stats_solve(frames, cur, 0, B, _dev.stream_handle(side), pm, None)
    ev = torch.cuda.Event()
    ev.record(side)
    if state["ev"] is not None:
        main.wait_event(state["ev"])
        ac3._apply(frames, out, prev, 0, B, _dev.stream_handle(main))
        e3 = torch.cuda.Event()
        e3.record(main)
        state["k3"][k] = e3
    state["ev"] = ev
    state["k"] = k + 1


print("pipe    ms/step", round(timeit(pipelined), 4))
