"""Config 5m (the attention tick, bench.py's AttendPipeline step): is the
step GPU- or host-bound?  Host wall time per submit() with no
synchronisation (the enqueue + the previous batch's Scheduler ticks) vs the
GPU's time per step (CUDA events), and the GPU time of the copies submit()
makes into its result slot.

    python tools/attend_probe.py [config5m|config5|config2] [--profile]
"""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

name = next((a for a in sys.argv[1:] if a.startswith("config")), "config5m")
prof = "--profile" in sys.argv[1:]
split = "--split" in sys.argv[1:]
sys.argv = [sys.argv[0], "--workload", name]
ap = bench.parse()
wl = bench.Workload(name, bench.WORKLOADS[name][3], ap, 1, 0, torch).run(20, 3,
                                                                       torch.cuda.synchronize)
print(f"bench step {wl.ms / wl.steps:.4f} ms (GPU events)")
s = wl.stream
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    host = []
    for _ in range(20):
        h0 = time.perf_counter()
        wl.step()
        host.append(time.perf_counter() - h0)
    e1.record(s)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / 20
    print(f"rep {rep}: host per submit {sum(host) / len(host) * 1e3:.3f} ms (max "
          f"{max(host) * 1e3:.3f}), wall per step {wall * 1e3:.3f} ms, GPU per step "
          f"{e0.elapsed_time(e1) / 20:.4f} ms", flush=True)
if name != "config5m":
    sys.exit(0)
if split:  # the pieces of one step, each timed alone on the step's stream
    ac, pipe = wl.ac, wl.pipe
    sl = pipe._slot(30, 0)

    def t_of(fn, n=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(n):
            fn()
        b.record(s)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n * 1e3
    with torch.cuda.stream(s):
        print(f"correct_with_motion into the slot: {t_of(lambda: ac.correct_with_motion(wl.frames, sl['out'], size=960, stream=s, _bufs=sl)):.1f} us")
        print(f"  (of it: the previous-frame copy {t_of(lambda: ac._motion_prev.copy_(wl.frames[29], non_blocking=True)):.1f} us)")
        cnt_h = torch.empty((30, 36), dtype=torch.int64, pin_memory=True)

        def with_d2h():
            _, c, _ = ac.correct_with_motion(wl.frames, sl["out"], size=960, stream=s, _bufs=sl)
            cnt_h.copy_(c, non_blocking=True)
        print(f"  + the counts D2H: {t_of(with_d2h):.1f} us")
        import numpy as np
        wins = torch.as_tensor(np.asarray([(b, 960 * (b % 16), 0) for b in range(30)
                                           for _ in range(4)], np.int32), device="cuda")
        tiles = torch.empty((120, 416, 416, 3), dtype=torch.uint8, device="cuda")
        from paper_1910_03517_b200 import _lib

        def with_tiles():
            with_d2h()
            _lib.call("camx_tiles", sl["out"].data_ptr(), 8, 1536, 2048, wins.data_ptr(), 120,
                      960, 416, tiles.data_ptr(), s.cuda_stream)
        print(f"  + 120 tiles: {t_of(with_tiles):.1f} us")
        print(f"full submit (steady state): {t_of(lambda: pipe.submit(wl.frames, frame_index=0, stream=s)):.1f} us")
# the slot copies alone (maps, stats, histograms of one 30-frame batch)
ac = wl.ac
res = ac._buffers(30)
sl = wl.pipe._slot(30, 0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    e0.record(s)
    for _ in range(20):
        sl["stats"].copy_(res["stats"].view_as(sl["stats"]), non_blocking=True)
        if sl["hist"] is not None:
            sl["hist"].copy_(res["hist"].view_as(sl["hist"]), non_blocking=True)
    e1.record(s)
torch.cuda.synchronize()
print(f"stats + histogram slot copies: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per batch")

if prof:
    import cProfile
    import pstats
    pr = cProfile.Profile()
    torch.cuda.synchronize()
    pr.enable()
    for _ in range(20):
        wl.step()
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
