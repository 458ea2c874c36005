"""Why does bench.py's config-5 roofline leg (K3 + tile kernel through
camx_correct_and_tile) sometimes read slower than tools/fused_probe.py on the
same call?  Builds the bench workload, then times the leg repeatedly and
variants of it in one process.

    python tools/leg_probe.py
"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

sys.argv = [sys.argv[0], "--workload", "config5"]
ap = bench.parse()
wl = bench.Workload("config5", bench.WORKLOADS["config5"][3], ap, 1, 0, torch).run(
    20, 3, torch.cuda.synchronize)
print(f"step {wl.ms / wl.steps:.4f} ms {wl.clocks}")
for r in range(4):
    wl.roofline_leg(20)
    print(f"leg run {r}: median {wl.k_ms:.4f} mean {wl.k_ms_mean:.4f} {wl.k_clocks}")
# same leg on a fresh side stream and on the default stream
for lbl, s in (("fresh stream", torch.cuda.Stream()), ("default stream", torch.cuda.default_stream())):
    wl.stream = s
    wl.roofline_leg(20)
    print(f"leg {lbl}: median {wl.k_ms:.4f} {wl.k_clocks}")
# fresh output buffer
wl.out = torch.empty_like(wl.out)
wl.roofline_leg(20)
print(f"leg fresh out: median {wl.k_ms:.4f}")
wl.tiles_buf = torch.empty_like(wl.tiles_buf)
wl.roofline_leg(20)
print(f"leg fresh tiles: median {wl.k_ms:.4f}")
wl.frames = wl.frames.clone()
wl.roofline_leg(20)
print(f"leg fresh frames: median {wl.k_ms:.4f}")
