"""Config-2 step (30 frames, STANDARD, histograms): the CUDA-graph step
(K1 -> K2 -> K3) vs camx_correct_step_pipelined (K3 of batch k -> K1 -> K2 of
batch k+1, PDL-chained across calls), eager and graph-captured; results
checked against the sequential path."""
import ctypes

import torch

from paper_1910_03517_b200 import _lib, _dev
from paper_1910_03517_b200.array import ArrayCorrector
from paper_1910_03517_b200.exposure import ExposureConfig, ExposureMode, _MODE_CODE
from paper_1910_03517_b200.synth import synthetic_batch

N, H, W, B, K = 8, 1536, 2048, 30, 16
cfg = ExposureConfig()
frames = [synthetic_batch(B, N, H, W, seed=100 + i) for i in range(2)]
outs = [torch.empty_like(frames[0]) for _ in range(2)]
S = N - 1


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


ac = ArrayCorrector(N, H, W, cfg, histograms=True)
k = [0]


def graph_step():
    i = k[0] & 1
    ac.correct_graphed(frames[i], outs[i])
    k[0] += 1


t_graph = timeit(graph_step)

bufs = [dict(stats=torch.empty((B, N, 2, K, _lib.STAT_BYTES), dtype=torch.uint8, device="cuda"),
             hist=torch.empty((B, N, 2, K, 3, 256), dtype=torch.int32, device="cuda"),
             gain=torch.empty((B, S, 2, K, 3), dtype=torch.float64, device="cuda"),
             offset=torch.empty((B, S, 2, K, 3), dtype=torch.float64, device="cuda"),
             fit_ok=torch.empty((B, S, K), dtype=torch.uint8, device="cuda")) for _ in range(2)]
state = {"k": 0, "have_prev": False}


def pipe_step(stream=None):
    """apply batch k-1 (if any), stats+solve batch k."""
    kk = state["k"]
    cur, prv = bufs[kk & 1], bufs[(kk - 1) & 1]
    sh = _dev.stream_handle(stream or torch.cuda.current_stream())
    have_prev = kk > 0
    sc = _lib.SolveConfig(_MODE_CODE[ExposureMode.STANDARD], K, int(cfg.min_band_pixels),
                          float(cfg.sigma_min), float(cfg.alpha), float(cfg.min_valid_fraction),
                          int(have_prev), 0)
    pg = prv["gain"][B - 1].data_ptr() if have_prev else None
    po = prv["offset"][B - 1].data_ptr() if have_prev else None
    fi, fp = frames[kk & 1], frames[(kk - 1) & 1]
    _lib.call("camx_correct_step_pipelined",
              fp.data_ptr() if have_prev else None, outs[(kk - 1) & 1].data_ptr(),
              B if have_prev else 0, prv["gain"].data_ptr(), prv["offset"].data_ptr(),
              fi.data_ptr(), None, B, N, 0, H, W, cfg.band_width, cfg.t_diff, ctypes.byref(sc),
              pg, po, cur["stats"].data_ptr(), cur["hist"].data_ptr(), cur["gain"].data_ptr(),
              cur["offset"].data_ptr(), cur["fit_ok"].data_ptr(), sh)
    state["k"] = kk + 1


t_pipe = timeit(pipe_step)

# correctness: batches 0, 1, 2 through the pipeline == sequential correct()
state["k"] = 0
ref = ArrayCorrector(N, H, W, cfg, histograms=True)
want = []
for i in range(3):
    r = ref.correct(frames[i & 1])
    want.append((r.out.clone(), r.gain.clone()))
pipe_step()
pipe_step()
o0 = outs[0].clone()
g0 = bufs[0]["gain"].clone()
pipe_step()
o1 = outs[1].clone()
g1 = bufs[1]["gain"].clone()
torch.cuda.synchronize()
ok = (torch.equal(o0, want[0][0]) and torch.equal(g0, want[0][1]) and torch.equal(o1, want[1][0])
      and torch.equal(g1, want[1][1]))
print(f"graph step {t_graph * 1e3:.1f} us ({B / t_graph * 1e3:.0f} array-fps); pipelined step "
      f"{t_pipe * 1e3:.1f} us ({B / t_pipe * 1e3:.0f} array-fps); pipelined == sequential: {ok}",
      flush=True)
