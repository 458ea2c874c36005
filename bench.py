#!/usr/bin/env python
"""Benchmark: corrected megapixels/s (and array-frames/s) of the seam
exposure correction path on B200, with the HBM roofline of the dominant
kernel and the reference CPU path timed beside it.

  python bench.py [--gpus N --steps K --warmup W] [--workload config2]
  python bench.py --impl reference ...   (reference algorithm on host CPU)

One step = one pass of the hot path (K1 band stats -> K2 seam solve ->
K3 apply, STANDARD mode, fresh maps every array-frame) over a batch of
synthetic array-frames resident in HBM.  Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: (n_cams, H, W, default batch, description)
    "config1": (2, 480, 640, 64, "2 cameras 640x480 (reference CPU oracle config)"),
    "config2": (8, 1536, 2048, 30, "8 cameras x 2048x1536 (25.17 MP array), 30-frame batch"),
    "config3": (8, 1536, 2048, 30, "8-camera 25 MP array sharded one camera group per GPU"),
    "config4": (14, 2160, 3840, 64, "14-camera 360-degree 4K array (wrap seam), 64-frame batches"),
    "config5": (8, 1536, 2048, 30, "config 2 + 36 attention tiles/array-frame, 960 -> 416x416"),
    "config5m": (8, 1536, 2048, 30, "config 2 + motion counts fused into the apply pass + "
                 "attention tick (Scheduler, budget 4) + 960 -> 416x416 tiles of the chosen "
                 "windows"),
}
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["camx", "reference"], default="camx")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=None)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--mode", choices=["standard", "object_removal", "smoothing"],
                    default="standard")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-batch", type=int, default=4)
    ap.add_argument("--e2e-steps", type=int, default=60)
    ap.add_argument("--e2e-slots", type=int, default=4)
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of a CUDA graph")
    ap.add_argument("--no-hist", action="store_true",
                    help="skip the seam-band histograms (K1 means/moments only)")
    ap.add_argument("--no-secondary", action="store_true",
                    help="only the primary workload (default N=1 run also times config4 and "
                         "config5 and reports them under 'secondary')")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return float(d["hbm_gbs"]), "measured"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback"


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """NVML SM clock / throttle-reason sampler running during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.power_w = []
        self._stop = threading.Event()
        self._th = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _sample(self):
        nv = self.nv
        try:
            self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
            self.power_w.append(nv.nvmlDeviceGetPowerUsage(self.h) / 1e3)
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for bit, name in self.REASONS.items():
                if r & bit and name != "gpu_idle":
                    self.reasons.add(name)
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            self._stop.wait(0.002)

    def __enter__(self):
        if self.nv is not None:
            self._th = threading.Thread(target=self._run, daemon=True)
            self._th.start()
        return self

    def mark(self):
        """One synchronous sample (the GPU is busy with the timed work)."""
        if self.nv is not None:
            self._sample()

    def __exit__(self, *a):
        self._stop.set()
        if self._th is not None:
            self._th.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        d = {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
             "reasons": sorted(self.reasons), "samples": len(self.samples)}
        if self.power_w:
            d["power_w"] = round(statistics.median(self.power_w), 1)
        return d


# ------------------------------------------------------------------ CPU baseline

def cpu_reference_sample(frames_np, n_frames: int, threads: int, wrap: bool = False):
    """The reference algorithm (numpy restatement in oracle/, fresh maps
    every frame: update_exposure per seam + apply_exposure per camera side)
    on host cores; returns seconds per array-frame."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import camarray_oracle as O
    n = frames_np.shape[1]
    S = n if wrap else n - 1

    def solve_one(args):
        b, s = args
        r = O.update_exposure(frames_np[b, s], frames_np[b, (s + 1) % n], None)
        return s, r

    times = []
    with ThreadPoolExecutor(threads) as ex:
        for i in range(n_frames):
            b = i % frames_np.shape[0]
            t0 = time.perf_counter()
            res = dict(ex.map(solve_one, [(b, s) for s in range(S)]))
            gain = O.np.stack([[res[s]["gl"], res[s]["gr"]] for s in range(S)])
            off = O.np.stack([[res[s]["ol"], res[s]["orr"]] for s in range(S)])
            O.apply_array(frames_np[b], gain, off, wrap=wrap, threads=threads)
            times.append(time.perf_counter() - t0)
    return times


def cpu_cached_apply_sample(frames_np, n_frames: int, threads: int, gain, offset,
                            wrap: bool = False):
    """Steady state of the reference (maps unchanged: the _apply_arrays cache
    hits, exposure.py:363-381): apply_exposure per camera side with the f32
    tables built once; seconds per array-frame."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import camarray_oracle as O
    n, H, W = frames_np.shape[1:4]
    S = n if wrap else n - 1
    tabs = {(s, side): O.apply_tables(gain[s, side], offset[s, side], H, W,
                                      O.LEFT if side == 0 else O.RIGHT)
            for s in range(S) for side in (0, 1)}

    def one(args):
        res, c = args
        if c < S:
            O.apply_exposure_inplace(res[c], gain[c, 0], offset[c, 0], O.LEFT, tables=tabs[(c, 0)])
        sr = c - 1 if c >= 1 else (S - 1 if wrap else -1)
        if sr >= 0:
            O.apply_exposure_inplace(res[c], gain[sr, 1], offset[sr, 1], O.RIGHT,
                                     tables=tabs[(sr, 1)])

    times = []
    with ThreadPoolExecutor(threads) as ex:
        for i in range(n_frames):
            t0 = time.perf_counter()
            res = frames_np[i % frames_np.shape[0]].copy()  # apply_exposure copies its input
            list(ex.map(one, [(res, c) for c in range(n)]))
            times.append(time.perf_counter() - t0)
    return times


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def bench_frames(name, batch, device):
    """The benchmark's synthetic array-frames: synth.synthetic_batch, seed
    100 - device-independent bytes, so the GPU arm and the CPU reference arm
    correct the same frames (the reference arm samples the first two)."""
    from paper_1910_03517_b200.synth import synthetic_batch
    n_cams, H, W, _, _ = WORKLOADS[name]
    return synthetic_batch(batch, n_cams, H, W, seed=100, device=device)


DATA = ("synthetic (synth.synthetic_batch seed 100: shared panorama + per-camera affine "
        "distortion + moving objects; identical bytes in both arms)")


def run_reference(args):
    """--impl reference: the reference CPU path, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    # the GPU arm's workload at this N (config 3 = config 2's array sharded
    # over the ranks; the same frames - the CPU reference has no shards)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    name = args.workload or ("config3" if world > 1 else "config2")
    n_cams, H, W, _, desc = WORKLOADS[name]
    frames = bench_frames(name, 2, "cpu").numpy()
    threads = os.cpu_count() or 1
    wrap = name == "config4"
    times = cpu_reference_sample(frames, args.warmup + args.steps, threads, wrap)[args.warmup:]
    sec = sum(times) / len(times)
    mp = n_cams * H * W / 1e6
    val = mp / sec
    line = {
        "impl": "reference", "metric": "corrected megapixels/sec", "value": round(val, 3),
        "unit": "MP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": DATA,
        "array_frames_per_sec": round(1.0 / sec, 4),
        "config": {"workload": f"{name}: {desc}", "step": "1 array-frame, STANDARD update + apply",
                   "frames": "array-frames 0-1 of the GPU arm's batch, alternating"},
        "cpu_baseline": {"value": round(val, 3), "unit": "MP/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} array-frames of {name} after {args.warmup} warm-up",
                         "cpu_model": cpu_model()},
        "e2e": {"value": round(val, 3), "unit": "MP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm

def traffic_for(name, kernel_bytes, batch):
    """ncu DRAM bytes (read + write) of the dominant kernel(s) per launch,
    from a capture of this workload at this batch size (profiles/
    traffic.json), else None."""
    tp = ROOT / "profiles" / "traffic.json"
    if not tp.exists():
        return None
    try:
        for d in json.loads(tp.read_text()).get("entries", []):
            if d.get("workload") == name and int(d.get("batch", -1)) == batch and \
                    int(d.get("algorithmic_bytes_per_launch", -1)) == kernel_bytes:
                return int(d["dram_bytes_per_launch"])
    except Exception:
        pass
    return None


class Workload:
    """One benchmarked configuration on this rank: frames resident in HBM,
    a step function, and the dominant kernel's roofline leg."""

    def __init__(self, name, B, args, world, rank, torch):
        from paper_1910_03517_b200.array import ArrayCorrector
        from paper_1910_03517_b200.dist import camera_partition, sharded_corrector
        from paper_1910_03517_b200.exposure import ExposureConfig, ExposureMode
        self.name, self.B, self.world, self.torch = name, B, world, torch
        n_cams, H, W, _, self.desc = WORKLOADS[name]
        self.n_cams, self.H, self.W = n_cams, H, W
        self.mode = ExposureMode(args.mode)
        self.cfg = ExposureConfig()
        self.wrap = name == "config4"
        self.hist = not args.no_hist
        if world > 1:
            self.ac = sharded_corrector(n_cams, H, W, self.cfg, self.mode, wrap=self.wrap,
                                        histograms=self.hist)
            self.begin, self.count = camera_partition(n_cams, world)[rank]
        else:
            self.ac = ArrayCorrector(n_cams, H, W, self.cfg, self.mode, wrap=self.wrap,
                                     histograms=self.hist)
            self.begin, self.count = 0, n_cams
        full = bench_frames(name, B, "cuda")
        self.frames = full[:, self.begin:self.begin + self.count].contiguous()
        del full
        self.out = torch.empty_like(self.frames)
        self.stream = torch.cuda.Stream()
        self.tiles = name == "config5"
        self.attend = name == "config5m"
        if self.attend:
            from paper_1910_03517_b200.array import AttendPipeline
            from paper_1910_03517_b200.attention import Scheduler
            self.scheduler = Scheduler((n_cams * W, H))
            # the step re-submits the same resident batch unchanged, so the
            # next batch's frame 0 reads its previous frame in place
            self.pipe = AttendPipeline(self.ac, self.scheduler, retain_frames=True)
            self.frame_index = 0
            self.tiles_attended = 0
        self.tiles_buf = None
        if self.tiles:
            n_tiles = len(self.ac.tile_windows(960)) * B
            self.tiles_buf = torch.empty((n_tiles, 416, 416, 3), dtype=torch.uint8, device="cuda")
        self.use_graph = not args.no_graph and world == 1 and not self.tiles and not self.attend
        # N > 1 over NCCL: the front half (K1 -> all-gather -> K2) of batch k on
        # a side stream under K3 of batch k-1 (ArrayCorrector.submit)
        self.use_pipe = (world > 1 and getattr(self.ac, "comm", None) is not None
                         and not self.tiles and os.environ.get("CAMX_SHARD_PIPE", "1") != "0")

    def step(self):
        ac = self.ac
        if self.attend:
            # batch k: K1 -> K2 -> K3 + motion counts, counts D2H (async); batch
            # k-1: Scheduler per array-frame on the host under k's kernels,
            # then its tiles (AttendPipeline)
            r = self.pipe.submit(self.frames, frame_index=self.frame_index, stream=self.stream)
            self.frame_index += self.B
            if r is None:
                return None
            self.tiles_attended += r.tiles.shape[0]
            self.frames_attended = r.frame_index + self.B
            return r.result
        if self.tiles:
            return ac.correct_and_tile(self.frames, out=self.out, tiles=self.tiles_buf,
                                       stream=self.stream)[0]
        if self.use_graph:  # CUDA graph replay of K1 -> K2 -> K3 (+ state carry)
            return ac.correct_graphed(self.frames, self.out)
        if self.use_pipe:
            return ac.submit(self.frames, self.out, stream=self.stream)
        return ac.correct(self.frames, self.out, stream=self.stream)

    def launches_per_call(self, fn, a):
        """Our kernels behind one _lib.call (camx entry points launch several)."""
        from paper_1910_03517_b200.exposure import ExposureMode
        removal = self.mode is ExposureMode.OBJECT_REMOVAL
        if fn == "camx_correct_batch_motion":  # K1 (x2 as above) + K2 + K3 with motion counts
            return 4 if (removal and a[3] > 1 and a[2] is None) else 3
        if fn == "camx_tiles":
            return 1
        if fn in ("camx_correct_batch", "camx_correct_batch_tiles"):
            # K1 (x2 for OBJECT_REMOVAL with B > 1 and no previous frame) + K2 + K3
            # (+ the tile kernel)
            n = 3 if (removal and a[3] > 1 and a[2] is None) else 2
            return n + (1 if fn == "camx_correct_batch" else 2)
        if fn == "camx_correct_batch_sharded":  # K1 (x2) + K2 + K3 (+ NCCL, not ours)
            return 4 if (removal and a[3] > 1 and a[2] is None) else 3
        if fn == "camx_correct_batch_sharded_step":
            n = 0
            if a[0] is not None:  # front half: K1 (x2 without a previous frame) + K2
                n += 3 if (removal and a[2] > 1 and a[1] is None) else 2
            if a[21] is not None:  # back half: K3 of the previous batch
                n += 1
            return n
        return 1 if fn.startswith("camx_") else 0

    def run(self, steps, warmup, barrier):
        torch = self.torch
        from paper_1910_03517_b200 import _lib
        with torch.cuda.stream(self.stream):
            for _ in range(warmup):
                self.step()
        barrier()
        n_launch = [0]
        orig_call = _lib.call

        def traced_call(fn, *a):
            n_launch[0] += self.launches_per_call(fn, a)
            orig_call(fn, *a)

        start = torch.cuda.Event(enable_timing=True)
        stop = torch.cuda.Event(enable_timing=True)
        _lib.call = traced_call
        try:
            with ClockSampler(torch.cuda.current_device()) as clk:
                barrier()
                start.record(self.stream)
                with torch.cuda.stream(self.stream):
                    for _ in range(steps):
                        res = self.step()
                stop.record(self.stream)
                clk.mark()  # the queued steps are running: sample under load
                stop.synchronize()
                barrier()
        finally:
            _lib.call = orig_call
        if self.attend:  # the last batch's ticks and tiles (outside the timed region)
            with torch.cuda.stream(self.stream):
                self.pipe.flush(stream=self.stream)
            torch.cuda.synchronize()
        if self.use_pipe:  # drain the pipeline (outside the timed region)
            with torch.cuda.stream(self.stream):
                res = self.ac.flush(stream=self.stream) or res
            torch.cuda.synchronize()
        if self.use_graph:  # replays do not pass through _lib.call: same kernels as an eager step
            n_launch[0] = 3 * steps  # K1 (the captured tick has a previous frame), K2, K3
        self.res = res
        self.ms = start.elapsed_time(stop)
        self.steps = steps
        self.launches = n_launch[0]
        self.clocks = clk.summary()
        return self

    def roofline_leg(self, reps):
        """The dominant kernel alone (K3 apply; config 5: K3 + the tile
        kernel, against the one-pass bytes), same buffers and maps as the last step,
        CUDA events on its stream around each launch."""
        import numpy as np
        torch = self.torch
        from paper_1910_03517_b200 import _lib
        B, H, W = self.B, self.H, self.W
        res, cfg, stream = self.res, self.cfg, self.stream
        nbytes = 6 * B * self.count * H * W
        kname = "camx apply_tma_kernel (K3)"
        if self.tiles:
            wins = sorted(((b, x, y) for b in range(B) for (x, y) in self.ac.tile_windows(960)),
                          key=lambda w: w[0])
            per_b = np.bincount(np.asarray([w[0] for w in wins]), minlength=B)
            w_dev = torch.as_tensor(np.asarray(wins, dtype=np.int32).reshape(-1, 3), device="cuda")
            off_dev = torch.as_tensor(np.concatenate([[0], np.cumsum(per_b)]).astype(np.int32),
                                      device="cuda")
            nbytes += self.tiles_buf.numel()
            kname = "camx apply_tma_kernel + tiles_tma_kernel (K3 then K5; one-pass bytes)"
        if self.attend:
            # K1 + K2 + K3 with the in-pass motion counts: apply (6 B/px) + the
            # previous frame (3 B/px) + the seam bands K1 reads
            bands = 2 * (self.n_cams - 1) * cfg.band_width * H * 3
            nbytes = B * (9 * self.n_cams * H * W + bands)
            kname = "camx K1 + K2 + apply_tma_kernel<motion> (camx_correct_batch_motion)"
            motion_call = self.motion_call()
        def launch():
            if self.attend:
                motion_call()
            elif self.tiles:
                _lib.call("camx_correct_and_tile", self.frames.data_ptr(), self.out.data_ptr(),
                          B, self.n_cams, int(self.wrap), H, W, cfg.blocks,
                          res.gain.data_ptr(), res.offset.data_ptr(), w_dev.data_ptr(),
                          off_dev.data_ptr(), len(wins), int(per_b.max()), 960, 416,
                          self.tiles_buf.data_ptr(), stream.cuda_stream)
            else:
                _lib.call("camx_apply_array", self.frames.data_ptr(), self.out.data_ptr(), B,
                          self.begin, self.count, self.n_cams, int(self.wrap), H, W,
                          cfg.blocks, res.gain.data_ptr(), res.offset.data_ptr(),
                          stream.cuda_stream)

        # per-launch CUDA events on the launch stream, after warm-up; the
        # median launch - a mean would also count the rare host
        # stall that leaves the GPU idle between an event and its launch
        import statistics
        ev = []
        with torch.cuda.stream(stream), ClockSampler(torch.cuda.current_device()) as clk:
            for _ in range(2):
                launch()
            for _ in range(reps):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                launch()
                e1.record(stream)
                ev.append((e0, e1))
            clk.mark()
            torch.cuda.synchronize()
        self.k_clocks = clk.summary()
        times = [a.elapsed_time(b) for a, b in ev]
        self.k_ms = statistics.median(times)
        self.k_ms_mean = sum(times) / len(times)
        self.k_bytes = nbytes
        self.k_name = kname
        self.k_reps = len(times)

    def motion_call(self):
        """camx_correct_batch_motion on this workload's buffers (roofline leg):
        fresh maps, frame 0's previous frame = the batch's last frame."""
        import ctypes
        from paper_1910_03517_b200 import _lib
        from paper_1910_03517_b200.array import _MODE_CODE
        torch, ac, cfg, B = self.torch, self.ac, self.cfg, self.B
        buf = ac._buffers(B)
        counts = torch.empty((B, len(ac.tile_windows(960))), dtype=torch.int64, device="cuda")
        sc = _lib.SolveConfig(_MODE_CODE[ac.mode], ac.K, int(cfg.min_band_pixels),
                              float(cfg.sigma_min), float(cfg.alpha),
                              float(cfg.min_valid_fraction), 0, 0)
        prev = self.frames[B - 1]
        self._keep = (counts, sc)

        def call():
            _lib.call("camx_correct_batch_motion", self.frames.data_ptr(), self.out.data_ptr(),
                      None, B, self.n_cams, int(self.wrap), self.H, self.W, cfg.band_width,
                      cfg.t_diff, ctypes.byref(sc), None, None, buf["stats"].data_ptr(),
                      None if buf["hist"] is None else buf["hist"].data_ptr(),
                      buf["gain"].data_ptr(), buf["offset"].data_ptr(), buf["fit_ok"].data_ptr(),
                      prev.data_ptr(), 960, 20, counts.data_ptr(), self.stream.cuda_stream)
        return call

    def summary(self, peak, peak_kind):
        """Throughput + roofline fields (after max-over-ranks timing)."""
        ms_step = self.ms / self.steps
        px = self.B * self.n_cams * self.H * self.W
        achieved = self.k_bytes / (self.k_ms / 1e3) / 1e9
        return {
            "workload": f"{self.name}: {self.desc}",
            "value": round(px / 1e6 / (ms_step / 1e3), 2), "unit": "MP/s",
            "ms_per_step": round(ms_step, 4),
            "array_frames_per_sec": round(self.B / (ms_step / 1e3), 2),
            "roofline": {"bound": "hbm", "kernel": self.k_name, "achieved": round(achieved, 1),
                         "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic_for(self.name, self.k_bytes, self.B),
                         "peak_kind": peak_kind, "k_ms_per_launch": round(self.k_ms, 4),
                         "k_ms_stat": "median of the timed launches (mean "
                                      f"{getattr(self, 'k_ms_mean', self.k_ms):.4f})",
                         "k_bytes_per_launch": self.k_bytes, "k_launches_timed": self.k_reps,
                         "k_clocks": getattr(self, "k_clocks", None),
                         "k_share_of_step": round(self.k_ms * self.steps / self.ms, 4)},
        }

    def config(self):
        return {"workload": f"{self.name}: {self.desc}", "batch": self.B,
                "global_batch": self.B, "camera_frames_per_gpu": self.B * self.count,
                "mode": self.mode.value, "histograms": self.hist, "wrap": self.wrap,
                "tiles_per_step": (self.tiles_buf.shape[0] if self.tiles else
                                   round(self.tiles_attended /
                                         max(1, getattr(self, "frames_attended", 0)) * self.B, 2)
                                   if self.attend else 0),
                "cameras_per_gpu": self.count, "frame": f"{self.W}x{self.H}",
                "step": ("K1 band stats" + (" + histograms" if self.hist else "") +
                         " + K2 seam solve + K3 apply" +
                         (" + 36 attention tiles 960->416 from the corrected frames" if self.tiles else "") +
                         (" with the motion counts of the 36 tiling windows in the same pass, "
                          "counts D2H; the previous batch's attention.Scheduler ticks (budget 4) "
                          "on the host under it, then its chosen windows 960->416 "
                          "(array.AttendPipeline, retain_frames: the re-submitted batch is the previous "
                          "batch, read in place)" if self.attend else "") +
                         " per array-frame"),
                "l2": "inputs larger than L2 (batch >> 126 MB)",
                "parallelism": f"camera-shard{self.world}" if self.world > 1 else "single",
                "launch": ("cuda-graph replay" if self.use_graph else
                           "software-pipelined: K1 -> NCCL all-gather -> K2 of batch k on "
                           "a side stream under K3 of batch k-1" if self.use_pipe else
                           "eager (PDL-chained)")}

    def free(self):
        for k in ("frames", "out", "tiles_buf", "res", "ac", "_keep"):
            if hasattr(self, k):
                delattr(self, k)
        self.torch.cuda.empty_cache()


def e2e_ring(wl, Be, steps, warmup, barrier, world, slots=4):
    """End to end through the streaming API (ring.FrameRing): frames sit in
    the ring's pinned host slots (the producer - a decoder - writes them
    there; the bench fills the R slots once, outside the timed region), and
    every step publishes one slot: H2D on the copy stream -> K1, K2, K3 on
    the compute stream -> D2H of the corrected batch and its maps into the
    slot's pinned output, then get() + release() by the consumer.  Wall
    clock from the first publish to the last completed D2H."""
    torch = wl.torch
    from paper_1910_03517_b200.ring import FrameRing
    ac = wl.ac
    ac.reset()
    # 4 slots of 4 array-frames: the shape that saturates PCIe both ways
    # (tools/ring_probe.py: 48.0 GB/s each way = the measured H2D || D2H ceiling)
    ring = FrameRing(ac, slots=slots, batch=Be)
    host = wl.frames[: min(wl.B, slots * Be)].cpu()
    for j in range(slots):  # the producer's writes (decode) - not timed
        lo = (j * Be) % max(1, host.shape[0] - Be + 1)
        ring.acquire(block=False)[...] = host[lo:lo + Be].numpy()
        ring.publish(tag=j)
    for r in ring.drain():
        ring.release(r)

    def run(n):
        done = 0
        for k in range(n):
            ring.acquire(block=False)  # the slot still holds its frames
            ring.publish(tag=k)
            if ring.pending() >= slots:
                ring.release(ring.get())
                done += 1
        for r in ring.drain():
            ring.release(r)

    run(max(1, warmup))
    barrier()
    t0 = time.perf_counter()
    run(steps)
    ms = (time.perf_counter() - t0) * 1e3
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt[0])
    ms_step = ms / steps
    px = Be * wl.n_cams * wl.H * wl.W
    ceiling = pcie_ceiling(torch, ring)
    return {"value": round(px / 1e6 / (ms_step / 1e3), 2), "unit": "MP/s",
            "h2d_bytes_per_step": ring.h2d_bytes_per_batch * world,
            "d2h_bytes_per_step": ring.d2h_bytes_per_batch * world,
            "array_frames_per_sec": round(Be / (ms_step / 1e3), 2),
            "batch": Be, "steps": steps, "slots": slots,
            "path": "ring.FrameRing (pinned host slots -> H2D copy stream -> K1/K2/K3 compute "
                    "stream -> D2H copy-back stream; wall clock)",
            "pcie_bytes_per_sec_each_way": round(ring.h2d_bytes_per_batch / (ms_step / 1e3) / 1e9,
                                                 2),
            "pcie_ceiling_gbs_each_way": ceiling,
            "pcie_ceiling_how": "plain H2D || D2H copies of one slot on two streams, same run"}


def pcie_ceiling(torch, ring, reps=8):
    """Bidirectional PCIe ceiling: a slot's pinned input -> device and a
    device buffer -> the slot's pinned output at the same time (GB/s each)."""
    src, dst = ring._in[0], ring._out[0]
    a = torch.empty(src.shape, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def both():
        with torch.cuda.stream(s1):
            a.copy_(src, non_blocking=True)
        with torch.cuda.stream(s2):
            dst.copy_(b, non_blocking=True)
    both()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        both()
    torch.cuda.synchronize()
    sec = (time.perf_counter() - t0) / reps
    return round(src.numel() / sec / 1e9, 2)


def cpu_baseline_line(wl, args):
    threads = os.cpu_count() or 1
    fr = bench_frames(wl.name, 2, "cpu").numpy()  # = the GPU arm's array-frames 0-1
    sample = 3 if wl.H * wl.W <= 4_000_000 else 2
    times = cpu_reference_sample(fr, sample + 1, threads, wl.wrap)[1:]
    sec = sum(times) / len(times)
    mp_frame = wl.n_cams * wl.H * wl.W / 1e6
    cpu = {"value": round(mp_frame / sec, 3), "unit": "MP/s", "cores": threads, "kind": "port",
           "sample": f"{sample} array-frames of {wl.name} (the GPU arm's frames 0-1; numpy "
                     f"restatement of the reference: update_exposure per seam + apply_exposure "
                     f"per side, fresh maps, {threads} threads)",
           "array_frames_per_sec": round(1.0 / sec, 4), "cpu_model": cpu_model(),
           "nproc": threads}
    try:  # SURVEY 8d variants: one thread, and steady state (cached maps)
        t1 = cpu_reference_sample(fr, 1, 1, wl.wrap)
        g = wl.res.gain[0].cpu().numpy()
        o = wl.res.offset[0].cpu().numpy()
        tc = cpu_cached_apply_sample(fr, sample + 1, threads, g, o, wl.wrap)[1:]
        tc1 = cpu_cached_apply_sample(fr, 2, 1, g, o, wl.wrap)[1:]
        cpu["variants"] = {
            "fresh_maps_all_threads_mp_s": cpu["value"],
            "fresh_maps_1_thread_mp_s": round(mp_frame / t1[0], 3),
            "cached_maps_all_threads_mp_s": round(mp_frame / (sum(tc) / len(tc)), 3),
            "cached_maps_1_thread_mp_s": round(mp_frame / tc1[0], 3),
        }
    except Exception as e:  # pragma: no cover
        cpu["variants"] = {"failed": str(e)}
    return cpu


def main_workload(args, world):
    """(name, batch, weak) of the primary line.  Config 3 at N GPUs: the
    8-camera array sharded one camera group per GPU, 30 N array-frames per
    step, so every GPU corrects the same 240 camera-frames per step as the
    single GPU does (weak scaling; --batch 30 gives the fixed batch)."""
    name = args.workload or ("config3" if world > 1 else "config2")
    weak = args.batch is None and name == "config3"
    B = args.batch or WORKLOADS[name][3] * (world if weak else 1)
    return name, B, weak


def run_camx(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if world > 1:
        # NCCL over NVLink/NVSwitch; CAMX_DIST_BACKEND=gloo exercises the same
        # code path with several ranks on one GPU (tests only)
        backend = os.environ.get("CAMX_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)

    def barrier():
        # drain this rank's GPU work first: the sharded path's own NCCL
        # all-gathers (camx's communicator, side stream) must not be in
        # flight while torch's communicator runs the barrier's collective
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_ranks(*vals):
        if world == 1:
            return vals
        tt = torch.tensor(vals, device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return tuple(float(v) for v in tt)

    peak, peak_kind = peaks()
    name, B, weak = main_workload(args, world)
    wl = Workload(name, B, args, world, rank, torch).run(args.steps, args.warmup, barrier)
    wl.roofline_leg(max(3, min(args.steps, 20)))
    wl.ms, wl.k_ms = max_ranks(wl.ms, wl.k_ms)
    main = wl.summary(peak, peak_kind)

    line_cfg = wl.config()
    clocks, launches = wl.clocks, wl.launches

    # the other single-GPU workloads BASELINE.json names, each timed and
    # rooflined the same way (same steps / warm-up, own clocks); before the
    # e2e and CPU legs, whose host-heavy phases were measured to slow the GPU
    # legs that follow them
    secondary = []
    if world == 1 and args.workload is None and not args.no_secondary:
        for nm in ("config5", "config5m", "config4"):  # the long, hot 4K run last
            w2 = Workload(nm, WORKLOADS[nm][3], args, world, rank, torch).run(
                args.steps, args.warmup, barrier)
            w2.roofline_leg(max(3, min(args.steps, 20)))
            d = w2.summary(peak, peak_kind)
            d.update(config=w2.config(), clocks=w2.clocks, gpu_launches=w2.launches,
                     steps=args.steps, warmup=args.warmup)
            secondary.append(d)
            w2.free()

    e2e = None
    if not args.no_e2e and not wl.tiles:
        e2e = e2e_ring(wl, min(args.e2e_batch, B), max(2, args.e2e_steps), args.warmup,
                       barrier, world, args.e2e_slots)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_line(wl, args)
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": "MP/s", "cores": 0, "kind": "port",
                   "sample": f"failed: {e}"}
    wl.free()

    if rank == 0:
        line = {
            "metric": "corrected megapixels/sec", "value": main["value"], "unit": "MP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": main["ms_per_step"], "higher_is_better": True,
            "scaling": "weak" if weak and world > 1 else "strong", "vs_baseline": None,
            "dtype": "u8", "data": DATA,
            "array_frames_per_sec": main["array_frames_per_sec"],
            "config": line_cfg,
            "roofline": main["roofline"],
            "clocks": clocks,
            "e2e": e2e,
            "gpu_launches": launches,
            "cpu_baseline": cpu,
        }
        if secondary:
            line["secondary"] = secondary
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_camx(args)


if __name__ == "__main__":
    sys.exit(main())
