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
    ap.add_argument("--e2e-batch", type=int, default=8)
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of a CUDA graph")
    ap.add_argument("--no-hist", action="store_true",
                    help="skip the seam-band histograms (K1 means/moments only)")
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

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.005)

    def __enter__(self):
        if self.nv is not None:
            self._th = threading.Thread(target=self._run, daemon=True)
            self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._th is not None:
            self._th.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ CPU baseline

def cpu_reference_sample(frames_np, n_frames: int, threads: int):
    """The reference algorithm (numpy restatement in oracle/, fresh maps
    every frame: update_exposure per seam + apply_exposure per camera side)
    on host cores; returns seconds per array-frame."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import camarray_oracle as O
    n = frames_np.shape[1]
    S = n - 1

    def solve_one(args):
        b, s = args
        r = O.update_exposure(frames_np[b, s], frames_np[b, s + 1], None)
        return s, r

    times = []
    with ThreadPoolExecutor(threads) as ex:
        for i in range(n_frames):
            b = i % frames_np.shape[0]
            t0 = time.perf_counter()
            res = dict(ex.map(solve_one, [(b, s) for s in range(S)]))
            gain = O.np.stack([[res[s]["gl"], res[s]["gr"]] for s in range(S)])
            off = O.np.stack([[res[s]["ol"], res[s]["orr"]] for s in range(S)])
            O.apply_array(frames_np[b], gain, off, threads=threads)
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


def run_reference(args):
    """--impl reference: the reference CPU path, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np
    name = args.workload or "config2"
    n_cams, H, W, _, desc = WORKLOADS[name]
    from oracle import camarray_oracle as O
    frames = np.stack([O.synthetic_array(n_cams, H, W, seed=100 + t, objects=4)
                       for t in range(2)])
    threads = os.cpu_count() or 1
    times = cpu_reference_sample(frames, args.warmup + args.steps, threads)[args.warmup:]
    sec = sum(times) / len(times)
    mp = n_cams * H * W / 1e6
    val = mp / sec
    line = {
        "impl": "reference", "metric": "corrected megapixels/sec", "value": round(val, 3),
        "unit": "MP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (panorama + per-camera affine distortion)",
        "array_frames_per_sec": round(1.0 / sec, 4),
        "config": {"workload": f"{name}: {desc}", "step": "1 array-frame, STANDARD update + apply"},
        "cpu_baseline": {"value": round(val, 3), "unit": "MP/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} array-frames of {name} after {args.warmup} warm-up",
                         "cpu_model": cpu_model()},
        "e2e": {"value": round(val, 3), "unit": "MP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm

def run_camx(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1910_03517_b200.array import ArrayCorrector
    from paper_1910_03517_b200.dist import camera_partition, sharded_corrector
    from paper_1910_03517_b200.exposure import ExposureConfig, ExposureMode
    from paper_1910_03517_b200.synth import synthetic_batch

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
    name = args.workload or ("config3" if world > 1 else "config2")
    n_cams, H, W, B0, desc = WORKLOADS[name]
    B = args.batch or B0
    mode = ExposureMode(args.mode)
    cfg = ExposureConfig()
    wrap = name == "config4"
    if world > 1:
        ac = sharded_corrector(n_cams, H, W, cfg, mode, wrap=wrap, histograms=not args.no_hist)
        begin, count = camera_partition(n_cams, world)[rank]
    else:
        ac = ArrayCorrector(n_cams, H, W, cfg, mode, wrap=wrap, histograms=not args.no_hist)
        begin, count = 0, n_cams
    full = synthetic_batch(B, n_cams, H, W, seed=100)
    frames = full[:, begin:begin + count].contiguous()
    del full
    out = torch.empty_like(frames)
    stream = torch.cuda.Stream()
    px_per_frame = n_cams * H * W                      # whole-job pixels per array-frame

    def barrier():
        # drain this rank's GPU work first: the sharded path's own NCCL
        # all-gathers (camx's communicator, side stream) must not be in
        # flight while torch's communicator runs the barrier's collective
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    tiles_mode = name == "config5"
    tiles_buf = None
    if tiles_mode:
        n_tiles = len(ac.tile_windows(960)) * B
        tiles_buf = torch.empty((n_tiles, 416, 416, 3), dtype=torch.uint8, device="cuda")

    use_graph = not args.no_graph and world == 1 and not tiles_mode
    # N > 1 over NCCL: the front half (K1 -> all-gather -> K2) of batch k on a
    # side stream under K3 of batch k-1 (ArrayCorrector.submit)
    use_pipe = (world > 1 and getattr(ac, "comm", None) is not None and not tiles_mode
                and os.environ.get("CAMX_SHARD_PIPE", "1") != "0")

    def step():
        if tiles_mode:
            return ac.correct_and_tile(frames, out=out, tiles=tiles_buf, stream=stream)[0]
        if use_graph:  # CUDA graph replay of K1 -> K2 -> K3 (+ state carry)
            return ac.correct_graphed(frames, out)
        if use_pipe:
            return ac.submit(frames, out, stream=stream)
        return ac.correct(frames, out, stream=stream)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    barrier()

    # timed region: K steps, events on the launching stream, every camx
    # kernel launch counted
    n_launch = [0]
    from paper_1910_03517_b200 import _lib
    orig_call = _lib.call

    def traced_call(fn, *a):
        if fn in ("camx_correct_batch", "camx_correct_batch_tiles"):
            # K1 (x2 for OBJECT_REMOVAL with B > 1 and no previous frame) + K2 + K3
            # (+ tile fix-up)
            two_k1 = mode is ExposureMode.OBJECT_REMOVAL and a[3] > 1 and a[2] is None
            n_launch[0] += 3 if two_k1 else 2
            n_launch[0] += 1 if fn == "camx_correct_batch" else 2
        elif fn == "camx_correct_batch_sharded":  # K1 (x2) + K2 + K3 (+ NCCL, not ours)
            two_k1 = mode is ExposureMode.OBJECT_REMOVAL and a[3] > 1 and a[2] is None
            n_launch[0] += 4 if two_k1 else 3
        elif fn == "camx_correct_batch_sharded_step":
            if a[0] is not None:  # front half: K1 (x2 without a previous frame) + K2
                two_k1 = mode is ExposureMode.OBJECT_REMOVAL and a[2] > 1 and a[1] is None
                n_launch[0] += 3 if two_k1 else 2
            if a[21] is not None:  # back half: K3 of the previous batch
                n_launch[0] += 1
        elif fn.startswith("camx_"):
            n_launch[0] += 1
        orig_call(fn, *a)

    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    _lib.call = traced_call
    try:
        with ClockSampler(torch.cuda.current_device()) as clk:
            barrier()
            start.record(stream)
            with torch.cuda.stream(stream):
                for _ in range(args.steps):
                    res = step()
            stop.record(stream)
            stop.synchronize()
            barrier()
    finally:
        _lib.call = orig_call
    if use_pipe:  # drain the pipeline (outside the timed region)
        with torch.cuda.stream(stream):
            res = ac.flush(stream=stream) or res
        torch.cuda.synchronize()
    if use_graph:  # replays do not pass through _lib.call: same kernels as an eager step
        per_step = 3  # K1 (one launch: the captured tick has a previous frame), K2, K3
        n_launch[0] = per_step * args.steps

    # roofline leg: the dominant kernel (K3 apply) alone, same buffers and
    # maps as the last step, CUDA events on its stream around each launch
    # (config 5: the fused apply+tile kernel and its fix-up, whose
    # algorithmic bytes add the tile writes to K3's read + write)
    k3_ev = []
    k3_launch_bytes = 6 * B * count * H * W
    k3_name = "camx apply_tma_kernel (K3)"
    if tiles_mode:
        wins = sorted((b, x, y) for b in range(B) for (x, y) in ac.tile_windows(960))
        wins = sorted(wins, key=lambda w: w[0])
        per_b = np.bincount(np.asarray([w[0] for w in wins]), minlength=B)
        w_dev = torch.as_tensor(np.asarray(wins, dtype=np.int32).reshape(-1, 3), device="cuda")
        off_dev = torch.as_tensor(np.concatenate([[0], np.cumsum(per_b)]).astype(np.int32),
                                  device="cuda")
        k3_launch_bytes += tiles_buf.numel()
        k3_name = "camx apply_tma_kernel<fused tiles> + tile_fixup (K3+K5)"
    with torch.cuda.stream(stream):
        for _ in range(max(3, min(args.steps, 20))):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if tiles_mode:
                _lib.call("camx_correct_and_tile", frames.data_ptr(), out.data_ptr(), B, n_cams,
                          int(wrap), H, W, cfg.blocks, res.gain.data_ptr(),
                          res.offset.data_ptr(), w_dev.data_ptr(), off_dev.data_ptr(),
                          len(wins), int(per_b.max()), 960, 416, tiles_buf.data_ptr(),
                          stream.cuda_stream)
            else:
                _lib.call("camx_apply_array", frames.data_ptr(), out.data_ptr(), B, begin, count,
                          n_cams, int(wrap), H, W, cfg.blocks, res.gain.data_ptr(),
                          res.offset.data_ptr(), stream.cuda_stream)
            e1.record(stream)
            k3_ev.append((e0, e1))
    torch.cuda.synchronize()
    ms = start.elapsed_time(stop)
    k3_ms = sum(a.elapsed_time(b) for a, b in k3_ev) / len(k3_ev)
    k3_share = k3_ms * args.steps / ms
    if world > 1:
        tt = torch.tensor([ms, k3_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms, k3_ms = float(tt[0]), float(tt[1])
        k3_share = k3_ms * args.steps / ms
    ms_per_step = ms / args.steps
    mp_per_s = B * px_per_frame / 1e6 / (ms_per_step / 1e3)
    afps = B / (ms_per_step / 1e3)
    peak, peak_kind = peaks()
    achieved = k3_launch_bytes / (k3_ms / 1e3) / 1e9
    traffic = None
    tp = ROOT / "profiles" / "apply_traffic.json"
    if tp.exists():
        try:
            entries = json.loads(tp.read_text())
            entries = entries.get("entries", [entries])
            for d in entries:
                if d.get("workload") == name:
                    # DRAM bytes per algorithmic byte of the captured launch,
                    # scaled to this run's launch size (streaming kernel)
                    traffic = int(d["dram_bytes_per_launch"] / d["algorithmic_bytes_per_launch"]
                                  * k3_launch_bytes)
        except Exception:
            pass

    # e2e through the public host API (pinned host in -> pinned host out)
    e2e = None
    if not args.no_e2e and not tiles_mode:
        Be = min(args.e2e_batch, B)
        host_in = frames[:Be].cpu().pin_memory()
        host_out = torch.empty_like(host_in).pin_memory()
        ac.reset()
        for _ in range(max(1, min(args.warmup, 2))):
            ac.correct_host(host_in, host_out)
        torch.cuda.synchronize()
        e_steps = max(2, min(args.steps, 10))
        barrier()
        t0 = time.perf_counter()
        e_start = torch.cuda.Event(enable_timing=True)
        e_stop = torch.cuda.Event(enable_timing=True)
        e_start.record()
        last = None
        for _ in range(e_steps):  # a stream of batches: consecutive calls pipeline
            _, last = ac.correct_host(host_in, host_out, wait=False)
        torch.cuda.current_stream().wait_event(last)
        e_stop.record()
        e_stop.synchronize()
        e_ms = e_start.elapsed_time(e_stop)
        if world > 1:
            tt = torch.tensor([e_ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_ms = float(tt[0])
        wall = time.perf_counter() - t0
        e_ms_step = e_ms / e_steps
        # every rank copies its camera shard: whole-job bytes = world x this rank's
        # (shards are equal for the benchmark configs)
        e2e = {"value": round(Be * px_per_frame / 1e6 / (e_ms_step / 1e3), 2), "unit": "MP/s",
               "h2d_bytes_per_step": int(host_in.numel()) * world,
               "d2h_bytes_per_step": int(host_out.numel()) * world,
               "array_frames_per_sec": round(Be / (e_ms_step / 1e3), 2),
               "batch": Be, "steps": e_steps, "wall_s": round(wall, 3),
               "path": "ArrayCorrector.correct_host (pinned ring, 3 streams, batches pipelined)",
               "pcie_bytes_per_sec_each_way": round(host_in.numel() / (e_ms_step / 1e3) / 1e9, 2)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            fr = frames[:2].cpu().numpy()
            sample = 3 if H * W <= 4_000_000 else 2
            times = cpu_reference_sample(fr, sample + 1, threads)[1:]
            sec = sum(times) / len(times)
            mp_frame = n_cams * H * W / 1e6
            cpu = {"value": round(mp_frame / sec, 3), "unit": "MP/s", "cores": threads,
                   "kind": "port",
                   "sample": f"{sample} array-frames of {name} (numpy restatement of the "
                             f"reference: update_exposure per seam + apply_exposure per side, "
                             f"fresh maps, {threads} threads)",
                   "array_frames_per_sec": round(1.0 / sec, 4),
                   "cpu_model": cpu_model(), "nproc": threads}
            # SURVEY 8d variants: one thread, and steady state (cached maps)
            try:
                t1 = cpu_reference_sample(fr, 1, 1)
                g = res.gain[0].cpu().numpy()
                o = res.offset[0].cpu().numpy()
                tc = cpu_cached_apply_sample(fr, sample + 1, threads, g, o, wrap)[1:]
                tc1 = cpu_cached_apply_sample(fr, 2, 1, g, o, wrap)[1:]
                cpu["variants"] = {
                    "fresh_maps_all_threads_mp_s": cpu["value"],
                    "fresh_maps_1_thread_mp_s": round(mp_frame / t1[0], 3),
                    "cached_maps_all_threads_mp_s": round(mp_frame / (sum(tc) / len(tc)), 3),
                    "cached_maps_1_thread_mp_s": round(mp_frame / tc1[0], 3),
                }
            except Exception as e:  # pragma: no cover
                cpu["variants"] = {"failed": str(e)}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": "MP/s", "cores": 0, "kind": "port", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": "corrected megapixels/sec", "value": round(mp_per_s, 2), "unit": "MP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (on-device panorama + per-camera affine distortion + moving objects)",
            "array_frames_per_sec": round(afps, 2),
            "config": {"workload": f"{name}: {desc}", "batch": B, "mode": mode.value,
                       "histograms": not args.no_hist,
                       "tiles_per_step": (tiles_buf.shape[0] if tiles_mode else 0),
                       "cameras_per_gpu": count, "frame": f"{W}x{H}",
                       "step": ("K1 band stats" + ("" if args.no_hist else " + histograms") +
                                " + K2 seam solve + K3 apply per array-frame"),
                       "l2": "inputs larger than L2 (batch >> 126 MB)",
                       "parallelism": f"camera-shard{world}" if world > 1 else "single",
                       "launch": ("cuda-graph replay" if use_graph else
                                  "software-pipelined: K1 -> NCCL all-gather -> K2 of batch k on "
                                  "a side stream under K3 of batch k-1" if use_pipe else
                                  "eager (PDL-chained)")},
            "roofline": {"bound": "hbm", "kernel": k3_name,
                         "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "peak_kind": peak_kind, "k3_ms_per_launch": round(k3_ms, 4),
                         "k3_bytes_per_launch": k3_launch_bytes,
                         "k3_launches_timed": len(k3_ev),
                         "k3_share_of_step": round(k3_share, 4)},
            "clocks": clk.summary(),
            "e2e": e2e,
            "gpu_launches": n_launch[0],
            "cpu_baseline": cpu,
        }
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
