"""Batched, device-resident array correction: the production path.

`ArrayCorrector` runs the whole seam pipeline for a batch of array-frames
(B array-frames x N cameras, uint8 (B, N, H, W, 3) in HBM) with three
kernel launches and no host round trip:

  K1 camx_band_stats  - both seam bands of every image, exact integer
                         moments (+ optional histograms; + fused in-band
                         mask_diff for OBJECT_REMOVAL)
  K2 camx_seam_solve  - update_exposure for every seam, batch as a tick loop
  K3 camx_apply_array - both seam corrections of every camera in one pass

No reference driver exists for a whole array: the semantics are
update_exposure per seam (exposure.py:245-344) followed by apply_exposure of
the seam's LEFT map on camera s and RIGHT map on camera s+1
(exposure.py:385-401).  Maps stay on the device; the previous batch's last
maps (and, for OBJECT_REMOVAL, its last frame) seed the next batch.

`correct_host` is the end-to-end entry point from pinned host memory: a
3-slot device ring with H2D, compute and D2H on separate streams so the
PCIe copies of chunk i+1 / i-1 overlap the kernels of chunk i.  The
streaming frame source with library-owned pinned slots and a producer /
consumer API is ring.FrameRing.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .exposure import (ExposureConfig, ExposureMap, ExposureMode, SeamMaps, Side, _MODE_CODE,
                       block_bounds)


@dataclass
class CorrectResult:
    out: object            # uint8 (B, N, H, W, 3) CUDA tensor
    gain: object           # float64 (B, S, 2, K, 3)
    offset: object         # float64 (B, S, 2, K, 3)
    fit_ok: object         # uint8 (B, S, K)
    stats: object          # uint8 (B, N, 2, K, 112) camx_band_stat records
    hist: object | None    # int32 (B, N, 2, K, 3, 256) (uint32 counts) or None


class _LocalComm:
    """The whole array on one GPU: no communicator (world 1)."""

    world, rank, handle = 1, 0, None


class ArrayCorrector:
    """Seam exposure correction of an N-camera array on one GPU."""

    def __init__(self, n_cams: int, height: int, width: int,
                 cfg: ExposureConfig = ExposureConfig(),
                 mode: ExposureMode = ExposureMode.STANDARD, *, wrap: bool = False,
                 histograms: bool = False, cam_begin: int = 0, cam_count: int | None = None,
                 exchange=None, comm=None):
        """cam_begin/cam_count: the cameras this GPU owns (default all).  A
        camera shard needs the other ranks' seam statistics, either through
        `comm` (dist.NcclComm: camx's own NCCL all-gather inside one
        camx_correct_batch_sharded call per batch) or `exchange(stats_local)
        -> stats_full` assembling the (B, n_cams, 2, K) records in Python
        (any torch.distributed backend, e.g. gloo)."""
        if n_cams < 1:
            raise ValueError("need at least one camera")
        if wrap and n_cams < 2:
            raise ValueError("a wrapped (360 degree) array needs two cameras")
        if not isinstance(mode, ExposureMode):
            raise ValueError(f"unknown exposure mode {mode!r}")
        if cfg.band_width > width // 2:
            raise ValueError(f"band width {cfg.band_width} exceeds half frame width {width // 2}")
        block_bounds(height, cfg.blocks)
        cam_count = n_cams - cam_begin if cam_count is None else cam_count
        if cam_begin < 0 or cam_count < 1 or cam_begin + cam_count > n_cams:
            raise ValueError("camera shard outside the array")
        if cam_count != n_cams and exchange is None and comm is None:
            raise ValueError("a camera shard needs a stats exchange")
        if comm is not None:
            from .dist import camera_partition
            if camera_partition(n_cams, comm.world)[comm.rank] != (cam_begin, cam_count):
                raise ValueError("camera shard does not match the communicator's rank")
        self.cam_begin, self.cam_count, self.exchange = cam_begin, cam_count, exchange
        self.comm = comm
        self.n_cams, self.height, self.width = n_cams, height, width
        self.cfg, self.mode, self.wrap = cfg, mode, bool(wrap)
        self.histograms = histograms
        self.S = n_cams if wrap else n_cams - 1
        self.K = cfg.blocks
        self._bufs: dict = {}
        self._prev_maps = None     # (gain, offset) device [S][2][K][3]
        self._prev_frame = None    # device (N, H, W, 3), OBJECT_REMOVAL only
        self._motion_prev = None   # device (N, H, W, 3): last frame of correct_with_motion
        self._motion_own = None    # the copy buffer behind _motion_prev (retain=False)
        self._ring = None

    # ------------------------------------------------------------ state
    def reset(self) -> None:
        """Forget previous maps / frames (next batch starts like tick 0).
        Captured CUDA graphs baked "has previous maps" in: drop them."""
        self._prev_maps = None
        self._prev_frame = None
        self._motion_prev = None
        self._graphs = {}

    def set_prev_maps(self, maps: list[SeamMaps]) -> None:
        """Seed the tick loop with host maps (seam s = cameras (s, s+1 mod N)).
        They are copied into the one device state buffer that every path -
        eager calls and captured graph replays alike - reads."""
        g = np.stack([[m.left.gain, m.right.gain] for m in maps])
        o = np.stack([[m.left.offset, m.right.offset] for m in maps])
        if g.shape != (self.S, 2, self.K, 3):
            raise ValueError("exposure map geometry mismatch")
        pg, po = self._state()
        pg.copy_(_dev.to_device(g))
        po.copy_(_dev.to_device(o))
        self._prev_maps = (pg, po)

    def _state(self):
        """Device tick-loop state: the last frame's maps (S, 2, K, 3), one
        pair of buffers for the corrector's lifetime (graph replays read
        them by address)."""
        st = getattr(self, "_state_bufs", None)
        if st is None:
            t = _dev.require_cuda()
            shape = (max(self.S, 1), 2, self.K, 3)
            st = (t.ones(shape, dtype=t.float64, device="cuda"),
                  t.zeros(shape, dtype=t.float64, device="cuda"))
            self._state_bufs = st
        return st

    def _buffers(self, B: int):
        buf = self._bufs.get(B)
        if buf is None:
            t = _dev.require_cuda()
            N, K, S = self.cam_count, self.K, self.S
            buf = dict(
                stats=t.empty((B, N, 2, K, _lib.STAT_BYTES), dtype=t.uint8, device="cuda"),
                gain=t.empty((B, max(S, 1), 2, K, 3), dtype=t.float64, device="cuda"),
                offset=t.empty((B, max(S, 1), 2, K, 3), dtype=t.float64, device="cuda"),
                fit_ok=t.empty((B, max(S, 1), K), dtype=t.uint8, device="cuda"),
                hist=(t.empty((B, N, 2, K, 3, 256), dtype=t.int32, device="cuda")
                      if self.histograms else None),
            )
            self._bufs[B] = buf
        return buf

    # ------------------------------------------------------------ device path
    def correct(self, frames, out=None, *, stream=None, prev_frames=None,
                _tile_args=None) -> CorrectResult:
        """Correct a (B, cam_count, H, W, 3) uint8 CUDA tensor (this GPU's
        cameras); returns device results.

        `prev_frames` (N, H, W, 3) overrides the remembered previous frame
        for OBJECT_REMOVAL's motion mask of array-frame 0."""
        t = _dev.require_cuda()
        if frames.dim() == 4:
            frames = frames[None]
        B, N, H, W, C = frames.shape
        if (N, H, W, C) != (self.cam_count, self.height, self.width, 3) or frames.dtype != t.uint8:
            raise ValueError(f"frames must be (B, {self.cam_count}, {self.height}, {self.width}, 3) "
                             f"uint8, got {tuple(frames.shape)} {frames.dtype}")
        if not frames.is_cuda or not frames.is_contiguous():
            raise ValueError("frames must be a contiguous CUDA tensor")
        if out is None:
            out = t.empty_like(frames)
        elif out.shape != frames.shape or not out.is_contiguous():
            raise ValueError("out must match frames")
        buf = self._buffers(B)
        main = stream if stream is not None else t.cuda.current_stream()
        removal = self.mode is ExposureMode.OBJECT_REMOVAL
        pf = prev_frames if prev_frames is not None else self._prev_frame
        if self.comm is not None and self.S > 0:
            self._correct_sharded(frames, out, buf, _dev.stream_handle(main), pf)
            return self._finish(frames, out, buf, main, removal)
        if self.exchange is None and self.S > 0 and self.fused:
            self._correct_fused(frames, out, buf, _dev.stream_handle(main), pf, _tile_args)
            return self._finish(frames, out, buf, main, removal)
        # separate launches: K1 (+ the Python stats exchange of a camera shard
        # on a non-NCCL backend) -> K2 -> K3, all on `main`
        sh = _dev.stream_handle(main)
        self._stats_solve(frames, buf, 0, B, sh, self._prev_maps, _dev.ptr(pf) if removal else None)
        self._apply(frames, out, buf, 0, B, sh)
        return self._finish(frames, out, buf, main, removal)

    def _finish(self, frames, out, buf, main, removal) -> CorrectResult:
        t = _dev.torch()
        B = frames.shape[0]
        gain, off = buf["gain"], buf["offset"]
        # carry the tick-loop state to the next batch
        with t.cuda.stream(main):
            if self.S > 0:
                pg, po = self._state()
                pg.copy_(gain[B - 1], non_blocking=True)
                po.copy_(off[B - 1], non_blocking=True)
                self._prev_maps = (pg, po)
            if removal:
                if self._prev_frame is None:
                    self._prev_frame = t.empty_like(frames[0])
                self._prev_frame.copy_(frames[B - 1], non_blocking=True)
        if self.comm is not None and "stats_all" in buf:
            R = _lib.STAT_BYTES
            with t.cuda.stream(main):
                full = buf["stats_all"].view(-1, 2, self.K, R).index_select(
                    0, buf["gather_index"]).view(B, self.n_cams, 2, self.K, R)
        else:
            full = buf["stats"] if self.exchange is None else buf["full"]
        return CorrectResult(out, gain[:, : self.S], off[:, : self.S], buf["fit_ok"][:, : self.S],
                             full, buf["hist"])

    # K1 -> K2 -> K3 as one camx_correct_batch call (K2, K3 programmatic
    # dependents).  False: the separate-launch path the Python stats
    # exchange needs (kept testable on one GPU).
    fused = True

    def _correct_fused(self, frames, out, buf, sh, pf, tile_args=None):
        """camx_correct_batch: K1 -> K2 -> K3 (PDL-chained) in one C call."""
        cfg = self.cfg
        B = frames.shape[0]
        removal = self.mode is ExposureMode.OBJECT_REMOVAL
        have_prev = self._prev_maps is not None
        sc = _lib.SolveConfig(_MODE_CODE[self.mode], self.K, int(cfg.min_band_pixels),
                              float(cfg.sigma_min), float(cfg.alpha),
                              float(cfg.min_valid_fraction), int(have_prev),
                              int(removal and pf is not None))
        pg, po = self._prev_maps if have_prev else (None, None)
        common = (frames.data_ptr(), out.data_ptr(), _dev.ptr(pf) if removal else None, B,
                  self.n_cams, int(self.wrap), self.height, self.width, cfg.band_width,
                  cfg.t_diff, ctypes.byref(sc), _dev.ptr(pg), _dev.ptr(po),
                  buf["stats"].data_ptr(), _dev.ptr(buf["hist"]), buf["gain"].data_ptr(),
                  buf["offset"].data_ptr(), buf["fit_ok"].data_ptr())
        if tile_args is not None:
            _lib.call("camx_correct_batch_tiles", *common, *tile_args, sh)
        else:
            _lib.call("camx_correct_batch", *common, None, sh)

    def _correct_sharded(self, frames, out, buf, sh, pf):
        """camx_correct_batch_sharded: K1 on this rank's cameras, NCCL
        all-gather of the records, K2 for all seams, K3 (one C call)."""
        cfg = self.cfg
        B = frames.shape[0]
        world = self.comm.world
        self._shard_bufs(buf, B)
        removal = self.mode is ExposureMode.OBJECT_REMOVAL
        have_prev = self._prev_maps is not None
        sc = _lib.SolveConfig(_MODE_CODE[self.mode], self.K, int(cfg.min_band_pixels),
                              float(cfg.sigma_min), float(cfg.alpha),
                              float(cfg.min_valid_fraction), int(have_prev),
                              int(removal and pf is not None))
        pg, po = self._prev_maps if have_prev else (None, None)
        _lib.call("camx_correct_batch_sharded", frames.data_ptr(), out.data_ptr(),
                  _dev.ptr(pf) if removal else None, B, self.n_cams, self.cam_begin,
                  self.cam_count, world, int(self.wrap), self.height, self.width, cfg.band_width,
                  cfg.t_diff, ctypes.byref(sc), _dev.ptr(pg), _dev.ptr(po),
                  buf["stats_local"].data_ptr(), buf["stats_all"].data_ptr(),
                  _dev.ptr(buf["hist"]), buf["gain"].data_ptr(), buf["offset"].data_ptr(),
                  buf["fit_ok"].data_ptr(), min(self.shard_chunks(world), B), self.comm.handle,
                  sh)

    def _shard_bufs(self, buf, B):
        """Record buffers of the sharded entry points: local records, the
        rank-major gathered records and their camera-order index."""
        t = _dev.torch()
        world = self.comm.world
        cmax = -(-self.n_cams // world)
        if "stats_all" not in buf:
            R = _lib.STAT_BYTES
            buf["stats_local"] = t.empty((B, cmax, 2, self.K, R), dtype=t.uint8, device="cuda")
            buf["stats_all"] = t.empty((world, B, cmax, 2, self.K, R), dtype=t.uint8,
                                       device="cuda")
            # gathered records (per chunk: rank-major [world][n_c][cmax]) ->
            # (B, n_cams) camera order
            from .dist import camera_partition
            parts = camera_partition(self.n_cams, world)
            nch = min(self.shard_chunks(world), B)
            idx = []
            for ci in range(nch):
                lo, hi = B * ci // nch, B * (ci + 1) // nch
                idx += [world * cmax * lo + (g * (hi - lo) + (b - lo)) * cmax + l
                        for b in range(lo, hi) for g, (_, c) in enumerate(parts) for l in range(c)]
            buf["gather_index"] = t.as_tensor(idx, dtype=t.int64, device="cuda")

    # ------------------------------------------------------------ pipelined stream
    def submit(self, frames, out=None, *, stream=None) -> CorrectResult | None:
        """Software-pipelined stream of batches for a camera shard (needs
        `comm`): this call runs the front half (K1 -> NCCL all-gather -> K2)
        of `frames` on a side stream while K3 of the previously submitted
        batch runs on `stream`; returns the previous batch's CorrectResult
        (complete in `stream` order), or None on the first call.  `flush()`
        applies the last batch.  Keep each batch's frames/out alive until
        its result is returned (the frames buffer may be refilled on
        `stream` right after the call: the call's end is joined into it).
        Maps and records are double-buffered: a returned result's gain /
        offset / fit_ok / stats / hist are views of the buffer the NEXT
        submit() refills, so they stay valid until the next submit() (copy
        them to keep them).  The tick-loop state carries across
        submits like correct()."""
        t = _dev.require_cuda()
        if self.S == 0:
            raise ValueError("submit() needs at least one seam")
        if self.comm is None and self.cam_count != self.n_cams:
            raise ValueError("a camera shard pipelines through its comm= (dist.NcclComm)")
        if frames.dim() == 4:
            frames = frames[None]
        B = frames.shape[0]
        if tuple(frames.shape[1:]) != (self.cam_count, self.height, self.width, 3) or \
                frames.dtype != t.uint8 or not frames.is_cuda or not frames.is_contiguous():
            raise ValueError("frames must be a contiguous uint8 CUDA tensor "
                             f"(B, {self.cam_count}, {self.height}, {self.width}, 3)")
        if out is None:
            out = t.empty_like(frames)
        elif out.shape != frames.shape or not out.is_contiguous():
            raise ValueError("out must match frames")
        old = getattr(self, "_pipe", None)
        if old is not None and old["pending"] is not None and old["B"] != B:
            raise ValueError("submit() batches must keep one size (flush() first)")
        pipe = self._pipe_state(B)
        main = stream if stream is not None else t.cuda.current_stream()
        k = pipe["k"]
        cur = pipe["bufs"][k % 2]
        removal = self.mode is ExposureMode.OBJECT_REMOVAL
        pending = pipe["pending"]
        if pending is not None and self.S > 0:  # maps of the previous batch's last frame
            pg, po = pending[2]["gain"][-1], pending[2]["offset"][-1]
        else:
            pg, po = self._prev_maps if self._prev_maps is not None else (None, None)
        pf = self._prev_frame if removal else None
        self._step_call(frames, B, cur, pg, po, pf, pending, main)
        res = self._pending_result(pending, main)
        pipe["pending"] = (frames, out, cur)
        pipe["k"] = k + 1
        if removal:  # raw last frame for the next batch's motion mask
            with t.cuda.stream(main):
                if self._prev_frame is None:
                    self._prev_frame = t.empty_like(frames[0])
                self._prev_frame.copy_(frames[B - 1], non_blocking=True)
        return res

    def flush(self, *, stream=None) -> CorrectResult | None:
        """K3 of the last submitted batch; returns its result.  The tick-loop
        state (maps, previous frame) carries on to correct()/submit()."""
        t = _dev.require_cuda()
        pipe = getattr(self, "_pipe", None)
        if pipe is None or pipe["pending"] is None:
            return None
        main = stream if stream is not None else t.cuda.current_stream()
        pending = pipe["pending"]
        self._step_call(None, 0, None, None, None, None, pending, main)
        res = self._pending_result(pending, main)
        pg, po = self._state()
        with t.cuda.stream(main):
            pg.copy_(pending[2]["gain"][-1], non_blocking=True)
            po.copy_(pending[2]["offset"][-1], non_blocking=True)
        self._prev_maps = (pg, po)
        pipe["pending"] = None
        return res

    def _pipe_state(self, B):
        pipe = getattr(self, "_pipe", None)
        if pipe is None or pipe["B"] != B:
            t = _dev.torch()
            world = self._pipe_comm().world
            cmax = -(-self.n_cams // world)
            R, K, S = _lib.STAT_BYTES, self.K, self.S

            def one():
                return dict(
                    stats_local=t.empty((B, cmax, 2, K, R), dtype=t.uint8, device="cuda"),
                    stats_all=t.empty((world, B, cmax, 2, K, R), dtype=t.uint8, device="cuda"),
                    hist=(t.empty((B, self.cam_count, 2, K, 3, 256), dtype=t.int32, device="cuda")
                          if self.histograms else None),
                    gain=t.empty((B, S, 2, K, 3), dtype=t.float64, device="cuda"),
                    offset=t.empty((B, S, 2, K, 3), dtype=t.float64, device="cuda"),
                    fit_ok=t.empty((B, S, K), dtype=t.uint8, device="cuda"))
            from .dist import camera_partition
            idx = [g * B * cmax + b * cmax + l for b in range(B)
                   for g, (_, c) in enumerate(camera_partition(self.n_cams, world))
                   for l in range(c)]
            pipe = dict(B=B, k=0, pending=None, bufs=[one(), one()],
                        index=t.as_tensor(idx, dtype=t.int64, device="cuda"))
            self._pipe = pipe
        return pipe

    def _step_call(self, frames, B, cur, pg, po, pf, pending, main):
        cfg = self.cfg
        removal = self.mode is ExposureMode.OBJECT_REMOVAL
        sc = _lib.SolveConfig(_MODE_CODE[self.mode], self.K, int(cfg.min_band_pixels),
                              float(cfg.sigma_min), float(cfg.alpha),
                              float(cfg.min_valid_fraction), int(pg is not None),
                              int(removal and pf is not None))
        front = () if frames is None else (
            frames.data_ptr(), _dev.ptr(pf) if removal else None, B)
        if not front:
            front = (None, None, 0)
        cb = cur if cur is not None else {}
        ap = (None, None, 0, None, None) if pending is None else (
            pending[0].data_ptr(), pending[1].data_ptr(), pending[0].shape[0],
            pending[2]["gain"].data_ptr(), pending[2]["offset"].data_ptr())
        comm = self._pipe_comm()
        _lib.call("camx_correct_batch_sharded_step", *front, self.n_cams, self.cam_begin,
                  self.cam_count, comm.world, int(self.wrap), self.height, self.width,
                  cfg.band_width, cfg.t_diff, ctypes.byref(sc), _dev.ptr(pg), _dev.ptr(po),
                  _dev.ptr(cb.get("stats_local")), _dev.ptr(cb.get("stats_all")),
                  _dev.ptr(cb.get("hist")), _dev.ptr(cb.get("gain")),
                  _dev.ptr(cb.get("offset")), _dev.ptr(cb.get("fit_ok")), *ap,
                  comm.handle, _dev.stream_handle(main))

    def _pipe_comm(self):
        """The shard's communicator, or a one-GPU stand-in (no collective)."""
        return self.comm if self.comm is not None else _LocalComm

    def _pending_result(self, pending, main):
        if pending is None:
            return None
        t = _dev.torch()
        frames, out, b = pending
        B = frames.shape[0]
        R = _lib.STAT_BYTES
        with t.cuda.stream(main):
            full = b["stats_all"].view(-1, 2, self.K, R).index_select(
                0, self._pipe["index"]).view(B, self.n_cams, 2, self.K, R)
        return CorrectResult(out, b["gain"], b["offset"], b["fit_ok"], full, b["hist"])

    # camx_correct_batch_sharded can split a batch into chunks (K1 + all-
    # gather + K2 of chunk c+1 on a side stream under K3 of chunk c); measured
    # slower at every N on B200 (smaller K3 launches, per-chunk launch and
    # collective latency: tools/shard_probe_native.py), so one chunk.
    shard_chunk_count = 1

    def shard_chunks(self, world: int) -> int:
        return max(1, min(8, int(self.shard_chunk_count)))

    def _stats_solve(self, frames, buf, lo, hi, sh, prev_maps, prev_frame_ptr):
        """K1 + (exchange) + K2 for array-frames [lo, hi) on stream `sh`."""
        cfg = self.cfg
        N, H, W = self.cam_count, self.height, self.width
        per_img = H * W * 3
        n = hi - lo
        stats, hist = buf["stats"], buf["hist"]
        rec_bytes = N * 2 * self.K * _lib.STAT_BYTES
        hist_bytes = N * 2 * self.K * 3 * 256 * 4
        base = frames.data_ptr() + lo * N * per_img
        st_ptr = stats.data_ptr() + lo * rec_bytes
        h_ptr = None if hist is None else hist.data_ptr() + lo * hist_bytes
        removal = self.mode is ExposureMode.OBJECT_REMOVAL
        # frames lo+1.. against their predecessors (a contiguous view, no
        # copy), frame lo against the previous chunk's / batch's last frame
        if removal and n > 1:
            _lib.call("camx_band_stats", base + N * per_img, base, None, (n - 1) * N, H, W,
                      cfg.band_width, self.K, cfg.t_diff, st_ptr + rec_bytes,
                      None if h_ptr is None else h_ptr + hist_bytes, sh)
            n0 = N
        else:
            n0 = n * N
        _lib.call("camx_band_stats", base, prev_frame_ptr if removal else None, None, n0, H, W,
                  cfg.band_width, self.K, cfg.t_diff, st_ptr, h_ptr, sh)
        if self.S == 0:
            return
        full_ptr = stats.data_ptr() + lo * rec_bytes
        if self.exchange is not None:
            # Python exchange (any torch.distributed backend): host-synchronous
            # on both sides (for gloo the records go through host copies:
            # dist._gather).  This path exists for portability, not speed -
            # the NCCL path is the stream-ordered camx_correct_batch_sharded.
            t = _dev.torch()
            ext = t.cuda.ExternalStream(sh)
            ext.synchronize()
            with t.cuda.stream(ext):
                full = self.exchange(stats[lo:hi])
                t.cuda.synchronize()
                if "full" not in buf:
                    buf["full"] = t.empty((buf["stats"].shape[0], self.n_cams, *full.shape[2:]),
                                          dtype=full.dtype, device=full.device)
                buf["full"][lo:hi].copy_(full)
            t.cuda.synchronize()  # the records are in place before K2 is enqueued
            full_ptr = buf["full"][lo].data_ptr()
        have_prev = prev_maps is not None
        sc = _lib.SolveConfig(_MODE_CODE[self.mode], self.K, int(cfg.min_band_pixels),
                              float(cfg.sigma_min), float(cfg.alpha),
                              float(cfg.min_valid_fraction), int(have_prev),
                              int(removal and prev_frame_ptr is not None))
        pg, po = prev_maps if have_prev else (None, None)
        _lib.call("camx_seam_solve", full_ptr, n, self.n_cams, int(self.wrap), ctypes.byref(sc),
                  _dev.ptr(pg), _dev.ptr(po), buf["gain"][lo].data_ptr(),
                  buf["offset"][lo].data_ptr(), buf["fit_ok"][lo].data_ptr(), sh)

    def _apply(self, frames, out, buf, lo, hi, sh):
        N, H, W = self.cam_count, self.height, self.width
        per_img = H * W * 3
        off = lo * N * per_img
        _lib.call("camx_apply_array", frames.data_ptr() + off, out.data_ptr() + off, hi - lo,
                  self.cam_begin, N, self.n_cams, int(self.wrap), H, W, self.K,
                  buf["gain"][lo].data_ptr(), buf["offset"][lo].data_ptr(), sh)

    # ------------------------------------------------------------ CUDA graphs
    def correct_graphed(self, frames, out) -> CorrectResult:
        """correct() for a stream of batches in fixed device buffers: the
        first call runs eagerly (establishing the tick-loop state) and
        captures the batch's launches - K1, K2, K3 with their programmatic
        dependencies, and the state carry - into a CUDA graph; later calls
        with the same (frames, out) buffers replay it, removing the per-call
        host cost (launch-bound small arrays).  Refill `frames` in place
        between calls.  The graphs read the tick-loop state from the
        corrector's fixed state buffers (_state: maps; the remembered
        previous frame), so set_prev_maps() and eager calls in between
        stay coherent; reset() drops the graphs."""
        t = _dev.require_cuda()
        key = (frames.data_ptr(), out.data_ptr(), tuple(frames.shape))
        if not hasattr(self, "_graphs"):
            self._graphs = {}
        hit = self._graphs.get(key) if self._prev_maps is not None or self.S == 0 else None
        if hit is not None:
            hit[0].replay()
            return hit[1]
        res = self.correct(frames, out)  # eager tick; state now "has previous"
        s = t.cuda.Stream()
        s.wait_stream(t.cuda.current_stream())
        g = t.cuda.CUDAGraph()
        with t.cuda.graph(g, stream=s):
            cap = self.correct(frames, out, stream=s)
        t.cuda.current_stream().wait_stream(s)
        self._graphs[key] = (g, cap)
        return res

    # ------------------------------------------------------------ tiles
    def tile_windows(self, size: int, overlap: float = 0.0):
        """Sliding-window origins over one array-frame's mosaic
        (attention.sliding_window_plan, attention.py:66-86)."""
        from .attention import window_origins
        return window_origins((self.n_cams * self.width, self.height), size, overlap)

    def correct_and_tile(self, frames, windows=None, *, size: int = 960, out_size: int = 416,
                         out=None, tiles=None, stream=None):
        """Correct a batch and cut detector tiles from the corrected mosaic of
        every array-frame (config 5).  windows: (x, y) origins applied to every
        frame (default: the sliding plan) or (b, x, y) triples.  Returns
        (CorrectResult, tiles uint8 (T, out_size, out_size, 3))."""
        t = _dev.require_cuda()
        if self.cam_count != self.n_cams:
            raise ValueError("tiles need the whole array on one GPU")
        B = frames.shape[0] if frames.dim() == 5 else 1
        wins = self.tile_windows(size) if windows is None else list(windows)
        if wins and len(wins[0]) == 2:
            wins = [(b, x, y) for b in range(B) for (x, y) in wins]
        for (b, x, y) in wins:
            if not (0 <= b < B and 0 <= x and 0 <= y and x + size <= self.n_cams * self.width
                    and y + size <= self.height):
                raise ValueError(f"window ({b}, {x}, {y}, {size}) outside the array")
        # grouped by array-frame (the fused kernel's contract), order kept within a frame
        wins = sorted(wins, key=lambda w: w[0])
        key = ("tiles", B, tuple(wins))
        wd = self._bufs.get(key)
        if wd is None:
            counts = np.bincount(np.asarray([w[0] for w in wins], dtype=np.int64), minlength=B)
            off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
            wd = (_dev.to_device(np.asarray(wins, dtype=np.int32).reshape(-1, 3)),
                  _dev.to_device(off), int(counts.max()) if len(wins) else 0)
            self._bufs[key] = wd
        T = len(wins)
        if tiles is None:
            tiles = t.empty((T, out_size, out_size, 3), dtype=t.uint8, device="cuda")
        tile_args = (wd[0].data_ptr(), wd[1].data_ptr(), T, wd[2], int(size), int(out_size),
                     tiles.data_ptr())
        if self.exchange is None and self.S > 0 and self.fused:
            if frames.dim() == 4:
                frames = frames[None]
            if out is None:
                out = t.empty_like(frames)
            res = self.correct(frames, out, stream=stream, _tile_args=tile_args)
        else:
            res = self.correct(frames, out, stream=stream)
            if T:
                _lib.call("camx_tiles", res.out.data_ptr(), self.n_cams, self.height, self.width,
                          wd[0].data_ptr(), T, int(size), int(out_size), tiles.data_ptr(),
                          _dev.stream_handle(stream))
        return res, tiles

    # ------------------------------------------------------------ attention
    def correct_with_motion(self, frames, out=None, *, size: int = 960, t_motion: int = 20,
                            stream=None, retain: bool = False, _bufs=None):
        """Correct a batch and, in the same pass over the pixels (K4 fused
        into K3: camx_correct_batch_motion), count per array-frame the
        motion-mask on-pixels of every window of the overlap-0 tiling - the
        counts of difference_plan(mask_diff(prev, cur, t_motion), size)
        (attention.py:89-103, core.py:191-196).  The previous array-frame
        of frame 0 is the last frame of the previous call (none after
        reset(): frame 0 then has no counts).  On a camera shard
        (comm=) each rank's K3 counts its cameras' pixels and the ranks'
        counts are all-gathered and summed (camx_correct_batch_sharded_motion):
        every rank returns the whole array's counts.

        Returns (CorrectResult, counts int64 CUDA tensor (B, n_windows) in
        window_origins order, has_counts list[bool] per frame).
        `retain=True`: the caller keeps `frames` unchanged until the next
        call's kernels have run (a ring of two or more batch buffers, or a
        batch re-submitted unchanged), so the next call's frame 0 reads its
        previous frame from this batch in place instead of from a copy (saves
        a device copy of one array-frame per call).  `_bufs`
        (internal, whole array only): result buffers (stats, gain, offset,
        fit_ok, hist) the kernels write directly - AttendPipeline's slots."""
        t = _dev.require_cuda()
        sharded = self.cam_count != self.n_cams
        if self.S == 0:
            raise ValueError("motion counts need an array of two or more cameras")
        if sharded and self.comm is None:
            raise ValueError("motion counts on a camera shard go through comm= (dist.NcclComm)")
        if not 0 <= int(t_motion) <= 255:
            raise ValueError("t_motion must be in 0..255")
        if frames.dim() == 4:
            frames = frames[None]
        B, N, H, W, C = frames.shape
        if (N, H, W, C) != (self.cam_count, self.height, self.width, 3) or frames.dtype != t.uint8:
            raise ValueError(f"frames must be (B, {self.cam_count}, {self.height}, {self.width}, "
                             "3) uint8")
        if not frames.is_cuda or not frames.is_contiguous():
            raise ValueError("frames must be a contiguous CUDA tensor")
        s = min(int(size), self.n_cams * W, H)  # the windows tile the whole mosaic
        origins = self.tile_windows(s)
        if out is None:
            out = t.empty_like(frames)
        elif out.shape != frames.shape or not out.is_contiguous():
            raise ValueError("out must match frames")
        buf = _bufs if _bufs is not None and not sharded else self._buffers(B)
        main = stream if stream is not None else t.cuda.current_stream()
        sh = _dev.stream_handle(main)
        counts = t.empty((B, len(origins)), dtype=t.int64, device="cuda")
        cfg = self.cfg
        removal = self.mode is ExposureMode.OBJECT_REMOVAL
        pf = self._prev_frame
        have_prev = self._prev_maps is not None
        sc = _lib.SolveConfig(_MODE_CODE[self.mode], self.K, int(cfg.min_band_pixels),
                              float(cfg.sigma_min), float(cfg.alpha),
                              float(cfg.min_valid_fraction), int(have_prev),
                              int(removal and pf is not None))
        pg, po = self._prev_maps if have_prev else (None, None)
        mp = self._motion_prev
        self.last_motion_fused = bool(_lib.load().camx_motion_supported(
            B, self.n_cams, self.cam_count, H, W, self.K, s))
        if sharded:
            # this rank's K3 counts its cameras' pixels; the ranks' counts are
            # all-gathered through comm and summed (identical on every rank)
            if not self.last_motion_fused or self.shard_chunks(self.comm.world) != 1:
                raise ValueError(f"window size {s} is too small for the fused counts on a "
                                 "camera shard: use dist.sharded_window_counts")
            self._shard_bufs(buf, B)
            key = ("counts_all", B, len(origins))
            call = self._bufs.get(key)
            if call is None:
                call = t.empty((self.comm.world, B, len(origins)), dtype=t.int64, device="cuda")
                self._bufs[key] = call
            _lib.call("camx_correct_batch_sharded_motion", frames.data_ptr(), out.data_ptr(),
                      _dev.ptr(pf) if removal else None, B, self.n_cams, self.cam_begin,
                      self.cam_count, self.comm.world, int(self.wrap), H, W, cfg.band_width,
                      cfg.t_diff, ctypes.byref(sc), _dev.ptr(pg), _dev.ptr(po),
                      buf["stats_local"].data_ptr(), buf["stats_all"].data_ptr(),
                      _dev.ptr(buf["hist"]), buf["gain"].data_ptr(), buf["offset"].data_ptr(),
                      buf["fit_ok"].data_ptr(), _dev.ptr(mp), s, int(t_motion), call.data_ptr(),
                      counts.data_ptr(), self.comm.handle, sh)
            res = self._finish(frames, out, buf, main, removal)
        elif self.last_motion_fused:
            _lib.call("camx_correct_batch_motion", frames.data_ptr(), out.data_ptr(),
                      _dev.ptr(pf) if removal else None, B, self.n_cams, int(self.wrap), H, W,
                      cfg.band_width, cfg.t_diff, ctypes.byref(sc), _dev.ptr(pg), _dev.ptr(po),
                      buf["stats"].data_ptr(), _dev.ptr(buf["hist"]), buf["gain"].data_ptr(),
                      buf["offset"].data_ptr(), buf["fit_ok"].data_ptr(), _dev.ptr(mp), s,
                      int(t_motion), counts.data_ptr(), sh)
            res = self._finish(frames, out, buf, main, removal)
        else:  # geometry outside the fused kernel: correct, then K4 per frame
            res = self.correct(frames, out, stream=stream)
            org = _dev.to_device(np.asarray(origins, dtype=np.int32).reshape(-1, 2))
            self._motion_org = org  # alive until the next call (the launches are async)
            with t.cuda.stream(main):
                counts.zero_()
            for b in range(B):
                prev = frames[b - 1] if b > 0 else mp
                if prev is None:
                    continue
                _lib.call("camx_window_counts", None, frames[b].data_ptr(), prev.data_ptr(),
                          int(t_motion), N, H, W, org.data_ptr(), len(origins), s,
                          counts[b].data_ptr(), sh)
        has = [mp is not None] + [True] * (B - 1)
        if retain:
            self._motion_prev = frames[B - 1]  # read in place by the next call
        else:
            with t.cuda.stream(main):
                if self._motion_own is None or self._motion_own.shape != frames[0].shape:
                    self._motion_own = t.empty_like(frames[0])
                self._motion_own.copy_(frames[B - 1], non_blocking=True)
            self._motion_prev = self._motion_own
        return res, counts, has

    def correct_and_attend(self, frames, scheduler, *, objects=(), frame_index: int = 0,
                           out_size: int = 416, t_motion: int = 20, out=None, stream=None):
        """One attention tick per array-frame (the paper's detector loop,
        attention.py:149-186): correct the batch with the fused motion counts
        (correct_with_motion), run `scheduler` (attention.Scheduler) on every
        frame in order - startup sweep, expectation windows of `objects`,
        then the difference windows ranked from the device counts, merged,
        cut to the budget - and resample the chosen windows of the corrected
        frames to out_size tiles (camx_tiles).

        Returns (CorrectResult, requests: list per frame of AttentionRequest,
        tiles uint8 (T, out_size, out_size, 3) in request order, counts)."""
        t = _dev.require_cuda()
        if tuple(scheduler.mosaic_size) != (self.n_cams * self.width, self.height):
            raise ValueError("scheduler mosaic does not match the array")
        size = scheduler.window_size
        res, counts, has = self.correct_with_motion(frames, out, size=size, t_motion=t_motion,
                                                    stream=stream)
        host = _dev.to_host(counts)  # one D2H of B x n_windows int64 (synchronises)
        requests, wins = [], []
        for b in range(host.shape[0]):
            fn = (lambda org, s, c=host[b]: c) if has[b] else None
            reqs = scheduler.schedule(frame_index=frame_index + b, objects=objects,
                                      window_counts_fn=fn)
            requests.append(reqs)
            wins += [(b, r.window.x, r.window.y) for r in reqs]
        tiles = t.empty((len(wins), out_size, out_size, 3), dtype=t.uint8, device="cuda")
        if wins:
            wd = _dev.to_device(np.asarray(wins, dtype=np.int32).reshape(-1, 3))
            _lib.call("camx_tiles", res.out.data_ptr(), self.n_cams, self.height, self.width,
                      wd.data_ptr(), len(wins), int(size), int(out_size), tiles.data_ptr(),
                      _dev.stream_handle(stream))
            self._attend_wins = wd  # alive until the next call (the launch is async)
        return res, requests, tiles, counts

    # ------------------------------------------------------------ results
    def maps(self, result: CorrectResult, b: int = -1, camera_ids=None) -> list[SeamMaps]:
        """Host SeamMaps of array-frame b (seam s = cameras (s, s+1 mod N))."""
        ids = list(camera_ids) if camera_ids is not None else list(range(self.n_cams))
        g = _dev.to_host(result.gain[b])
        o = _dev.to_host(result.offset[b])
        bw = self.cfg.band_width
        maps = []
        for s in range(self.S):
            sid = (ids[s], ids[(s + 1) % self.n_cams])
            maps.append(SeamMaps(ExposureMap(sid, Side.LEFT, bw, g[s, 0], o[s, 0]),
                                 ExposureMap(sid, Side.RIGHT, bw, g[s, 1], o[s, 1])))
        return maps

    # ------------------------------------------------------------ host path
    def correct_host(self, frames_host, out_host=None, *, chunk: int = 1, wait: bool = True,
                     stage: bool = False):
        """End-to-end correction of host frames (B, N, H, W, 3) uint8.

        frames_host/out_host: PINNED torch CPU tensors (async copies at full
        PCIe speed; ring.FrameRing hands out such buffers).  Pageable input
        (numpy arrays, unpinned tensors) is rejected with ValueError unless
        stage=True, which copies it into a pinned staging tensor first -
        explicitly, never silently.  H2D, kernels and D2H of consecutive
        chunks overlap on three streams.  wait=True returns out_host once
        it is filled; wait=False returns (out_host, event) right away so
        consecutive calls pipeline (the next batch's H2D overlaps this
        batch's D2H) - synchronize the event before reading out_host or
        reusing frames_host."""
        t = _dev.require_cuda()
        src = frames_host if isinstance(frames_host, t.Tensor) else t.from_numpy(
            np.ascontiguousarray(frames_host))
        if src.is_cuda:
            raise ValueError("correct_host takes host frames; use correct() for CUDA tensors")
        if not src.is_pinned():
            if not stage:
                raise ValueError("frames_host is pageable memory: pass a pinned tensor "
                                 "(tensor.pin_memory(), ring.FrameRing) or stage=True")
            src = src.pin_memory()
        if src.dim() == 4:
            src = src[None]
        B = src.shape[0]
        if out_host is None:
            out_host = t.empty(src.shape, dtype=t.uint8, pin_memory=True)
        dst = out_host if isinstance(out_host, t.Tensor) else t.from_numpy(out_host)
        if not dst.is_pinned():
            raise ValueError("out_host must be pinned memory (a D2H into pageable memory "
                             "is synchronous)")
        ring = self._host_ring(chunk)
        n_chunks = (B + chunk - 1) // chunk
        cur = t.cuda.current_stream()
        ring["h2d"].wait_stream(cur)  # inputs produced on the caller's stream
        for i in range(n_chunks):
            lo, hi = i * chunk, min(B, (i + 1) * chunk)
            slot = i % ring["slots"]
            dev_in = ring["in"][slot][: hi - lo]
            dev_out = ring["out"][slot][: hi - lo]
            with t.cuda.stream(ring["h2d"]):
                ring["h2d"].wait_event(ring["in_free"][slot])
                dev_in.copy_(src[lo:hi], non_blocking=True)
                ring["h2d_done"][slot].record(ring["h2d"])
            ring["comp"].wait_event(ring["h2d_done"][slot])
            ring["comp"].wait_event(ring["out_free"][slot])
            self.correct(dev_in, dev_out, stream=ring["comp"])
            ring["in_free"][slot].record(ring["comp"])
            ring["comp_done"][slot].record(ring["comp"])
            with t.cuda.stream(ring["d2h"]):
                ring["d2h"].wait_event(ring["comp_done"][slot])
                dst[lo:hi].copy_(dev_out, non_blocking=True)
                ring["out_free"][slot].record(ring["d2h"])
        done = t.cuda.Event()
        done.record(ring["d2h"])
        if wait:
            done.synchronize()
            return out_host
        return out_host, done

    def _host_ring(self, chunk: int):
        ring = self._ring
        if ring is not None and ring["chunk"] == chunk:
            return ring
        t = _dev.require_cuda()
        slots = 3
        shape = (chunk, self.cam_count, self.height, self.width, 3)
        ring = dict(chunk=chunk, slots=slots,
                    h2d=t.cuda.Stream(), comp=t.cuda.Stream(), d2h=t.cuda.Stream(),
                    **{"in": [t.empty(shape, dtype=t.uint8, device="cuda") for _ in range(slots)]},
                    out=[t.empty(shape, dtype=t.uint8, device="cuda") for _ in range(slots)],
                    in_free=[t.cuda.Event() for _ in range(slots)],
                    out_free=[t.cuda.Event() for _ in range(slots)],
                    h2d_done=[t.cuda.Event() for _ in range(slots)],
                    comp_done=[t.cuda.Event() for _ in range(slots)])
        self._ring = ring
        return ring


@dataclass
class AttendResult:
    """One batch through the attention tick (AttendPipeline)."""

    result: CorrectResult   # corrected frames and maps
    requests: list          # per array-frame: the Scheduler's AttentionRequests
    tiles: object           # uint8 (T, out, out, 3) CUDA tensor, request order
    counts: np.ndarray      # int64 (B, n_windows) motion counts (host)
    frame_index: int        # of the batch's first array-frame


class AttendPipeline:
    """The attention tick as a stream (the paper's detector loop: maps and
    pixels on the GPU, the per-tick decision on the host, in parallel).

    submit(batch k) launches k's correction with the fused motion counts
    (ArrayCorrector.correct_with_motion, writing straight into a result
    slot) and an async copy of the counts to pinned host memory (on a side
    stream), then finishes batch k-1: waits for its counts (its kernels ran
    before k's), runs `scheduler` on each of its array-frames on the host
    while the GPU corrects batch k, and launches k-1's tiles (camx_tiles on
    k-1's corrected frames) on a second side stream beside k's kernels; the
    caller's stream waits for those tiles before anything enqueued after the
    call.  It returns k-1's AttendResult (None for the first batch); flush()
    returns the last one.  A result's buffers (frames, maps) are reused two
    submits later."""

    def __init__(self, corrector, scheduler, *, out_size: int = 416, t_motion: int = 20,
                 retain_frames: bool = False):
        if tuple(scheduler.mosaic_size) != (corrector.n_cams * corrector.width, corrector.height):
            raise ValueError("scheduler mosaic does not match the array")
        self.ac, self.scheduler = corrector, scheduler
        self.out_size, self.t_motion = int(out_size), int(t_motion)
        # True: each submitted batch stays unchanged until the next batch's
        # kernels have run (ArrayCorrector.correct_with_motion(retain=True))
        self.retain_frames = bool(retain_frames)
        self._slots: dict = {}
        self._k = 0
        self._pending = None
        self._copy = None  # side stream of the counts' D2H
        self._tile_stream = None  # side stream of the previous batch's tiles

    def _slot(self, B: int, i: int):
        key = (B, i)
        sl = self._slots.get(key)
        if sl is None:
            t = _dev.require_cuda()
            ac = self.ac
            n_win = len(ac.tile_windows(self.scheduler.window_size))
            shape = (B, ac.n_cams, ac.height, ac.width, 3)
            mshape = (B, max(ac.S, 1), 2, ac.K, 3)
            sl = dict(out=t.empty(shape, dtype=t.uint8, device="cuda"),
                      gain=t.empty(mshape, dtype=t.float64, device="cuda"),
                      offset=t.empty(mshape, dtype=t.float64, device="cuda"),
                      fit_ok=t.empty((B, max(ac.S, 1), ac.K), dtype=t.uint8, device="cuda"),
                      stats=t.empty((B, ac.n_cams, 2, ac.K, _lib.STAT_BYTES), dtype=t.uint8,
                                    device="cuda"),
                      hist=(t.empty((B, ac.n_cams, 2, ac.K, 3, 256), dtype=t.int32,
                                    device="cuda") if ac.histograms else None),
                      counts=t.empty((B, n_win), dtype=t.int64, pin_memory=True),
                      # the chosen windows go up through pinned memory on the
                      # caller's stream: a pageable upload would synchronise the
                      # host with the batch just submitted (the GPU then idles
                      # while the host returns and launches the next batch)
                      wins_host=t.empty((B * n_win, 3), dtype=t.int32, pin_memory=True),
                      wins_dev=t.empty((B * n_win, 3), dtype=t.int32, device="cuda"),
                      event=t.cuda.Event())
            self._slots[key] = sl
        return sl

    def submit(self, frames, *, frame_index: int, objects=(), stream=None):
        t = _dev.require_cuda()
        main = stream if stream is not None else t.cuda.current_stream()
        if frames.dim() == 4:
            frames = frames[None]
        B = frames.shape[0]
        sl = self._slot(B, self._k % 2)
        # the fused kernels write maps, stats and histograms straight into the
        # slot (no per-batch device copies of ~100 MB of histograms)
        res, counts, has = self.ac.correct_with_motion(
            frames, sl["out"], size=self.scheduler.window_size, t_motion=self.t_motion,
            stream=main, retain=self.retain_frames, _bufs=sl)
        S = self.ac.S
        with t.cuda.stream(main):
            if res.gain.data_ptr() != sl["gain"].data_ptr():  # a shard or the unfused path
                sl["gain"][:, :S].copy_(res.gain, non_blocking=True)
                sl["offset"][:, :S].copy_(res.offset, non_blocking=True)
                sl["fit_ok"][:, :S].copy_(res.fit_ok, non_blocking=True)
                sl["stats"].copy_(res.stats, non_blocking=True)
                if sl["hist"] is not None:
                    sl["hist"].copy_(res.hist, non_blocking=True)
        # the counts' D2H runs on a side stream: on the compute stream the
        # small copy would sit between batch k and the next kernels (~30 us
        # of copy-engine round trip per step); the host waits for its event
        if self._copy is None:
            self._copy = t.cuda.Stream()
        self._copy.wait_stream(main)
        with t.cuda.stream(self._copy):
            sl["counts"].copy_(counts, non_blocking=True)
            sl["event"].record(self._copy)
        counts.record_stream(self._copy)
        prev, self._pending = self._pending, (sl, B, int(frame_index), tuple(objects), has)
        self._k += 1
        return self._finish(prev, main) if prev is not None else None

    def flush(self, stream=None):
        t = _dev.require_cuda()
        main = stream if stream is not None else t.cuda.current_stream()
        prev, self._pending = self._pending, None
        return self._finish(prev, main) if prev is not None else None

    def _finish(self, pend, main) -> AttendResult:
        t = _dev.torch()
        sl, B, f0, objects, has = pend
        sl["event"].synchronize()
        host = sl["counts"].numpy().copy()
        ac, sched = self.ac, self.scheduler
        requests, wins = [], []
        for b in range(B):
            fn = (lambda org, s, c=host[b]: c) if has[b] else None
            reqs = sched.schedule(frame_index=f0 + b, objects=objects, window_counts_fn=fn)
            requests.append(reqs)
            wins += [(b, r.window.x, r.window.y) for r in reqs]
        tiles = t.empty((len(wins), self.out_size, self.out_size, 3), dtype=t.uint8,
                        device="cuda")
        if wins:
            n = len(wins)
            if n > sl["wins_host"].shape[0]:  # more windows than the tiling (large budgets)
                sl["wins_host"] = t.empty((n, 3), dtype=t.int32, pin_memory=True)
                sl["wins_dev"] = t.empty((n, 3), dtype=t.int32, device="cuda")
            # the slot's previous upload (two submits ago) ran before the batch
            # whose event was synchronised above, so its host buffer is free
            sl["wins_host"][:n].numpy()[:] = np.asarray(wins, dtype=np.int32).reshape(-1, 3)
            wd = sl["wins_dev"]
            # batch k-1's frames are complete (its event was synchronised
            # above), so its tiles need not queue behind batch k on `main`:
            # they run beside k's kernels on a side stream, and `main` waits
            # for them before anything enqueued after this call
            if self._tile_stream is None:
                self._tile_stream = t.cuda.Stream()
            ts = self._tile_stream
            with t.cuda.stream(ts):
                wd[:n].copy_(sl["wins_host"][:n], non_blocking=True)
                _lib.call("camx_tiles", sl["out"].data_ptr(), ac.n_cams, ac.height, ac.width,
                          wd.data_ptr(), n, int(sched.window_size), self.out_size,
                          tiles.data_ptr(), _dev.stream_handle(ts))
                done = t.cuda.Event()
                done.record(ts)
            tiles.record_stream(ts)
            main.wait_event(done)
        S = ac.S
        res = CorrectResult(sl["out"], sl["gain"][:, :S], sl["offset"][:, :S],
                            sl["fit_ok"][:, :S], sl["stats"], sl["hist"])
        return AttendResult(res, requests, tiles, host, f0)


def correct_array(frames, cfg: ExposureConfig = ExposureConfig(), prev_maps=None,
                  mode: ExposureMode = ExposureMode.STANDARD, *, prev_frames=None,
                  wrap: bool = False, histograms: bool = False, camera_ids=None):
    """One array-frame through update_exposure (every seam) + apply_exposure
    (both halves of every camera) - the batched extension of SURVEY 8b.

    frames: (N, H, W, 3) uint8, host numpy (copied to the GPU and back) or a
    CUDA tensor (stays on the device).  prev_maps: list of SeamMaps of the
    previous tick (seam s = cameras (s, s+1 mod N)) or None; prev_frames:
    (N, H, W, 3) of the previous tick for OBJECT_REMOVAL.  Returns
    (corrected, maps, histograms): corrected like `frames`, maps a list of
    SeamMaps with seam_id from `camera_ids` (default 0..N-1), histograms
    uint32 (N, 2, K, 3, 256) of the band pixels (side 0 = LEFT band, cols
    [W-bw, W); side 1 = RIGHT band) as numpy, or None."""
    t = _dev.require_cuda()
    on_host = isinstance(frames, np.ndarray)
    dev = _dev.to_device(np.ascontiguousarray(frames)) if on_host else frames
    if dev.dim() != 4 or dev.shape[-1] != 3 or dev.dtype != t.uint8:
        raise ValueError("frames must be uint8 (N, H, W, 3)")
    N, H, W = (int(v) for v in dev.shape[:3])
    ac = ArrayCorrector(N, H, W, cfg, mode, wrap=wrap, histograms=histograms)
    if prev_maps is not None:
        ac.set_prev_maps(list(prev_maps))
    pf = None
    if prev_frames is not None:
        pf = (_dev.to_device(np.ascontiguousarray(prev_frames))
              if isinstance(prev_frames, np.ndarray) else prev_frames)
        if tuple(pf.shape) != (N, H, W, 3):
            raise ValueError("prev_frames must match frames")
    res = ac.correct(dev[None].contiguous(), prev_frames=pf)
    maps = ac.maps(res, 0, camera_ids)
    hist = None
    if res.hist is not None:
        hist = _dev.to_host(res.hist[0]).view(np.uint32)
    out = res.out[0]
    return (_dev.to_host(out) if on_host else out), maps, hist
