"""Drop-in for `camarray.exposure` (reference exposure.py) on the GPU.

Same public names, signatures, shapes, dtypes and ValueError conditions as
the reference module; the arithmetic runs in libcamx.so:

  band_stats        -> camx_band_stats + camx_band_moments   (K1)
  fit_affine        -> camx_fit_affine                         (K2)
  smooth_exposure   -> camx_smooth_maps                        (K2)
  update_exposure   -> camx_band_stats + camx_seam_solve       (K1 + K2)
  apply_exposure(_inplace) -> camx_apply_map                   (K3)
  seam_cost         -> camx_seam_cost

The per-call functions move numpy arrays host<->device like the
reference's per-call numpy API; the batched device-resident path is
`paper_1910_03517_b200.array.ArrayCorrector`.
"""

from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _dev, _lib
from .core import Frame

__all__ = [
    "Side",
    "ExposureMode",
    "ExposureConfig",
    "ExposureMap",
    "SeamMaps",
    "BandStats",
    "band_stats",
    "fit_affine",
    "smooth_exposure",
    "update_exposure",
    "apply_exposure",
    "seam_cost",
    "identity_map",
    "write_maps_table",
    "read_maps_table",
]

CHANNELS = "rgb"


class Side(enum.Enum):
    """LEFT: the seam is at the frame's right edge; RIGHT: at its left edge."""

    LEFT = "left"
    RIGHT = "right"


class ExposureMode(enum.Enum):
    STANDARD = "standard"
    OBJECT_REMOVAL = "object_removal"
    SMOOTHING = "smoothing"


_SIDE_CODE = {Side.LEFT: _lib.SIDE_LEFT, Side.RIGHT: _lib.SIDE_RIGHT}
_MODE_CODE = {ExposureMode.STANDARD: _lib.MODE_STANDARD,
              ExposureMode.OBJECT_REMOVAL: _lib.MODE_OBJECT_REMOVAL,
              ExposureMode.SMOOTHING: _lib.MODE_SMOOTHING}


@dataclass(frozen=True)
class ExposureConfig:
    """exposure.py:54-63."""

    band_width: int = 32
    blocks: int = 16
    alpha: float = 0.05
    t_diff: int = 20
    min_valid_fraction: float = 0.25
    min_band_pixels: int = 64
    sigma_min: float = 1e-3
    downsample: int = 8


@dataclass(eq=False)
class ExposureMap:
    """(K, 3) float64 gain/offset of one seam side (exposure.py:66-101).

    `_cache` memoises the device copy of the coefficients (the reference
    memoises its per-shape f32 apply tables there)."""

    seam_id: tuple[int, int]
    side: Side
    band_width: int
    gain: np.ndarray
    offset: np.ndarray
    _cache: dict = field(default_factory=dict, repr=False)

    def __post_init__(self) -> None:
        self.gain = np.asarray(self.gain, dtype=np.float64)
        self.offset = np.asarray(self.offset, dtype=np.float64)
        g, o = self.gain, self.offset
        if g.shape != o.shape or g.ndim != 2 or g.shape[1] != 3:
            raise ValueError("gain/offset must both be (K, 3)")
        if not (np.isfinite(g).all() and np.isfinite(o).all()):
            raise ValueError("non-finite exposure coefficients")
        if (g <= 0).any():
            raise ValueError("gains must be positive")

    @property
    def block_count(self) -> int:
        return self.gain.shape[0]

    def same_geometry(self, other: "ExposureMap") -> bool:
        return (self.seam_id, self.side, self.block_count) == \
            (other.seam_id, other.side, other.block_count)

    def device_coeffs(self):
        """Cached contiguous CUDA float64 copies of (gain, offset)."""
        hit = self._cache.get("camx")
        if hit is None:
            hit = (_dev.to_device(self.gain), _dev.to_device(self.offset))
            self._cache["camx"] = hit
        return hit


@dataclass(frozen=True, eq=False)
class SeamMaps:
    """The LEFT/RIGHT side maps of one seam (exposure.py:104-109)."""

    left: ExposureMap
    right: ExposureMap


def identity_map(seam_id: tuple[int, int], side: Side, blocks: int,
                 band_width: int) -> ExposureMap:
    return ExposureMap(seam_id, side, band_width, np.ones((blocks, 3)), np.zeros((blocks, 3)))


def block_bounds(height: int, blocks: int) -> list[tuple[int, int]]:
    """K row ranges of floor(H/K) rows, remainder in the last (exposure.py:123-135)."""
    if blocks < 1:
        raise ValueError("need at least one block")
    if blocks > height:
        raise ValueError(f"more blocks ({blocks}) than rows ({height})")
    bh = height // blocks
    return [(k * bh, (k + 1) * bh if k < blocks - 1 else height) for k in range(blocks)]


@dataclass(frozen=True, eq=False)
class BandStats:
    """Per-block, per-channel band moments (exposure.py:138-149)."""

    mean: np.ndarray
    std: np.ndarray
    valid_count: np.ndarray
    band_area: np.ndarray


# ----------------------------------------------------------------- helpers

def _check_band(width: int, band_width: int) -> None:
    if band_width > width // 2:
        raise ValueError(f"band width {band_width} exceeds half frame width {width // 2}")


def _stats_device(images, prev=None, masks=None, *, band_width, blocks, t_diff=20,
                  hist=False):
    """Run K1 on a (n, H, W, 3) uint8 CUDA tensor -> (records uint8 tensor, hist)."""
    t = _dev.require_cuda()
    n, h, w = images.shape[:3]
    _check_band(w, band_width)
    block_bounds(h, blocks)
    rec = t.empty((n, 2, blocks, _lib.STAT_BYTES), dtype=t.uint8, device="cuda")
    hs = t.empty((n, 2, blocks, 3, 256), dtype=t.int32, device="cuda") if hist else None
    _lib.call("camx_band_stats", images.data_ptr(), _dev.ptr(prev), _dev.ptr(masks), n, h, w,
              band_width, blocks, int(t_diff), rec.data_ptr(), _dev.ptr(hs),
              _dev.stream_handle())
    return rec, hs


def _moments(rec, use_raw=False):
    t = _dev.require_cuda()
    n = rec.numel() // _lib.STAT_BYTES
    mean = t.empty((n, 3), dtype=t.float64, device="cuda")
    std = t.empty((n, 3), dtype=t.float64, device="cuda")
    valid = t.empty((n,), dtype=t.int64, device="cuda")
    area = t.empty((n,), dtype=t.int64, device="cuda")
    _lib.call("camx_band_moments", rec.data_ptr(), n, int(use_raw), mean.data_ptr(),
              std.data_ptr(), valid.data_ptr(), area.data_ptr(), _dev.stream_handle())
    return mean, std, valid, area


def _pixels(frame) -> np.ndarray:
    return frame.pixels if isinstance(frame, Frame) else np.asarray(frame)


def _bands(px: np.ndarray, band_width: int) -> np.ndarray:
    """The two seam bands of a frame packed side by side, (H, 2*bw[, 3]):
    K1 over this image (width 2*bw) reads exactly the columns it would read
    in the full frame (LEFT side = the last bw columns, RIGHT side = the
    first bw), so the per-call drop-in ships ~2*bw/W of the frame over PCIe
    instead of all of it."""
    w = px.shape[1]
    if 2 * band_width >= w:
        return np.ascontiguousarray(px)
    return np.concatenate((px[:, :band_width], px[:, w - band_width:]), axis=1)


# ----------------------------------------------------------------- stage 1

def band_stats(frame: Frame, side: Side, band_width: int, blocks: int,
               exclusion_mask: np.ndarray | None = None) -> BandStats:
    """Moments of the `band_width` columns nearest the seam, per row block,
    with masked pixels dropped (exposure.py:152-185).  Computed from exact
    integer sums on the GPU (K1)."""
    h, w = frame.height, frame.width
    _check_band(w, band_width)
    block_bounds(h, blocks)
    img = _dev.to_device(_bands(frame.pixels, band_width))[None]
    msk = None
    if exclusion_mask is not None:
        # the reference slices the mask like the band (exposure.py:163-168)
        # and boolean-indexes each block's pixels with it (:178-180): any
        # mask whose band slice covers the band's rows and columns works
        # (extra rows are never read); otherwise numpy raises IndexError
        m = np.asarray(exclusion_mask, dtype=bool)
        mb = m[:, w - band_width:] if side is Side.LEFT else m[:, :band_width]
        if mb.ndim != 2 or mb.shape[0] < h or mb.shape[1] != band_width:
            raise IndexError(f"boolean index did not match the band: mask {m.shape}, "
                             f"band {(h, band_width)}")
        mb = np.ascontiguousarray(mb[:h]).view(np.uint8)
        full = np.zeros((h, 2 * band_width) if 2 * band_width < w else (h, w), dtype=np.uint8)
        if 2 * band_width < w:  # the packed layout of _bands: RIGHT band, then LEFT band
            if side is Side.LEFT:
                full[:, band_width:] = mb
            else:
                full[:, :band_width] = mb
        elif side is Side.LEFT:
            full[:, w - band_width:] = mb
        else:
            full[:, :band_width] = mb
        msk = _dev.to_device(full)[None]
    rec, _ = _stats_device(img, masks=msk, band_width=band_width, blocks=blocks)
    s = 0 if side is Side.LEFT else 1
    mean, std, valid, area = (_dev.to_host(x) for x in _moments(rec[0, s]))
    return BandStats(mean=mean, std=std, valid_count=valid, band_area=area)


def band_histograms(frames, band_width: int, blocks: int, exclusion_masks=None):
    """uint32 (n, 2 sides, K, 3, 256) band histograms of n frames (builder-
    defined product of K1).  `frames`: (n, H, W, 3)."""
    px = np.asarray(frames, dtype=np.uint8)
    img = _dev.to_device(px)
    msk = None if exclusion_masks is None else _dev.to_device(
        np.asarray(exclusion_masks, dtype=bool).view(np.uint8))
    _, hs = _stats_device(img, masks=msk, band_width=band_width, blocks=blocks, hist=True)
    return _dev.to_host(hs).view(np.uint32)


# ----------------------------------------------------------------- stage 2

def fit_affine(left: BandStats, right: BandStats, *,
               sigma_min: float = 1e-3,
               min_band_pixels: int = 64,
               seam_id: tuple[int, int] = (0, 1),
               band_width: int = 32) -> tuple[ExposureMap, ExposureMap, np.ndarray]:
    """Moment-matching affine fit to the shared spectrum (exposure.py:188-229),
    on the GPU (camx_fit_affine)."""
    k = left.mean.shape[0]
    if right.mean.shape[0] != k:
        raise ValueError("block counts differ between sides")
    t = _dev.require_cuda()
    dv = [_dev.to_device(np.asarray(a, dtype=np.float64)) for a in
          (left.mean, left.std, right.mean, right.std)]
    cv = [_dev.to_device(np.asarray(a, dtype=np.int64)) for a in
          (left.valid_count, right.valid_count)]
    gain = t.empty((2, k, 3), dtype=t.float64, device="cuda")
    off = t.empty((2, k, 3), dtype=t.float64, device="cuda")
    ok = t.empty((k,), dtype=t.uint8, device="cuda")
    _lib.call("camx_fit_affine", dv[0].data_ptr(), dv[1].data_ptr(), cv[0].data_ptr(),
              dv[2].data_ptr(), dv[3].data_ptr(), cv[1].data_ptr(), k, float(sigma_min),
              int(min_band_pixels), gain.data_ptr(), off.data_ptr(), ok.data_ptr(),
              _dev.stream_handle())
    g, o, okh = _dev.to_host(gain), _dev.to_host(off), _dev.to_host(ok).astype(bool)
    return (ExposureMap(seam_id, Side.LEFT, band_width, g[0], o[0]),
            ExposureMap(seam_id, Side.RIGHT, band_width, g[1], o[1]), okh)


def smooth_exposure(prev: ExposureMap, new: ExposureMap, alpha: float = 0.05) -> ExposureMap:
    """(1 - alpha) * prev + alpha * new, coefficient-wise (exposure.py:232-242)."""
    if not prev.same_geometry(new):
        raise ValueError("exposure map geometry mismatch")
    t = _dev.require_cuda()
    pg, po = prev.device_coeffs()
    ng, no = new.device_coeffs()
    g = t.empty_like(ng)
    o = t.empty_like(no)
    _lib.call("camx_smooth_maps", pg.data_ptr(), po.data_ptr(), ng.data_ptr(), no.data_ptr(),
              ng.numel(), float(alpha), g.data_ptr(), o.data_ptr(), _dev.stream_handle())
    return ExposureMap(new.seam_id, new.side, new.band_width, _dev.to_host(g), _dev.to_host(o))


def _solve_config(mode: ExposureMode, cfg: ExposureConfig, have_prev_maps: bool,
                  have_prev_frames: bool) -> _lib.SolveConfig:
    return _lib.SolveConfig(_MODE_CODE[mode], cfg.blocks, int(cfg.min_band_pixels),
                            float(cfg.sigma_min), float(cfg.alpha),
                            float(cfg.min_valid_fraction), int(have_prev_maps),
                            int(have_prev_frames))


def update_exposure(frames: tuple[Frame, Frame],
                    prev_maps: SeamMaps | None,
                    mode: ExposureMode = ExposureMode.STANDARD,
                    cfg: ExposureConfig = ExposureConfig(),
                    prev_frames: tuple[Frame, Frame] | None = None) -> SeamMaps:
    """This tick's seam maps from a synchronized frame pair
    (exposure.py:245-344): K1 band statistics (with the in-band motion mask
    for OBJECT_REMOVAL) and the K2 solve, both on the GPU."""
    left_f, right_f = frames
    seam_id = (left_f.camera_id, right_f.camera_id)
    if left_f.height != right_f.height:
        raise ValueError("seam frames differ in height")
    if not isinstance(mode, ExposureMode):
        raise ValueError(f"unknown exposure mode {mode!r}")
    if left_f.width != right_f.width:
        # the array kernels index one geometry; fall back to per-side calls
        return _update_mixed_width(frames, prev_maps, mode, cfg, prev_frames)
    t = _dev.require_cuda()
    _check_band(left_f.width, cfg.band_width)
    bw = cfg.band_width
    imgs = _dev.to_device(np.stack([_bands(left_f.pixels, bw), _bands(right_f.pixels, bw)]))
    use_prev = mode is ExposureMode.OBJECT_REMOVAL and prev_frames is not None
    if use_prev and any(pf.pixels.shape != f.pixels.shape for pf, f in zip(prev_frames, frames)):
        raise ValueError("pixel dimensions differ")
    prev = _dev.to_device(np.stack([_bands(prev_frames[0].pixels, bw),
                                    _bands(prev_frames[1].pixels, bw)])) if use_prev else None
    rec, _ = _stats_device(imgs, prev=prev, band_width=cfg.band_width, blocks=cfg.blocks,
                           t_diff=cfg.t_diff)
    return _solve_pair(rec.view(1, 2, 2, cfg.blocks, _lib.STAT_BYTES), prev_maps, mode, cfg,
                       use_prev, seam_id)


def _solve_pair(rec, prev_maps, mode, cfg, use_prev, seam_id) -> SeamMaps:
    """K2 for one seam, with the reference's checks on `prev_maps`:
    * where the reference blends into them (SMOOTHING; OBJECT_REMOVAL with
      prev_frames) smooth_exposure requires the same seam_id, side and K
      (exposure.py:234-235, 304-307, 332-335);
    * elsewhere they are only resolve()'s fallback (exposure.py:275-293):
      no check at all when every block fits (:280-281), else numpy's
      np.where broadcast of (K, 1) against the fallback's (K', 3), which
      accepts K' in {1, K} and raises ValueError otherwise."""
    t = _dev.torch()
    K = cfg.blocks
    blends = mode is ExposureMode.SMOOTHING or (mode is ExposureMode.OBJECT_REMOVAL and use_prev)
    pg = po = None
    deferred = False  # a fallback that only fails if some block needs it
    if prev_maps is not None:
        sides = ((prev_maps.left, Side.LEFT), (prev_maps.right, Side.RIGHT))
        if blends:
            for pm, side in sides:
                if (pm.seam_id, pm.side, pm.block_count) != (seam_id, side, K):
                    raise ValueError("exposure map geometry mismatch")
        coeffs = []
        for pm, _ in sides:
            if pm.block_count == K:
                coeffs.append((pm.gain, pm.offset))
            elif pm.block_count == 1:  # broadcasts against (K, 1) like np.where
                coeffs.append((np.broadcast_to(pm.gain, (K, 3)),
                               np.broadcast_to(pm.offset, (K, 3))))
            else:
                deferred = True
        if not deferred:
            pg = _dev.to_device(np.stack([c[0] for c in coeffs]))
            po = _dev.to_device(np.stack([c[1] for c in coeffs]))
    gain = t.empty((1, 1, 2, K, 3), dtype=t.float64, device="cuda")
    off = t.empty_like(gain)
    ok = t.empty((1, 1, K), dtype=t.uint8, device="cuda")
    sc = _solve_config(mode, cfg, pg is not None, use_prev)
    _lib.call("camx_seam_solve", rec.data_ptr(), 1, 2, 0, ctypes.byref(sc), _dev.ptr(pg),
              _dev.ptr(po), gain.data_ptr(), off.data_ptr(), ok.data_ptr(), _dev.stream_handle())
    g, o = _dev.to_host(gain)[0, 0], _dev.to_host(off)[0, 0]
    if deferred and not _dev.to_host(ok).all():
        kp = [pm.block_count for pm, _ in sides if pm.block_count not in (1, K)][0]
        raise ValueError(f"operands could not be broadcast together with shapes ({K},1) "
                         f"({K},3) ({kp},3)")
    bw = cfg.band_width
    return SeamMaps(ExposureMap(seam_id, Side.LEFT, bw, g[0], o[0]),
                    ExposureMap(seam_id, Side.RIGHT, bw, g[1], o[1]))


def _update_mixed_width(frames, prev_maps, mode, cfg, prev_frames) -> SeamMaps:
    """Seam frames of different widths: K1 per frame, records joined for K2."""
    t = _dev.require_cuda()
    use_prev = mode is ExposureMode.OBJECT_REMOVAL and prev_frames is not None
    recs = []
    bw = cfg.band_width
    for i, f in enumerate(frames):
        _check_band(f.width, bw)
        img = _dev.to_device(_bands(f.pixels, bw))[None]
        prev = None
        if use_prev:
            if prev_frames[i].pixels.shape != f.pixels.shape:
                raise ValueError("pixel dimensions differ")
            prev = _dev.to_device(_bands(prev_frames[i].pixels, bw))[None]
        r, _ = _stats_device(img, prev=prev, band_width=cfg.band_width, blocks=cfg.blocks,
                             t_diff=cfg.t_diff)
        recs.append(r)
    rec = t.cat(recs, 0).view(1, 2, 2, cfg.blocks, _lib.STAT_BYTES)
    return _solve_pair(rec, prev_maps, mode, cfg, use_prev,
                       (frames[0].camera_id, frames[1].camera_id))


# ----------------------------------------------------------------- stage 3

def _apply_device(img, out, emap: ExposureMap) -> None:
    n, h, w = img.shape[:3]
    block_bounds(h, emap.block_count)
    g, o = emap.device_coeffs()
    _lib.call("camx_apply_map", img.data_ptr(), out.data_ptr(), n, h, w, _SIDE_CODE[emap.side],
              emap.block_count, g.data_ptr(), o.data_ptr(), _dev.stream_handle())


def apply_exposure(frame: Frame, emap: ExposureMap) -> Frame:
    """Correct the half of the frame nearest the seam (exposure.py:385-401);
    the far half is returned untouched (K3, bit-exact with the reference)."""
    t = _dev.require_cuda()
    img = _dev.to_device(frame.pixels)[None]
    out = t.empty_like(img)
    _apply_device(img, out, emap)
    return Frame(frame.camera_id, frame.frame_index, frame.timestamp_ms, _dev.to_host(out[0]))


def apply_exposure_inplace(pixels: np.ndarray, emap: ExposureMap) -> None:
    """apply_exposure mutating a raw (H, W, 3) pixel array (exposure.py:404-414).
    CUDA tensors are corrected in place on the device."""
    t = _dev.torch()
    if isinstance(pixels, t.Tensor) and pixels.is_cuda:
        img = pixels if pixels.dim() == 4 else pixels[None]
        _apply_device(img, img, emap)
        return
    img = _dev.to_device(pixels)[None]
    _apply_device(img, img, emap)
    pixels[...] = _dev.to_host(img[0])


# ------------------------------------------------------------- seam quality

def seam_cost(left, right, downsample_factor: int = 8) -> float:
    """Gradient-trend discrepancy across the seam (exposure.py:417-445,
    Eq. 1 of the paper), on the GPU (camx_seam_cost)."""
    lp, rp = _pixels(left), _pixels(right)
    if lp.shape[0] != rp.shape[0]:
        raise ValueError("seam frames differ in height")
    f = int(downsample_factor)
    h = lp.shape[0]
    if f < 1 or h // f < 1 or lp.shape[1] // f < 2 or rp.shape[1] // f < 2:
        raise ValueError(f"frame too small for downsample factor {downsample_factor}")
    t = _dev.require_cuda()
    a = _dev.to_device(np.asarray(lp, dtype=np.uint8))
    b = _dev.to_device(np.asarray(rp, dtype=np.uint8))
    out = t.empty((1,), dtype=t.float64, device="cuda")
    _lib.call("camx_seam_cost", a.data_ptr(), b.data_ptr(), 1, h, lp.shape[1], rp.shape[1], f,
              out.data_ptr(), _dev.stream_handle())
    return float(_dev.to_host(out)[0])


# ---------------------------------------------------------- maps table I/O

_TABLE_VERSION = "camarray-exposure-v1"


def write_maps_table(maps: list[SeamMaps]) -> str:
    """Versioned text table, one line per (seam, side, block, channel)
    with repr floats so values round-trip exactly (exposure.py:448-463)."""
    out = [f"# {_TABLE_VERSION}", "# seam side block channel gain offset"]
    for sm in maps:
        for em in (sm.left, sm.right):
            sid = "%d-%d" % tuple(em.seam_id)
            out.extend(f"{sid} {em.side.value} {k} {CHANNELS[c]} "
                       f"{float(em.gain[k, c])!r} {float(em.offset[k, c])!r}"
                       for k in range(em.block_count) for c in range(3))
    return "\n".join(out) + "\n"


def read_maps_table(text: str, band_width: int = 32) -> list[SeamMaps]:
    """Parse write_maps_table output (exposure.py:466-493); ValueError on a
    missing or unknown version line."""
    lines = text.strip().splitlines()
    if not lines or lines[0] != f"# {_TABLE_VERSION}":
        raise ValueError("missing or unknown exposure table version")
    table: dict = {}
    for ln in lines[1:]:
        if not ln or ln.startswith("#"):
            continue
        sid_s, side_s, k_s, ch, a_s, b_s = ln.split()
        lo, hi = (int(v) for v in sid_s.split("-"))
        table.setdefault(((lo, hi), Side(side_s)), []).append(
            (int(k_s), CHANNELS.index(ch), float(a_s), float(b_s)))
    sides: dict = {}
    for (sid, side), rows in table.items():
        k = max(r[0] for r in rows) + 1
        gain, off = np.ones((k, 3)), np.zeros((k, 3))
        for bi, ci, a, b in rows:
            gain[bi, ci], off[bi, ci] = a, b
        sides.setdefault(sid, {})[side] = ExposureMap(sid, side, band_width, gain, off)
    return [SeamMaps(sides[s][Side.LEFT], sides[s][Side.RIGHT]) for s in sorted(sides)]


# ------------------------------------------------- band statistics export

_STATS_VERSION = "camarray-bandstats-v1"
_STAT_FIELDS = ("area", "valid", "sum", "sumsq", "raw_sum", "raw_sumsq")


def write_stats_table(stats, hist=None, camera_ids=None, frame_indices=None) -> str:
    """Versioned text export of K1's exact band statistics (and, when given,
    the 256-bin histograms) - the stage-1 counterpart of the maps table
    (exposure.py:448-463 is the model: a version line, one record per line,
    exact values).  stats: camx_band_stat records (B, N, 2, K) as the
    structured _lib.STAT_DTYPE array or the raw (B, N, 2, K, 112) uint8
    bytes of CorrectResult.stats; hist: uint32/int32 (B, N, 2, K, 3, 256).
    Lines:
      rec  frame camera side block area valid sum[3] sumsq[3] raw_sum[3] raw_sumsq[3]
      hist frame camera side block channel <256 counts>
    side is the reference's Side value ("left" = band at the frame's right
    edge, exposure.py:163-168); every value is an exact integer, so the
    table round-trips bit for bit.  BandStats' mean / std follow exactly
    from (valid, sum, sumsq)."""
    rec = _as_records(stats)
    B, N, _, K = rec.shape
    cams = list(camera_ids) if camera_ids is not None else list(range(N))
    frames = list(frame_indices) if frame_indices is not None else list(range(B))
    if len(cams) != N or len(frames) != B:
        raise ValueError("camera_ids / frame_indices do not match the records")
    h = None
    if hist is not None:
        if hasattr(hist, "detach"):  # torch tensor (device or host)
            hist = hist.detach().cpu().numpy()
        h = np.asarray(hist)
        h = h.view(np.uint32) if h.dtype == np.int32 else h.astype(np.uint32)
        if h.shape != (B, N, 2, K, 3, 256):
            raise ValueError(f"histograms must be {(B, N, 2, K, 3, 256)}, got {h.shape}")
    sides = (Side.LEFT.value, Side.RIGHT.value)
    out = [f"# {_STATS_VERSION}", f"# frames {B} cameras {N} blocks {K} histograms "
           f"{'yes' if h is not None else 'no'}",
           "# rec frame camera side block area valid sum[rgb] sumsq[rgb] raw_sum[rgb] "
           "raw_sumsq[rgb]", "# hist frame camera side block channel counts[256]"]
    for b in range(B):
        for n in range(N):
            for s in range(2):
                for k in range(K):
                    r = rec[b, n, s, k]
                    vals = [int(r["area"]), int(r["valid"])]
                    for f in _STAT_FIELDS[2:]:
                        vals.extend(int(v) for v in r[f])
                    out.append(f"rec {frames[b]} {cams[n]} {sides[s]} {k} " +
                               " ".join(map(str, vals)))
                    if h is not None:
                        for c in range(3):
                            out.append(f"hist {frames[b]} {cams[n]} {sides[s]} {k} "
                                       f"{CHANNELS[c]} " + " ".join(map(str, h[b, n, s, k, c])))
    return "\n".join(out) + "\n"


def read_stats_table(text: str):
    """Parse write_stats_table output -> (records (B, N, 2, K) _lib.STAT_DTYPE,
    histograms uint32 (B, N, 2, K, 3, 256) or None, camera_ids,
    frame_indices).  ValueError on a missing / unknown version line or a
    malformed record."""
    lines = text.strip().splitlines()
    if not lines or lines[0] != f"# {_STATS_VERSION}":
        raise ValueError("missing or unknown band statistics table version")
    recs, hists = {}, {}
    for ln in lines[1:]:
        if not ln or ln.startswith("#"):
            continue
        parts = ln.split()
        key = (int(parts[1]), int(parts[2]), Side(parts[3]), int(parts[4]))
        if parts[0] == "rec":
            if len(parts) != 19:
                raise ValueError(f"malformed record line: {ln[:60]}")
            recs[key] = [int(v) for v in parts[5:]]
        elif parts[0] == "hist":
            if len(parts) != 262:
                raise ValueError(f"malformed histogram line: {ln[:60]}")
            hists[key + (CHANNELS.index(parts[5]),)] = [int(v) for v in parts[6:]]
        else:
            raise ValueError(f"unknown line kind {parts[0]!r}")
    frames = sorted({k[0] for k in recs})
    cams = sorted({k[1] for k in recs})
    K = max(k[3] for k in recs) + 1 if recs else 0
    rec = np.zeros((len(frames), len(cams), 2, K), dtype=_lib.STAT_DTYPE)
    fi = {f: i for i, f in enumerate(frames)}
    ci = {c: i for i, c in enumerate(cams)}
    si = {Side.LEFT: 0, Side.RIGHT: 1}
    for (f, c, s, k), v in recs.items():
        r = rec[fi[f], ci[c], si[s], k]
        r["area"], r["valid"] = v[0], v[1]
        for j, name in enumerate(_STAT_FIELDS[2:]):
            r[name] = v[2 + 3 * j: 5 + 3 * j]
    if len(recs) != rec.size:
        raise ValueError("band statistics table is missing records")
    h = None
    if hists:
        h = np.zeros((len(frames), len(cams), 2, K, 3, 256), dtype=np.uint32)
        for (f, c, s, k, ch), v in hists.items():
            h[fi[f], ci[c], si[s], k, ch] = v
    return rec, h, cams, frames


def _as_records(stats) -> np.ndarray:
    a = stats
    if hasattr(a, "detach"):  # torch tensor (device or host)
        a = a.detach().cpu().numpy()
    a = np.asarray(a)
    if a.dtype == _lib.STAT_DTYPE:
        return a
    if a.dtype == np.uint8 and a.shape[-1] == _lib.STAT_BYTES:
        return np.ascontiguousarray(a).view(_lib.STAT_DTYPE)[..., 0]
    raise ValueError("stats must be camx_band_stat records (STAT_DTYPE or (..., 112) bytes)")
