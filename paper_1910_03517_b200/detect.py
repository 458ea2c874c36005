"""Detector-input side of the tile path: `DetectorWindow` (reference
detect.py:60-72) and the batched tile crop/resize (the crop of
ExternalDetector.detect, detect.py:297-300, plus the builder-defined
resize to the detector input size) on the GPU (K5).

The detectors themselves (nms, Oracle/Blob/External detectors) consume
tiles and are out of scope ("tile consumer").
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .core import BBox, Mosaic

__all__ = ["DetectorWindow", "crop_window", "tiles", "encode_ppm", "encode_ppm_tiles",
           "detect_requests"]


@dataclass(frozen=True)
class DetectorWindow:
    """Square detector input region in mosaic coordinates (detect.py:60-72)."""

    x: int
    y: int
    size: int

    def as_bbox(self) -> BBox:
        return BBox(self.x, self.y, self.size, self.size)

    def contains_point(self, px: float, py: float) -> bool:
        return (self.x <= px < self.x + self.size) and (self.y <= py < self.y + self.size)


def _check_windows(wins, size, mosaic_w, mosaic_h):
    for (_, x, y) in wins:
        if x < 0 or y < 0 or x + size > mosaic_w or y + size > mosaic_h:
            raise ValueError(f"window ({x}, {y}, {size}) not inside the {mosaic_w}x{mosaic_h} mosaic")


def tiles(images, windows, size: int, out_size: int = 416, *, stream=None, out=None):
    """Crop + resize windows of a device-resident array (K5).

    images: uint8 CUDA tensor (B, N, H, W, 3) — the virtual mosaic of each
    array-frame is its N cameras side by side.  windows: iterable of
    (batch_index, x, y) or DetectorWindow (batch 0).  Returns a uint8 CUDA
    tensor (T, out_size, out_size, 3)."""
    t = _dev.require_cuda()
    if images.dim() == 4:
        images = images[None]
    B, N, H, W = images.shape[:4]
    wins = [(0, w.x, w.y) if isinstance(w, DetectorWindow) else tuple(int(v) for v in w)
            for w in windows]
    for w in windows:
        if isinstance(w, DetectorWindow) and w.size != size:
            raise ValueError("all windows of one batch share the window size")
    _check_windows(wins, size, N * W, H)
    for (b, _, _) in wins:
        if not 0 <= b < B:
            raise ValueError(f"batch index {b} outside [0, {B})")
    T = len(wins)
    res = out if out is not None else t.empty((T, out_size, out_size, 3), dtype=t.uint8,
                                              device="cuda")
    if T == 0:
        return res
    wd = _dev.to_device(np.asarray(wins, dtype=np.int32).reshape(T, 3))
    _lib.call("camx_tiles", images.data_ptr(), N, H, W, wd.data_ptr(), T, int(size),
              int(out_size), res.data_ptr(), _dev.stream_handle(stream))
    return res


def crop_window(mosaic: Mosaic, window: DetectorWindow, out_size: int | None = None) -> np.ndarray:
    """The contiguous (S, S, 3) crop ExternalDetector sends (detect.py:297-300),
    optionally resized to out_size; computed on the GPU from the mosaic."""
    px = mosaic.pixels
    h, w = px.shape[:2]
    y0, x0 = max(window.y, 0), max(window.x, 0)
    y1, x1 = min(window.y + window.size, h), min(window.x + window.size, w)
    if (y1 - y0, x1 - x0) != (window.size, window.size):
        if out_size not in (None, window.size):
            raise ValueError("resize needs a window fully inside the mosaic")
        # clipped crop at the mosaic border: exact slice, as the reference
        img = _dev.to_device(np.ascontiguousarray(px[y0:y1, x0:x1]))[None, None]
        return _dev.to_host(img[0, 0]).copy()
    img = _dev.to_device(px)[None, None]
    res = tiles(img, [(0, window.x, window.y)], window.size,
                window.size if out_size is None else out_size)
    return _dev.to_host(res[0])


# ------------------------------------------------ tile wire format
# The detector consumes tiles as netpbm P6 payloads (imgio.encode_ppm,
# imgio.py:14-18) framed by ExternalDetector's request line (detect.py:252-301):
#   "DETECT v1 <x> <y> <size> <w> <h>\n" + PPM bytes of the crop.

def encode_ppm(pixels) -> bytes:
    """P6 payload of one (H, W, 3) uint8 image (header + raw RGB rows)."""
    px = np.asarray(pixels)
    if px.ndim != 3 or px.shape[2] != 3 or px.dtype != np.uint8:
        raise ValueError("PPM payload must be (H, W, 3) uint8")
    return b"P6\n%d %d\n255\n" % (px.shape[1], px.shape[0]) + np.ascontiguousarray(px).tobytes()


def encode_ppm_tiles(tile_batch) -> list[bytes]:
    """P6 payloads of a (T, S, S, 3) tile batch.  A CUDA batch is brought to
    the host in ONE copy (the tiles are already the payload bytes: a P6 body
    is raw row-major RGB), then each payload is header + a slice."""
    t = _dev.torch()
    if isinstance(tile_batch, t.Tensor):
        host = tile_batch.detach().to("cpu", non_blocking=False).numpy()
    else:
        host = np.asarray(tile_batch)
    if host.ndim != 4 or host.shape[-1] != 3 or host.dtype != np.uint8:
        raise ValueError("tile batch must be (T, H, W, 3) uint8")
    head = b"P6\n%d %d\n255\n" % (host.shape[2], host.shape[1])
    return [head + host[i].tobytes() for i in range(host.shape[0])]


def detect_requests(windows, tile_batch) -> list[bytes]:
    """Full wire requests (header line + PPM) for windows and their tiles, as
    ExternalDetector.detect would send them (detect.py:297-301); the tile's
    own dimensions (resized or not) are the reported crop size."""
    payloads = encode_ppm_tiles(tile_batch)
    if len(payloads) != len(windows):
        raise ValueError("one tile per window")
    out = []
    for w, ppm in zip(windows, payloads):
        x, y, size = (w.x, w.y, w.size) if isinstance(w, DetectorWindow) else w
        dims = ppm.split(b"\n", 2)[1].split()
        out.append(b"DETECT v1 %d %d %d %s %s\n" % (x, y, size, dims[0], dims[1]) + ppm)
    return out
