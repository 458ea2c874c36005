"""Detector-input side of the tile path: `DetectorWindow` (reference
detect.py:60-72) and the batched tile crop/resize (the crop of
ExternalDetector.detect, detect.py:297-300, plus the builder-defined
resize to the detector input size) on the GPU (K5).

Tile consumers: nms, the motion-blob detector (GPU connected
components) and the external-detector wire adapter (`ExternalDetector`,
plus `detect_tiles` feeding it whole device tile batches).  The
ground-truth OracleDetector projects the scene generator's 3-D objects
(world3d) and stays out of scope.
"""

from __future__ import annotations

import abc
import enum
import socket
import threading
from dataclasses import dataclass, replace

import numpy as np

from . import _dev, _lib
from .core import BBox, Category, Mosaic, iou

__all__ = ["DetectorWindow", "crop_window", "tiles", "encode_ppm", "encode_ppm_tiles",
           "detect_requests", "Detection", "DetectionSource", "Detector", "BlobDetector",
           "ExternalDetector", "nms", "TOL_DETECT", "TOL_NMS"]


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


# ------------------------------------------------ motion-blob detector

TOL_DETECT = 0.65   # detect.py:35
TOL_NMS = 0.45      # detect.py:36


class DetectionSource(enum.Enum):
    ORACLE = "oracle"
    BLOB = "blob"
    EXTERNAL = "external"


@dataclass(frozen=True)
class Detection:
    """Classified box in mosaic coordinates with confidence (detect.py:45-57)."""

    category: Category
    bbox: BBox
    probability: float
    frame_index: int
    source: DetectionSource

    def __post_init__(self) -> None:
        if not (0.0 <= self.probability <= 1.0):
            raise ValueError(f"probability {self.probability} outside [0, 1]")


def nms(dets: list[Detection], tol_nms: float = TOL_NMS) -> list[Detection]:
    """Greedy per-category suppression, highest probability first, ties by
    input order (detect.py:75-95).  Host logic on a handful of boxes."""
    order = sorted(range(len(dets)), key=lambda i: (-dets[i].probability, i))
    dead = set()
    kept = []
    for i in order:
        if i in dead:
            continue
        kept.append(dets[i])
        dead.update(j for j in order if j != i and j not in dead
                    and dets[j].category is dets[i].category
                    and iou(dets[j].bbox, dets[i].bbox) > tol_nms)
    return kept


def _finalize(dets, mosaic_w, mosaic_h, tol_detect, tol_nms):
    """Clip to the mosaic, confidence gate, NMS (detect.py:104-114)."""
    keep = []
    for d in dets:
        box = d.bbox.clipped(mosaic_w, mosaic_h)
        if box.area > 0 and d.probability > tol_detect:
            keep.append(replace(d, bbox=box))
    return nms(keep, tol_nms)


def blob_components(mask, window: DetectorWindow, n_cams: int = 1, max_comp: int = 4096,
                    stream=None):
    """8-connected components of the motion mask inside `window` (GPU,
    camx_blob_components).  mask: (n_cams, H, W) (or (H, W)) bool/uint8,
    numpy or CUDA; the mosaic of the n_cams masks is virtual.  Returns an
    int array (n, 6): raster index of the first pixel, xmin, ymin, xmax,
    ymax (window coordinates, inclusive), on-pixels inside the box - in
    scipy.ndimage.label order."""
    t = _dev.require_cuda()
    m = mask if isinstance(mask, t.Tensor) else _dev.to_device(
        np.asarray(mask, dtype=bool).view(np.uint8))
    if m.dtype == t.bool:
        m = m.view(t.uint8)
    m = m.reshape(n_cams, *m.shape[-2:]).contiguous()
    H, W = m.shape[-2:]
    S = int(window.size)
    scratch = t.empty((6 * S * S + 2 * S + 1 + (S * S + 1023) // 1024 + 3,), dtype=t.int32,
                      device="cuda")
    comp = t.empty((max_comp, 6), dtype=t.int32, device="cuda")
    n = t.zeros((1,), dtype=t.int32, device="cuda")
    _lib.call("camx_blob_components", m.data_ptr(), int(n_cams), int(H), int(W), int(window.x),
              int(window.y), S, scratch.data_ptr(), comp.data_ptr(), int(max_comp), n.data_ptr(),
              _dev.stream_handle(stream))
    count = int(n.item())
    if count > max_comp:
        return blob_components(mask, window, n_cams, count, stream)
    return _dev.to_host(comp[:count])


class Detector(abc.ABC):
    """Detections in one window of one mosaic tick (detect.py:117-129)."""

    @abc.abstractmethod
    def detect(self, window: DetectorWindow, mosaic: Mosaic) -> list[Detection]:
        ...


class BlobDetector(Detector):
    """Motion-blob detector (detect.py:192-249): connected components of the
    frame-difference mask of consecutive mosaics, one detection per
    component of at least `min_area` on-pixels (counted over its box, as
    the reference).  The mask and the components are computed on the GPU."""

    def __init__(self, *, t_diff: int = 20, min_area: int = 4,
                 category: Category = Category.VEHICLE, p_saturation_area: float = 400.0,
                 tol_detect: float = TOL_DETECT, tol_nms: float = TOL_NMS):
        self.t_diff = t_diff
        self.min_area = min_area
        self.category = category
        self.p_saturation_area = p_saturation_area
        self.tol_detect = tol_detect
        self.tol_nms = tol_nms
        self._lock = threading.Lock()
        self._prev = None          # previous mosaic pixels on the device
        self._prev_index = None
        self._mask = None          # (H, W) uint8 CUDA mask of this tick
        self._mask_index = None

    def _mask_for(self, mosaic: Mosaic):
        t = _dev.require_cuda()
        with self._lock:
            if self._mask_index == mosaic.frame_index:
                return self._mask
            cur = _dev.to_device(mosaic.pixels)
            mask = None
            if self._prev is not None and self._prev_index < mosaic.frame_index:
                if self._prev.shape != cur.shape:
                    raise ValueError("pixel dimensions differ")
                h, w = cur.shape[:2]
                mask = t.empty((h, w), dtype=t.uint8, device="cuda")
                _lib.call("camx_mask_diff", cur.data_ptr(), self._prev.data_ptr(), h * w,
                          int(self.t_diff), mask.data_ptr(), _dev.stream_handle())
            self._prev, self._prev_index = cur, mosaic.frame_index
            self._mask, self._mask_index = mask, mosaic.frame_index
            return mask

    def detect(self, window: DetectorWindow, mosaic: Mosaic) -> list[Detection]:
        mask = self._mask_for(mosaic)
        if mask is None:
            return []
        x0, y0 = max(window.x, 0), max(window.y, 0)
        x1 = min(window.x + window.size, mosaic.width)
        y1 = min(window.y + window.size, mosaic.height)
        if x1 - x0 != y1 - y0:  # clipped non-square window: label the exact slice
            sub = mask[y0:y1, x0:x1].contiguous()
            side = max(x1 - x0, y1 - y0)
            pad = _dev.torch().zeros((side, side), dtype=sub.dtype, device="cuda")
            pad[: y1 - y0, : x1 - x0] = sub
            comps = blob_components(pad, DetectorWindow(0, 0, side))
        else:
            comps = blob_components(mask, DetectorWindow(x0, y0, x1 - x0))
        dets = []
        for _, bx0, by0, bx1, by1, area in comps:
            if area < self.min_area:
                continue
            box = BBox(x0 + int(bx0), y0 + int(by0), int(bx1 - bx0 + 1), int(by1 - by0 + 1))
            p = min(1.0, 0.66 + 0.34 * min(1.0, int(area) / self.p_saturation_area))
            dets.append(Detection(self.category, box, p, mosaic.frame_index,
                                  DetectionSource.BLOB))
        return _finalize(dets, mosaic.width, mosaic.height, self.tol_detect, self.tol_nms)


class ExternalDetector(Detector):
    """Adapter to an external detector process over a local socket, the
    reference's wire protocol (detect.py:252-349): per request
      -> "DETECT v1 <x> <y> <size> <w> <h>\n" + P6 bytes of the crop
      <- "OK <n>\n" + n lines "<category> <x> <y> <w> <h> <p>" (crop-local
         coordinates) or "ERR <message>\n".
    A missed deadline or a broken connection gives an empty result and sets
    `degraded` (the pipeline is never blocked).  `detect` sends the window's
    crop of a host mosaic exactly as the reference; `detect_tiles` feeds a
    whole device tile batch (K5 crops / resizes: one D2H copy, then one
    request per tile) and maps the replies back to mosaic coordinates."""

    def __init__(self, address, *, deadline_s: float = 0.1,
                 tol_detect: float = TOL_DETECT, tol_nms: float = TOL_NMS):
        self.address = address
        self.deadline_s = deadline_s
        self.tol_detect = tol_detect
        self.tol_nms = tol_nms
        self.degraded = False
        self._sock = None
        self._lock = threading.Lock()

    def _connect(self):
        fam = socket.AF_UNIX if isinstance(self.address, str) else socket.AF_INET
        s = socket.socket(fam, socket.SOCK_STREAM)
        s.settimeout(self.deadline_s)
        s.connect(self.address)
        return s

    def close(self) -> None:
        with self._lock:
            self._drop()

    def _drop(self) -> None:
        if self._sock is not None:
            try:
                self._sock.close()
            finally:
                self._sock = None

    @staticmethod
    def _line(sock) -> str:
        buf = bytearray()
        while True:
            c = sock.recv(1)
            if not c:
                raise OSError("connection closed")
            if c == b"\n":
                return buf.decode()
            buf += c

    def _exchange(self, payload: bytes):
        """One request/reply; None on a missed deadline / broken peer."""
        with self._lock:
            try:
                if self._sock is None:
                    self._sock = self._connect()
                self._sock.settimeout(self.deadline_s)
                self._sock.sendall(payload)
                status = self._line(self._sock)
                if status.startswith("ERR"):
                    raise ValueError(status)
                if not status.startswith("OK "):
                    raise ValueError(f"malformed reply {status!r}")
                rows = []
                for _ in range(int(status.split()[1])):
                    f = self._line(self._sock).split()
                    rows.append((f[0], *(float(v) for v in f[1:6])))
            except (OSError, ValueError):
                self._drop()
                self.degraded = True
                return None
        self.degraded = False
        return rows

    def _to_dets(self, rows, ox, oy, scale, frame_index):
        dets = []
        for cat_s, bx, by, bw, bh, p in rows:
            try:
                cat = Category(cat_s)
            except ValueError:
                continue
            box = BBox(ox + bx * scale, oy + by * scale, bw * scale, bh * scale)
            dets.append(Detection(cat, box, min(max(p, 0.0), 1.0), frame_index,
                                  DetectionSource.EXTERNAL))
        return dets

    def detect(self, window: DetectorWindow, mosaic: Mosaic) -> list[Detection]:
        x0, y0 = max(window.x, 0), max(window.y, 0)
        x1 = min(window.x + window.size, mosaic.width)
        y1 = min(window.y + window.size, mosaic.height)
        crop = np.ascontiguousarray(mosaic.pixels[y0:y1, x0:x1])
        req = (b"DETECT v1 %d %d %d %d %d\n" % (window.x, window.y, window.size, crop.shape[1],
                                                crop.shape[0]) + encode_ppm(crop))
        rows = self._exchange(req)
        if rows is None:
            return []
        return _finalize(self._to_dets(rows, x0, y0, 1.0, mosaic.frame_index), mosaic.width,
                         mosaic.height, self.tol_detect, self.tol_nms)

    def detect_tiles(self, windows, tile_batch, *, frame_index: int, mosaic_w: int,
                     mosaic_h: int) -> list[list[Detection]]:
        """Detections of every window from its K5 tile (T, S', S', 3) - a
        crop resized to S' (or the exact crop when S' = size).  Reply
        coordinates are tile-local and scaled by size / S' back to the
        mosaic; per window: clip, confidence gate and NMS as `detect`."""
        reqs = detect_requests(windows, tile_batch)
        out = []
        for w, req in zip(windows, reqs):
            x, y, size = (w.x, w.y, w.size) if isinstance(w, DetectorWindow) else w
            side = int(req.split(b"\n", 1)[0].split()[5])
            rows = self._exchange(req)
            if rows is None:
                out.append([])
                continue
            dets = self._to_dets(rows, max(x, 0), max(y, 0), size / side, frame_index)
            out.append(_finalize(dets, mosaic_w, mosaic_h, self.tol_detect, self.tol_nms))
        return out
