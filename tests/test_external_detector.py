"""ExternalDetector: the reference's socket wire protocol (detect.py:252-349)
against a fake detector process, on CPU; and detect_tiles feeding a tile
batch.  When the reference package is importable here, its own
ExternalDetector is run against the same fake server and must give the same
detections."""
import socket
import threading
import time

import numpy as np
import pytest

from paper_1910_03517_b200 import core, detect


def _read_line(conn):
    buf = b""
    while not buf.endswith(b"\n"):
        c = conn.recv(1)
        if not c:
            raise OSError("closed")
        buf += c
    return buf[:-1].decode()


def _recv_exact(conn, n):
    out = bytearray()
    while len(out) < n:
        c = conn.recv(n - len(out))
        if not c:
            raise OSError("closed")
        out += c
    return bytes(out)


class FakeDetector:
    """Replies with boxes derived from the request: a 'vehicle' box at crop-local
    (w/4, h/4, w/2, h/2) with p from the crop's mean red value, a box of an
    unknown category (dropped by the adapter), and one below the confidence
    gate.  mode='slow' misses the deadline; mode='err' answers ERR."""

    def __init__(self, mode="ok"):
        self.mode = mode
        self.srv = socket.socket(socket.AF_INET, socket.SOCK_STREAM)
        self.srv.bind(("127.0.0.1", 0))
        self.srv.listen(4)
        self.address = self.srv.getsockname()
        self.requests = []
        threading.Thread(target=self._serve, daemon=True).start()

    def _serve(self):
        while True:
            try:
                conn, _ = self.srv.accept()
            except OSError:
                return
            threading.Thread(target=self._client, args=(conn,), daemon=True).start()

    def _client(self, conn):
        try:
            while True:
                head = _read_line(conn).split()
                assert head[:2] == ["DETECT", "v1"]
                x, y, size, w, h = map(int, head[2:])
                assert _read_line(conn) == "P6"
                assert _read_line(conn).split() == [str(w), str(h)]
                assert _read_line(conn) == "255"
                px = np.frombuffer(_recv_exact(conn, w * h * 3), np.uint8).reshape(h, w, 3)
                self.requests.append((x, y, size, w, h))
                if self.mode == "slow":
                    time.sleep(0.3)
                if self.mode == "err":
                    conn.sendall(b"ERR busy\n")
                    continue
                p = 0.7 + 0.3 * float(px[..., 0].mean()) / 255.0
                rows = [f"vehicle {w / 4} {h / 4} {w / 2} {h / 2} {p:.6f}",
                        f"unicorn 1 1 2 2 0.99",
                        f"person 0 0 3 3 0.10"]
                conn.sendall(("OK %d\n" % len(rows) + "".join(r + "\n" for r in rows)).encode())
        except OSError:
            conn.close()

    def close(self):
        self.srv.close()


def _mosaic(seed=0, h=120, w=300):
    px = np.random.default_rng(seed).integers(0, 256, (h, w, 3), dtype=np.uint8)
    return core.Mosaic(frame_index=7, timestamp_ms=0, camera_ids=(0, 1), frame_width=w // 2,
                       pixels=px)


def test_detect_matches_protocol_and_reference():
    srv = FakeDetector()
    m = _mosaic()
    det = detect.ExternalDetector(srv.address, deadline_s=2.0)
    wins = [detect.DetectorWindow(10, 20, 64), detect.DetectorWindow(260, 80, 64)]  # 2nd clipped
    got = [det.detect(w, m) for w in wins]
    assert not det.degraded
    assert srv.requests[0] == (10, 20, 64, 64, 64) and srv.requests[1] == (260, 80, 64, 40, 40)
    for w, dets in zip(wins, got):
        assert len(dets) == 1 and dets[0].category is core.Category.VEHICLE
        assert dets[0].source is detect.DetectionSource.EXTERNAL and dets[0].frame_index == 7
    assert got[0][0].bbox == core.BBox(10 + 16.0, 20 + 16.0, 32.0, 32.0)
    det.close()
    import sys
    from pathlib import Path
    ref_src = Path("/root/reference/pkg/src")  # present in the build container only
    if ref_src.exists() and str(ref_src) not in sys.path:
        sys.path.append(str(ref_src))
    try:
        from camarray import detect as rdet
        from camarray.core import Mosaic as RMosaic
    except ImportError:
        return  # reference not importable (GPU box): protocol checks above stand
    rd = rdet.ExternalDetector(srv.address, deadline_s=2.0)
    rm = RMosaic(frame_index=7, timestamp_ms=0, camera_ids=(0, 1), frame_width=m.frame_width,
                 pixels=m.pixels)
    for w, dets in zip(wins, got):
        want = rd.detect(rdet.DetectorWindow(w.x, w.y, w.size), rm)
        assert [(d.category.value, d.bbox.x, d.bbox.y, d.bbox.w, d.bbox.h, d.probability)
                for d in want] == [(d.category.value, d.bbox.x, d.bbox.y, d.bbox.w, d.bbox.h,
                                    d.probability) for d in dets]
    rd.close()
    srv.close()


def test_detect_tiles_scales_back_to_mosaic():
    srv = FakeDetector()
    det = detect.ExternalDetector(srv.address, deadline_s=2.0)
    tiles = np.full((2, 16, 16, 3), 200, np.uint8)  # two 64-px windows resized to 16
    wins = [(0, 0, 64), (100, 10, 64)]
    out = det.detect_tiles(wins, tiles, frame_index=3, mosaic_w=300, mosaic_h=120)
    assert [r[2:] for r in srv.requests] == [(64, 16, 16), (64, 16, 16)]
    assert out[1][0].bbox == core.BBox(100 + 4 * 4.0, 10 + 4 * 4.0, 8 * 4.0, 8 * 4.0)
    det.close()
    srv.close()


@pytest.mark.parametrize("mode", ["slow", "err"])
def test_missed_deadline_or_error_degrades(mode):
    srv = FakeDetector(mode)
    det = detect.ExternalDetector(srv.address, deadline_s=0.05)
    assert det.detect(detect.DetectorWindow(0, 0, 32), _mosaic()) == []
    assert det.degraded
    det.close()
    srv.close()
