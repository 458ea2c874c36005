"""Generate the golden fixtures by running the REAL reference package.

Run here (the build container), where the reference is mounted read-only:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports `camarray` (the reference, arXiv 1910.03517 remote-tower
package) and records its outputs on seeded inputs into small compressed
.npz files next to this script.  The reference does not exist on the GPU
box; the fixtures travel instead.  They pin (1) the numpy oracle in
`oracle/` (tests/test_oracle_golden.py) and (2) the CUDA path
(tests/test_gpu_parity.py).
"""

from __future__ import annotations

import math
import os
import sys
from pathlib import Path

import numpy as np

REF = os.environ.get("CAMARRAY_REF", "/root/reference/pkg/src")
if REF not in sys.path:
    sys.path.insert(0, REF)

from camarray import exposure as xp                    # noqa: E402
from camarray.attention import difference_plan, sliding_window_plan  # noqa: E402
from camarray.core import Category, Frame, mask_diff  # noqa: E402
from camarray.scenegen import (ExposureDistortion, Scenario, SceneObject,  # noqa: E402
                               render_tick)
from camarray.world3d import CameraModel              # noqa: E402

OUT = Path(__file__).resolve().parent
MODES = {"standard": xp.ExposureMode.STANDARD,
         "object_removal": xp.ExposureMode.OBJECT_REMOVAL,
         "smoothing": xp.ExposureMode.SMOOTHING}


def frame(px, cam=0, idx=0):
    return Frame(cam, idx, 0, np.ascontiguousarray(px, dtype=np.uint8))


def scenario(n, width, height, seed, distort_all, objects=(), drift=0.0):
    hfov = math.pi / 3 if n <= 2 else 2 * math.pi / max(n, 7)
    cams = [CameraModel(camera_id=k, position=(0.0, 0.0, 50.0), yaw=k * hfov,
                        pitch=0.0, roll=0.0, hfov=hfov, width=width, height=height)
            for k in range(n)]
    dist = {}
    for k in range(n):
        if k == 0 and not distort_all:
            continue
        r = np.random.default_rng(1000 + k)
        dist[k] = ExposureDistortion(gain=tuple(r.uniform(0.5, 2.0, 3)),
                                     offset=tuple(r.uniform(-40.0, 40.0, 3)),
                                     drift_amplitude=drift * (k + 1), drift_period=20.0)
    return Scenario(seed=seed, tick_rate=30.0, duration=60, cameras=cams,
                    distortions=dist, objects=list(objects))


def small_cases():
    rng = np.random.default_rng(20191008)
    d = {}
    # ---- band_stats: shapes, sides, masks (exposure.py:152-185)
    bs = []
    for i, (h, w, bw, k) in enumerate([(32, 64, 8, 4), (17, 18, 4, 3), (48, 40, 16, 5),
                                       (96, 128, 32, 16), (30, 22, 11, 7), (5, 6, 3, 5)]):
        px = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        if i == 1:
            px[:] = 77          # constant image: sigma exactly 0
        m = rng.random((h, w)) > 0.6 if i % 2 == 0 else None
        for side in (xp.Side.LEFT, xp.Side.RIGHT):
            s = xp.band_stats(frame(px), side, bw, k, m)
            bs.append(dict(px=px, mask=m, bw=bw, k=k, side=side.value,
                           mean=s.mean, std=s.std, valid=s.valid_count, area=s.band_area))
    d["band_stats"] = bs
    # ---- fit_affine on float moments (exposure.py:188-229)
    fa = []
    for i in range(12):
        k = int(rng.integers(1, 6))
        mk = lambda: rng.uniform(20, 230, (k, 3))                      # noqa: E731
        sd = lambda: np.where(rng.random((k, 3)) < 0.2, rng.uniform(0, 2e-3, (k, 3)),  # noqa: E731
                              rng.uniform(0.5, 40, (k, 3)))
        cnt = lambda: rng.integers(0, 200, k).astype(np.int64)         # noqa: E731
        L = xp.BandStats(mk(), sd(), cnt(), np.full(k, 200, np.int64))
        R = xp.BandStats(mk(), sd(), cnt(), np.full(k, 200, np.int64))
        lm, rm, ok = xp.fit_affine(L, R, sigma_min=1e-3, min_band_pixels=64)
        fa.append(dict(lmean=L.mean, lstd=L.std, lvalid=L.valid_count,
                       rmean=R.mean, rstd=R.std, rvalid=R.valid_count,
                       gl=lm.gain, ol=lm.offset, gr=rm.gain, orr=rm.offset, ok=ok))
    d["fit_affine"] = fa
    # ---- apply_exposure (exposure.py:385-401): odd/even widths, both sides
    ap = []
    for (h, w, k) in [(16, 9, 2), (12, 16, 3), (6, 8, 1), (31, 27, 4), (48, 64, 16),
                      (40, 2048 // 16, 8), (7, 5, 7), (33, 60, 5)]:
        px = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        for side in (xp.Side.LEFT, xp.Side.RIGHT):
            g = rng.uniform(0.3, 2.5, (k, 3))
            b = rng.uniform(-60, 60, (k, 3))
            if h == 6:
                g[:] = 2.0
                b[:] = 0.0
            em = xp.ExposureMap((0, 1), side, 4, g, b)
            out = xp.apply_exposure(frame(px), em).pixels
            ap.append(dict(px=px, side=side.value, gain=g, offset=b, out=out))
    d["apply"] = ap
    # ---- mask_diff (core.py:191-196)
    md = []
    for (h, w, t) in [(6, 8, 20), (13, 7, 0), (32, 32, 50), (9, 11, 254)]:
        a = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        b = np.clip(a.astype(int) + rng.integers(-40, 41, a.shape), 0, 255).astype(np.uint8)
        md.append(dict(a=a, b=b, t=t, out=mask_diff(a, b, t)))
    d["mask_diff"] = md
    # ---- sliding_window_plan / difference_plan (attention.py:53-103)
    sw = []
    for (w, h, s, ov) in [(1920, 1080, 960, 0.0), (960, 960, 960, 0.0), (1920, 960, 960, 0.5),
                          (500, 300, 128, 0.25), (16384, 1536, 960, 0.0),
                          (16384, 1536, 416, 0.0), (53760, 2160, 960, 0.0), (300, 300, 100, 0.0),
                          (1280, 480, 416, 0.0), (777, 555, 111, 0.3)]:
        reqs = sliding_window_plan((w, h), s, ov)
        sw.append(dict(w=w, h=h, s=s, ov=ov,
                       xy=np.array([(r.window.x, r.window.y) for r in reqs], dtype=np.int64)))
    d["sliding"] = sw
    dp = []
    for (h, w, s, thr, p) in [(300, 500, 128, 50, 0.002), (256, 256, 256, 50, 0.0008),
                              (128, 256, 128, 50, 0.01), (480, 1280, 416, 50, 0.0004),
                              (192, 640, 64, 10, 0.003)]:
        m = rng.random((h, w)) < p
        m[10:20, 30:40] = True
        plan = difference_plan(m, s, thr)
        dp.append(dict(mask=m, s=s, thr=thr,
                       plan=np.array([(r.window.x, r.window.y, r.priority) for r in plan],
                                     dtype=np.int64).reshape(-1, 3)))
    d["difference"] = dp
    # ---- seam_cost (exposure.py:417-445)
    sc = []
    for (h, wl, wr, f) in [(64, 64, 64, 8), (32, 24, 40, 4), (16, 16, 16, 1), (50, 33, 35, 3)]:
        a = rng.integers(0, 256, (h, wl, 3), dtype=np.uint8)
        b = rng.integers(0, 256, (h, wr, 3), dtype=np.uint8)
        sc.append(dict(a=a, b=b, f=f, cost=xp.seam_cost(a, b, f)))
    d["seam_cost"] = sc
    return d


def scene_cases():
    """Tick loops over a reference scenegen scene for all three modes: a
    2-camera and a 3-camera array with a moving object crossing a seam."""
    out = {}
    def crossing(oid, az0, az1, dist, size, height):
        a0, a1 = math.radians(az0), math.radians(az1)
        return SceneObject(oid, Category.AIRCRAFT, size,
                           ((0.0, dist * math.sin(a0), dist * math.cos(a0), height),
                            (0.6, dist * math.sin(a1), dist * math.cos(a1), height)))

    for n, (w, h) in [(2, (256, 192)), (3, (160, 120))]:
        hfov = 60.0 if n <= 2 else 360.0 / 7
        seam = hfov / 2
        objs = [crossing(1, seam - 12, seam + 12, 150.0, (60.0, 30.0), 40.0),
                crossing(2, seam + hfov + 9, seam + hfov - 9, 400.0, (20.0, 10.0), 55.0)]
        sc = scenario(n, w, h, seed=100 + n, distort_all=True, objects=objs, drift=6.0)
        ticks = [render_tick(sc, t)[0] for t in range(0, 20, 5)]
        frames = np.stack([np.stack([f.pixels for f in tk]) for tk in ticks])  # (T,N,H,W,3)
        cfg = xp.ExposureConfig(band_width=16, blocks=8, min_band_pixels=64)
        res = {"frames": frames, "band_width": 16, "blocks": 8}
        for name, mode in MODES.items():
            prev_maps = [None] * (n - 1)
            prev_tick = None
            g_all, o_all, corr = [], [], []
            for tk in ticks:
                gs, os_, maps = [], [], []
                for s in range(n - 1):
                    pf = None if prev_tick is None else (prev_tick[s], prev_tick[s + 1])
                    sm = xp.update_exposure((tk[s], tk[s + 1]), prev_maps[s], mode, cfg, pf)
                    maps.append(sm)
                    gs.append([sm.left.gain, sm.right.gain])
                    os_.append([sm.left.offset, sm.right.offset])
                cams = []
                for c in range(n):
                    f = tk[c]
                    if c < n - 1:
                        f = xp.apply_exposure(f, maps[c].left)
                    if c >= 1:
                        f = xp.apply_exposure(f, maps[c - 1].right)
                    cams.append(f.pixels)
                corr.append(np.stack(cams))
                g_all.append(gs)
                o_all.append(os_)
                prev_maps = maps
                prev_tick = tk
            res[f"{name}_gain"] = np.array(g_all)
            res[f"{name}_offset"] = np.array(o_all)
            res[f"{name}_out"] = np.stack(corr)
        out[f"n{n}"] = res
    return out


def config1_case():
    """BASELINE config 1: 2 cameras 640x480, default ExposureConfig, STANDARD."""
    sc = scenario(2, 640, 480, seed=100, distort_all=False)
    sc.distortions[1] = ExposureDistortion(gain=(1.4, 0.8, 1.1), offset=(-12.0, 18.0, 4.0))
    f0, f1 = render_tick(sc, 0)[0]
    maps = xp.update_exposure((f0, f1), None)
    a = xp.apply_exposure(f0, maps.left).pixels
    b = xp.apply_exposure(f1, maps.right).pixels
    return dict(frames=np.stack([f0.pixels, f1.pixels]), out=np.stack([a, b]),
                gain=np.stack([maps.left.gain, maps.right.gain]),
                offset=np.stack([maps.left.offset, maps.right.offset]),
                cost_before=xp.seam_cost(f0, f1), cost_after=xp.seam_cost(a, b))


def flatten(prefix, obj, into):
    if isinstance(obj, dict):
        for k, v in obj.items():
            flatten(f"{prefix}.{k}" if prefix else k, v, into)
    elif isinstance(obj, list):
        into[f"{prefix}.__len__"] = np.array(len(obj))
        for i, v in enumerate(obj):
            flatten(f"{prefix}.{i}", v, into)
    elif obj is None:
        into[f"{prefix}.__none__"] = np.array(0)
    else:
        into[prefix] = np.asarray(obj)


def main():
    small = {}
    flatten("", small_cases(), small)
    np.savez_compressed(OUT / "golden_small.npz", **small)
    scene = {}
    flatten("", scene_cases(), scene)
    np.savez_compressed(OUT / "golden_scene.npz", **scene)
    c1 = {}
    flatten("", config1_case(), c1)
    np.savez_compressed(OUT / "golden_config1.npz", **c1)
    text_maps = []
    r = np.random.default_rng(7)
    for seam in [(0, 1), (1, 2)]:
        lm = xp.ExposureMap(seam, xp.Side.LEFT, 32, r.uniform(0.5, 2, (4, 3)), r.uniform(-40, 40, (4, 3)))
        rm = xp.ExposureMap(seam, xp.Side.RIGHT, 32, r.uniform(0.5, 2, (4, 3)), r.uniform(-40, 40, (4, 3)))
        text_maps.append(xp.SeamMaps(lm, rm))
    (OUT / "maps_table.txt").write_text(xp.write_maps_table(text_maps))
    for p in sorted(OUT.glob("golden_*.npz")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
