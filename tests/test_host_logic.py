"""CPU tests of the host-side logic of the drop-in API (no GPU needed):
value types, window plans, expectation plan, scheduler, maps table.
Known-answer cases restate the reference's tests (pkg/tests/test_core.py,
test_attention.py, test_exposure.py) - cited per test."""

import numpy as np
import pytest
from hypothesis import given, strategies as st

from golden_io import GOLDEN, load
from paper_1910_03517_b200 import attention as at
from paper_1910_03517_b200 import exposure as xp
from paper_1910_03517_b200.core import BBox, Category, Frame, Mosaic, concat_mosaic, iou
from paper_1910_03517_b200.detect import DetectorWindow

SMALL = load("small")


class Obj:
    """Minimal tracked object (the reference's tracker.TrackedObject fields
    the attention module reads)."""

    def __init__(self, oid, entries):
        self.id = oid
        self.history = [(f, BBox(x, y, 10, 10)) for f, x, y in entries]

    @property
    def last_seen(self):
        return self.history[-1][0]


def gray(w, h, v, cam=0, idx=0):
    return Frame(cam, idx, 0, np.full((h, w, 3), v, np.uint8))


class TestValueTypes:                 # test_core.py:11-127
    def test_iou_cases(self):
        assert iou(BBox(0, 0, 4, 4), BBox(0, 0, 4, 4)) == 1.0
        assert iou(BBox(0, 0, 2, 2), BBox(10, 10, 2, 2)) == 0.0
        assert iou(BBox(0, 0, 2, 2), BBox(1, 1, 2, 2)) == pytest.approx(1.0 / 7.0)
        z = BBox(3, 3, 0, 0)
        assert iou(z, z) == 0.0 and iou(z, BBox(0, 0, 10, 10)) == 0.0
        with pytest.raises(ValueError):
            BBox(0, 0, -1, 5)

    @given(st.tuples(*[st.floats(-100, 100)] * 2, *[st.floats(0, 50)] * 2),
           st.tuples(*[st.floats(-100, 100)] * 2, *[st.floats(0, 50)] * 2))
    def test_iou_symmetric_in_range(self, t1, t2):
        v = iou(BBox(*t1), BBox(*t2))
        assert v == iou(BBox(*t2), BBox(*t1)) and 0.0 <= v <= 1.0

    def test_bbox_helpers(self):
        b = BBox(-5, 2, 20, 10)
        assert b.area == 200 and b.center == (5.0, 7.0)
        assert b.translated(5, -2) == BBox(0, 0, 20, 10)
        assert b.clipped(10, 8) == BBox(0.0, 2.0, 10.0, 6.0)

    def test_frame_checks(self):
        with pytest.raises(ValueError):
            Frame(0, 0, 0, np.zeros((4, 4), np.uint8))
        with pytest.raises(ValueError):
            Frame(0, 0, 0, np.zeros((4, 4, 3), np.float32))
        f = gray(5, 3, 1)
        assert (f.width, f.height) == (5, 3)

    def test_mosaic(self):
        m = concat_mosaic([gray(4, 3, 10, 0, 5), gray(4, 3, 20, 1, 5)])
        assert isinstance(m, Mosaic) and m.width == 8 and m.height == 3
        assert m.camera_at(0) == 0 and m.camera_at(5) == 1 and m.camera_at(99) == 1
        assert m.camera_at(-3) == 0
        assert (m.pixels[:, :4] == 10).all() and (m.pixels[:, 4:] == 20).all()
        with pytest.raises(ValueError):
            concat_mosaic([gray(4, 3, 0, idx=1), gray(4, 3, 0, idx=2)])
        with pytest.raises(ValueError):
            concat_mosaic([gray(4, 3, 0), gray(5, 3, 0)])
        with pytest.raises(ValueError):
            concat_mosaic([])

    def test_category(self):
        assert {c.value for c in Category} == {"aircraft", "vehicle", "person"}
        assert len({c.color for c in Category}) == 3
        assert Category.AIRCRAFT.color == (235, 80, 60)

    def test_window(self):
        w = DetectorWindow(10, 20, 5)
        assert w.as_bbox() == BBox(10, 20, 5, 5)
        assert w.contains_point(10, 24.9) and not w.contains_point(15, 20)


class TestPlans:                      # test_attention.py:20-51
    def test_golden_sliding(self):
        for c in SMALL["sliding"]:
            reqs = at.sliding_window_plan((int(c["w"]), int(c["h"])), int(c["s"]), float(c["ov"]))
            xy = np.array([(r.window.x, r.window.y) for r in reqs], dtype=np.int64).reshape(-1, 2)
            np.testing.assert_array_equal(xy, c["xy"])
            assert [r.priority for r in reqs] == list(range(len(reqs)))

    def test_kat(self):
        o = [(r.window.x, r.window.y) for r in at.sliding_window_plan((1920, 1080), 960)]
        assert o == [(0, 0), (960, 0), (0, 120), (960, 120)]
        assert len(at.sliding_window_plan((960, 960), 960)) == 1
        xs = sorted({r.window.x for r in at.sliding_window_plan((1920, 960), 960, 0.5)})
        assert xs == [0, 480, 960]
        with pytest.raises(ValueError):
            at.sliding_window_plan((500, 300), 512)

    def test_full_coverage(self):
        w, h, s = 500, 300, 128
        cover = np.zeros((h, w), bool)
        for r in at.sliding_window_plan((w, h), s, 0.25):
            cover[r.window.y:r.window.y + s, r.window.x:r.window.x + s] = True
        assert cover.all()

    def test_rank_windows_stable(self):
        origins = [(0, 0), (10, 0), (20, 0), (30, 0)]
        plan = at.rank_windows(origins, np.array([60, 500, 60, 10]), 10, 50)
        assert [(p.window.x, p.priority) for p in plan] == [(10, 0), (0, 1), (20, 2)]
        assert all(p.mechanism is at.Mechanism.DIFFERENCE for p in plan)


class TestExpectation:                # test_attention.py:81-121
    def test_linear_extrapolation(self):
        win = at.expectation_plan([Obj(1, [(10, 95, 95), (11, 105, 95)])], 12, 64,
                                  (1000, 1000))[0].window
        assert (win.x + 32, win.y + 32) == (120, 100)

    def test_single_observation(self):
        win = at.expectation_plan([Obj(1, [(10, 95, 95)])], 15, 64, (1000, 1000))[0].window
        assert (win.x + 32, win.y + 32) == (100, 100)

    def test_clamped(self):
        r = at.expectation_plan([Obj(1, [(10, 0, 0), (11, -20, 0)])], 20, 64, (200, 200))[0]
        assert r.window.x == 0 and 0 <= r.window.y <= 136

    def test_staleness_order(self):
        reqs = at.expectation_plan([Obj(1, [(50, 10, 10)]), Obj(2, [(30, 100, 100)])], 51, 64,
                                   (1000, 1000))
        assert [r.target_object_id for r in reqs] == [2, 1]


class TestScheduler:                  # test_attention.py:124-183
    def test_startup_spills(self):
        sched = at.Scheduler((300, 300), at.AttentionConfig(budget=3, window_size=100))
        seen = []
        for tick in range(3):
            batch = sched.schedule(frame_index=tick)
            assert len(batch) == 3
            assert all(r.mechanism is at.Mechanism.SLIDING_WINDOW for r in batch)
            seen += [(r.window.x, r.window.y) for r in batch]
        assert not sched.in_startup
        assert seen == [(x, y) for y in (0, 100, 200) for x in (0, 100, 200)]

    def test_empty_tick_and_restart(self):
        sched = at.Scheduler((128, 128), at.AttentionConfig(budget=4, window_size=128))
        sched.schedule(frame_index=0)
        assert sched.schedule(frame_index=1) == []
        sched.restart()
        assert sched.in_startup

    def test_duplicates_merged(self):
        sched = at.Scheduler((640, 64), at.AttentionConfig(budget=4, window_size=64))
        while sched.in_startup:
            sched.schedule(frame_index=0)
        batch = sched.schedule(frame_index=6, objects=[Obj(1, [(5, 100, 20)]),
                                                       Obj(2, [(5, 101, 20)])])
        assert len(batch) == 1

    def test_counts_callback_and_budget(self):
        cfg = at.AttentionConfig(budget=2, window_size=64, diff_threshold=10)
        sched = at.Scheduler((640, 64), cfg)
        while sched.in_startup:
            sched.schedule(frame_index=0)
        counts = np.zeros(10, np.int64)
        counts[[2, 4, 7]] = [100, 50, 30]
        batch = sched.schedule(frame_index=6, objects=[Obj(1, [(5, 30, 20)])],
                               window_counts_fn=lambda org, s: counts)
        assert [r.mechanism for r in batch] == [at.Mechanism.EXPECTATION, at.Mechanism.DIFFERENCE]
        assert batch[1].window.x == 128
        with pytest.raises(ValueError):
            at.Scheduler((128, 128), at.AttentionConfig(budget=0)).schedule(frame_index=0)


class TestMapsTable:                  # test_exposure.py:382-399
    def test_reference_table_round_trip(self):
        text = (GOLDEN / "maps_table.txt").read_text()
        maps = xp.read_maps_table(text)
        assert len(maps) == 2 and maps[0].left.seam_id == (0, 1)
        assert xp.write_maps_table(maps) == text

    def test_random_round_trip_exact(self):
        rng = np.random.default_rng(1234)
        maps = [xp.SeamMaps(xp.ExposureMap(s, xp.Side.LEFT, 32, rng.uniform(0.5, 2, (4, 3)),
                                           rng.uniform(-40, 40, (4, 3))),
                            xp.ExposureMap(s, xp.Side.RIGHT, 32, rng.uniform(0.5, 2, (4, 3)),
                                           rng.uniform(-40, 40, (4, 3))))
                for s in [(0, 1), (1, 2)]]
        back = xp.read_maps_table(xp.write_maps_table(maps))
        for a, b in zip(maps, back):
            assert np.array_equal(a.left.gain, b.left.gain)
            assert np.array_equal(a.right.offset, b.right.offset)
        with pytest.raises(ValueError):
            xp.read_maps_table("0-1 left 0 r 1.0 0.0\n")

    def test_map_validation(self):
        with pytest.raises(ValueError):
            xp.ExposureMap((0, 1), xp.Side.LEFT, 32, np.ones((2, 3)), np.zeros((2, 2)))
        with pytest.raises(ValueError):
            xp.ExposureMap((0, 1), xp.Side.LEFT, 32, np.full((1, 3), np.nan), np.zeros((1, 3)))
        with pytest.raises(ValueError):
            xp.ExposureMap((0, 1), xp.Side.LEFT, 32, np.zeros((1, 3)), np.zeros((1, 3)))
        assert xp.block_bounds(1080, 16)[-1] == (1005, 1080)
        with pytest.raises(ValueError):
            xp.block_bounds(4, 5)
        with pytest.raises(ValueError):
            xp.block_bounds(4, 0)


class TestTileWire:                   # imgio.py:14-18, detect.py:297-301
    def test_ppm_framing_matches_reference_format(self):
        from paper_1910_03517_b200 import detect
        rng = np.random.default_rng(3)
        tiles = rng.integers(0, 256, (3, 4, 5, 3), dtype=np.uint8)
        pp = detect.encode_ppm_tiles(tiles)
        assert pp[1] == b"P6\n5 4\n255\n" + tiles[1].tobytes()
        assert pp[2] == detect.encode_ppm(tiles[2])
        req = detect.detect_requests([DetectorWindow(7, 8, 9), (1, 2, 3), DetectorWindow(0, 0, 4)],
                                     tiles)
        assert req[0].startswith(b"DETECT v1 7 8 9 5 4\nP6\n5 4\n255\n")
        assert req[1][len(b"DETECT v1 1 2 3 5 4\n"):] == pp[1]
        with pytest.raises(ValueError):
            detect.encode_ppm(np.zeros((4, 4), np.uint8))
        with pytest.raises(ValueError):
            detect.detect_requests([DetectorWindow(0, 0, 1)], tiles)


class TestBandPacking:                # the drop-in's per-call band transfer
    def test_packed_bands_are_the_band_columns(self):
        """K1 over the packed (H, 2 bw) image reads exactly the columns it
        reads in the full frame: RIGHT side = the first bw columns, LEFT side
        = the last bw (exposure.py:163-168), for frames and 2-D masks."""
        rng = np.random.default_rng(5)
        for (h, w, bw) in [(12, 40, 8), (7, 9, 4), (5, 16, 8)]:
            px = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
            pk = xp._bands(px, bw)
            assert pk.shape == ((h, 2 * bw, 3) if 2 * bw < w else (h, w, 3))
            assert pk.flags["C_CONTIGUOUS"]
            np.testing.assert_array_equal(pk[:, :bw], px[:, :bw])
            np.testing.assert_array_equal(pk[:, -bw:], px[:, w - bw:])
            m = rng.random((h, w)) < 0.5
            pm = xp._bands(m.view(np.uint8), bw)
            np.testing.assert_array_equal(pm[:, :bw], m[:, :bw].view(np.uint8))
            np.testing.assert_array_equal(pm[:, -bw:], m[:, w - bw:].view(np.uint8))


class TestStatsTable:                 # band-statistics export
    def _records(self, B=2, N=3, K=4, seed=0):
        from paper_1910_03517_b200 import _lib
        rng = np.random.default_rng(seed)
        rec = np.zeros((B, N, 2, K), dtype=_lib.STAT_DTYPE)
        rec["area"] = rng.integers(0, 10**6, rec.shape)
        rec["valid"] = rng.integers(0, 10**6, rec.shape)
        for f in ("sum", "sumsq", "raw_sum", "raw_sumsq"):
            rec[f] = rng.integers(0, 2**63, rec.shape + (3,), dtype=np.uint64) * 2 + 1
        hist = rng.integers(0, 2**32, (B, N, 2, K, 3, 256), dtype=np.uint64).astype(np.uint32)
        return rec, hist

    def test_round_trip_exact(self):
        rec, hist = self._records()
        text = xp.write_stats_table(rec, hist, camera_ids=[4, 5, 6], frame_indices=[10, 11])
        assert text.startswith("# camarray-bandstats-v1\n")
        got, gh, cams, frames = xp.read_stats_table(text)
        assert cams == [4, 5, 6] and frames == [10, 11]
        assert got.tobytes() == rec.tobytes()
        np.testing.assert_array_equal(gh, hist)

    def test_raw_record_bytes_and_int32_hist(self):
        rec, hist = self._records(B=1, N=2, K=2, seed=3)
        raw = rec.view(np.uint8).reshape(1, 2, 2, 2, 112)  # CorrectResult.stats layout
        text = xp.write_stats_table(raw, hist.view(np.int32))
        got, gh, _, _ = xp.read_stats_table(text)
        assert got.tobytes() == rec.tobytes()
        np.testing.assert_array_equal(gh, hist)

    def test_without_histograms(self):
        rec, _ = self._records(B=1, N=1, K=3)
        got, gh, _, _ = xp.read_stats_table(xp.write_stats_table(rec))
        assert gh is None and got.tobytes() == rec.tobytes()

    def test_version_and_shape_errors(self):
        rec, hist = self._records(B=1, N=1, K=2)
        with pytest.raises(ValueError):
            xp.read_stats_table("rec 0 0 left 0 " + "1 " * 14)
        with pytest.raises(ValueError):
            xp.write_stats_table(rec, hist[:, :, :, :1])
        text = xp.write_stats_table(rec).splitlines()
        with pytest.raises(ValueError):
            xp.read_stats_table("\n".join(text[:-1]) + "\n")  # a record missing


@given(st.lists(st.tuples(st.integers(0, 400), st.integers(0, 400), st.integers(20, 200)),
                min_size=0, max_size=40),
       st.integers(1, 8), st.floats(0.0, 1.0))
def test_merge_with_budget_cut_is_exact(wins, budget, merge_iou):
    """Scheduler cuts the merged list to its budget with an early exit
    (_merge_duplicates(..., limit)): identical to merging everything and
    slicing, as in attention.py:149-186."""
    reqs = [at.AttentionRequest(DetectorWindow(x, y, s), at.Mechanism.DIFFERENCE, i)
            for i, (x, y, s) in enumerate(wins)]
    full = at._merge_duplicates(reqs, merge_iou)[:budget]
    cut = at._merge_duplicates(reqs, merge_iou, budget)
    assert [r.priority for r in cut] == [r.priority for r in full]


def _merge_by_core_iou(reqs, merge_iou):
    """attention.py:140-146 as written: core.iou on BBox objects."""
    from paper_1910_03517_b200.core import iou
    kept, boxes = [], []
    for r in reqs:
        b = r.window.as_bbox()
        if not any(iou(b, k) > merge_iou for k in boxes):
            kept.append(r)
            boxes.append(b)
    return kept


@given(st.lists(st.tuples(st.integers(0, 400), st.integers(0, 400), st.integers(1, 200)),
                min_size=0, max_size=40),
       st.floats(0.0, 1.0))
def test_merge_inlined_iou_matches_core_iou(wins, merge_iou):
    """_merge_duplicates' inlined integer IoU keeps exactly the requests the
    reference's core.iou comparison keeps (mixed window sizes)."""
    reqs = [at.AttentionRequest(DetectorWindow(x, y, s), at.Mechanism.DIFFERENCE, i)
            for i, (x, y, s) in enumerate(wins)]
    assert at._merge_duplicates(reqs, merge_iou) == _merge_by_core_iou(reqs, merge_iou)


@given(st.integers(0, 2**31), st.sampled_from([(16384, 1536), (4000, 1200), (2980, 960)]),
       st.sampled_from([960, 416, 300]), st.integers(1, 12), st.sampled_from([0, 50, 1000]),
       st.sampled_from([0.3, 0.8, 0.95]))
def test_scheduler_tick_matches_reference_restatement(seed, mosaic, size, budget, thr, miou):
    """A post-startup tick with device counts (lazy ranking, cached tiling,
    inlined IoU) equals rank-all-then-merge with core.iou (attention.py:89-103,
    140-146, 175-186)."""
    rng = np.random.default_rng(seed)
    cfg = at.AttentionConfig(budget=budget, window_size=size, diff_threshold=thr, merge_iou=miou)
    sch = at.Scheduler(mosaic, cfg)
    sch._startup.clear()
    s = sch.window_size
    org = at.window_origins(mosaic, s, 0.0)
    counts = rng.choice([0, 10, 60, 500, 5000], size=len(org))
    got = sch.schedule(frame_index=0, window_counts_fn=lambda o, ss: counts)
    order = sorted((i for i, c in enumerate(counts) if c > thr), key=lambda i: -int(counts[i]))
    ranked = [at.AttentionRequest(DetectorWindow(*org[i], s), at.Mechanism.DIFFERENCE, r)
              for r, i in enumerate(order)]
    assert got == _merge_by_core_iou(ranked, miou)[:budget]
