"""Pin the numpy oracle against outputs of the real reference (CPU only).

The fixtures were produced by tests/golden/make_golden.py importing the
reference `camarray` package; this suite proves oracle/camarray_oracle.py
reproduces them, so the oracle can stand in for the reference on the GPU
box (where /root/reference does not exist)."""

import numpy as np
import pytest

from oracle import camarray_oracle as O
from golden_io import GOLDEN, load

SMALL = load("small")
SCENE = load("scene")
C1 = load("config1")


def test_band_stats_match_reference():
    for case in SMALL["band_stats"]:
        side = O.LEFT if str(case["side"]) == "left" else O.RIGHT
        mean, std, valid, area = O.band_stats(case["px"], side, int(case["bw"]), int(case["k"]),
                                              case["mask"])
        np.testing.assert_array_equal(valid, case["valid"])
        np.testing.assert_array_equal(area, case["area"])
        np.testing.assert_allclose(mean, case["mean"], rtol=1e-14, atol=1e-12)
        np.testing.assert_allclose(std, case["std"], rtol=1e-12, atol=1e-12)


def test_histograms_give_reference_moments():
    # Builder-defined histograms: their exact moments equal band_stats.
    for case in SMALL["band_stats"]:
        side = O.LEFT if str(case["side"]) == "left" else O.RIGHT
        h = O.band_histograms(case["px"], side, int(case["bw"]), int(case["k"]), case["mask"])
        v = np.arange(256, dtype=np.float64)
        n = h.sum(axis=2).astype(np.float64)
        assert (n[:, 0] == case["valid"]).all()
        with np.errstate(invalid="ignore", divide="ignore"):
            mean = np.where(n > 0, (h * v).sum(axis=2) / n, 0.0)
            var = np.where(n > 0, (h * v * v).sum(axis=2) / n - mean ** 2, 0.0)
        np.testing.assert_allclose(mean, case["mean"], rtol=1e-13, atol=1e-11)
        np.testing.assert_allclose(np.sqrt(np.maximum(var, 0)), case["std"], rtol=1e-6, atol=1e-6)


def test_fit_affine_match_reference():
    for c in SMALL["fit_affine"]:
        gl, ol, gr, orr, ok = O.fit_affine((c["lmean"], c["lstd"], c["lvalid"]),
                                           (c["rmean"], c["rstd"], c["rvalid"]), 1e-3, 64)
        np.testing.assert_array_equal(ok, c["ok"])
        for got, want in ((gl, c["gl"]), (ol, c["ol"]), (gr, c["gr"]), (orr, c["orr"])):
            np.testing.assert_array_equal(got, want)


def test_apply_bit_exact_with_reference():
    for c in SMALL["apply"]:
        side = O.LEFT if str(c["side"]) == "left" else O.RIGHT
        out = O.apply_exposure(c["px"], c["gain"], c["offset"], side)
        np.testing.assert_array_equal(out, c["out"])


def test_mask_diff_match_reference():
    for c in SMALL["mask_diff"]:
        np.testing.assert_array_equal(O.mask_diff(c["a"], c["b"], int(c["t"])), c["out"])


def test_window_plans_match_reference():
    for c in SMALL["sliding"]:
        xy = O.sliding_window_plan(int(c["w"]), int(c["h"]), int(c["s"]), float(c["ov"]))
        np.testing.assert_array_equal(np.array(xy, dtype=np.int64).reshape(-1, 2), c["xy"])
    for c in SMALL["difference"]:
        plan = O.difference_plan(c["mask"], int(c["s"]), int(c["thr"]))
        got = np.array([(x, y, r) for r, (x, y, _) in enumerate(plan)], dtype=np.int64).reshape(-1, 3)
        np.testing.assert_array_equal(got, c["plan"])


def test_seam_cost_match_reference():
    for c in SMALL["seam_cost"]:
        assert O.seam_cost(c["a"], c["b"], int(c["f"])) == pytest.approx(float(c["cost"]), rel=1e-12)


@pytest.mark.parametrize("name,mode", [("standard", O.STANDARD),
                                       ("object_removal", O.OBJECT_REMOVAL),
                                       ("smoothing", O.SMOOTHING)])
@pytest.mark.parametrize("arr", ["n2", "n3"])
def test_tick_loop_matches_reference(arr, name, mode):
    sc = SCENE[arr]
    cfg = O.Cfg(band_width=int(sc["band_width"]), blocks=int(sc["blocks"]))
    out, gain, off, _ = O.correct_sequence(sc["frames"], None, mode, cfg, None)
    np.testing.assert_allclose(gain, sc[f"{name}_gain"], rtol=1e-12, atol=1e-9)
    np.testing.assert_allclose(off, sc[f"{name}_offset"], rtol=1e-12, atol=1e-9)
    np.testing.assert_array_equal(out, sc[f"{name}_out"])


def test_config1_matches_reference():
    frames = C1["frames"]
    g, o, _ = O.solve_array(frames)
    np.testing.assert_allclose(g[0], C1["gain"], rtol=1e-12)
    np.testing.assert_allclose(o[0], C1["offset"], rtol=1e-12, atol=1e-9)
    out = O.apply_array(frames, g, o)
    np.testing.assert_array_equal(out, C1["out"])
    before = O.seam_cost(frames[0], frames[1])
    after = O.seam_cost(out[0], out[1])
    assert before == pytest.approx(float(C1["cost_before"]), rel=1e-12)
    assert after == pytest.approx(float(C1["cost_after"]), rel=1e-12)
    assert after <= 0.5 * before


def test_maps_table_fixture_present():
    text = (GOLDEN / "maps_table.txt").read_text()
    assert text.startswith("# camarray-exposure-v1")
