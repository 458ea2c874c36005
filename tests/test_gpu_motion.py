"""K4 fused into K3 (camx_correct_batch_motion) and the device attention tick
(ArrayCorrector.correct_and_attend), against the oracle:

* window counts bit-exact against the oracle's difference-plan counts of
  mask_diff(prev, cur) on the concatenated mosaic (attention.py:89-103,
  core.py:191-196), for frames inside a batch and across calls;
* the corrected frames, maps and histograms identical to correct();
* the attention tick's requests identical to the host Scheduler fed with the
  oracle mask, and its tiles bit-exact against the oracle crop + resize of
  the oracle-corrected frames."""

import numpy as np
import pytest

from oracle import camarray_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1910_03517_b200 import attention as at  # noqa: E402
from paper_1910_03517_b200 import exposure as xp  # noqa: E402
from paper_1910_03517_b200.core import BBox  # noqa: E402
from paper_1910_03517_b200.array import ArrayCorrector  # noqa: E402
from paper_1910_03517_b200.synth import synthetic_batch  # noqa: E402


def mosaic(frame):
    return np.concatenate(list(frame), axis=1)


def oracle_counts(prev, cur, size, t):
    m = np.concatenate([O.mask_diff(cur[c], prev[c], t) for c in range(cur.shape[0])], axis=1)
    return O.window_counts(m, size)


def moving_batch(B, N, H, W, seed):
    """Frames with sparse changes (and a dense patch straddling camera seams)."""
    rng = np.random.default_rng(seed)
    base = rng.integers(0, 256, (N, H, W, 3), dtype=np.uint8)
    out = []
    for b in range(B):
        f = base.copy()
        f[rng.random((N, H, W)) < 0.03] += np.uint8(40 + b)
        # single-channel changes of exactly t and t + 1 (strict > t)
        ys, xs = rng.integers(0, H, 200), rng.integers(0, W, 200)
        f[0, ys, xs, 1] = (f[0, ys, xs, 1].astype(int) + 20 + (b % 2)).clip(0, 255)
        x0 = (b * 37) % (N * W - 40)
        for c in range(N):
            lo, hi = max(x0 - c * W, 0), min(x0 + 40 - c * W, W)
            if lo < hi:
                f[c, 10:40, lo:hi] = 255 - f[c, 10:40, lo:hi]
        out.append(f)
    return np.stack(out)


@pytest.mark.parametrize("N,H,W,size,t,fused", [
    (3, 96, 128, 64, 20, True),      # one column group per row, clamped last windows
    (2, 500, 1024, 500, 20, True),   # rows of 3072 B: a pixel straddles the column groups
    (4, 100, 688, 100, 0, False),    # > 3 windows per CTA: correct() + camx_window_counts
    (3, 64, 704, 64, 254, False),
    (3, 360, 704, 360, 0, True),     # 2112-byte rows (partial second group), t = 0
    (2, 350, 1360, 350, 254, True),  # 4080-byte rows, t = 254, clamped windows
    (3, 96, 128, 96, 255, True),     # t = 255: nothing moves
])
def test_motion_counts_vs_oracle(N, H, W, size, t, fused):
    B = 4
    frames = moving_batch(B, N, H, W, seed=N * 1000 + W)
    d = torch.from_numpy(frames).cuda()
    cfg = xp.ExposureConfig(band_width=16, blocks=4)
    ac = ArrayCorrector(N, H, W, cfg, histograms=True)
    res, counts, has = ac.correct_with_motion(d[:2], size=size, t_motion=t)
    assert ac.last_motion_fused is fused
    res2, counts2, has2 = ac.correct_with_motion(d[2:], size=size, t_motion=t)
    torch.cuda.synchronize()
    assert has == [False, True] and has2 == [True, True]
    c = np.concatenate([counts.cpu().numpy(), counts2.cpu().numpy()])
    for b in range(1, B):
        wins, want = oracle_counts(frames[b - 1], frames[b], size, t)
        assert list(map(tuple, ac.tile_windows(min(size, N * W, H)))) == wins
        np.testing.assert_array_equal(c[b], want, err_msg=f"frame {b}")
    # the correction itself is the plain path's, bit for bit
    ref = ArrayCorrector(N, H, W, cfg, histograms=True)
    r1 = ref.correct(d[:2])
    r2 = ref.correct(d[2:])
    for got, want in ((res, r1), (res2, r2)):
        assert torch.equal(got.out, want.out)
        assert torch.equal(got.gain, want.gain) and torch.equal(got.offset, want.offset)
        assert torch.equal(got.hist, want.hist)


def test_motion_counts_full_size_config2():
    """Config-2 geometry (8 x 2048x1536, 36 windows of 960): frame 1's
    counts against frame 0, bit-exact."""
    N, H, W = 8, 1536, 2048
    d = synthetic_batch(2, N, H, W, seed=7)
    ac = ArrayCorrector(N, H, W)
    _, counts, has = ac.correct_with_motion(d, size=960)
    assert ac.last_motion_fused
    frames = d.cpu().numpy()
    wins, want = oracle_counts(frames[0], frames[1], 960, 20)
    assert len(wins) == 36 and has == [False, True]
    got = counts.cpu().numpy()[1]
    assert want.sum() > 0
    np.testing.assert_array_equal(got, want)


def test_attention_tick_matches_host_scheduler_and_oracle_tiles():
    N, H, W, B = 3, 200, 256, 6
    frames = moving_batch(B, N, H, W, seed=3)
    d = torch.from_numpy(frames).cuda()
    cfg = xp.ExposureConfig(band_width=16, blocks=4)
    ac = ArrayCorrector(N, H, W, cfg)
    acfg = at.AttentionConfig(window_size=200, budget=3, diff_threshold=5)  # 4-window sweep
    sched = at.Scheduler((N * W, H), acfg)
    host = at.Scheduler((N * W, H), acfg)
    # one tracked object, so expectation windows mix with difference ones
    obj = type("Obj", (), {})()
    obj.id, obj.last_seen = 7, 1
    obj.history = [(0, BBox(100, 50, 30, 20)), (1, BBox(110, 52, 30, 20))]
    res, reqs, tiles, _ = ac.correct_and_attend(d, sched, objects=[obj], frame_index=0,
                                                out_size=48)
    want_out, _, _, _ = O.correct_sequence(frames, None, O.STANDARD,
                                           O.Cfg(band_width=16, blocks=4))
    np.testing.assert_array_equal(res.out.cpu().numpy(), want_out)
    tiles = tiles.cpu().numpy()
    k = 0
    n_diff = 0
    for b in range(B):
        mask = None
        if b > 0:
            mask = np.concatenate([O.mask_diff(frames[b][c], frames[b - 1][c], 20)
                                   for c in range(N)], axis=1)
        want = host.schedule(frame_index=b, objects=[obj], diff_mask=mask)
        assert [(r.window.x, r.window.y, r.window.size, r.mechanism) for r in reqs[b]] == \
               [(r.window.x, r.window.y, r.window.size, r.mechanism) for r in want]
        n_diff += sum(r.mechanism is at.Mechanism.DIFFERENCE for r in want)
        for r in reqs[b]:
            c = O.crop(mosaic(want_out[b]), r.window.x, r.window.y, 200)
            np.testing.assert_array_equal(tiles[k], O.resize_bilinear(c, 48))
            k += 1
    assert k == tiles.shape[0]
    assert n_diff > 0  # the difference mechanism was exercised


def test_motion_rejects_bad_arguments():
    N, H, W = 2, 64, 128
    ac = ArrayCorrector(N, H, W, xp.ExposureConfig(band_width=16, blocks=4))
    d = torch.zeros((1, N, H, W, 3), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        ac.correct_with_motion(d, t_motion=-1)
    with pytest.raises(ValueError):
        ac.correct_with_motion(d, t_motion=256)
    sched = at.Scheduler((N * W + 1, H))
    with pytest.raises(ValueError):
        ac.correct_and_attend(d, sched)


@pytest.mark.parametrize("geom", [(3, 200, 256, 3, 3, 200), (4, 1024, 1024, 6, 6, 960)],
                         ids=["small", "long-stream"])
def test_attend_pipeline_matches_sequential_ticks(geom):
    """AttendPipeline (batch k's kernels under batch k-1's host ticks; the
    counts' D2H and k-1's tiles on side streams) gives the same requests,
    tiles, maps and frames as correct_and_attend called batch by batch -
    "long-stream" reuses every result slot several times with kernels long
    enough for the side streams to overlap them."""
    from paper_1910_03517_b200.array import AttendPipeline
    N, H, W, B, n_b, win = geom
    frames = moving_batch(n_b * B, N, H, W, seed=11)
    d = torch.from_numpy(frames).cuda()
    cfg = xp.ExposureConfig(band_width=16, blocks=4)
    acfg = at.AttentionConfig(window_size=win, budget=2, diff_threshold=5)
    seq_ac = ArrayCorrector(N, H, W, cfg, histograms=True)
    seq_s = at.Scheduler((N * W, H), acfg)
    want = []
    for k in range(n_b):  # the corrector's map buffers are reused by the next call: clone now
        r, q, tl, _ = seq_ac.correct_and_attend(d[k * B:(k + 1) * B], seq_s, frame_index=k * B,
                                                out_size=40)
        want.append((r.out.clone(), r.gain.clone(), r.hist.clone(), q, tl.clone()))
    pipe = AttendPipeline(ArrayCorrector(N, H, W, cfg, histograms=True),
                          at.Scheduler((N * W, H), acfg), out_size=40)
    got = []
    for k in range(n_b + 1):  # results arrive one submit late; compare before slot reuse
        r = pipe.submit(d[k * B:(k + 1) * B], frame_index=k * B) if k < n_b else pipe.flush()
        if k == 0:
            assert r is None
            continue
        got.append((r.frame_index, r.result.out.clone(), r.result.gain.clone(),
                    r.result.hist.clone(), r.requests, r.tiles.clone()))
    assert pipe.flush() is None
    if win == 960:  # the fused counts, written straight into the pipeline's slots
        assert pipe.ac.last_motion_fused
    for k, (g, (out, gain, hist, reqs, tiles)) in enumerate(zip(got, want)):
        f0, g_out, g_gain, g_hist, g_reqs, g_tiles = g
        assert f0 == k * B
        assert torch.equal(g_out, out) and torch.equal(g_gain, gain)
        assert torch.equal(g_hist, hist)
        assert [[(r.window.x, r.window.y, r.mechanism) for r in f] for f in g_reqs] == \
               [[(r.window.x, r.window.y, r.mechanism) for r in f] for f in reqs]
        assert torch.equal(g_tiles, tiles)


@pytest.mark.parametrize("mode", [xp.ExposureMode.OBJECT_REMOVAL, xp.ExposureMode.SMOOTHING],
                         ids=lambda m: m.value)
def test_motion_counts_with_wrap_and_stateful_modes(mode):
    """The in-pass counts on a 360-degree array (wrap seam) in the stateful
    modes: counts bit-exact; frames, maps and histograms identical to
    correct() across two calls (the OBJECT_REMOVAL previous frame and the
    smoothing state carry exactly as without the counts)."""
    N, H, W, S = 3, 96, 128, 64
    frames = moving_batch(4, N, H, W, seed=77)
    d = torch.from_numpy(frames).cuda()
    cfg = xp.ExposureConfig(band_width=16, blocks=4)
    ac = ArrayCorrector(N, H, W, cfg, mode, wrap=True, histograms=True)
    ref = ArrayCorrector(N, H, W, cfg, mode, wrap=True, histograms=True)
    c = []
    for lo, hi in ((0, 2), (2, 4)):
        got, counts, _ = ac.correct_with_motion(d[lo:hi], size=S)
        assert ac.last_motion_fused
        want = ref.correct(d[lo:hi])
        assert torch.equal(got.out, want.out) and torch.equal(got.gain, want.gain)
        assert torch.equal(got.offset, want.offset) and torch.equal(got.hist, want.hist)
        c.append(counts.cpu().numpy())
    c = np.concatenate(c)
    for b in range(1, 4):
        _, want_c = oracle_counts(frames[b - 1], frames[b], S, 20)
        np.testing.assert_array_equal(c[b], want_c)


def test_retain_reads_previous_batch_in_place():
    """correct_with_motion(retain=True) over alternating batch buffers (a
    two-slot ring) gives the same frames, maps and counts as the copying
    default: frame 0's previous frame is read from the previous buffer."""
    N, H, W, B, S = 3, 96, 128, 2, 64
    frames = moving_batch(3 * B, N, H, W, seed=5)
    d = [torch.from_numpy(frames[k * B:(k + 1) * B]).cuda() for k in range(3)]
    cfg = xp.ExposureConfig(band_width=16, blocks=4)
    a = ArrayCorrector(N, H, W, cfg)
    b = ArrayCorrector(N, H, W, cfg)
    ring = [torch.empty_like(d[0]), torch.empty_like(d[0])]
    for k in range(3):
        ra, ca, ha = a.correct_with_motion(d[k], size=S)
        buf = ring[k % 2]
        buf.copy_(d[k])
        rb, cb, hb = b.correct_with_motion(buf, size=S, retain=True)
        assert ha == hb
        assert torch.equal(ca, cb)
        assert torch.equal(ra.out, rb.out) and torch.equal(ra.gain, rb.gain)
