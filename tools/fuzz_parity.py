"""Randomised parity sweep of the production paths against the oracle
(CUDA; checker = oracle/camarray_oracle.py).  Each case draws a geometry
(cameras, height, width incl. unaligned widths, blocks, band width), a mode,
wrap, batch size and seed, then checks:

* ArrayCorrector.correct (two consecutive batches, histograms on) against the
  oracle tick loop: gains/offsets within 1e-12 relative, fit_ok identical,
  pixels identical except for the documented +-1 LSB tolerance (counted);
* histograms of sampled bands against np.bincount of the oracle's band slices
  (OBJECT_REMOVAL: of the pixels its in-band mask_diff keeps);
* correct_with_motion counts against the oracle's difference-plan counts;
* camx_tiles (random windows, random out size) against oracle crop + resize.

    python tools/fuzz_parity.py [n_cases] [seed]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import camarray_oracle as O  # noqa: E402
from paper_1910_03517_b200 import _lib  # noqa: E402
from paper_1910_03517_b200 import exposure as xp  # noqa: E402
from paper_1910_03517_b200.array import ArrayCorrector  # noqa: E402

MODES = [(xp.ExposureMode.STANDARD, O.STANDARD), (xp.ExposureMode.OBJECT_REMOVAL, O.OBJECT_REMOVAL),
         (xp.ExposureMode.SMOOTHING, O.SMOOTHING)]


def one_case(rng, idx):
    N = int(rng.integers(2, 6))
    W = int(rng.choice([64, 96, 100, 128, 130, 160, 250, 256, 342, 512, 700, 704]))
    H = int(rng.integers(40, 200))
    K = int(rng.integers(1, min(12, H) + 1))
    bw = int(rng.integers(2, max(3, min(32, W // 2)) + 1))
    mode, om = MODES[int(rng.integers(0, 3))]
    wrap = bool(rng.integers(0, 2)) and N >= 2
    B = int(rng.integers(1, 5))
    seed = int(rng.integers(0, 10**6))
    cfg = xp.ExposureConfig(band_width=bw, blocks=K, min_band_pixels=int(rng.integers(1, 80)))
    ocfg = O.Cfg(band_width=bw, blocks=K, min_band_pixels=cfg.min_band_pixels)
    frames = np.stack([O.synthetic_array(N, H, W, seed=seed, objects=int(rng.integers(0, 3)),
                                         frame_index=t) for t in range(2 * B)])
    d = torch.from_numpy(frames).cuda()
    ac = ArrayCorrector(N, H, W, cfg, mode, wrap=wrap, histograms=True)
    r1 = ac.correct(d[:B])
    o1, g1 = r1.out.cpu().numpy(), r1.gain.cpu().numpy()
    of1, ok1, h1 = r1.offset.cpu().numpy(), r1.fit_ok.cpu().numpy(), r1.hist.cpu().numpy()
    r2 = ac.correct(d[B:])
    got_out = np.concatenate([o1, r2.out.cpu().numpy()])
    got_g = np.concatenate([g1, r2.gain.cpu().numpy()])
    got_o = np.concatenate([of1, r2.offset.cpu().numpy()])
    got_ok = np.concatenate([ok1, r2.fit_ok.cpu().numpy()])
    got_h = np.concatenate([h1, r2.hist.cpu().numpy()])
    want_out, wg, wo, wok = O.correct_sequence(frames, None, om, ocfg, wrap=wrap)
    tag = f"case {idx}: N={N} H={H} W={W} K={K} bw={bw} {mode.value} wrap={wrap} B={B} seed={seed}"
    np.testing.assert_allclose(got_g, wg, rtol=1e-12, atol=1e-9, err_msg=tag)
    np.testing.assert_allclose(got_o, wo, rtol=1e-12, atol=1e-9, err_msg=tag)
    np.testing.assert_array_equal(got_ok.astype(bool), wok, err_msg=tag)
    diff = np.abs(got_out.astype(int) - want_out.astype(int))
    assert diff.max() <= 1, f"{tag}: pixel diff {diff.max()}"
    flips = int((diff > 0).sum())
    # histograms of a few bands (OBJECT_REMOVAL: the pixels kept by the
    # in-band mask_diff against the previous array-frame; frame 0 unmasked)
    for _ in range(3):
        b = int(rng.integers(0, 2 * B))
        c = int(rng.integers(0, N))
        mask = None
        if om == O.OBJECT_REMOVAL and b > 0:
            mask = O.mask_diff(frames[b, c], frames[b - 1, c], cfg.t_diff)
        for s, side in ((0, O.LEFT), (1, O.RIGHT)):
            want_h = O.band_histograms(frames[b, c], side, bw, K, mask)
            np.testing.assert_array_equal(got_h[b, c, s], want_h, err_msg=f"{tag} hist b={b}")
    # motion counts (fused or fallback path)
    size = int(rng.integers(8, min(H, N * W) + 1))
    t = int(rng.integers(0, 256))
    mc = ArrayCorrector(N, H, W, cfg, wrap=wrap)
    _, counts, has = mc.correct_with_motion(d[:B + 1], size=size, t_motion=t)
    cnt = counts.cpu().numpy()
    for b in range(1, B + 1):
        m = np.concatenate([O.mask_diff(frames[b][k], frames[b - 1][k], t) for k in range(N)],
                           axis=1)
        _, wc = O.window_counts(m, size)
        np.testing.assert_array_equal(cnt[b], wc, err_msg=f"{tag} counts size={size} t={t}")
    # tiles
    S = int(rng.integers(4, min(H, N * W) + 1))
    out = int(rng.integers(2, 2 * S + 1))
    wins = [(int(rng.integers(0, B)), int(rng.integers(0, N * W - S + 1)),
             int(rng.integers(0, H - S + 1))) for _ in range(int(rng.integers(1, 12)))]
    wd = torch.as_tensor(np.asarray(wins, np.int32), device="cuda")
    tiles = torch.empty((len(wins), out, out, 3), dtype=torch.uint8, device="cuda")
    _lib.call("camx_tiles", d.data_ptr(), N, H, W, wd.data_ptr(), len(wins), S, out,
              tiles.data_ptr(), None)
    tl = tiles.cpu().numpy()
    for i, (b, x, y) in enumerate(wins):
        crop = O.crop(np.concatenate(list(frames[b]), axis=1), x, y, S)
        want_t = crop if out == S else O.resize_bilinear(crop, out)
        np.testing.assert_array_equal(tl[i], want_t, err_msg=f"{tag} tile {i} S={S} out={out}")
    return flips, mc.last_motion_fused


def shard_case(rng, idx):
    """The camera-sharded native path at world 2..min(N, 4) with the loopback
    communicator (one thread + stream per rank): every rank's frames, maps,
    records and histograms byte-identical to the whole-array corrector over
    two batches (correct and submit/flush alternately); sharded tiles summed
    over the ranks identical to camx_tiles."""
    import threading
    from paper_1910_03517_b200.dist import camera_partition, loopback_comms
    N = int(rng.integers(2, 7))
    world = int(rng.integers(2, min(N, 4) + 1))
    W = int(rng.choice([96, 128, 160, 256, 342]))
    H = int(rng.integers(48, 160))
    K = int(rng.integers(1, min(8, H) + 1))
    bw = int(rng.integers(2, min(24, W // 2) + 1))
    mode = MODES[int(rng.integers(0, 3))][0]
    wrap = bool(rng.integers(0, 2))
    B = int(rng.integers(1, 4))
    piped = bool(rng.integers(0, 2))
    seed = int(rng.integers(0, 10**6))
    cfg = xp.ExposureConfig(band_width=bw, blocks=K)
    frames = np.stack([O.synthetic_array(N, H, W, seed=seed, objects=2, frame_index=t)
                       for t in range(2 * B)])
    d = torch.from_numpy(frames).cuda()
    tag = (f"shard case {idx}: N={N} world={world} H={H} W={W} K={K} bw={bw} {mode.value} "
           f"wrap={wrap} B={B} piped={piped} seed={seed}")
    whole = ArrayCorrector(N, H, W, cfg, mode, wrap=wrap, histograms=True)
    keys = ("out", "gain", "offset", "fit_ok", "stats", "hist")
    want = []
    for lo, hi in ((0, B), (B, 2 * B)):
        r = whole.correct(d[lo:hi])
        want.append({k: getattr(r, k).clone() for k in keys})
    comms = loopback_comms(world)
    parts = camera_partition(N, world)
    got, errs = [None] * world, []

    def rank(r):
        try:
            torch.cuda.set_device(0)
            b0, c = parts[r]
            ac = ArrayCorrector(N, H, W, cfg, mode, wrap=wrap, histograms=True, cam_begin=b0,
                                cam_count=c, comm=comms[r])
            st = torch.cuda.Stream()
            res = []
            with torch.cuda.stream(st):
                locs = [d[lo:hi, b0:b0 + c].contiguous() for lo, hi in ((0, B), (B, 2 * B))]
                if piped:
                    ac.submit(locs[0], stream=st)
                    outs = [ac.submit(locs[1], stream=st), ac.flush(stream=st)]
                    for o in outs:
                        res.append({k: getattr(o, k).clone() for k in keys})
                        st.synchronize()
                else:
                    for loc in locs:
                        o = ac.correct(loc, stream=st)
                        res.append({k: getattr(o, k).clone() for k in keys})
            st.synchronize()
            got[r] = res
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    ths = [threading.Thread(target=rank, args=(r,), daemon=True) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(240)
    for c in comms:
        c.close()
    if errs:
        raise errs[0]
    for r, (b0, c) in enumerate(parts):
        for i in range(2):
            g, w = got[r][i], want[i]
            for k in ("gain", "offset", "fit_ok", "stats"):
                assert torch.equal(g[k], w[k]), f"{tag} rank {r} batch {i} {k}"
            for k in ("out", "hist"):
                assert torch.equal(g[k], w[k][:, b0:b0 + c]), f"{tag} rank {r} batch {i} {k}"
    # sharded attention-tick counts (when the geometry takes the fused path)
    size = int(rng.integers(max(8, min(H, N * W) // 2), min(H, N * W) + 1))
    tm = int(rng.integers(0, 256))
    motion = all(_lib.load().camx_motion_supported(B + 1, N, c, H, W, K, size) for _, c in parts)
    if motion:
        comms = loopback_comms(world)
        cnts = [None] * world

        def rank_m(r):
            try:
                torch.cuda.set_device(0)
                b0, c = parts[r]
                ac = ArrayCorrector(N, H, W, cfg, mode, wrap=wrap, cam_begin=b0, cam_count=c,
                                    comm=comms[r])
                st = torch.cuda.Stream()
                with torch.cuda.stream(st):
                    _, cc, _ = ac.correct_with_motion(d[:B + 1, b0:b0 + c].contiguous(), size=size,
                                                      t_motion=tm, stream=st)
                    cnts[r] = cc.cpu().numpy()
            except BaseException as e:  # noqa: BLE001
                errs.append(e)

        ths = [threading.Thread(target=rank_m, args=(r,), daemon=True) for r in range(world)]
        for t in ths:
            t.start()
        for t in ths:
            t.join(240)
        for c in comms:
            c.close()
        if errs:
            raise errs[0]
        for b in range(1, B + 1):
            m = np.concatenate([O.mask_diff(frames[b][k], frames[b - 1][k], tm) for k in range(N)],
                               axis=1)
            _, wc = O.window_counts(m, size)
            for r in range(world):
                np.testing.assert_array_equal(cnts[r][b], wc,
                                              err_msg=f"{tag} rank {r} counts size={size} t={tm}")
    # sharded tiles: disjoint owned columns summing to the whole-array tiles
    S = int(rng.integers(4, min(H, N * W) + 1))
    out = int(rng.integers(2, 2 * S + 1))
    wins = [(int(rng.integers(0, B)), int(rng.integers(0, N * W - S + 1)),
             int(rng.integers(0, H - S + 1))) for _ in range(int(rng.integers(1, 10)))]
    wd = torch.as_tensor(np.asarray(wins, np.int32), device="cuda")
    full = want[0]["out"]
    ref = torch.empty((len(wins), out, out, 3), dtype=torch.uint8, device="cuda")
    _lib.call("camx_tiles", full.data_ptr(), N, H, W, wd.data_ptr(), len(wins), S, out,
              ref.data_ptr(), None)
    acc = torch.zeros((len(wins), out, out, 3), dtype=torch.int32, device="cuda")
    for g, (b0, c) in enumerate(parts):
        local = full[:, b0:b0 + c].contiguous()
        halo = full[:, b0 + c, :, 0, :].contiguous() if g + 1 < world else None
        part = torch.zeros_like(ref)
        _lib.call("camx_tiles_shard", local.data_ptr(), c, H, W, b0 * W,
                  0 if halo is None else halo.data_ptr(), wd.data_ptr(), len(wins), S, out,
                  part.data_ptr(), None)
        acc += part.to(torch.int32)
    torch.cuda.synchronize()
    assert torch.equal(acc.to(torch.uint8), ref), f"{tag} sharded tiles S={S} out={out}"
    return motion


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2024)
    total_flips = fused = 0
    for i in range(n):
        f, fu = one_case(rng, i)
        total_flips += f
        fused += int(fu)
    print(f"{n} cases OK; LSB flips {total_flips}; fused motion path in {fused} cases")
    ns = max(1, n // 4)
    nm = sum(bool(shard_case(rng, i)) for i in range(ns))
    print(f"{ns} camera-shard cases OK (loopback world 2..4, correct and submit/flush, tiles; "
          f"sharded motion counts in {nm})")


if __name__ == "__main__":
    main()
