"""The pinned host frame ring (ring.FrameRing) and the
host entry point's pinned-memory contract, on the GPU, against the oracle's
tick loop (oracle.correct_sequence restates update_exposure + apply_exposure
per array-frame, exposure.py:245-414)."""

import threading

import numpy as np
import pytest

from oracle import camarray_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1910_03517_b200 import exposure as xp  # noqa: E402
from paper_1910_03517_b200.array import ArrayCorrector  # noqa: E402
from paper_1910_03517_b200.ring import FrameRing, RingFull  # noqa: E402

MODES = [(xp.ExposureMode.STANDARD, O.STANDARD), (xp.ExposureMode.OBJECT_REMOVAL, O.OBJECT_REMOVAL),
         (xp.ExposureMode.SMOOTHING, O.SMOOTHING)]
GAIN_RTOL, GAIN_ATOL = 1e-12, 1e-9


def _stream(N, H, W, n_batches, B, seed):
    return np.stack([O.synthetic_array(N, H, W, seed=seed, objects=3, frame_index=t)
                     for t in range(n_batches * B)])


def _check(out, gain, frames, om, ocfg, wrap=False):
    want, want_g, _, _ = O.correct_sequence(frames, None, om, ocfg, None, wrap)
    np.testing.assert_allclose(gain, want_g, rtol=GAIN_RTOL, atol=GAIN_ATOL)
    d = np.abs(out.astype(int) - want.astype(int))
    assert d.max() <= 1, f"max |diff| {d.max()}"
    return int((d > 0).sum())


@pytest.mark.parametrize("mode,om", MODES, ids=lambda m: getattr(m, "value", str(m)))
def test_ring_streams_batches_in_order_vs_oracle(mode, om):
    """Single-threaded producer/consumer: 5 batches of 2 array-frames through
    a 3-slot ring (slots reused), results in publish order, tick-loop state
    carried across batches; pixels and maps against the oracle's tick loop
    over the whole 10-frame stream."""
    N, H, W, B, T = 4, 96, 128, 2, 5
    cfg = xp.ExposureConfig(band_width=16, blocks=4)
    ocfg = O.Cfg(band_width=16, blocks=4)
    frames = _stream(N, H, W, T, B, seed=31)
    ring = FrameRing(ArrayCorrector(N, H, W, cfg, mode), slots=3, batch=B)
    outs, gains, tags = [], [], []

    def consume():
        r = ring.get()
        outs.append(r.pixels.copy())
        gains.append(r.gain.copy())
        tags.append(r.tag)
        ring.release(r)

    for k in range(T):
        try:
            view = ring.acquire(block=False)
        except RingFull:
            consume()
            view = ring.acquire(block=False)
        view[...] = frames[k * B:(k + 1) * B]   # the producer writes into the pinned slot
        ring.publish(tag=k * B)
    while ring.pending():
        consume()
    assert tags == [k * B for k in range(T)]
    flips = _check(np.concatenate(outs), np.concatenate(gains), frames, om, ocfg)
    assert flips == 0, f"{flips} LSB flips"


def test_ring_threaded_producer_consumer_vs_oracle():
    """Producer and consumer threads (acquire blocks until the consumer
    releases); 8 batches through 2 slots, OBJECT_REMOVAL with the previous
    frame carried across batches."""
    N, H, W, B, T = 3, 64, 96, 1, 8
    cfg = xp.ExposureConfig(band_width=8, blocks=4)
    ocfg = O.Cfg(band_width=8, blocks=4)
    frames = _stream(N, H, W, T, B, seed=5)
    ring = FrameRing(ArrayCorrector(N, H, W, cfg, xp.ExposureMode.OBJECT_REMOVAL), slots=2,
                     batch=B)
    got = {}
    err = []

    def producer():
        try:
            torch.cuda.set_device(0)
            for k in range(T):
                view = ring.acquire(timeout=60)
                view[...] = frames[k * B:(k + 1) * B]
                ring.publish(tag=k)
        except BaseException as e:  # noqa: BLE001
            err.append(e)

    def consumer():
        try:
            torch.cuda.set_device(0)
            n = 0
            while n < T:
                r = ring.get()
                if r is None:
                    threading.Event().wait(0.001)
                    continue
                got[r.tag] = (r.pixels.copy(), r.gain.copy())
                ring.release(r)
                n += 1
        except BaseException as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=producer), threading.Thread(target=consumer)]
    for x in th:
        x.start()
    for x in th:
        x.join(120)
        assert not x.is_alive()
    assert not err, err
    assert sorted(got) == list(range(T))
    out = np.concatenate([got[k][0] for k in range(T)])
    gain = np.concatenate([got[k][1] for k in range(T)])
    flips = _check(out, gain, frames, O.OBJECT_REMOVAL, ocfg)
    assert flips == 0, f"{flips} LSB flips"


def test_ring_wrap_array_and_release_errors():
    N, H, W, B = 3, 64, 96, 2
    cfg = xp.ExposureConfig(band_width=8, blocks=4)
    frames = _stream(N, H, W, 2, B, seed=9)
    ring = FrameRing(ArrayCorrector(N, H, W, cfg, wrap=True), slots=2, batch=B)
    with pytest.raises(ValueError):
        ring.publish()  # nothing acquired
    for k in range(2):
        ring.acquire(block=False)[...] = frames[k * B:(k + 1) * B]
        ring.publish(k)
    with pytest.raises(RingFull):
        ring.acquire(block=False)
    res = ring.drain()
    ring.release(res[0])
    with pytest.raises(ValueError):
        ring.release(res[0])  # second release of the same slot
    ring.release(res[1])
    out = np.concatenate([r.pixels.copy() for r in res])
    gain = np.concatenate([r.gain.copy() for r in res])
    assert gain.shape == (2 * B, N, 2, 4, 3)  # wrap: N seams
    _check(out, gain, frames, O.STANDARD, O.Cfg(band_width=8, blocks=4), wrap=True)


def test_correct_host_rejects_pageable_unless_staged():
    N, H, W = 2, 64, 96
    frames = _stream(N, H, W, 1, 2, seed=3)
    ac = ArrayCorrector(N, H, W, xp.ExposureConfig(band_width=8, blocks=4))
    with pytest.raises(ValueError, match="pageable"):
        ac.correct_host(frames)  # numpy: pageable
    with pytest.raises(ValueError, match="pageable"):
        ac.correct_host(torch.from_numpy(frames))
    with pytest.raises(ValueError, match="pinned"):
        ac.correct_host(torch.from_numpy(frames).pin_memory(), torch.empty(frames.shape,
                                                                           dtype=torch.uint8))
    ac.reset()
    staged = ac.correct_host(frames, stage=True).numpy()
    ac.reset()
    pinned = ac.correct_host(torch.from_numpy(frames).pin_memory()).numpy()
    np.testing.assert_array_equal(staged, pinned)
