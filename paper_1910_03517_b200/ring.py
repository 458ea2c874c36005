"""Pinned host frame ring: the frame source of the streaming path (SURVEY
8a row a16).

The reference has no frame source beyond `scenegen.render_tick`
(scenegen.py:243-270: fresh numpy frames per tick); the paper's system
decodes camera streams and applies the maps per frame while the maps are
refreshed a few times per second.
`FrameRing` is the B200-side buffer between a producer (decoder, renderer,
capture card) and the corrector:

  R slots, each one batch of B array-frames (B, N, H, W, 3) uint8 in
  page-locked host memory for the input and another for the corrected
  output (+ the batch's maps).

  producer:  view = ring.acquire()     a free slot's pinned input array
             ... write / decode frames into view ...
             ring.publish(tag)          enqueue: H2D (copy stream) ->
                                        K1 -> K2 -> K3 (compute stream) ->
                                        D2H into the slot's pinned output
                                        (copy-back stream), event handoff
                                        between the three streams
  consumer:  res = ring.get()          oldest published batch, once its
                                        D2H completed (pixels, gain, offset
                                        as numpy views of the slot)
             ring.release(res)         slot back to the producer

Batches are corrected in publish order (the tick-loop state - previous
maps, previous frame - carries from one batch to the next exactly as in
consecutive ArrayCorrector.correct calls), and the copies of batch k+1
(H2D) and k-1 (D2H) overlap the kernels of batch k.  acquire() blocks
(threading.Condition) until a slot is released, so a producer thread and a
consumer thread can run freely; a single-threaded loop calls get() /
release() before acquiring more slots than the ring has (acquire(block=
False) raises RingFull instead of waiting).  Frames never
pass through pageable memory: the slots are the only host buffers.
"""

from __future__ import annotations

import threading
from collections import deque
from dataclasses import dataclass

import numpy as np

from . import _dev


@dataclass
class RingResult:
    slot: int
    tag: object               # whatever publish() was given (e.g. the first frame index)
    pixels: np.ndarray        # uint8 (B, N, H, W, 3), a view of the slot's pinned output
    gain: np.ndarray          # float64 (B, S, 2, K, 3), pinned
    offset: np.ndarray        # float64 (B, S, 2, K, 3), pinned


class RingFull(RuntimeError):
    """acquire() would block forever: every slot is filled, in flight or
    held by the consumer, and no other thread can release one."""


_FREE, _FILLING, _IN_FLIGHT, _HELD = range(4)


class FrameRing:
    """R pinned slots of B array-frames feeding an ArrayCorrector (one GPU,
    the corrector's cameras)."""

    def __init__(self, corrector, slots: int = 4, batch: int = 1, *, device_buffers: int = 2):
        t = _dev.require_cuda()
        if slots < 2:
            raise ValueError("a ring needs at least two slots")
        if batch < 1 or device_buffers < 1:
            raise ValueError("batch and device_buffers must be >= 1")
        self.ac = corrector
        self.R, self.B, self.D = int(slots), int(batch), int(device_buffers)
        shape = (self.B, corrector.cam_count, corrector.height, corrector.width, 3)
        mshape = (self.B, max(corrector.S, 1), 2, corrector.K, 3)
        self.shape = shape
        pin = dict(dtype=t.uint8, pin_memory=True)
        self._in = [t.empty(shape, **pin) for _ in range(self.R)]
        self._out = [t.empty(shape, **pin) for _ in range(self.R)]
        self._gain = [t.empty(mshape, dtype=t.float64, pin_memory=True) for _ in range(self.R)]
        self._off = [t.empty(mshape, dtype=t.float64, pin_memory=True) for _ in range(self.R)]
        self._dev_in = [t.empty(shape, dtype=t.uint8, device="cuda") for _ in range(self.D)]
        self._dev_out = [t.empty(shape, dtype=t.uint8, device="cuda") for _ in range(self.D)]
        self._dev_gain = [t.empty(mshape, dtype=t.float64, device="cuda") for _ in range(self.D)]
        self._dev_off = [t.empty(mshape, dtype=t.float64, device="cuda") for _ in range(self.D)]
        self.h2d, self.comp, self.d2h = t.cuda.Stream(), t.cuda.Stream(), t.cuda.Stream()
        ev = t.cuda.Event
        self._dev_in_free = [ev() for _ in range(self.D)]   # K1..K3 done reading dev_in[d]
        self._dev_in_ready = [ev() for _ in range(self.D)]  # H2D into dev_in[d] done
        self._dev_out_free = [ev() for _ in range(self.D)]  # D2H out of dev_out/gain/off[d] done
        self._comp_done = [ev() for _ in range(self.D)]
        self._d2h_done = [ev() for _ in range(self.R)]      # slot's pinned output complete
        self._state = [_FREE] * self.R
        self._tags = [None] * self.R
        self._queue: deque[int] = deque()   # published slots, oldest first
        self._filling: deque[int] = deque()
        self._next = 0                       # round-robin slot cursor
        self._k = 0                          # batches published (device buffer cursor)
        self._cv = threading.Condition()

    # ------------------------------------------------------------ producer
    def acquire(self, block: bool = True, timeout: float | None = None) -> np.ndarray:
        """A free slot's pinned input (B, N, H, W, 3) uint8 numpy array to
        fill; publish() hands it to the GPU.  With every slot filled, in
        flight or held, block=True waits for another thread's release()
        (TimeoutError after `timeout` s) and block=False raises RingFull
        (a single-threaded loop get()s and release()s first)."""
        with self._cv:
            while True:
                for j in range(self.R):
                    i = (self._next + j) % self.R
                    if self._state[i] == _FREE:
                        self._next = (i + 1) % self.R
                        self._state[i] = _FILLING
                        self._filling.append(i)
                        return self._in[i].numpy()
                if not block:
                    raise RingFull(f"all {self.R} slots are filled, in flight or held: "
                                   "get() and release() results first")
                if not self._cv.wait(timeout):
                    raise TimeoutError("no ring slot released in time")

    def publish(self, tag=None) -> None:
        """Enqueue the oldest acquired slot: H2D -> correct -> D2H, all
        asynchronous on the ring's three streams."""
        t = _dev.torch()
        with self._cv:
            if not self._filling:
                raise ValueError("publish() without a matching acquire()")
            i = self._filling.popleft()
            self._state[i] = _IN_FLIGHT
            self._tags[i] = tag
        d = self._k % self.D
        self._k += 1
        dev_in, dev_out = self._dev_in[d], self._dev_out[d]
        # H2D of the pinned slot once the device buffer's previous batch was consumed
        self.h2d.wait_event(self._dev_in_free[d])
        with t.cuda.stream(self.h2d):
            dev_in.copy_(self._in[i], non_blocking=True)
        self._dev_in_ready[d].record(self.h2d)
        # K1 -> K2 -> K3 (the corrector's own launches, on the compute stream)
        self.comp.wait_event(self._dev_in_ready[d])
        self.comp.wait_event(self._dev_out_free[d])
        res = self.ac.correct(dev_in, dev_out, stream=self.comp)
        if self.ac.S > 0:  # the corrector's map buffers are reused by the next batch
            with t.cuda.stream(self.comp):
                self._dev_gain[d].copy_(res.gain, non_blocking=True)
                self._dev_off[d].copy_(res.offset, non_blocking=True)
        self._dev_in_free[d].record(self.comp)
        self._comp_done[d].record(self.comp)
        # D2H of the corrected batch and its maps into the slot
        self.d2h.wait_event(self._comp_done[d])
        with t.cuda.stream(self.d2h):
            self._out[i].copy_(dev_out, non_blocking=True)
            if self.ac.S > 0:
                self._gain[i].copy_(self._dev_gain[d], non_blocking=True)
                self._off[i].copy_(self._dev_off[d], non_blocking=True)
        self._dev_out_free[d].record(self.d2h)
        self._d2h_done[i].record(self.d2h)
        with self._cv:  # visible to get() only once its completion event is recorded
            self._queue.append(i)

    # ------------------------------------------------------------ consumer
    def pending(self) -> int:
        """Published batches not yet returned by get()."""
        with self._cv:
            return len(self._queue)

    def ready(self) -> bool:
        """The oldest published batch's result is complete (get() won't block)."""
        with self._cv:
            if not self._queue:
                return False
            i = self._queue[0]
        return self._d2h_done[i].query()

    def get(self) -> RingResult | None:
        """The oldest published batch (blocks on its D2H event); None when
        nothing is published.  The arrays are views of the slot's pinned
        memory, valid until release()."""
        with self._cv:
            if not self._queue:
                return None
            i = self._queue.popleft()
        self._d2h_done[i].synchronize()
        with self._cv:
            self._state[i] = _HELD
        S = self.ac.S
        return RingResult(i, self._tags[i], self._out[i].numpy(), self._gain[i].numpy()[:, :S],
                          self._off[i].numpy()[:, :S])

    def release(self, res: RingResult) -> None:
        """Return a result's slot to the producer."""
        with self._cv:
            if self._state[res.slot] != _HELD:
                raise ValueError("slot is not held by the consumer")
            self._state[res.slot] = _FREE
            self._cv.notify_all()

    def drain(self) -> list[RingResult]:
        """get() every published batch (the caller releases them)."""
        out = []
        while True:
            r = self.get()
            if r is None:
                return out
            out.append(r)

    @property
    def h2d_bytes_per_batch(self) -> int:
        return int(np.prod(self.shape))

    @property
    def d2h_bytes_per_batch(self) -> int:
        g = self._gain[0]
        return int(np.prod(self.shape)) + 2 * g.numel() * g.element_size() * (self.ac.S > 0)
