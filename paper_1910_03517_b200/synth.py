"""Synthetic multi-camera input (the role of the reference's scenegen.py):
a smooth shared panorama cut into N adjacent cameras, a per-camera affine
exposure distortion (scenegen.py:37-53) and moving rectangles, generated
directly in HBM with torch so full-size benchmark batches (8 x 2048x1536,
14 x 3840x2160) take milliseconds to make.  Test/bench data only."""

from __future__ import annotations

import math

from . import _dev


def synthetic_batch(batch: int, n_cams: int, height: int, width: int, *, seed: int = 100,
                    objects: int = 4, device="cuda", first: int = 0):
    """uint8 (batch, n_cams, height, width, 3) tensor; frame t shows the
    objects moved by first + t ticks.  The panorama (the only
    transcendental part) is always computed on the CPU and the rest is
    IEEE-exact float32 elementwise work, so the same seed gives the same
    bytes on any device: bench.py's GPU arm and its CPU reference arm
    correct identical frames."""
    t = _dev.torch()
    g = t.Generator(device="cpu").manual_seed(seed)

    def u(lo, hi, *shape):
        return (t.rand(*shape, generator=g, dtype=t.float64) * (hi - lo) + lo)

    total_w = n_cams * width
    az = ((t.arange(total_w, dtype=t.float32) + 0.5) / total_w * 2 * math.pi)
    el = 0.5 - (t.arange(height, dtype=t.float32) + 0.5) / height
    base = t.tensor([118.0, 132.0, 150.0]) + u(-8, 8, 3)
    chans = []
    for c in range(3):
        acc = float(base[c]) + 50.0 * el[:, None] + t.zeros(1, total_w)
        for _ in range(3):
            fa, fe, ph, amp = (float(v) for v in (u(1, 6, 1), u(0.5, 3, 1), u(0, 2 * math.pi, 1),
                                                   u(4, 12, 1)))
            acc = acc + amp * t.sin(fa * az[None, :] + fe * 6 * el[:, None] + ph)
        chans.append(acc)
    pano = t.stack(chans, -1).to(device)                        # (H, total_w, 3) f32
    gains = u(0.5, 2.0, n_cams, 3).float().to(device)
    offs = u(-40.0, 40.0, n_cams, 3).float().to(device)
    ow = [int(v) for v in u(8, max(9, width // 6), objects)]
    oh = [int(v) for v in u(6, max(7, height // 6), objects)]
    ox = [int(v) for v in u(0, total_w - 16, objects)]
    oy = [int(v) for v in u(0, height - 8, objects)]
    vx = [int(v) for v in u(-6, 7, objects)]
    col = [u(0, 255, 3).float().to(device) for _ in range(objects)]
    out = t.empty((batch, n_cams, height, width, 3), dtype=t.uint8, device=device)
    for b in range(batch):
        img = pano.clone()
        for i in range(objects):
            x0 = (ox[i] + vx[i] * (first + b)) % max(1, total_w - ow[i])
            img[oy[i]:oy[i] + oh[i], x0:x0 + ow[i]] = col[i]
        cams = img.view(height, n_cams, width, 3).permute(1, 0, 2, 3)
        v = t.round(cams * gains[:, None, None, :] + offs[:, None, None, :])
        out[b] = v.clamp_(0, 255).to(t.uint8)
    return out
