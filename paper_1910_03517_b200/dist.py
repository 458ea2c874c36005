"""Camera sharding across the GPUs of one NVLink/NVSwitch box.

Every stage but the seam solve is per camera; the solve of seam (s, s+1)
needs only the two band-statistic records adjacent to it.  GPU g owns a
contiguous group of cameras, runs K1 on them, all-gathers the fixed-size
stat records (112 B x 2 sides x K blocks per camera-frame: ~3.5 KB, latency-
bound) over NCCL, runs the tiny K2 solve for all seams redundantly, and
applies K3 to its own cameras only - so the corrected output is
byte-identical to the 1-GPU result.  The reference has no
parallelism; this is the one exchange step the path really has.
"""

from __future__ import annotations

from . import _dev
from .array import ArrayCorrector
from .exposure import ExposureConfig, ExposureMode


def camera_partition(n_cams: int, world: int) -> list[tuple[int, int]]:
    """Contiguous (begin, count) per rank; counts differ by at most one."""
    if world < 1 or n_cams < world:
        raise ValueError(f"cannot shard {n_cams} cameras over {world} ranks")
    q, r = divmod(n_cams, world)
    out, b = [], 0
    for g in range(world):
        c = q + (1 if g < r else 0)
        out.append((b, c))
        b += c
    return out


def make_stats_exchange(n_cams: int, group=None):
    """Return exchange(stats_local (B, c_local, 2, K, R) uint8) ->
    stats_full (B, n_cams, 2, K, R): an all-gather of every rank's records,
    padded to the largest shard, re-assembled in camera order."""
    import torch.distributed as dist
    t = _dev.torch()
    world = dist.get_world_size(group)
    parts = camera_partition(n_cams, world)
    cmax = max(c for _, c in parts)
    nccl = dist.get_backend(group) == "nccl"

    def exchange(stats_local):
        B = stats_local.shape[0]
        tail = stats_local.shape[2:]
        send = stats_local
        if stats_local.shape[1] != cmax:
            send = t.zeros((B, cmax, *tail), dtype=stats_local.dtype, device=stats_local.device)
            send[:, : stats_local.shape[1]] = stats_local
        send = send.contiguous()
        if nccl:
            recv = t.empty((world, *send.shape), dtype=send.dtype, device=send.device)
            dist.all_gather_into_tensor(recv, send, group=group)
            chunks = list(recv.unbind(0))
        else:
            chunks = [t.empty_like(send) for _ in range(world)]
            dist.all_gather(chunks, send, group=group)
        return t.cat([chunks[g][:, :c] for g, (_, c) in enumerate(parts)], dim=1).contiguous()

    return exchange


def sharded_corrector(n_cams: int, height: int, width: int,
                      cfg: ExposureConfig = ExposureConfig(),
                      mode: ExposureMode = ExposureMode.STANDARD, *, wrap: bool = False,
                      histograms: bool = False, group=None) -> ArrayCorrector:
    """ArrayCorrector for this rank's camera shard of an n_cams array."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    begin, count = camera_partition(n_cams, world)[rank]
    ex = make_stats_exchange(n_cams, group) if world > 1 else None
    return ArrayCorrector(n_cams, height, width, cfg, mode, wrap=wrap, histograms=histograms,
                          cam_begin=begin, cam_count=count, exchange=ex)


def sharded_window_counts(origins, size: int, *, cur=None, prev=None, mask=None,
                          t_diff: int = 20, n_cams: int, width: int, group=None, counts_fn=None):
    """difference_plan's per-window on-pixel counts (attention.py:96-100) over
    a camera-sharded array: this rank counts the window pixels that fall on
    its own cameras (origins shifted into its local mosaic; columns outside
    it are skipped by K4), then one all-reduce(sum) of the int64 counts gives
    every rank the whole-array counts - and so the same ranking.
    cur/prev (or mask) hold only this rank's cameras.  `counts_fn` replaces
    the K4 call (tests)."""
    import numpy as np
    import torch.distributed as dist
    t = _dev.torch()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    begin, count = camera_partition(n_cams, world)[rank]
    local = [(x - begin * width, y) for (x, y) in origins]
    if counts_fn is None:
        from .attention import window_counts
        counts_fn = lambda org, s: window_counts(org, s, cur=cur, prev=prev, mask=mask,  # noqa: E731
                                                 t_diff=t_diff, n_cams=count)
    part = t.as_tensor(np.asarray(counts_fn(local, size), dtype=np.int64))
    if dist.get_backend(group) == "nccl":
        part = part.cuda()
    dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)
    return part.cpu().numpy()
