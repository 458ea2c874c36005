"""Camera sharding across the GPUs of one NVLink/NVSwitch box.

Every stage but the seam solve is per camera; the solve of seam (s, s+1)
needs only the two band-statistic records adjacent to it.  GPU g owns a
contiguous group of cameras, runs K1 on them, all-gathers the fixed-size
stat records (112 B x 2 sides x K blocks per camera-frame: ~3.5 KB, latency-
bound) over NCCL, runs the tiny K2 solve for all seams redundantly, and
applies K3 to its own cameras only - so the corrected output is
byte-identical to the 1-GPU result.  The reference has no
parallelism; this is the one exchange step the path really has.

With NCCL the exchange runs in C (NcclComm + camx_correct_batch_sharded:
K1 -> ncclAllGather -> K2 -> K3 from one call, ~no host work per batch);
make_stats_exchange is the backend-agnostic Python form (gloo tests).
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
            _gather(chunks, send, nccl, group)
        return t.cat([chunks[g][:, :c] for g, (_, c) in enumerate(parts)], dim=1).contiguous()

    return exchange


class NcclComm:
    """camx's own NCCL communicator over the ranks of `group` (camx_comm_*):
    the unique id is made on the group's first rank and broadcast with
    torch.distributed; afterwards every batch's seam-stat all-gather is
    issued from C inside camx_correct_batch_sharded (no Python, no
    torch.distributed call on the per-batch path).  Call on every rank
    (NCCL init is collective), with this rank's CUDA device current."""

    def __init__(self, group=None):
        import ctypes

        import torch.distributed as dist

        from . import _lib
        t = _dev.require_cuda()
        if not _lib.load().camx_comm_available():
            raise RuntimeError("camx: libnccl.so.2 not loadable, cannot build an NCCL comm")
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        uid = t.zeros(128, dtype=t.uint8)
        if self.rank == 0:
            _lib.call("camx_comm_unique_id", uid.data_ptr())
        src = dist.get_global_rank(group, 0) if group is not None else 0
        if dist.get_backend(group) == "nccl":
            d = uid.cuda()
            dist.broadcast(d, src=src, group=group)
            uid = d.cpu()
        else:
            dist.broadcast(uid, src=src, group=group)
        h = ctypes.c_void_p()
        _lib.call("camx_comm_init", ctypes.byref(h), uid.data_ptr(), self.world, self.rank)
        self.handle = h.value

    def close(self) -> None:
        if getattr(self, "handle", None):
            from . import _lib
            _lib.call("camx_comm_destroy", self.handle)
            self.handle = None


class LoopbackComm:
    """Rank `rank` of a test-only loopback group (camx_comm_loopback_create):
    the W ranks of a camera-sharded array live in ONE process on one GPU,
    each driven from its own host thread and CUDA stream.  Same attributes
    as NcclComm (rank, world, handle), so ArrayCorrector(comm=...) runs its
    world > 1 native path unchanged; the all-gather goes through a shared
    device buffer with event waits and host barriers instead of NCCL (which
    refuses two ranks per device)."""

    def __init__(self, handle: int, rank: int, world: int):
        self.handle, self.rank, self.world = handle, rank, world

    def close(self) -> None:
        if self.handle:
            from . import _lib
            _lib.call("camx_comm_destroy", self.handle)
            self.handle = None


def loopback_comms(world: int) -> list[LoopbackComm]:
    """`world` LoopbackComm handles of one group (use each from its own
    thread; every rank must enter every collective)."""
    import ctypes

    from . import _lib
    _dev.require_cuda()
    hs = (ctypes.c_void_p * world)()
    _lib.call("camx_comm_loopback_create", world, hs)
    return [LoopbackComm(hs[r], r, world) for r in range(world)]


def sharded_corrector(n_cams: int, height: int, width: int,
                      cfg: ExposureConfig = ExposureConfig(),
                      mode: ExposureMode = ExposureMode.STANDARD, *, wrap: bool = False,
                      histograms: bool = False, group=None, native: bool | None = None
                      ) -> ArrayCorrector:
    """ArrayCorrector for this rank's camera shard of an n_cams array.

    native (default: the group's backend is NCCL): exchange the seam stats
    with camx's own NCCL communicator inside one C call per batch
    (camx_correct_batch_sharded); otherwise through torch.distributed
    all-gathers in Python (make_stats_exchange; any backend)."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    begin, count = camera_partition(n_cams, world)[rank]
    if world == 1:
        return ArrayCorrector(n_cams, height, width, cfg, mode, wrap=wrap, histograms=histograms)
    if native is None:
        native = dist.get_backend(group) == "nccl"
    if native:
        return ArrayCorrector(n_cams, height, width, cfg, mode, wrap=wrap, histograms=histograms,
                              cam_begin=begin, cam_count=count, comm=NcclComm(group))
    return ArrayCorrector(n_cams, height, width, cfg, mode, wrap=wrap, histograms=histograms,
                          cam_begin=begin, cam_count=count,
                          exchange=make_stats_exchange(n_cams, group))


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
    _reduce_sum(part, dist.get_backend(group) == "nccl", group)
    return part.cpu().numpy()


def _gather(outs, x, nccl: bool, group=None) -> None:
    """all_gather of `x` into `outs`.  NCCL: on the device, stream-ordered.
    Other backends (gloo): through host copies - gloo's CUDA collectives do
    not reliably order their device copies against the caller's stream (a
    K2 launched after the exchange was measured reading records that had
    not landed), so the device tensors are copied to the host (synchronous),
    gathered there, and copied back (stream-ordered before later kernels)."""
    import torch.distributed as dist
    if nccl:
        dist.all_gather(outs, x, group=group)
        return
    xc = x.cpu()
    hs = [_dev.torch().empty_like(xc) for _ in outs]
    dist.all_gather(hs, xc, group=group)
    for o, h in zip(outs, hs):
        o.copy_(h)


def _reduce_sum(x, nccl: bool, group=None):
    """all_reduce(SUM) of `x` (host copies for non-NCCL backends; see _gather)."""
    import torch.distributed as dist
    if nccl or not getattr(x, "is_cuda", False):
        dist.all_reduce(x, op=dist.ReduceOp.SUM, group=group)
        return x
    xc = x.cpu()
    dist.all_reduce(xc, op=dist.ReduceOp.SUM, group=group)
    x.copy_(xc)
    return x


def tile_homes(windows, size: int, n_cams: int, width: int, world: int):
    """Per window (b, x, y): (home rank, straddles).  Home = the rank holding
    the window's first column; a window straddles when its last column lies
    on another rank (its output columns are then split by first-tap owner)."""
    parts = camera_partition(n_cams, world)
    owner = [0] * n_cams
    for g, (b0, c) in enumerate(parts):
        for cam in range(b0, b0 + c):
            owner[cam] = g
    out = []
    for (_, x, _) in windows:
        h = owner[x // width]
        out.append((h, owner[(x + size - 1) // width] != h))
    return out


def sharded_tiles(out_local, windows, *, size: int = 960, out_size: int = 416, n_cams: int,
                  group=None, tiles_fn=None):
    """Attention tiles over a camera-sharded array.

    out_local: this rank's corrected cameras, (B, c_local, H, W, 3) uint8;
    windows: (b, x, y) in global mosaic coordinates (the same list on every
    rank).  Steps: (1) all-gather of every rank's first corrected column
    (B x H x 3 bytes) - the 1-pixel halo the previous rank's last output
    columns tap; (2) each rank resamples the output columns whose first tap
    it holds (camx_tiles_shard) - whole tiles for windows inside its
    cameras, column slices of straddling ones into a zero-filled buffer;
    (3) one all-reduce(sum) of the straddling partials (disjoint columns, so
    the sum is the assembled tile).  Returns (ids, tiles): the indices into
    `windows` of the tiles homed on this rank (first column here), ascending,
    and those tiles (len(ids), out_size, out_size, 3) - byte-identical to the
    1-GPU tiles.  `tiles_fn(local, halo, wins, col_begin, size, out_size,
    dst)` replaces the kernel call (CPU tests)."""
    import numpy as np
    import torch.distributed as dist
    t = _dev.torch()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    B, c_local, H, W = (int(v) for v in out_local.shape[:4])
    begin, count = camera_partition(n_cams, world)[rank]
    if count != c_local:
        raise ValueError(f"rank {rank} holds {c_local} cameras, partition says {count}")
    wins = [tuple(int(v) for v in w) for w in windows]
    for (b, x, y) in wins:
        if not (0 <= b < B and 0 <= x and 0 <= y and x + size <= n_cams * W and y + size <= H):
            raise ValueError(f"window ({b}, {x}, {y}, {size}) outside the array")
    col_begin = begin * W
    dev = out_local.device
    nccl = dist.get_backend(group) == "nccl"

    # (1) halo: every rank's first corrected column
    first = out_local[:, 0, :, 0, :].contiguous()  # (B, H, 3)
    cols = [t.empty_like(first) for _ in range(world)]
    _gather(cols, first, nccl, group)
    halo = cols[rank + 1] if rank + 1 < world else None

    if tiles_fn is None:
        def tiles_fn(local, hal, wl, cb, s, o, dst):
            from . import _lib
            wd = t.as_tensor(np.asarray(wl, dtype=np.int32).reshape(-1, 3), device=local.device)
            _lib.call("camx_tiles_shard", local.data_ptr(), local.shape[1], local.shape[2],
                      local.shape[3], cb, 0 if hal is None else hal.data_ptr(), wd.data_ptr(),
                      len(wl), s, o, dst.data_ptr(), _dev.stream_handle(None))

    homes = tile_homes(wins, size, n_cams, W, world)
    lo, hi = col_begin, col_begin + count * W
    touches = [x < hi and x + size > lo for (_, x, _) in wins]
    own = [i for i, (h, s) in enumerate(homes) if h == rank and not s]
    strad = [i for i, (_, s) in enumerate(homes) if s]
    tile_shape = (out_size, out_size, 3)

    whole = t.empty((len(own), *tile_shape), dtype=t.uint8, device=dev)
    if own:
        tiles_fn(out_local, halo, [wins[i] for i in own], col_begin, size, out_size, whole)
    part = t.zeros((len(strad), *tile_shape), dtype=t.uint8, device=dev)
    mine = [k for k, i in enumerate(strad) if touches[i]]
    if mine:
        sub = t.zeros((len(mine), *tile_shape), dtype=t.uint8, device=dev)
        tiles_fn(out_local, halo, [wins[strad[k]] for k in mine], col_begin, size, out_size, sub)
        part[t.as_tensor(mine, device=dev)] = sub
    if strad:
        if not nccl and part.dtype == t.uint8:  # gloo sums int32
            part = _reduce_sum(part.to(t.int32), nccl, group).to(t.uint8)
        else:
            _reduce_sum(part, nccl, group)

    ids = sorted(own + [i for i in strad if homes[i][0] == rank])
    pos_own = {i: k for k, i in enumerate(own)}
    pos_str = {i: k for k, i in enumerate(strad)}
    res = t.empty((len(ids), *tile_shape), dtype=t.uint8, device=dev)
    for k, i in enumerate(ids):
        res[k] = whole[pos_own[i]] if i in pos_own else part[pos_str[i]]
    return ids, res
