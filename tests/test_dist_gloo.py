"""Multi-process (gloo, world_size 2, CPU) checks of the camera-sharding
host logic: partition, the stat-record all-gather + re-assembly, and that
the assembled records equal the 1-process records of the whole array."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1910_03517_b200.dist import camera_partition, make_stats_exchange


def test_partition_contiguous_and_balanced():
    for n in range(1, 17):
        for w in range(1, n + 1):
            parts = camera_partition(n, w)
            assert sum(c for _, c in parts) == n
            assert [b for b, _ in parts] == list(np.cumsum([0] + [c for _, c in parts])[:-1])
            assert max(c for _, c in parts) - min(c for _, c in parts) <= 1
    with pytest.raises(ValueError):
        camera_partition(2, 3)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def records(B, n_cams, K, seed=0):
    """Deterministic fake stat records for the whole array (B, N, 2, K, 112)."""
    g = torch.Generator().manual_seed(seed)
    return torch.randint(0, 256, (B, n_cams, 2, K, 112), generator=g, dtype=torch.uint8)


def _worker(rank, world, port, n_cams, B, K, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = records(B, n_cams, K)
        begin, count = camera_partition(n_cams, world)[rank]
        ex = make_stats_exchange(n_cams)
        got = ex(full[:, begin:begin + count].contiguous())
        q.put((rank, bool(torch.equal(got, full)), tuple(got.shape)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_cams", [8, 5, 2])
def test_stats_allgather_reassembles_array(n_cams):
    world, B, K = 2, 3, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_cams, B, K, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, shape in res:
        assert same, f"rank {rank} re-assembled records differ"
        assert shape == (B, n_cams, 2, K, 112)


def _counts_worker(rank, world, port, q):
    """Each rank counts its own cameras' share of every window on the CPU
    (numpy stand-in for K4 with the same local-coordinate clipping), then the
    all-reduce must give the whole-array counts."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1910_03517_b200.dist import camera_partition, sharded_window_counts
        n_cams, H, W, S = 5, 40, 30, 25
        rng = np.random.default_rng(7)
        mosaic = rng.random((H, n_cams * W)) < 0.3
        origins = [(x, y) for y in (0, 15) for x in range(0, n_cams * W - S + 1, 17)]
        begin, count = camera_partition(n_cams, world)[rank]
        local_mask = mosaic[:, begin * W:(begin + count) * W]

        def cpu_counts(org, s):
            out = []
            for (x, y) in org:
                x0, x1 = max(x, 0), min(x + s, local_mask.shape[1])
                out.append(int(local_mask[y:y + s, x0:x1].sum()) if x1 > x0 else 0)
            return out

        got = sharded_window_counts(origins, S, n_cams=n_cams, width=W, counts_fn=cpu_counts)
        want = [int(mosaic[y:y + S, x:x + S].sum()) for (x, y) in origins]
        q.put((rank, list(map(int, got)) == want))
    finally:
        dist.destroy_process_group()


def test_sharded_window_counts_allreduce():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_counts_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res), res


def _tiles_worker(rank, world, port, n_cams, q):
    """Camera-sharded tiles: each rank resamples the output columns whose
    first tap it holds (numpy stand-in for camx_tiles_shard, same ownership
    rule, halo column from the next rank), straddling partials are summed;
    every window's tile must equal the whole-array oracle tile exactly, and
    every window must be homed on exactly one rank."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.camarray_oracle import resize_bilinear, resize_coords
        from paper_1910_03517_b200.dist import camera_partition, sharded_tiles
        B, H, W, S, O = 2, 30, 40, 24, 10
        rng = np.random.default_rng(11)
        full = rng.integers(0, 256, (B, n_cams, H, W, 3), dtype=np.uint8)
        mosaic = np.concatenate(list(full.transpose(1, 0, 2, 3, 4)), axis=2)  # (B, H, N*W, 3)
        wins = [(b, x, y) for b in range(B) for y in (0, 6)
                for x in list(range(0, n_cams * W - S + 1, 13)) + [W - S // 2, 2 * W - 1]]
        begin, count = camera_partition(n_cams, world)[rank]
        local = torch.from_numpy(full[:, begin:begin + count].copy())
        i0, _, _ = resize_coords(S, O)

        def cpu_tiles(loc, halo, wl, cb, s, o, dst):
            lm = np.concatenate(list(loc.numpy().transpose(1, 0, 2, 3, 4)), axis=2)
            if halo is not None:
                lm = np.concatenate([lm, halo.numpy()[:, :, None, :]], axis=2)
            glob = np.zeros((B, H, n_cams * W + 1, 3), np.uint8)
            glob[:, :, cb:cb + lm.shape[2]] = lm
            for k, (b, x, y) in enumerate(wl):
                tile = resize_bilinear(glob[b, y:y + s, x:x + s], o)
                owned = (x + i0 >= cb) & (x + i0 < cb + loc.shape[1] * loc.shape[3])
                d = dst[k].numpy()
                d[:, owned] = tile[:, owned]

        ids, tiles = sharded_tiles(local, wins, size=S, out_size=O, n_cams=n_cams,
                                   tiles_fn=cpu_tiles)
        ok = all(np.array_equal(tiles[k].numpy(),
                                resize_bilinear(mosaic[wins[i][0], wins[i][2]:wins[i][2] + S,
                                                       wins[i][1]:wins[i][1] + S], O))
                 for k, i in enumerate(ids))
        q.put((rank, ok, ids, len(wins)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_cams", [(2, 4), (3, 5)])
def test_sharded_tiles_assemble_exactly(world, n_cams):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tiles_worker, args=(r, world, port, n_cams, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _, _ in res), res
    homed = sorted(i for _, _, ids, _ in res for i in ids)
    assert homed == list(range(res[0][3]))  # every window on exactly one rank
