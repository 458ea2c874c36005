"""The camera-sharded native path at world > 1, run on ONE GPU.

NCCL refuses two ranks on one device, so these tests drive the production
sharded entry points - camx_correct_batch_sharded (ArrayCorrector.correct
with comm=), camx_correct_batch_sharded_step (submit / flush), the
rank-major gather_index of ArrayCorrector._finish and the _pipe_state index
- with W ranks in one process: one host thread and one CUDA stream per rank
and camx's loopback communicator (camx_comm_loopback_create), whose
all-gather stages the records through a shared device buffer with event
waits and host barriers.  Every rank's output must be byte-identical to
the whole-array one-GPU ArrayCorrector: pixels, maps, fit_ok, the gathered
stat records and the rank's histograms.

A 2-process gloo test runs the Python exchange path (sharded_corrector with
native=False) and sharded_tiles with the real kernels on cuda:0."""

import os
import socket
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
from paper_1910_03517_b200.dist import camera_partition, loopback_comms  # noqa: E402

MODES = [xp.ExposureMode.STANDARD, xp.ExposureMode.OBJECT_REMOVAL, xp.ExposureMode.SMOOTHING]


def keep(r):
    """Results alias the corrector's buffers between calls: copy them."""
    return dict(out=r.out.clone(), gain=r.gain.clone(), offset=r.offset.clone(),
                fit_ok=r.fit_ok.clone(), stats=r.stats.clone(),
                hist=None if r.hist is None else r.hist.clone())


def run_ranks(world, fn, timeout=240):
    """fn(rank) on `world` threads; re-raises the first failure."""
    res, err = [None] * world, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            res[r] = fn(r)
        except BaseException as e:  # noqa: BLE001 - surfaced below
            err.append(e)

    ths = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout)
        assert not t.is_alive(), "a rank hung (loopback collective not entered by every rank?)"
    if err:
        raise err[0]
    return res


def whole_array(frames_d, batches, N, H, W, cfg, mode, wrap):
    ac = ArrayCorrector(N, H, W, cfg, mode, wrap=wrap, histograms=True)
    return [keep(ac.correct(frames_d[lo:hi].contiguous())) for lo, hi in batches]


def assert_rank_matches(got, want, begin, count, what):
    for i, (g, w) in enumerate(zip(got, want)):
        tag = f"{what} batch {i}"
        np.testing.assert_array_equal(g["out"].cpu().numpy(),
                                      w["out"][:, begin:begin + count].cpu().numpy(), tag)
        for key in ("gain", "offset", "fit_ok", "stats"):
            np.testing.assert_array_equal(g[key].cpu().numpy(), w[key].cpu().numpy(),
                                          f"{tag} {key}")
        np.testing.assert_array_equal(g["hist"].cpu().numpy(),
                                      w["hist"][:, begin:begin + count].cpu().numpy(),
                                      f"{tag} hist")


CASES = [  # (n_cams, world, wrap)
    (5, 2, False),
    (7, 3, True),
    (8, 8, False),
    (4, 3, True),
]


@pytest.mark.parametrize("mode", MODES, ids=lambda m: m.value)
@pytest.mark.parametrize("N,world,wrap", CASES)
def test_sharded_correct_world_gt1_matches_one_gpu(N, world, wrap, mode):
    """ArrayCorrector.correct(comm=loopback rank): K1 on the rank's cameras
    -> record padding (uneven partitions) -> in-place all-gather -> K2 on
    rank-major records -> K3 on the rank's cameras; two consecutive batches
    (tick-loop state carried), histograms on."""
    H, W, K = 96, 128, 4
    cfg = xp.ExposureConfig(band_width=16, blocks=K)
    frames = np.stack([O.synthetic_array(N, H, W, seed=91, objects=3, frame_index=t)
                       for t in range(5)])
    d = torch.from_numpy(frames).cuda()
    batches = [(0, 2), (2, 5)]
    want = whole_array(d, batches, N, H, W, cfg, mode, wrap)
    comms = loopback_comms(world)
    parts = camera_partition(N, world)

    def rank_fn(r):
        begin, count = parts[r]
        ac = ArrayCorrector(N, H, W, cfg, mode, wrap=wrap, histograms=True, cam_begin=begin,
                            cam_count=count, comm=comms[r])
        s = torch.cuda.Stream()
        out = []
        with torch.cuda.stream(s):
            for lo, hi in batches:
                loc = d[lo:hi, begin:begin + count].contiguous()
                out.append(keep(ac.correct(loc, stream=s)))
        s.synchronize()
        return out

    try:
        got = run_ranks(world, rank_fn)
    finally:
        for c in comms:
            c.close()
    for r, (begin, count) in enumerate(parts):
        assert_rank_matches(got[r], want, begin, count, f"rank {r}/{world}")


@pytest.mark.parametrize("mode", MODES, ids=lambda m: m.value)
@pytest.mark.parametrize("N,world,wrap", [(5, 2, False), (7, 3, True), (8, 8, False)])
def test_sharded_submit_flush_world_gt1(N, world, wrap, mode):
    """The software-pipelined stream (camx_correct_batch_sharded_step: front
    half of batch k on the per-communicator side stream under K3 of batch
    k-1) at world > 1: results arrive one call late and equal the one-GPU
    sequential results; the state carries into a following correct()."""
    H, W, K, B = 96, 128, 4, 2
    cfg = xp.ExposureConfig(band_width=16, blocks=K)
    frames = np.stack([O.synthetic_array(N, H, W, seed=57, objects=3, frame_index=t)
                       for t in range(4 * B)])
    d = torch.from_numpy(frames).cuda()
    batches = [(i * B, (i + 1) * B) for i in range(4)]
    want = whole_array(d, batches, N, H, W, cfg, mode, wrap)
    comms = loopback_comms(world)
    parts = camera_partition(N, world)

    def rank_fn(r):
        begin, count = parts[r]
        ac = ArrayCorrector(N, H, W, cfg, mode, wrap=wrap, histograms=True, cam_begin=begin,
                            cam_count=count, comm=comms[r])
        s = torch.cuda.Stream()
        loc = [d[lo:hi, begin:begin + count].contiguous() for lo, hi in batches]
        outs = [torch.empty_like(x) for x in loc]
        got = []
        with torch.cuda.stream(s):
            for i in range(3):
                res = ac.submit(loc[i], outs[i], stream=s)
                assert (res is None) == (i == 0)
                if res is not None:
                    got.append(keep(res))  # valid until the next submit()
            got.append(keep(ac.flush(stream=s)))
            got.append(keep(ac.correct(loc[3], stream=s)))
        s.synchronize()
        return got

    try:
        got = run_ranks(world, rank_fn)
    finally:
        for c in comms:
            c.close()
    for r, (begin, count) in enumerate(parts):
        assert_rank_matches(got[r], want, begin, count, f"rank {r}/{world} (pipelined)")


def test_loopback_all_gather_many_calls():
    """50 back-to-back one-frame batches on 3 rank streams, no host sync
    between calls: the loopback all-gather's staging buffer is reused every
    call, ordered only by its events (one camera per rank)."""
    world = N = 3
    H, W, K, T = 64, 64, 2, 50
    cfg = xp.ExposureConfig(band_width=8, blocks=K)
    frames = np.stack([O.synthetic_array(N, H, W, seed=s, objects=1) for s in range(T)])
    d = torch.from_numpy(frames).cuda()
    want_ac = ArrayCorrector(N, H, W, cfg, xp.ExposureMode.STANDARD)
    want = [want_ac.correct(d[i:i + 1].contiguous()).gain.clone() for i in range(T)]
    comms = loopback_comms(world)

    def rank_fn(r):
        ac = ArrayCorrector(N, H, W, cfg, xp.ExposureMode.STANDARD, cam_begin=r, cam_count=1,
                            comm=comms[r])
        s = torch.cuda.Stream()
        gains = []
        with torch.cuda.stream(s):
            for i in range(T):
                gains.append(ac.correct(d[i:i + 1, r:r + 1].contiguous(), stream=s).gain.clone())
        s.synchronize()
        return gains

    try:
        got = run_ranks(world, rank_fn)
    finally:
        for c in comms:
            c.close()
    for r in range(world):
        for i in range(T):
            assert torch.equal(got[r][i], want[i]), f"rank {r} call {i}"


# ------------------------------------------------------- 2 processes, gloo

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_gpu_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1910_03517_b200 import _lib
        from paper_1910_03517_b200.dist import sharded_corrector, sharded_tiles
        N, H, W, K, B = 5, 128, 160, 4, 3
        cfg = xp.ExposureConfig(band_width=16, blocks=K)
        frames = np.stack([O.synthetic_array(N, H, W, seed=23, objects=3, frame_index=t)
                           for t in range(B)])
        d = torch.from_numpy(frames).cuda()
        ok = []
        for mode in MODES:
            whole = ArrayCorrector(N, H, W, cfg, mode, histograms=True)
            w = whole.correct(d)
            ac = sharded_corrector(N, H, W, cfg, mode, histograms=True, native=False)
            begin, count = camera_partition(N, world)[rank]
            g = ac.correct(d[:, begin:begin + count].contiguous())
            ok.append(torch.equal(g.out, w.out[:, begin:begin + count]))
            ok.append(torch.equal(g.gain, w.gain) and torch.equal(g.offset, w.offset))
            ok.append(torch.equal(g.hist, w.hist[:, begin:begin + count]))
        # tiles over the shards (halo all-gather + straddling partials summed)
        size, out = 96, 40
        wins = [(b, x, y) for b in range(B) for y in (0, 31)
                for x in list(range(0, N * W - size + 1, 57)) + [W - size // 2, 3 * W - 7]]
        full = w.out  # last mode's corrected array-frames (B, N, H, W, 3)
        ref = torch.empty((len(wins), out, out, 3), dtype=torch.uint8, device="cuda")
        wd = torch.as_tensor(np.asarray(wins, dtype=np.int32), device="cuda")
        _lib.call("camx_tiles", full.data_ptr(), N, H, W, wd.data_ptr(), len(wins), size, out,
                  ref.data_ptr(), None)
        begin, count = camera_partition(N, world)[rank]
        ids, tiles = sharded_tiles(full[:, begin:begin + count].contiguous(), wins, size=size,
                                   out_size=out, n_cams=N)
        ok.append(all(torch.equal(tiles[k], ref[i]) for k, i in enumerate(ids)))
        torch.cuda.synchronize()
        q.put((rank, ok, ids, len(wins)))
    finally:
        dist.destroy_process_group()


def test_two_process_gloo_sharded_path_on_gpu():
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_gpu_worker, args=(r, world, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, _, _ in res:
        assert all(ok), (rank, ok)
    homed = sorted(i for _, _, ids, _ in res for i in ids)
    assert homed == list(range(res[0][3]))


def _nccl_one_rank_worker(port, q):
    """One process, torch.distributed over NCCL with world 1: dist.NcclComm
    (the unique id broadcast over NCCL, camx_comm_init) and the sharded entry
    points with a real one-rank NCCL all-gather, against ArrayCorrector."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_1910_03517_b200.dist import NcclComm
        N, H, W, K, B = 4, 96, 160, 4, 3
        cfg = xp.ExposureConfig(band_width=16, blocks=K)
        frames = np.stack([O.synthetic_array(N, H, W, seed=31, objects=2, frame_index=t)
                           for t in range(2 * B)])
        d = torch.from_numpy(frames).cuda()
        ok = []
        comm = NcclComm()
        for mode in MODES:
            want = whole_array(d, [(0, B), (B, 2 * B)], N, H, W, cfg, mode, False)
            ac = ArrayCorrector(N, H, W, cfg, mode, histograms=True, cam_begin=0, cam_count=N,
                                comm=comm)
            got = [keep(ac.correct(d[lo:hi].contiguous())) for lo, hi in ((0, B), (B, 2 * B))]
            ap = ArrayCorrector(N, H, W, cfg, mode, histograms=True, cam_begin=0, cam_count=N,
                                comm=comm)
            piped = [ap.submit(d[:B].contiguous())]
            piped = [keep(ap.submit(d[B:].contiguous())), keep(ap.flush())]
            for g, w in list(zip(got, want)) + list(zip(piped, want)):
                ok.append(all(torch.equal(g[k], w[k]) for k in
                              ("out", "gain", "offset", "fit_ok", "stats", "hist")))
        comm.close()
        torch.cuda.synchronize()
        q.put(ok)
    finally:
        dist.destroy_process_group()


def test_nccl_comm_one_rank_sharded_entry_points():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_one_rank_worker, args=(_free_port(), q))
    p.start()
    ok = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert ok and all(ok), ok


@pytest.mark.parametrize("mode", [xp.ExposureMode.STANDARD, xp.ExposureMode.OBJECT_REMOVAL],
                         ids=lambda m: m.value)
@pytest.mark.parametrize("N,world,wrap", [(5, 2, False), (6, 3, True), (4, 4, False)])
def test_sharded_motion_counts_world_gt1(N, world, wrap, mode):
    """correct_with_motion on camera shards (camx_correct_batch_sharded_motion,
    loopback communicator): every rank's counts are the whole array's
    difference-plan counts (the ranks' K3 counts all-gathered and summed),
    and its frames / maps / histograms equal the whole-array corrector's."""
    H, W, K, S = 128, 128, 4, 128
    cfg = xp.ExposureConfig(band_width=16, blocks=K)
    frames = np.stack([O.synthetic_array(N, H, W, seed=57, objects=3, frame_index=t)
                       for t in range(5)])
    d = torch.from_numpy(frames).cuda()
    batches = [(0, 2), (2, 5)]
    want = whole_array(d, batches, N, H, W, cfg, mode, wrap)
    comms = loopback_comms(world)
    parts = camera_partition(N, world)

    def rank_fn(r):
        begin, count = parts[r]
        ac = ArrayCorrector(N, H, W, cfg, mode, wrap=wrap, histograms=True, cam_begin=begin,
                            cam_count=count, comm=comms[r])
        s = torch.cuda.Stream()
        out, cnt, has = [], [], []
        with torch.cuda.stream(s):
            for lo, hi in batches:
                loc = d[lo:hi, begin:begin + count].contiguous()
                res, c, h = ac.correct_with_motion(loc, size=S, stream=s)
                assert ac.last_motion_fused
                out.append(keep(res))
                cnt.append(c.clone())
                has += h
        s.synchronize()
        return out, torch.cat(cnt).cpu().numpy(), has

    try:
        got = run_ranks(world, rank_fn)
    finally:
        for c in comms:
            c.close()
    for r, (begin, count) in enumerate(parts):
        res, cnt, has = got[r]
        assert_rank_matches(res, want, begin, count, f"rank {r}/{world}")
        assert has == [False, True, True, True, True]
        for b in range(1, 5):
            m = np.concatenate([O.mask_diff(frames[b][c], frames[b - 1][c], 20)
                                for c in range(N)], axis=1)
            _, wc = O.window_counts(m, S)
            np.testing.assert_array_equal(cnt[b], wc, f"rank {r} frame {b}")
