"""Debug: 2 gloo ranks on cuda:0, exchange path vs whole array."""
import os, sys
import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def worker(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import camarray_oracle as O
    from paper_1910_03517_b200 import exposure as xp
    from paper_1910_03517_b200.array import ArrayCorrector
    from paper_1910_03517_b200.dist import camera_partition, sharded_corrector, make_stats_exchange
    N, H, W, K, B = 5, 128, 160, 4, 3
    cfg = xp.ExposureConfig(band_width=16, blocks=K)
    frames = np.stack([O.synthetic_array(N, H, W, seed=23, objects=3, frame_index=t) for t in range(B)])
    d = torch.from_numpy(frames).cuda()
    mode = xp.ExposureMode.STANDARD
    w = ArrayCorrector(N, H, W, cfg, mode, histograms=True).correct(d)
    begin, count = camera_partition(N, world)[rank]
    ex = make_stats_exchange(N)
    full = ex(w.stats[:, begin:begin + count].contiguous())
    torch.cuda.synchronize()
    print(rank, "exchange alone equal:", torch.equal(full, w.stats), flush=True)
    ac = sharded_corrector(N, H, W, cfg, mode, histograms=True, native=False)
    g = ac.correct(d[:, begin:begin + count].contiguous())
    torch.cuda.synchronize()
    print(rank, "stats", torch.equal(g.stats, w.stats), "gain", torch.equal(g.gain, w.gain),
          "out", torch.equal(g.out, w.out[:, begin:begin + count]), flush=True)
    if not torch.equal(g.gain, w.gain):
        dd = (g.gain != w.gain)
        print(rank, "gain diff at (b, s, side, k, c):", dd.nonzero().tolist()[:12], "n", int(dd.sum()),
              "maxabs", float((g.gain - w.gain).abs().max()), flush=True)
        import ctypes
        from paper_1910_03517_b200 import _lib
        from paper_1910_03517_b200.exposure import _MODE_CODE
        sc = _lib.SolveConfig(_MODE_CODE[mode], K, int(cfg.min_band_pixels), float(cfg.sigma_min),
                              float(cfg.alpha), float(cfg.min_valid_fraction), 0, 0)
        gg = torch.empty((B, N - 1, 2, K, 3), dtype=torch.float64, device="cuda")
        oo = torch.empty_like(gg)
        okk = torch.empty((B, N - 1, K), dtype=torch.uint8, device="cuda")
        _lib.call("camx_seam_solve", g.stats.data_ptr(), B, N, 0, ctypes.byref(sc), None, None,
                  gg.data_ptr(), oo.data_ptr(), okk.data_ptr(), None)
        torch.cuda.synchronize()
        print(rank, "re-solve on gathered records == whole:", torch.equal(gg, w.gain),
              "== sharded:", torch.equal(gg, g.gain), flush=True)
    if not torch.equal(g.stats, w.stats):
        diff = (g.stats != w.stats).any(-1).any(-1).any(-1)
        print(rank, "differing (b, cam):", diff.nonzero().tolist(), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    import socket
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    mp.spawn(worker, args=(2, port), nprocs=2)
