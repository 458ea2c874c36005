"""Wall time of the per-call drop-in API on config-2 frames (host numpy in,
host numpy out, like the reference's functions): update_exposure for one
seam and apply_exposure of one map, vs the numpy oracle port of the
reference on the same frames."""
import time

import numpy as np

from oracle import camarray_oracle as O
from paper_1910_03517_b200 import core
from paper_1910_03517_b200 import exposure as xp

H, W = 1536, 2048
arr = O.synthetic_array(2, H, W, seed=3, objects=2)
prev = O.synthetic_array(2, H, W, seed=3, objects=2, frame_index=1)
fr = [core.Frame(i, 0, 0, arr[i]) for i in range(2)]
pf = [core.Frame(i, 0, 0, prev[i]) for i in range(2)]


def best(fn, reps=10):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3


m = xp.update_exposure((fr[0], fr[1]), None)
print(f"update_exposure STANDARD: {best(lambda: xp.update_exposure((fr[0], fr[1]), None)):.2f} ms")
print(f"update_exposure OBJECT_REMOVAL: "
      f"{best(lambda: xp.update_exposure((fr[0], fr[1]), m, xp.ExposureMode.OBJECT_REMOVAL, prev_frames=(pf[0], pf[1]))):.2f} ms")
print(f"apply_exposure (one map): {best(lambda: xp.apply_exposure(fr[0], m.left)):.2f} ms")
cfg = O.Cfg()
print(f"reference port update_exposure STANDARD: "
      f"{best(lambda: O.update_exposure(arr[0], arr[1], None, O.STANDARD, cfg), 3):.2f} ms")
