"""ctypes binding of libcamx.so (include/camx.h) — the product's only
compute path.

There is no CPU fallback: if the library or a CUDA device is missing, every
compute entry point raises.  Device buffers are torch CUDA tensors (torch is
the allocator/stream plumbing); the ABI itself only sees raw pointers,
sizes and a cudaStream_t.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libcamx.so"

CAMX_OK = 0
CAMX_EINVAL = -1
CAMX_EALIGN = -2
CAMX_ENCCL_BASE = 100000
CAMX_ENONCCL = 199999
SIDE_LEFT, SIDE_RIGHT = 0, 1
MODE_STANDARD, MODE_OBJECT_REMOVAL, MODE_SMOOTHING = 0, 1, 2


class BandStatRecord(ctypes.Structure):
    """camx_band_stat (112 bytes)."""

    _fields_ = [("area", ctypes.c_int64), ("valid", ctypes.c_int64),
                ("sum", ctypes.c_uint64 * 3), ("sumsq", ctypes.c_uint64 * 3),
                ("raw_sum", ctypes.c_uint64 * 3), ("raw_sumsq", ctypes.c_uint64 * 3)]


STAT_BYTES = ctypes.sizeof(BandStatRecord)
STAT_DTYPE = np.dtype([("area", "<i8"), ("valid", "<i8"), ("sum", "<u8", 3), ("sumsq", "<u8", 3),
                       ("raw_sum", "<u8", 3), ("raw_sumsq", "<u8", 3)])
assert STAT_DTYPE.itemsize == STAT_BYTES == 112


class SolveConfig(ctypes.Structure):
    """camx_solve_config."""

    _fields_ = [("mode", ctypes.c_int32), ("blocks", ctypes.c_int32),
                ("min_band_pixels", ctypes.c_int64), ("sigma_min", ctypes.c_double),
                ("alpha", ctypes.c_double), ("min_valid_fraction", ctypes.c_double),
                ("have_prev_maps", ctypes.c_int32), ("have_prev_frames", ctypes.c_int32)]


P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
F64 = ctypes.c_double

# name -> argtypes (all return int)
SIGNATURES = {
    "camx_abi_version": [],
    "camx_status_string": [ctypes.c_int],
    "camx_device_sm_count": [P],
    "camx_band_stats": [P, P, P, I64, I32, I32, I32, I32, I32, P, P, P],
    "camx_band_moments": [P, I64, I32, P, P, P, P, P],
    "camx_seam_solve": [P, I32, I32, I32, P, P, P, P, P, P, P],
    "camx_seam_solve_sharded": [P, I32, I32, I32, I32, P, P, P, P, P, P, P],
    "camx_comm_available": [],
    "camx_comm_unique_id": [P],
    "camx_comm_init": [P, P, I32, I32],
    "camx_comm_destroy": [P],
    "camx_comm_loopback_create": [I32, P],
    "camx_correct_batch_sharded": [P, P, P, I32, I32, I32, I32, I32, I32, I32, I32, I32, I32,
                                   P, P, P, P, P, P, P, P, P, I32, P, P],
    "camx_correct_batch_sharded_step": [P, P, I32, I32, I32, I32, I32, I32, I32, I32, I32, I32,
                                        P, P, P, P, P, P, P, P, P, P, P, I32, P, P, P, P],
    "camx_correct_batch": [P, P, P, I32, I32, I32, I32, I32, I32, I32, P, P, P, P, P, P, P, P, P,
                           P],
    "camx_fit_affine": [P, P, P, P, P, P, I32, F64, I64, P, P, P, P],
    "camx_smooth_maps": [P, P, P, P, I64, F64, P, P, P],
    "camx_apply_array": [P, P, I32, I32, I32, I32, I32, I32, I32, I32, P, P, P],
    "camx_apply_map": [P, P, I64, I32, I32, I32, I32, P, P, P],
    "camx_mask_diff": [P, P, I64, I32, P, P],
    "camx_mask_diff_channels": [P, P, I64, I32, I32, P, P],
    "camx_window_counts": [P, P, P, I32, I32, I32, I32, P, I32, I32, P, P],
    "camx_tiles": [P, I32, I32, I32, P, I32, I32, I32, P, P],
    "camx_tiles_shard": [P, I32, I32, I32, I32, P, P, I32, I32, I32, P, P],
    "camx_correct_and_tile": [P, P, I32, I32, I32, I32, I32, I32, P, P, P, P, I32, I32, I32, I32,
                              P, P],
    "camx_correct_batch_tiles": [P, P, P, I32, I32, I32, I32, I32, I32, I32, P, P, P, P, P, P, P,
                                 P, P, P, I32, I32, I32, I32, P, P],
    "camx_correct_batch_motion": [P, P, P, I32, I32, I32, I32, I32, I32, I32, P, P, P, P, P, P,
                                  P, P, P, I32, I32, P, P],
    "camx_tiling_size": [I32, I32, I32, P, P],
    "camx_motion_supported": [I32, I32, I32, I32, I32, I32, I32],
    "camx_correct_batch_sharded_motion": [P, P, P, I32, I32, I32, I32, I32, I32, I32, I32, I32,
                                          I32, P, P, P, P, P, P, P, P, P, P, I32, I32, P, P, P,
                                          P],
    "camx_seam_cost": [P, P, I64, I32, I32, I32, I32, P, P],
    "camx_blob_components": [P, I32, I32, I32, I32, I32, I32, P, P, I32, P, P],
}

_lib = None


def load():
    """Load libcamx.so (fails loudly when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("CAMX_LIB", LIB_PATH))
    if not path.exists():
        raise RuntimeError(
            f"camx CUDA library not found at {path}; build it with "
            "`python -m paper_1910_03517_b200.build` (there is no CPU fallback)")
    lib = ctypes.CDLL(str(path))
    for name, argt in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argt
        fn.restype = ctypes.c_char_p if name == "camx_status_string" else ctypes.c_int
    _lib = lib
    return lib


def check(status: int, what: str) -> None:
    if status == CAMX_OK:
        return
    msg = load().camx_status_string(status).decode()
    if status < 0:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: CUDA error {status} ({msg})")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
