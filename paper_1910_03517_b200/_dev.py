"""Device plumbing: torch supplies CUDA memory, streams and copies; all
arithmetic happens in libcamx.so kernels."""

from __future__ import annotations

import numpy as np

from . import _lib

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("paper_1910_03517_b200 needs a CUDA device (B200); "
                           "there is no CPU fallback")
    _lib.load()
    return t


def ptr(x) -> int | None:
    if x is None:
        return None
    return x.data_ptr()


def stream_handle(stream=None) -> int:
    t = torch()
    s = stream if stream is not None else t.cuda.current_stream()
    return s.cuda_stream


def to_device(a, dtype=None):
    """numpy array (or torch tensor) -> contiguous CUDA tensor."""
    t = require_cuda()
    if isinstance(a, t.Tensor):
        x = a
    else:
        arr = np.ascontiguousarray(a)
        if arr.dtype == np.bool_:
            arr = arr.view(np.uint8)
        x = t.from_numpy(arr)
    if dtype is not None:
        x = x.to(dtype)
    return x.to("cuda", non_blocking=False).contiguous()


def empty(shape, dtype):
    t = require_cuda()
    return t.empty(shape, dtype=dtype, device="cuda")


def to_host(x) -> np.ndarray:
    return x.detach().cpu().numpy()
