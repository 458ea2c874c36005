"""CPU-side checks of the C ABI boundary: the library loads without a GPU
and exports every function include/camx.h declares; struct layouts agree;
host-side validation raises ValueError like the reference."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1910_03517_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = (ROOT / "include" / "camx.h").read_text()


def declared_functions():
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(camx_\w+)\s*\(", HEADER, re.M)))


@pytest.fixture(scope="module")
def lib():
    if not _lib.LIB_PATH.exists():
        from paper_1910_03517_b200 import build
        build.build()
    return _lib.load()


def test_header_declares_expected_api():
    names = declared_functions()
    assert "camx_apply_array" in names and "camx_band_stats" in names
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_abi_version_and_status_strings(lib):
    assert lib.camx_abi_version() == 1
    assert lib.camx_status_string(0) == b"ok"
    assert lib.camx_status_string(-1) == b"invalid argument"


def test_struct_layouts():
    assert ctypes.sizeof(_lib.BandStatRecord) == 112
    assert ctypes.sizeof(_lib.SolveConfig) == 48
    m = re.search(r"typedef struct camx_band_stat \{(.*?)\}", HEADER, re.S).group(1)
    assert "int64_t area" in m and "raw_sumsq[3]" in m


def test_invalid_arguments_are_rejected_before_any_launch(lib):
    # band wider than W/2, K > H, bad side: negative status, no CUDA needed
    rec = np.zeros(8 * 112, np.uint8)
    assert lib.camx_band_stats(rec.ctypes.data, None, None, 1, 16, 10, 6, 1, 20,
                               rec.ctypes.data, None, None) == _lib.CAMX_EINVAL
    assert lib.camx_band_stats(rec.ctypes.data, None, None, 1, 4, 10, 2, 5, 20,
                               rec.ctypes.data, None, None) == _lib.CAMX_EINVAL
    g = np.ones(3)
    assert lib.camx_apply_map(rec.ctypes.data, rec.ctypes.data, 1, 4, 4, 7, 1, g.ctypes.data,
                              g.ctypes.data, None) == _lib.CAMX_EINVAL
    # the round-2 entry points: window grid / support queries and argument checks
    import ctypes
    nx, ny = ctypes.c_int32(), ctypes.c_int32()
    assert lib.camx_tiling_size(16384, 1536, 960, ctypes.byref(nx), ctypes.byref(ny)) == 0
    assert (nx.value, ny.value) == (18, 2)  # the 36-window config-2 plan
    assert lib.camx_tiling_size(100, 50, 60, ctypes.byref(nx), ctypes.byref(ny)) == _lib.CAMX_EINVAL
    assert lib.camx_motion_supported(30, 8, 8, 1536, 2048, 16, 960) == 1
    assert lib.camx_motion_supported(30, 8, 8, 1536, 2046, 16, 960) == 0  # unaligned rows
    assert lib.camx_motion_supported(30, 8, 8, 1536, 2048, 16, 64) == 0   # > 3 x 3 per CTA
    cnt = np.zeros(64, np.int64)
    sc = _lib.SolveConfig(0, 4, 64, 1e-3, 0.05, 0.5, 0, 0)
    args = [rec.ctypes.data, rec.ctypes.data, None, 1, 2, 0, 8, 16, 4, 20, ctypes.byref(sc), None,
            None, rec.ctypes.data, None, rec.ctypes.data, rec.ctypes.data, rec.ctypes.data, None]
    assert lib.camx_correct_batch_motion(*args, 8, 256, cnt.ctypes.data, None) == _lib.CAMX_EINVAL
    assert lib.camx_correct_batch_motion(*args, 99, 20, cnt.ctypes.data, None) == _lib.CAMX_EINVAL
    with pytest.raises(ValueError):
        _lib.check(_lib.CAMX_EINVAL, "x")
    with pytest.raises(RuntimeError):
        _lib.check(100, "x")


def test_product_fails_loudly_without_cuda():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1910_03517_b200 import exposure as xp
    from paper_1910_03517_b200.core import Frame
    f = Frame(0, 0, 0, np.zeros((8, 8, 3), np.uint8))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        xp.apply_exposure(f, xp.identity_map((0, 1), xp.Side.LEFT, 1, 4))
    # host-side validation still raises ValueError first, like the reference
    with pytest.raises(ValueError):
        xp.band_stats(f, xp.Side.LEFT, band_width=6, blocks=1)
