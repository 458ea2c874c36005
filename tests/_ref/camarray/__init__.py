"""Test shim: the `camarray` package the reference's own tests import,
with the hot-path modules replaced by this repository's drop-in.

camarray.exposure, .core, .attention and .detect ARE
paper_1910_03517_b200.exposure / .core / .attention / .detect (sys.modules
aliases), so the vendored reference tests in tests/_ref exercise the CUDA
path.  camarray.scenegen / .world3d / .tracker / .imgio are the reference's
fixture modules vendored beside this file (make_ref_tests.py); their
relative imports (`from .core import Frame`) resolve to the drop-in types.
"""

import sys

from paper_1910_03517_b200 import attention, core, detect, exposure

for _name, _mod in (("core", core), ("exposure", exposure), ("attention", attention),
                    ("detect", detect)):
    sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod

from paper_1910_03517_b200.core import (  # noqa: E402  (camarray/__init__.py:3)
    BBox, Category, Frame, Mosaic, abs_diff_threshold, concat_mosaic, iou)

__version__ = "0.1.0"
__all__ = ["BBox", "Category", "Frame", "Mosaic", "abs_diff_threshold", "concat_mosaic", "iou",
           "__version__"]
