"""B200-native seam-exposure + attention-tile path of the arXiv 1910.03517
remote-tower pipeline (drop-in for the `camarray` reference's hot path).

Modules mirror the reference package:
  core       - Frame / Mosaic / BBox value types, GPU mask_diff
  exposure   - band_stats / fit_affine / smooth / update / apply on the GPU
  attention  - window plans, GPU window counts, Scheduler
  detect     - DetectorWindow, GPU tile crop/resize
  array      - ArrayCorrector: batched device-resident pipeline (+ host e2e)
  dist       - camera sharding across GPUs (NCCL all-gather of seam stats)

All arithmetic runs in libcamx.so (sm_100a); see include/camx.h.
"""

__version__ = "0.1.0"

from .core import BBox, Category, Frame, Mosaic, abs_diff_threshold, concat_mosaic, iou

__all__ = ["BBox", "Category", "Frame", "Mosaic", "abs_diff_threshold", "concat_mosaic", "iou"]
