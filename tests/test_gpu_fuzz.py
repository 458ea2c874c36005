"""Randomised parity sweep (tools/fuzz_parity.py) in the GPU tier: random
geometries (incl. unaligned widths, wrap arrays, 1..12 blocks), modes and
batches through ArrayCorrector (two consecutive batches) against the oracle
tick loop, band histograms, the attention-tick motion counts (fused and
fallback paths) and camx_tiles (random windows and output sizes); and
random camera-sharded arrays through the native world > 1 path.  Round-2
runs: 400 + 120 + 300 single-GPU cases (0 LSB flips) and 30 + 75 shard
cases, all equal."""

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


@pytest.mark.parametrize("seed", [21, 22])
def test_random_camera_shard_cases_match_whole_array(seed):
    """Random camera-sharded arrays (loopback world 2..4, correct or
    submit/flush, sharded tiles) against the whole-array corrector."""
    rng = np.random.default_rng(seed)
    for i in range(4):
        fuzz_parity.shard_case(rng, i)
