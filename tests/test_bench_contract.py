"""bench.py's driver contract on CPU: the reference arm prints one JSON line
with the required keys; non-zero ranks of the reference arm stay silent; the
camx arm refuses to run without a GPU (no CPU fallback)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _run(args, env_extra=None, timeout=300):
    env = dict(os.environ)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=timeout)


def test_reference_arm_json_line():
    r = _run(["--impl", "reference", "--workload", "config1", "--steps", "1", "--warmup", "0"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    d = json.loads(lines[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["unit"] == d["unit"]


def test_reference_arm_nonzero_rank_is_silent():
    r = _run(["--impl", "reference", "--workload", "config1", "--steps", "1", "--warmup", "0"],
             {"RANK": "1", "WORLD_SIZE": "2"})
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_camx_arm_needs_a_gpu():
    pytest.importorskip("torch")
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r = _run(["--steps", "1", "--warmup", "0", "--no-e2e", "--no-cpu-baseline"])
    assert r.returncode != 0
    assert "CUDA" in (r.stderr + r.stdout) or "cuda" in (r.stderr + r.stdout)


@pytest.mark.gpu
def test_camx_arm_json_line_on_gpu():
    """The camx arm's line carries the contract keys: roofline (measured K3
    launches), clocks sampled in the timed region, e2e through the host path,
    and a non-zero count of our own kernel launches."""
    r = _run(["--steps", "3", "--warmup", "3", "--batch", "4", "--e2e-batch", "2",
              "--no-cpu-baseline", "--no-secondary"])
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.strip()][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "clocks", "e2e", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["achieved"] <= 1.2 * rf["peak"]
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-3
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 3 * d["steps"]
    assert "workload" in d["config"]
    assert "FrameRing" in d["e2e"]["path"]


@pytest.mark.gpu
def test_camx_arm_secondary_workloads_on_gpu():
    """The default N=1 line also carries config4, config5 and config5m (the
    attention tick with the in-pass motion counts), each with its own
    roofline and clocks."""
    r = _run(["--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e"], timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.strip()][-1])
    sec = {x["workload"].split(":")[0]: x for x in d["secondary"]}
    assert set(sec) == {"config4", "config5", "config5m"}
    for x in sec.values():
        assert x["value"] > 0 and x["roofline"]["bound"] == "hbm" and "clocks" in x
        assert 0 < x["roofline"]["frac"] <= 1.2 and x["gpu_launches"] >= 3 * x["steps"]
    assert sec["config4"]["config"]["wrap"] and sec["config4"]["config"]["batch"] == 64
    assert sec["config5"]["config"]["tiles_per_step"] == 36 * 30
    assert 0 < sec["config5m"]["config"]["tiles_per_step"] <= 4 * 30  # Scheduler budget 4


def test_primary_workload_and_weak_scaling_batch():
    """N = 1: config 2, 30 frames.  N GPUs: config 3 with 30 N frames per
    step (each GPU corrects 240 camera-frames, like N = 1: "weak"); --batch
    and --workload override."""
    import argparse
    import bench
    ns = lambda **kw: argparse.Namespace(**{"workload": None, "batch": None, **kw})  # noqa: E731
    assert bench.main_workload(ns(), 1) == ("config2", 30, False)
    assert bench.main_workload(ns(), 8) == ("config3", 240, True)
    assert bench.main_workload(ns(batch=30), 8) == ("config3", 30, False)
    assert bench.main_workload(ns(workload="config4"), 1) == ("config4", 64, False)
