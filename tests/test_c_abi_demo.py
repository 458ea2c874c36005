"""The C ABI from plain C (examples/c_abi_demo.c): compiled with gcc against
include/camx.h and the in-tree libcamx.so, no Python on the compute path."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CUDA = Path("/usr/local/cuda")


def _build(tmp_path):
    if shutil.which("gcc") is None or not (CUDA / "include" / "cuda_runtime.h").exists():
        pytest.skip("gcc / CUDA headers not available")
    lib = ROOT / "paper_1910_03517_b200"
    if not (lib / "libcamx.so").exists():
        pytest.skip("libcamx.so not built")
    exe = tmp_path / "c_abi_demo"
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-I", str(ROOT / "include"), "-I", str(CUDA / "include"),
           str(ROOT / "examples" / "c_abi_demo.c"), "-L", str(lib), "-lcamx",
           "-L", str(CUDA / "lib64"), "-lcudart", f"-Wl,-rpath,{lib}:{CUDA / 'lib64'}", "-lm",
           "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_demo_compiles(tmp_path):
    """Header + library link cleanly from C (no GPU needed)."""
    _build(tmp_path)


@pytest.mark.gpu
def test_c_demo_runs(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith("OK")
