"""The C ABI from a non-Python host: tools/c_host_demo.c is compiled with gcc
-std=c99 against include/kvmig.h and libkvmig.so (checks the header is valid
C and the symbols resolve), then run: the native scheduler on CPU, and one
paged-KV move checked byte for byte on the GPU."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2501_06709_b200", "_lib")
CUDA_LIB = "/usr/local/cuda/lib64"


def _build(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    exe = str(tmp_path / "c_host_demo")
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tools", "c_host_demo.c"), "-L", LIB, "-lkvmig", "-L", CUDA_LIB, "-lcudart",
           f"-Wl,-rpath,{LIB}:{CUDA_LIB}", "-o", exe]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    return exe


def test_c_host_scheduler(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([exe, "--cpu-only"], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "4 placements" in out.stdout and "depart(999) -> -4" in out.stdout


@pytest.mark.gpu
def test_c_host_migration(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "migration: 5 blocks" in out.stdout and "foreign layout: 3 blocks" in out.stdout
    assert "MISMATCH" not in out.stdout and out.stdout.count("bit-exact") == 2


@pytest.mark.gpu
def test_c_host_one_block_latency(tmp_path):
    """--latency: a tracked one-block 7B move issued from C lands (event to event) in tens of microseconds
    and reports its host issue time; the JSON line is what DESIGN.md quotes for a C/C++ host."""
    import json
    exe = _build(tmp_path)
    out = subprocess.run([exe, "--latency"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    d = json.loads(out.stdout.strip().splitlines()[-1])["one_block_7b_move"]
    assert d["bytes"] == 8 << 20 and 0 < d["host_issue_us_p50"] < d["issue_to_landed_us_p50"] < 200
