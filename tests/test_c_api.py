"""The C ABI from plain C: examples/c_api_demo.c compiles and links against
libsd.so with include/sd.h alone, and runs (host-only calls here; the full
calendar on a GPU box)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    exe = str(tmp_path / "c_api_demo")
    cmd = ["gcc", "-std=c99", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "examples", "c_api_demo.c"), "-L", os.path.join(ROOT, "paper_2501_18512_b200"), "-lsd",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_2501_18512_b200"), "-L", "/usr/local/cuda/lib64", "-lcudart",
           "-lm", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_demo_builds_and_runs_host_calls(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert "c_api_demo:" in r.stdout


@pytest.mark.gpu
def test_c_demo_runs_calendar_on_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert "status OK" in r.stdout, r.stdout
