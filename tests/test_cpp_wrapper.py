"""The C++ host interface (include/fsil/silhouette.hpp) compiled with g++ and linked
against libfsil.so, as a fastsil caller would use it (compute_silhouette,
PointScore/SilhouetteReport, ValidationError, plan_shards, assemble_score)."""
import os
import subprocess

import pytest

from paper_2303_14102_b200 import api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    lib_dir = os.path.dirname(api.LIB_PATH)
    exe = str(tmp_path / "wrapper_check")
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "wrapper_check.cpp"), "-L", lib_dir, "-lfsil",
           f"-Wl,-rpath,{lib_dir}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_wrapper_without_device(tmp_path):
    if os.path.exists("/dev/nvidia0"):
        pytest.skip("a GPU is present")
    exe = _build(tmp_path)
    r = subprocess.run([exe, "no-device"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_wrapper_golden(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "golden"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
