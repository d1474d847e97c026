"""The C++ facade (include/hpsim_b200.hpp) compiles against the C ABI and
behaves like the reference's hpsim::Cluster on its host-side error paths."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1404_5997_b200", "lib")


def build(tmp_path):
    exe = str(tmp_path / "facade_check")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "facade_check.cpp"), "-L", LIBDIR, "-lhpsim_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_facade_host_paths(tmp_path):
    out = subprocess.run([build(tmp_path)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "facade ok" in out.stdout


@pytest.mark.gpu
def test_facade_step(tmp_path):
    out = subprocess.run([build(tmp_path), "gpu"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
