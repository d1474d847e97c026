"""The C++ facade (include/hpsim_b200.hpp) compiles against the C ABI and
behaves like the reference's hpsim::Cluster on its host-side error paths."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1404_5997_b200", "lib")


def build(tmp_path, std="c++17"):
    exe = str(tmp_path / f"facade_check_{std}")
    subprocess.run(["g++", f"-std={std}", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "facade_check.cpp"), "-L", LIBDIR, "-lhpsim_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


@pytest.mark.parametrize("std", ["c++17", "c++20"])
def test_facade_host_paths(tmp_path, std):
    out = subprocess.run([build(tmp_path, std)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "facade ok" in out.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("std", ["c++17", "c++20"])
def test_facade_step(tmp_path, std):
    """Pointer and Tensor run_step overloads, worker(i), gathered_model() (cluster.hpp:190-201)."""
    out = subprocess.run([build(tmp_path, std), "gpu"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
