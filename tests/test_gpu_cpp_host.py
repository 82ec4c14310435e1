"""The host C++ layer (include/porodg_b200.hpp) over the C ABI on the GPU:
examples/slab_solve.cpp compiles against the header, links the in-tree
library and solves config 0's first slab."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    exe = str(tmp_path / "slab_solve")
    lib = os.path.join(ROOT, "paper_1801_04984_b200", "_lib")
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "slab_solve.cpp"), "-L", lib, "-lporodg_b200",
                    f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    return exe


def test_cpp_host_layer_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_cpp_host_layer_solves_config0_slab(tmp_path):
    out = subprocess.run([_build(tmp_path)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "converged=1 iterations=3" in out.stdout
    assert "fixed-stress: converged=1" in out.stdout
    worst = float(out.stdout.split("max|res|/scale=")[1].split()[0])
    assert worst < 1e-8
