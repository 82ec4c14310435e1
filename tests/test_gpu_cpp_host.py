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


def _build3d(tmp_path):
    exe = str(tmp_path / "slab_solve3d")
    lib = os.path.join(ROOT, "paper_1801_04984_b200", "_lib")
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "slab_solve3d.cpp"), "-L", lib, "-lporodg_b200",
                    f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    return exe


def test_cpp_host_layer_3d_compiles_and_links(tmp_path):
    assert os.path.exists(_build3d(tmp_path))


@pytest.mark.gpu
def test_cpp_host_layer_solves_3d_slab(tmp_path):
    """examples/slab_solve3d.cpp: pdg_ops_assemble3 + SlabSolver through the C++ layer (config-2 type, 8^3)."""
    out = subprocess.run([_build3d(tmp_path), "8"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "iterations=4" in out.stdout
    assert float(out.stdout.split("max|res|/scale=")[1].split()[0]) < 1e-8
    assert float(out.stdout.split("min u_z=")[1].split()[0]) < 0.0
    # SolveOptions::fast through the C++ layer, at a size whose displacement solve streams (16^3)
    uz = {}
    for mode in ("parity", "fast"):
        o = subprocess.run([_build3d(tmp_path), "16", mode], capture_output=True, text=True, timeout=300)
        assert o.returncode == 0, o.stdout + o.stderr
        assert f"({mode} mode)" in o.stdout and "iterations=4" in o.stdout
        uz[mode] = float(o.stdout.split("min u_z=")[1].split()[0])
    assert abs(uz["fast"] - uz["parity"]) <= 1e-6 * abs(uz["parity"])


def _build_adapter(tmp_path):
    exe = str(tmp_path / "adapter_main")
    lib = os.path.join(ROOT, "paper_1801_04984_b200", "_lib")
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "integration", "adapter_main.cpp"), "-L", lib, "-lporodg_b200",
                    f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    return exe


def test_reference_binding_compiles_and_links(tmp_path):
    """integration/porodg_gpu_slab.hpp (the slab.hpp binding of INTEGRATION.md) against
    stand-ins with the reference's member names."""
    assert os.path.exists(_build_adapter(tmp_path))


@pytest.mark.gpu
def test_reference_binding_solves_config0_slab_bitwise(tmp_path):
    """Reference-shaped operators -> pdg_ops_upload (mesh inferred) -> GPU slab solve:
    the same bits as the solve on the device-assembled operators."""
    out = subprocess.run([_build_adapter(tmp_path)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "mesh 16x16" in out.stdout and "bitwise 1" in out.stdout
