"""The C-ABI library: loads, exports every symbol include/porodg_b200.h
declares, and its host-only utilities agree with the oracle. No GPU compute."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1801_04984_b200 import _lib, problem as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "porodg_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pdg_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    names = declared_symbols()
    assert len(names) >= 25
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(_lib.EXPORTED)


def test_version_and_error_string_without_gpu():
    L = _lib.lib()
    assert b"sm_100a" in L.pdg_version()
    assert isinstance(L.pdg_last_error(), bytes)


def test_generators_match_oracle(oracle):
    k = P.lognormal_field(P.K_SEED, 5000)
    assert np.array_equal(k, oracle.lognormal(P.K_SEED, 5000, 1.0))
    x = P.uniform_vector(P.X_SEED, 5000)
    assert np.array_equal(x, oracle.uniform(P.X_SEED, 5000))


def test_problem_struct_roundtrip():
    spec = P.config1(8)
    s, keep = spec.to_struct()
    assert s.nx == 8 and s.ny == 8 and abs(s.lam - 5769.230769230769) < 1e-9
    assert abs(s.mu - 3846.153846153846) < 1e-9
    assert list(s.disp_kind) == [1, 1, 0, 1] and list(s.flow_kind) == [1, 1, 1, 0]
    assert s.disp_data[3][1] == -1.0
    assert spec.sizes == (8 * 64, 8 * 9 * 2, 64)


def test_missing_gpu_is_loud():
    """Without a CUDA device the product path raises instead of falling back."""
    import torch
    if torch.cuda.is_available():
        return
    h = ctypes.c_void_p()
    rc = _lib.lib().pdg_ctx_create(0, ctypes.byref(h))
    assert rc != 0


def test_ctx_device_list_argument_errors():
    """pdg_ctx_create_devices (SURVEY 8(b) signature): null / empty lists are invalid arguments;
    without a GPU every listed device fails loudly and nothing is kept."""
    import torch
    L = _lib.lib()
    out = (ctypes.c_void_p * 2)()
    assert L.pdg_ctx_create_devices(None, 1, out) == _lib.PDG_INVALID_ARGUMENT
    devs = (ctypes.c_int * 2)(0, 0)
    assert L.pdg_ctx_create_devices(devs, 0, out) == _lib.PDG_INVALID_ARGUMENT
    rc = L.pdg_ctx_create_devices(devs, 2, out)
    if torch.cuda.is_available():
        assert rc == 0 and out[0] and out[1]
        L.pdg_ctx_destroy(out[0])
        L.pdg_ctx_destroy(out[1])
    else:
        assert rc != 0 and not out[0] and not out[1]


@pytest.mark.parametrize("nx,ny", [(12, 7), (7, 12), (16, 16), (5, 1), (1, 5), (1, 1), (3, 2)])
def test_mesh_dims_inferred_from_reference_operators(oracle, nx, ny):
    """pdg_ops_upload(nx = ny = 0) infers the structured mesh (mesh.hpp:42-60)
    from reference-assembled operators, so the slab.hpp adapter
    needs nothing beyond SpatialOperators. Host-only, no GPU."""
    spec = P.config1(4)
    spec.nx, spec.ny = nx, ny
    spec.k_perm_cells = P.lognormal_field(P.K_SEED, nx * ny)
    rp = oracle.RefProblem(spec.to_dict())
    off, idx, val = rp.csr("B")
    off = np.ascontiguousarray(off, np.int32)
    idx = np.ascontiguousarray(idx, np.int32)
    val = np.ascontiguousarray(val, np.float64)
    csr = _lib.CSR(rp.n_q, rp.n_p, len(val), off.ctypes.data_as(_lib.IP), idx.ctypes.data_as(_lib.IP),
                   val.ctypes.data_as(_lib.DP))
    dims = (ctypes.c_int * 2)()
    _lib.check(_lib.lib().pdg_mesh_dims_from_operators(ctypes.byref(csr), rp.n_q, dims))
    assert (dims[0], dims[1]) == (nx, ny)


def test_library_real_schur_on_random_matrices(tmp_path):
    """The library's Hessenberg + Francis double-shift QR (csrc/timebasis.hpp), which stands where
    the reference calls Eigen::RealSchur for r >= 2, on 360 seeded random matrices (n = 2..7, a
    third of them symmetric so that every 2x2 block has to split): Q orthogonal and Q T Q^T = A to
    1e-12, T quasi-upper-triangular, 2x2 blocks only for complex pairs. Host-only."""
    import subprocess
    exe = str(tmp_path / "schur_check")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "paper_1801_04984_b200", "csrc"),
                    os.path.join(ROOT, "tests", "integration", "schur_check.cpp"), "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "cases 360" in out.stdout and "bad_blocks 0" in out.stdout


@pytest.mark.parametrize("r", [0, 1, 2, 3, 4, 5])
def test_library_time_constants_match_oracle_host_only(oracle, r):
    """pdg_time_constants / pdg_time_schur_blocks are host code: checked here without a GPU. Nodes,
    weights, phi(0), G_hat agree with the oracle to roundoff (bit for bit for r <= 1, where T and Q
    are compared directly too); for r >= 2 the ordered block structure and the block eigenvalues
    agree and Q T Q^T = W."""
    from paper_1801_04984_b200 import solver as S
    lib, ref = S.time_constants(r), oracle.time_constants(r)
    n = r + 1
    for k in ("nodes", "weights", "phi_at0", "G_hat"):
        assert np.allclose(lib[k], ref[k], rtol=1e-13, atol=1e-14), k
    if r <= 1:
        for k in ("nodes", "weights", "phi_at0", "T", "Q"):
            assert np.array_equal(lib[k], ref[k]), k
    sizes, starts = oracle.schur_blocks(r) if r >= 2 else (np.array([n]), np.array([0]))
    assert np.array_equal(lib["block_sizes"], sizes) and np.array_equal(lib["block_starts"], starts)
    W = lib["G_hat"] / lib["weights"][:, None]
    assert abs(lib["Q"].T @ lib["Q"] - np.eye(n)).max() <= 1e-12
    assert abs(lib["Q"] @ lib["T"] @ lib["Q"].T - W).max() <= 1e-10 * (1 + abs(W).max())
    assert np.allclose(np.diag(lib["T"]), np.diag(ref["T"]), rtol=1e-11)


def test_new_entry_points_reject_bad_arguments():
    """Argument errors of the round-2 entry points surface as PDG_INVALID_ARGUMENT with a message,
    before any device work (no GPU needed)."""
    L = _lib.lib()
    rep = _lib.Report()
    assert L.pdg_slab_step_device(None, 0.0, 0.1, None, None, ctypes.byref(rep)) == _lib.PDG_INVALID_ARGUMENT
    assert b"null" in L.pdg_last_error()
    assert L.pdg_ops_assemble3(None, None, None) == _lib.PDG_INVALID_ARGUMENT
    assert L.pdg_ops_upload3(None, 2, 2, 2, None, None, None, None, None, None, 0.8, 0.1, 2.0, None) == _lib.PDG_INVALID_ARGUMENT
    assert L.pdg_ops_rhs_sampled(None, None, None, None, None) == _lib.PDG_INVALID_ARGUMENT
    assert L.pdg_rhs_sample_points(None, None, None, None) == _lib.PDG_INVALID_ARGUMENT
    nb = ctypes.c_int()
    assert L.pdg_slab_block_reports(None, ctypes.byref(nb), None, None, None) == _lib.PDG_INVALID_ARGUMENT
    buf = (ctypes.c_double * 64)()
    assert L.pdg_time_constants(6, buf, buf, buf, buf, buf) == _lib.PDG_INVALID_ARGUMENT
    assert L.pdg_time_constants(-1, buf, buf, buf, buf, buf) == _lib.PDG_INVALID_ARGUMENT
    assert L.pdg_time_schur_blocks(2, None, None, None, None) == _lib.PDG_INVALID_ARGUMENT
