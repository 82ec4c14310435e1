"""ctypes binding of libporodg_b200.so (C ABI declared in include/porodg_b200.h).

The library is built in-tree by paper_1801_04984_b200/csrc/Makefile (sm_100a).
There is no CPU fallback: if the library cannot be loaded, or no CUDA device is
present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libporodg_b200.so")
_lib = None

PDG_OK, PDG_INVALID_ARGUMENT, PDG_NOT_CONVERGED, PDG_CUDA_ERROR, PDG_NCCL_ERROR, PDG_OUT_OF_MEMORY = range(6)


class PdgError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


class SolverError(PdgError):
    """porodg::SolverError (errors.hpp:10-13): non-convergence, singular factor."""


class InvalidArgument(PdgError, ValueError):
    """std::invalid_argument in the reference."""


class CSR(C.Structure):
    _fields_ = [("rows", C.c_int), ("cols", C.c_int), ("nnz", C.c_int), ("row_offsets", C.POINTER(C.c_int)),
                ("col_indices", C.POINTER(C.c_int)), ("values", C.POINTER(C.c_double))]


class Problem(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("lx", C.c_double), ("ly", C.c_double),
                ("lam", C.c_double), ("mu", C.c_double), ("k_perm", C.c_double), ("eta", C.c_double),
                ("biot_m", C.c_double), ("biot_b", C.c_double), ("k_perm_cells", C.POINTER(C.c_double)),
                ("penalty", C.c_double), ("disp_kind", C.c_int * 4), ("disp_data", (C.c_double * 2) * 4),
                ("flow_kind", C.c_int * 4), ("flow_data", C.c_double * 4)]


class Problem3(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("lx", C.c_double), ("ly", C.c_double),
                ("lz", C.c_double), ("lam", C.c_double), ("mu", C.c_double), ("k_perm", C.c_double),
                ("eta", C.c_double), ("biot_m", C.c_double), ("biot_b", C.c_double),
                ("k_perm_cells", C.POINTER(C.c_double)), ("penalty", C.c_double), ("disp_kind", C.c_int * 6),
                ("disp_data", (C.c_double * 3) * 6), ("flow_kind", C.c_int * 6), ("flow_data", C.c_double * 6)]


class RhsSamples(C.Structure):
    _fields_ = [("momentum", C.POINTER(C.c_double)), ("darcy", C.POINTER(C.c_double)), ("mass", C.POINTER(C.c_double)),
                ("traction", C.POINTER(C.c_double)), ("dirichlet", C.POINTER(C.c_double)),
                ("flow", C.POINTER(C.c_double))]


class GmresOpts(C.Structure):
    _fields_ = [("tol", C.c_double), ("restart", C.c_int), ("max_iter", C.c_int), ("sweeps", C.c_int),
                ("stab", C.c_double), ("candidate", C.c_int), ("mode", C.c_int)]


class FsOpts(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_sweeps", C.c_int), ("stab", C.c_double)]


class Report(C.Structure):
    _fields_ = [("converged", C.c_int), ("iterations", C.c_int), ("final_rel_res", C.c_double),
                ("history", C.POINTER(C.c_double)), ("history_cap", C.c_int), ("history_len", C.c_int),
                ("device_ms", C.c_double), ("kernel_launches", C.c_int)]


VP = C.c_void_p
DP = C.POINTER(C.c_double)
IP = C.POINTER(C.c_int)
LLP = C.POINTER(C.c_longlong)

_SIGS = {
    "pdg_last_error": (C.c_char_p, []),
    "pdg_version": (C.c_char_p, []),
    "pdg_ctx_create": (C.c_int, [C.c_int, C.POINTER(VP)]),
    "pdg_ctx_create_devices": (C.c_int, [IP, C.c_int, C.POINTER(VP)]),
    "pdg_ctx_destroy": (None, [VP]),
    "pdg_ops_upload": (C.c_int, [VP, C.c_int, C.c_int, C.POINTER(CSR), C.POINTER(CSR), C.POINTER(CSR),
                                 C.POINTER(CSR), DP, C.POINTER(C.c_byte), C.c_double, C.c_double, C.c_double,
                                 C.POINTER(VP)]),
    "pdg_mesh_dims_from_operators": (C.c_int, [C.POINTER(CSR), C.c_int, IP]),
    "pdg_ops_assemble": (C.c_int, [VP, C.POINTER(Problem), C.POINTER(VP)]),
    "pdg_ops_assemble3": (C.c_int, [VP, C.POINTER(Problem3), C.POINTER(VP)]),
    "pdg_ops_upload3": (C.c_int, [VP, C.c_int, C.c_int, C.c_int, C.POINTER(CSR), C.POINTER(CSR), C.POINTER(CSR),
                                  C.POINTER(CSR), DP, C.POINTER(C.c_byte), C.c_double, C.c_double, C.c_double,
                                  C.POINTER(VP)]),
    "pdg_ops_sizes": (C.c_int, [VP, LLP]),
    "pdg_ops_download": (C.c_int, [VP, C.c_int, IP, IP, DP]),
    "pdg_ops_rhs": (C.c_int, [VP, C.c_double, DP, DP, DP]),
    "pdg_rhs_sample_points": (C.c_int, [VP, DP, IP, DP]),
    "pdg_ops_rhs_sampled": (C.c_int, [VP, C.POINTER(RhsSamples), DP, DP, DP]),
    "pdg_ops_destroy": (None, [VP]),
    "pdg_block_create": (C.c_int, [VP, C.c_int, DP, C.c_double, C.c_double, C.POINTER(GmresOpts), C.POINTER(VP)]),
    "pdg_block_rows": (C.c_int, [VP, LLP, LLP]),
    "pdg_block_solve": (C.c_int, [VP, DP, DP, C.POINTER(Report)]),
    "pdg_block_solve_device": (C.c_int, [VP, C.c_void_p, C.c_void_p, C.POINTER(Report)]),
    "pdg_block_apply": (C.c_int, [VP, C.c_int, DP, DP]),
    "pdg_block_apply_device": (C.c_int, [VP, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_float)]),
    "pdg_block_precondition": (C.c_int, [VP, DP, DP]),
    "pdg_block_download_csr": (C.c_int, [VP, LLP, IP, DP]),
    "pdg_block_destroy": (None, [VP]),
    "pdg_slab_create": (C.c_int, [VP, C.c_int, C.c_double, C.POINTER(GmresOpts), C.POINTER(VP)]),
    "pdg_slab_solve": (C.c_int, [VP, DP, DP, C.POINTER(Report)]),
    "pdg_slab_solve_device": (C.c_int, [VP, C.c_void_p, C.c_void_p, C.POINTER(Report)]),
    "pdg_slab_rhs_device": (C.c_int, [VP, C.c_double, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]),
    "pdg_slab_block_reports": (C.c_int, [VP, IP, IP, IP, DP]),
    "pdg_slab_step_device": (C.c_int, [VP, C.c_double, C.c_double, C.c_void_p, C.c_void_p, C.POINTER(Report)]),
    "pdg_slab_rhs_sampled_device": (C.c_int, [VP, C.c_double, C.POINTER(RhsSamples), C.c_void_p, C.c_void_p, C.c_void_p]),
    "pdg_slab_destroy": (None, [VP]),
    "pdg_fs_create": (C.c_int, [VP, C.c_int, C.c_double, C.POINTER(FsOpts), C.POINTER(VP)]),
    "pdg_fs_solve": (C.c_int, [VP, DP, DP, DP, C.POINTER(Report)]),
    "pdg_fs_solve_device": (C.c_int, [VP, VP, VP, VP, C.POINTER(Report)]),
    "pdg_fs_destroy": (None, [VP]),
    "pdg_spmv_csr_device": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "pdg_op_create": (C.c_int, [VP, C.c_int, DP, C.c_double, C.POINTER(VP)]),
    "pdg_op_rows": (C.c_int, [VP, LLP, LLP]),
    "pdg_op_apply_device": (C.c_int, [VP, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_float)]),
    "pdg_op_set_strip": (C.c_int, [VP, C.c_int, C.c_int, C.c_int, C.c_int]),
    "pdg_op_apply_strip_device": (C.c_int, [VP, VP, VP, C.c_int, C.POINTER(C.c_float)]),
    "pdg_op_download_csr": (C.c_int, [VP, LLP, IP, DP]),
    "pdg_op_destroy": (None, [VP]),
    "pdg_nccl_unique_id": (C.c_int, [C.POINTER(C.c_ubyte)]),
    "pdg_comm_create_nccl": (C.c_int, [VP, C.c_int, C.c_int, C.POINTER(C.c_ubyte), C.POINTER(VP)]),
    "pdg_comm_create_host": (C.c_int, [VP, C.c_int, C.c_int, C.c_void_p, C.c_void_p, VP, C.POINTER(VP)]),
    "pdg_comm_destroy": (None, [VP]),
    "pdg_dblock_create": (C.c_int, [VP, VP, C.c_int, DP, C.c_double, C.c_double, C.POINTER(GmresOpts), C.POINTER(VP)]),
    "pdg_dblock_rows": (C.c_int, [VP, LLP, LLP]),
    "pdg_dblock_owned_rows": (C.c_int, [VP, LLP]),
    "pdg_dblock_solve_device": (C.c_int, [VP, VP, VP, C.POINTER(Report)]),
    "pdg_dblock_apply_device": (C.c_int, [VP, VP, VP]),
    "pdg_dblock_precondition_device": (C.c_int, [VP, VP, VP]),
    "pdg_dblock_destroy": (None, [VP]),
    "pdg_setup_reset": (None, []),
    "pdg_setup_read": (C.c_int, [C.POINTER(C.c_double), C.c_int]),
    "pdg_profile_enable": (None, [C.c_int]),
    "pdg_profile_reset": (None, []),
    "pdg_profile_read": (C.c_int, [C.c_int, C.POINTER(C.c_double), LLP, C.POINTER(C.c_double)]),
    "pdg_tri_create": (C.c_int, [VP, C.POINTER(CSR), IP, IP, C.c_int, C.c_int, C.POINTER(VP)]),
    "pdg_tri_solve_device": (C.c_int, [VP, VP, VP, C.c_int]),
    "pdg_tri_destroy": (None, [VP]),
    "pdg_mass_residual": (C.c_int, [VP, C.c_int, C.c_double, DP, DP, DP, DP]),
    "pdg_mass_residual_device": (C.c_int, [VP, C.c_int, C.c_double, VP, VP, VP, DP]),
    "pdg_time_constants": (C.c_int, [C.c_int, DP, DP, DP, DP, DP]),
    "pdg_time_schur_blocks": (C.c_int, [C.c_int, IP, IP, IP, DP]),
    "pdg_debug_recurrence_timing": (C.c_int, [VP, C.c_int, C.POINTER(C.c_ulonglong), C.c_longlong, IP, IP]),
    "pdg_util_uniform": (None, [C.c_ulonglong, C.c_longlong, DP]),
    "pdg_util_lognormal": (None, [C.c_ulonglong, C.c_longlong, C.c_double, DP]),
    "pdg_util_launch_count": (C.c_longlong, []),
}

EXPORTED = tuple(_SIGS)


def build() -> None:
    subprocess.run(["make", "-s", "-j8", "-C", os.path.join(_HERE, "csrc")], check=True)


def lib():
    """Load the CUDA library (raises if it is missing: no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"porodg_b200 CUDA library not built: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != PDG_OK:
        msg = lib().pdg_last_error().decode()
        if rc == PDG_NOT_CONVERGED:
            raise SolverError(rc, msg)
        if rc == PDG_INVALID_ARGUMENT:
            raise InvalidArgument(rc, msg)
        raise PdgError(rc, msg)
