"""Host-side mirror of the reference's slab-solve interface over the C ABI.

Names and argument meaning follow porodg (paths relative to
/root/reference/proj/include/porodg/):
  SpatialOperators       assembly.hpp:38-52   (device-resident here)
  GmresOptions           gmres.hpp:24-28
  FixedStressConfig      fixed_stress.hpp:17-22
  SolveOptions           slab.hpp:123-127     (block_solver is always the GPU gmres_fs path)
  SolverReport           gmres.hpp:15-20
  BlockSolver            one SlabSolver diagonal block (slab.hpp:154-171, :220-234)
  SlabSolver             slab.hpp:133-274 (r <= 1)
  march                  march.hpp:45-79,109-117 (monolithic-spectral branch)
Errors: SolverError for non-convergence (slab.hpp:228-230, same message text),
InvalidArgument for the reference's std::invalid_argument cases.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import InvalidArgument, SolverError, check, lib  # noqa: F401

_ctx_cache = {}


def context(device: int = 0):
    """One library context (device + stream) per device."""
    if device not in _ctx_cache:
        h = C.c_void_p()
        check(lib().pdg_ctx_create(device, C.byref(h)))
        _ctx_cache[device] = h
    return _ctx_cache[device]


def _dp(a):
    return a.ctypes.data_as(_lib.DP)


def _ip(a):
    return a.ctypes.data_as(_lib.IP)


@dataclass
class GmresOptions:
    tol: float = 1e-10
    restart: int = 100
    max_iter: int = 400


@dataclass
class FixedStressConfig:
    """FixedStressConfig (fixed_stress.hpp:17-35)."""
    stab: float = -1.0  # < 0: b^2 / K_dr
    truncation_sweeps: int = 1  # sweeps per preconditioner application
    tol: float = 1e-10  # fixed-stress march: true-residual tolerance
    max_sweeps: int = 200  # fixed-stress march: sweep limit


@dataclass
class SolveOptions:
    gmres: GmresOptions = field(default_factory=GmresOptions)
    fs: FixedStressConfig = field(default_factory=FixedStressConfig)
    # "reference": candidate x + P(V y) (gmres.hpp:116); "flexible": x + Z y (gmres_flexible)
    candidate: str = "reference"
    # "parity": exact fp64 inner solves (the reference's sparse-direct LU); "fast": the streamed
    # displacement factor of 3D meshes stored in fp32 (pdg_gmres_opts.mode; no effect in 2D)
    mode: str = "parity"

    def to_struct(self):
        o = _lib.GmresOpts()
        o.tol, o.restart, o.max_iter = self.gmres.tol, self.gmres.restart, self.gmres.max_iter
        o.sweeps, o.stab = self.fs.truncation_sweeps, self.fs.stab
        o.candidate = {"reference": 0, "flexible": 1}[self.candidate]
        o.mode = {"parity": 0, "fast": 1}[self.mode]
        return o


@dataclass
class SolverReport:
    converged: bool
    iterations: int
    final_relative_residual: float
    residual_history: np.ndarray
    device_ms: float
    kernel_launches: int
    mass_rel: float | None = None  # max per-cell local mass residual / scale (march(..., mass_check=True))


def _report(cap):
    rep = _lib.Report()
    hist = np.zeros(cap, dtype=np.float64)
    rep.history = _dp(hist)
    rep.history_cap = cap
    return rep, hist


def _to_report(rep, hist):
    return SolverReport(bool(rep.converged), rep.iterations, rep.final_rel_res, hist[:rep.history_len].copy(),
                        rep.device_ms, rep.kernel_launches)


def _csr_struct(off, idx, val, rows, cols):
    off = np.ascontiguousarray(off, np.int32)
    idx = np.ascontiguousarray(idx, np.int32)
    val = np.ascontiguousarray(val, np.float64)
    s = _lib.CSR(rows, cols, len(val), _ip(off), _ip(idx), _dp(val))
    return s, (off, idx, val)


def time_constants(r: int):
    """dG(r) constants (nodes, weights, phi(0), Schur T and Q) as the library computes them."""
    n = r + 1
    nodes, w, phi = np.empty(n), np.empty(n), np.empty(n)
    T, Q = np.empty((n, n)), np.empty((n, n))
    check(lib().pdg_time_constants(r, _dp(nodes), _dp(w), _dp(phi), _dp(T), _dp(Q)))
    nb = C.c_int()
    sizes, starts, G = np.zeros(n, np.int32), np.zeros(n, np.int32), np.empty((n, n))
    check(lib().pdg_time_schur_blocks(r, C.byref(nb), _ip(sizes), _ip(starts), _dp(G)))
    return dict(nodes=nodes, weights=w, phi_at0=phi, T=T, Q=Q, G_hat=G, block_sizes=sizes[:nb.value].copy(),
                block_starts=starts[:nb.value].copy())


class SpaceTimeOperator:
    """The canonical assembled space-time operator alone (pdg_op_*): the object
    of the SpMV bandwidth sweep (BASELINE config 3)."""

    def __init__(self, ops, theta, tau):
        self.theta = np.ascontiguousarray(np.atleast_2d(theta), np.float64)
        h = C.c_void_p()
        check(lib().pdg_op_create(ops._h, self.theta.shape[0], _dp(self.theta), tau, C.byref(h)))
        self._h = h
        rows, nnz = C.c_longlong(), C.c_longlong()
        check(lib().pdg_op_rows(self._h, C.byref(rows), C.byref(nnz)))
        self.rows, self.nnz = rows.value, nnz.value

    def apply_device(self, x_ptr: int, y_ptr: int, repeats: int = 1, times: bool = False):
        buf = (C.c_float * max(repeats, 1))() if times else None
        check(lib().pdg_op_apply_device(self._h, x_ptr, y_ptr, repeats, buf))
        return [buf[i] for i in range(repeats)] if times else None

    def csr(self):
        off = np.empty(self.rows + 1, np.int64)
        idx = np.empty(self.nnz, np.int32)
        val = np.empty(self.nnz, np.float64)
        check(lib().pdg_op_download_csr(self._h, off.ctypes.data_as(_lib.LLP), _ip(idx), _dp(val)))
        return off, idx, val

    def set_strip(self, nx: int, ny: int, r0: int, r1: int):
        """Own the rows of the strip of cell rows [r0, r1) (multi-GPU partitioning)."""
        check(lib().pdg_op_set_strip(self._h, nx, ny, r0, r1))

    def apply_strip_device(self, x_ptr: int, y_ptr: int, repeats: int = 1, times: bool = False):
        buf = (C.c_float * max(repeats, 1))() if times else None
        check(lib().pdg_op_apply_strip_device(self._h, x_ptr, y_ptr, repeats, buf))
        return [buf[i] for i in range(repeats)] if times else None

    def __del__(self):
        try:
            if getattr(self, "_h", None) and _lib._lib is not None:
                _lib._lib.pdg_op_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass


def profile(enable: bool | None = None, reset: bool = False):
    """Per-phase device timing (pdg_profile_*). Returns {phase: (ms, calls, alg_bytes)}."""
    L = lib()
    if reset:
        L.pdg_profile_reset()
    if enable is not None:
        L.pdg_profile_enable(1 if enable else 0)
    out = {}
    for i, nm in enumerate(PROFILE_PHASES):
        ms, calls, by = C.c_double(), C.c_longlong(), C.c_double()
        L.pdg_profile_read(i, C.byref(ms), C.byref(calls), C.byref(by))
        out[nm] = (ms.value, calls.value, by.value)
    return out


PROFILE_PHASES = ("spmv", "a_solve", "flow_solve", "precond_other", "krylov", "slab_transforms")


class SpatialOperators:
    """Device-resident A, M_q, B, E, m_p (SpatialOperators, assembly.hpp:38-52)."""

    def __init__(self, handle, nx, ny, nz=0):
        self._h = handle
        self.nx, self.ny, self.nz = nx, ny, nz  # nz > 0: 3D extension (24 displacement dofs per cell)
        sz = (C.c_longlong * 7)()
        check(lib().pdg_ops_sizes(self._h, sz))
        self.n_u, self.n_q, self.n_p = sz[0], sz[1], sz[2]
        self.nnz = dict(A=sz[3], M_q=sz[4], B=sz[5], E=sz[6])
        self.n_total = self.n_u + self.n_q + self.n_p

    @classmethod
    def assemble(cls, spec, device: int = 0):
        """assemble_operators (assembly.hpp:177-395) on the device."""
        p, keep = spec.to_struct()
        h = C.c_void_p()
        if isinstance(p, _lib.Problem3):  # 3D extension (assembly3d.cu)
            check(lib().pdg_ops_assemble3(context(device), C.byref(p), C.byref(h)))
            return cls(h, spec.nx, spec.ny, spec.nz)
        check(lib().pdg_ops_assemble(context(device), C.byref(p), C.byref(h)))
        del keep
        return cls(h, spec.nx, spec.ny)

    @classmethod
    def upload(cls, nx, ny, blocks, m_p_diag, q_constrained, biot_b, inv_m, k_dr, device: int = 0, nz: int = 0):
        """Upload host CSR blocks {'A','M_q','B','E': (off, idx, val)} (nz > 0: a 3D mesh)."""
        if nz > 0:
            n_u, n_p = 24 * nx * ny * nz, nx * ny * nz
            n_q = nx * ny * (nz + 1) + nx * (ny + 1) * nz + (nx + 1) * ny * nz
        else:
            n_u, n_p = 8 * nx * ny, nx * ny
            n_q = nx * (ny + 1) + (nx + 1) * ny
        dims = dict(A=(n_u, n_u), M_q=(n_q, n_q), B=(n_q, n_p), E=(n_u, n_p))
        structs, keep = {}, []
        for k, (r, c) in dims.items():
            structs[k], arrs = _csr_struct(*blocks[k], r, c)
            keep.append(arrs)
        mp = np.ascontiguousarray(m_p_diag, np.float64)
        qc = np.ascontiguousarray(q_constrained, np.int8)
        h = C.c_void_p()
        if nz > 0:
            check(lib().pdg_ops_upload3(context(device), nx, ny, nz, C.byref(structs["A"]), C.byref(structs["M_q"]),
                                        C.byref(structs["B"]), C.byref(structs["E"]), _dp(mp),
                                        qc.ctypes.data_as(C.POINTER(C.c_byte)), biot_b, inv_m, k_dr, C.byref(h)))
            return cls(h, nx, ny, nz)
        check(lib().pdg_ops_upload(context(device), nx, ny, C.byref(structs["A"]), C.byref(structs["M_q"]),
                                   C.byref(structs["B"]), C.byref(structs["E"]), _dp(mp),
                                   qc.ctypes.data_as(C.POINTER(C.c_byte)), biot_b, inv_m, k_dr, C.byref(h)))
        return cls(h, nx, ny)

    def download(self, name):
        rows = dict(A=self.n_u, M_q=self.n_q, B=self.n_q, E=self.n_u)[name]
        nnz = self.nnz[name]
        off, idx, val = np.empty(rows + 1, np.int32), np.empty(nnz, np.int32), np.empty(nnz, np.float64)
        check(lib().pdg_ops_download(self._h, ("A", "M_q", "B", "E").index(name), _ip(off), _ip(idx), _dp(val)))
        return off, idx, val

    def rhs(self, t):
        """assemble_rhs at time t (constant boundary data)."""
        u, q, p = np.empty(self.n_u), np.empty(self.n_q), np.empty(self.n_p)
        check(lib().pdg_ops_rhs(self._h, t, _dp(u), _dp(q), _dp(p)))
        return u, q, p

    def sample_points(self):
        """Quadrature points at which assemble_rhs evaluates its data (pdg_rhs_sample_points):
        cell points (n_cells, 36, 2), boundary face ids (2 nx + 2 ny,), face points (n_bfaces, 6, 2)."""
        if self.nz > 0:
            nb = 2 * (self.nx * self.ny + self.nx * self.nz + self.ny * self.nz)
            cxy, ids, fxy = np.empty((self.n_p, 216, 3)), np.empty(nb, np.int32), np.empty((nb, 36, 3))
        else:
            nb = 2 * (self.nx + self.ny)
            cxy, ids, fxy = np.empty((self.n_p, 36, 2)), np.empty(nb, np.int32), np.empty((nb, 6, 2))
        check(lib().pdg_rhs_sample_points(self._h, _dp(cxy), _ip(ids), _dp(fxy)))
        return cxy, ids, fxy

    @staticmethod
    def _samples_struct(samples):
        """samples: dict with 'traction', 'dirichlet', 'flow' and optionally 'momentum', 'darcy', 'mass'."""
        st, keep = _lib.RhsSamples(), []
        for k in ("momentum", "darcy", "mass", "traction", "dirichlet", "flow"):
            v = samples.get(k)
            if v is not None:
                a = np.ascontiguousarray(v, np.float64)
                keep.append(a)
                setattr(st, k, _dp(a))
        return st, keep

    def rhs_sampled(self, samples):
        """assemble_rhs (assembly.hpp:467-563) from fields sampled at sample_points()."""
        st, keep = self._samples_struct(samples)
        u, q, p = np.empty(self.n_u), np.empty(self.n_q), np.empty(self.n_p)
        check(lib().pdg_ops_rhs_sampled(self._h, C.byref(st), _dp(u), _dp(q), _dp(p)))
        del keep
        return u, q, p

    def mass_residual(self, r, tau, rhs, state):
        """local_mass_residual (slab.hpp:292-318) of one slab on the GPU: rhs and
        state are (r+1, n_total) (slab right-hand side and solution per Radau
        node). Returns (|residual| per cell, scale)."""
        rhs = np.ascontiguousarray(rhs, np.float64).reshape(-1)
        state = np.ascontiguousarray(state, np.float64).reshape(-1)
        if rhs.size != (r + 1) * self.n_total or state.size != (r + 1) * self.n_total:
            raise InvalidArgument("mass_residual: rhs/state must hold (r+1)*n_total values")
        res = np.empty(self.n_p)
        sc = C.c_double()
        check(lib().pdg_mass_residual(self._h, r, tau, _dp(rhs), _dp(state), _dp(res), C.byref(sc)))
        return res, sc.value

    def __del__(self):
        try:
            if getattr(self, "_h", None) and _lib._lib is not None:
                _lib._lib.pdg_ops_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass


class BlockSolver:
    """One transformed diagonal block (Theta = T_gg, kappa = 1, preconditioner
    lambda = T_gg(0,0)) solved by right-preconditioned GMRES on the GPU."""

    def __init__(self, ops: SpatialOperators, theta, tau, lambda_pre=None, opt: SolveOptions | None = None):
        self.ops = ops
        self.theta = np.ascontiguousarray(np.atleast_2d(theta), np.float64)
        self.m = self.theta.shape[0]
        self.tau = tau
        self.opt = opt or SolveOptions()
        lam = self.theta[0, 0] if lambda_pre is None else lambda_pre
        h = C.c_void_p()
        o = self.opt.to_struct()
        check(lib().pdg_block_create(ops._h, self.m, _dp(self.theta), tau, lam, C.byref(o), C.byref(h)))
        self._h = h
        rows, nnz = C.c_longlong(), C.c_longlong()
        check(lib().pdg_block_rows(self._h, C.byref(rows), C.byref(nnz)))
        self.rows, self.nnz = rows.value, nnz.value

    def solve(self, rhs):
        rhs = np.ascontiguousarray(rhs, np.float64)
        assert rhs.size == self.rows
        x = np.empty_like(rhs)
        rep, hist = _report(self.opt.gmres.max_iter + 2)
        check(lib().pdg_block_solve(self._h, _dp(rhs), _dp(x), C.byref(rep)))
        return x, _to_report(rep, hist)

    def solve_device(self, rhs_ptr: int, x_ptr: int):
        rep, hist = _report(self.opt.gmres.max_iter + 2)
        check(lib().pdg_block_solve_device(self._h, rhs_ptr, x_ptr, C.byref(rep)))
        return _to_report(rep, hist)

    def apply(self, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty_like(x)
        check(lib().pdg_block_apply(self._h, 0, _dp(x), _dp(y)))
        return y

    def apply_device(self, x_ptr: int, y_ptr: int, repeats: int = 1) -> float:
        ms = C.c_float()
        check(lib().pdg_block_apply_device(self._h, 0, x_ptr, y_ptr, repeats, C.byref(ms)))
        return ms.value

    def precondition(self, r):
        r = np.ascontiguousarray(r, np.float64)
        z = np.empty_like(r)
        check(lib().pdg_block_precondition(self._h, _dp(r), _dp(z)))
        return z

    def csr(self):
        off = np.empty(self.rows + 1, np.int64)
        idx = np.empty(self.nnz, np.int32)
        val = np.empty(self.nnz, np.float64)
        check(lib().pdg_block_download_csr(self._h, off.ctypes.data_as(_lib.LLP), _ip(idx), _dp(val)))
        return off, idx, val

    def __del__(self):
        try:
            if getattr(self, "_h", None) and _lib._lib is not None:
                _lib._lib.pdg_block_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass


class SlabSolver:
    """SlabSolver (slab.hpp:133-274) for dG(r), 0 <= r <= 5: Schur transform, one GMRES
    solve per diagonal Schur block with the back-substitution couplings, and the
    back-transform, all on the device."""

    def __init__(self, ops: SpatialOperators, r: int, tau: float, opt: SolveOptions | None = None):
        self.ops, self.r, self.tau = ops, r, tau
        self.opt = opt or SolveOptions()
        h = C.c_void_p()
        o = self.opt.to_struct()
        check(lib().pdg_slab_create(ops._h, r, tau, C.byref(o), C.byref(h)))
        self._h = h
        self.n = (r + 1) * ops.n_total

    def solve(self, rhs, out=None):
        """rhs: (r+1) * n_total stacked SlabSystem::rhs -> (r+1) * n_total state
        (written into `out` when given: a contiguous float64 host array, e.g. pinned)."""
        rhs = np.ascontiguousarray(rhs, np.float64)
        assert rhs.size == self.n
        if out is None:
            out = np.empty_like(rhs)
        elif out.dtype != np.float64 or out.size != self.n or not out.flags["C_CONTIGUOUS"]:
            raise InvalidArgument(_lib.PDG_INVALID_ARGUMENT, "slab solve: out must be a contiguous float64 array of the slab size")
        rep, hist = _report(self.opt.gmres.max_iter + 2)
        check(lib().pdg_slab_solve(self._h, _dp(rhs), _dp(out), C.byref(rep)))
        return out, _to_report(rep, hist)

    def solve_device(self, rhs_ptr: int, out_ptr: int):
        rep, hist = _report(self.opt.gmres.max_iter + 2)
        check(lib().pdg_slab_solve_device(self._h, rhs_ptr, out_ptr, C.byref(rep)))
        return _to_report(rep, hist)

    def block_reports(self):
        """Per Schur block of the last solve: (block size, GMRES iterations, final relative
        residual), blocks in ascending order (BlockReport, slab.hpp:113-119)."""
        nb = C.c_int()
        n = self.r + 1
        sizes, its, res = np.zeros(n, np.int32), np.zeros(n, np.int32), np.zeros(n)
        check(lib().pdg_slab_block_reports(self._h, C.byref(nb), _ip(sizes), _ip(its), _dp(res)))
        return [(int(sizes[g]), int(its[g]), float(res[g])) for g in range(nb.value)]

    def rhs_device(self, t0: float, u_prev_ptr: int, p_prev_ptr: int, rhs_ptr: int, tau: float | None = None):
        """build_slab_system on the device for the slab [t0, t0 + tau] (tau defaults
        to the solver's)."""
        check(lib().pdg_slab_rhs_device(self._h, t0, self.tau if tau is None else tau, u_prev_ptr, p_prev_ptr,
                                        rhs_ptr))

    def step_device(self, t0: float, prev_state_ptr: int | None, out_ptr: int, tau: float | None = None):
        """One slab of the march on the device (pdg_slab_step_device): right-hand side from the
        previous end trace (None = zero initial data) and solve, one synchronization."""
        rep, hist = _report(self.opt.gmres.max_iter + 2)
        check(lib().pdg_slab_step_device(self._h, t0, self.tau if tau is None else tau, prev_state_ptr, out_ptr,
                                         C.byref(rep)))
        return _to_report(rep, hist)

    def rhs_sampled_device(self, samples_per_node, u_prev_ptr: int, p_prev_ptr: int, rhs_ptr: int,
                           tau: float | None = None):
        """build_slab_system from sampled data: samples_per_node[i] = the fields at t0 + nodes[i] tau."""
        assert len(samples_per_node) == self.r + 1
        arr = (_lib.RhsSamples * (self.r + 1))()
        keep = []
        for i, sm in enumerate(samples_per_node):
            st, k = SpatialOperators._samples_struct(sm)
            arr[i] = st
            keep.append(k)
        check(lib().pdg_slab_rhs_sampled_device(self._h, self.tau if tau is None else tau, arr, u_prev_ptr, p_prev_ptr,
                                                rhs_ptr))
        del keep

    def mass_residual_device(self, rhs_ptr: int, state_ptr: int, residual_ptr: int, tau: float | None = None) -> float:
        """local_mass_residual (slab.hpp:292-318) of a device slab system/state
        (slab length tau, default the solver's) into residual_ptr (n_p doubles);
        returns the scale."""
        sc = C.c_double()
        check(lib().pdg_mass_residual_device(self.ops._h, self.r, self.tau if tau is None else tau, rhs_ptr,
                                             state_ptr, residual_ptr, C.byref(sc)))
        return sc.value

    def __del__(self):
        try:
            if getattr(self, "_h", None) and _lib._lib is not None:
                _lib._lib.pdg_slab_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass


class FixedStressSolver:
    """FixedStressSolver::solve (fixed_stress.hpp:144-172) of the fixed-stress
    march (march.hpp:80-108): Theta = G_hat, kappa = Radau weights, sweeps on the
    untransformed slab block from a warm start. Device path: dG(0) and dG(1)."""

    def __init__(self, ops: SpatialOperators, r: int, tau: float, cfg: FixedStressConfig | None = None):
        self.ops, self.r, self.tau = ops, r, tau
        self.cfg = cfg or FixedStressConfig()
        o = _lib.FsOpts()
        o.tol, o.max_sweeps, o.stab = self.cfg.tol, self.cfg.max_sweeps, self.cfg.stab
        h = C.c_void_p()
        check(lib().pdg_fs_create(ops._h, r, tau, C.byref(o), C.byref(h)))
        self._h = h
        self.n = (r + 1) * ops.n_total

    def solve(self, rhs, x0=None):
        rhs = np.ascontiguousarray(rhs, np.float64)
        assert rhs.size == self.n
        x0p = None if x0 is None else _dp(np.ascontiguousarray(x0, np.float64))
        out = np.empty_like(rhs)
        rep, hist = _report(self.cfg.max_sweeps + 2)
        check(lib().pdg_fs_solve(self._h, _dp(rhs), x0p, _dp(out), C.byref(rep)))
        return out, _to_report(rep, hist)

    def solve_device(self, rhs_ptr: int, x0_ptr: int | None, out_ptr: int):
        rep, hist = _report(self.cfg.max_sweeps + 2)
        check(lib().pdg_fs_solve_device(self._h, rhs_ptr, x0_ptr, out_ptr, C.byref(rep)))
        return _to_report(rep, hist)

    def __del__(self):
        try:
            if getattr(self, "_h", None) and _lib._lib is not None:
                _lib._lib.pdg_fs_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass


def uniform_partition(T: float, n_slabs: int):
    """TimePartition t_points of uniform_partition (time_basis.hpp:33-40): T*n/N, last = T."""
    if not T > 0.0 or n_slabs < 1:
        raise InvalidArgument("uniform_partition: bad arguments")
    pts = [T * n / n_slabs for n in range(n_slabs + 1)]
    pts[-1] = T
    return pts


def march(ops: SpatialOperators, r: int, T: float, n_slabs: int, opt: SolveOptions | None = None,
          keep_states: bool = False, mass_check: bool = False, method: str = "monolithic-spectral"):
    """Monolithic-spectral march (march.hpp:45-79,109-117) with a device-resident
    slab loop: the slab right-hand side, the Schur transforms and the jump data
    never leave the GPU. Returns per-slab reports (and states if asked). With
    mass_check, each report carries the slab's local mass balance
    max_c |residual_c| / scale (slab.hpp:292-318, computed on the device).
    method "fixed-stress" runs the fixed-stress branch (march.hpp:80-108): one
    FixedStressSolver per tau, warm-started from the previous end trace in every
    component; report.iterations is then the sweep count (fs_sweeps)."""
    if method not in ("monolithic-spectral", "fixed-stress"):
        raise InvalidArgument(f"march: unknown method {method!r}")
    import torch

    opt = opt or SolveOptions()
    t_points = uniform_partition(T, n_slabs)
    slab, cached_tau = None, -1.0
    nt = ops.n_total
    dev = torch.device("cuda")
    u_prev = torch.zeros(ops.n_u, dtype=torch.float64, device=dev)
    p_prev = torch.zeros(ops.n_p, dtype=torch.float64, device=dev)
    rhs = torch.empty((r + 1) * nt, dtype=torch.float64, device=dev)
    out = torch.empty_like(rhs)
    reports, states = [], []
    x0 = None
    # monolithic branch without the mass check: one library call per slab (pdg_slab_step_device:
    # right-hand side from the previous end trace + solve, one synchronization), two output
    # buffers used alternately so the previous end trace never aliases the current output
    fused = method == "monolithic-spectral" and not mass_check
    outs = (out, torch.empty_like(out)) if fused else (out, out)
    prev_ptr = None
    for n in range(n_slabs):
        # the slab's own length and start (march.hpp:63-64); the solver is rebuilt
        # only when tau changes by more than 1e-12 tau (march.hpp:72)
        tau, t0 = t_points[n + 1] - t_points[n], t_points[n]
        if slab is None or abs(tau - cached_tau) > 1e-12 * tau:
            slab = SlabSolver(ops, r, tau, opt)
            fs = FixedStressSolver(ops, r, tau, opt.fs) if method == "fixed-stress" else None
        cached_tau = tau
        out = outs[n % 2]
        if fused:
            try:
                rep = slab.step_device(t0, prev_ptr, out.data_ptr(), tau=tau)
            except SolverError as e:
                raise SolverError(e.status, f"slab {n} (t_n = {t_points[n + 1]:f}): {e}") from None
            reports.append(rep)
            prev_ptr = out.data_ptr() + 8 * r * nt
            if keep_states:
                states.append(out.cpu().numpy().copy())
            continue
        torch.cuda.synchronize()
        slab.rhs_device(t0, u_prev.data_ptr(), p_prev.data_ptr(), rhs.data_ptr(), tau=tau)
        try:
            if fs is None:
                rep = slab.solve_device(rhs.data_ptr(), out.data_ptr())
            else:  # warm start: the previous end trace in every component (march.hpp:87-93)
                rep = fs.solve_device(rhs.data_ptr(), None if x0 is None else x0.data_ptr(), out.data_ptr())
        except SolverError as e:
            raise SolverError(e.status, f"slab {n} (t_n = {t_points[n + 1]:f}): {e}") from None
        if mass_check:
            res = torch.empty(ops.n_p, dtype=torch.float64, device=dev)
            scale = slab.mass_residual_device(rhs.data_ptr(), out.data_ptr(), res.data_ptr(), tau=tau)
            rep.mass_rel = float(res.max().item()) / scale if scale > 0.0 else 0.0
        reports.append(rep)
        end = out[r * nt:(r + 1) * nt]
        u_prev.copy_(end[:ops.n_u])
        p_prev.copy_(end[ops.n_u + ops.n_q:])
        if method == "fixed-stress":
            x0 = end.repeat(r + 1)  # made before the next slab's synchronize
        if keep_states:
            states.append(out.cpu().numpy().copy())
    return reports, states
