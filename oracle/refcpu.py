"""ORACLE / TEST INFRASTRUCTURE ONLY -- ctypes view of the CPU restatement.

Loads oracle/_build/librefcpu.so (built by oracle/Makefile from
oracle/refcpu/*.{hpp,cpp}). Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this module, and
only as the checker / CPU baseline; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "librefcpu.so")
_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.refcpu_last_error.restype = C.c_char_p
    return _lib


class _Problem(C.Structure):
    _fields_ = [
        ("nx", C.c_int), ("ny", C.c_int), ("lx", C.c_double), ("ly", C.c_double),
        ("lam", C.c_double), ("mu", C.c_double), ("k_perm", C.c_double), ("eta", C.c_double),
        ("biot_m", C.c_double), ("biot_b", C.c_double), ("k_perm_cells", C.POINTER(C.c_double)),
        ("penalty", C.c_double), ("disp_kind", C.c_int * 4), ("disp_data", (C.c_double * 2) * 4),
        ("flow_kind", C.c_int * 4), ("flow_data", C.c_double * 4),
    ]


class _Problem3(C.Structure):
    _fields_ = [
        ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("lx", C.c_double), ("ly", C.c_double), ("lz", C.c_double),
        ("lam", C.c_double), ("mu", C.c_double), ("k_perm", C.c_double), ("eta", C.c_double),
        ("biot_m", C.c_double), ("biot_b", C.c_double), ("k_perm_cells", C.POINTER(C.c_double)),
        ("penalty", C.c_double), ("disp_kind", C.c_int * 6), ("disp_data", (C.c_double * 3) * 6),
        ("flow_kind", C.c_int * 6), ("flow_data", C.c_double * 6),
    ]


class _Opts(C.Structure):
    _fields_ = [("tol", C.c_double), ("restart", C.c_int), ("max_iter", C.c_int), ("sweeps", C.c_int),
                ("stab", C.c_double), ("backend", C.c_int), ("flexible", C.c_int)]


class _Report(C.Structure):
    _fields_ = [("converged", C.c_int), ("iterations", C.c_int), ("history_len", C.c_int),
                ("final_rel_res", C.c_double), ("setup_seconds", C.c_double), ("solve_seconds", C.c_double)]


class OracleError(RuntimeError):
    pass


def _check(rc):
    if rc != 0:
        raise OracleError(lib().refcpu_last_error().decode())


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


DISP = {"fixed": 0, "traction": 1, "roller_x": 2, "roller_y": 3, "roller_z": 4}
FLOW = {"pressure": 0, "no_flow": 1}
TAGS = ("left", "right", "bottom", "top")
TAGS3 = ("xlo", "xhi", "ylo", "yhi", "zlo", "zhi")


class RefProblem:
    """Assembled operators of one problem description (see
    paper_1801_04984_b200.problem.ProblemSpec.to_dict for the fields)."""

    def __init__(self, spec: dict):
        three_d = spec.get("nz") is not None
        p = _Problem3() if three_d else _Problem()
        p.nx, p.ny, p.lx, p.ly = spec["nx"], spec["ny"], spec["lx"], spec["ly"]
        if three_d:
            p.nz, p.lz = spec["nz"], spec["lz"]
        p.lam, p.mu, p.k_perm, p.eta = spec["lam"], spec["mu"], spec["k_perm"], spec["eta"]
        p.biot_m, p.biot_b, p.penalty = spec["biot_m"], spec["biot_b"], spec["penalty"]
        self._k = None
        if spec.get("k_perm_cells") is not None:
            self._k = np.ascontiguousarray(spec["k_perm_cells"], dtype=np.float64)
            p.k_perm_cells = _dp(self._k)
        for s, tag in enumerate(TAGS3 if three_d else TAGS):
            kind, data = spec["disp"][tag]
            p.disp_kind[s] = DISP[kind]
            for k, v in enumerate(data):
                p.disp_data[s][k] = v
            fk, fd = spec["flow"][tag]
            p.flow_kind[s] = FLOW[fk]
            p.flow_data[s] = fd
        self.spec = spec
        h = C.c_void_p()
        _check((lib().refcpu_create3 if three_d else lib().refcpu_create)(C.byref(p), C.byref(h)))
        self._h = h
        sz = (C.c_longlong * 8)()
        _check(lib().refcpu_sizes(self._h, sz))
        self.n_u, self.n_q, self.n_p = sz[0], sz[1], sz[2]
        self.nnz = dict(zip(("A", "M_q", "B", "E", "M_p"), sz[3:8]))
        self.n_total = self.n_u + self.n_q + self.n_p

    def __del__(self):
        if getattr(self, "_h", None):
            lib().refcpu_destroy(self._h)
            self._h = None

    def csr(self, name):
        rows = {"A": self.n_u, "M_q": self.n_q, "B": self.n_q, "E": self.n_u, "M_p": self.n_p}[name]
        which = ("A", "M_q", "B", "E", "M_p").index(name)
        nnz = self.nnz[name]
        off = np.empty(rows + 1, np.int32)
        idx = np.empty(nnz, np.int32)
        val = np.empty(nnz, np.float64)
        _check(lib().refcpu_export_csr(self._h, which, _ip(off), _ip(idx), _dp(val)))
        return off, idx, val

    def misc(self):
        mp = np.empty(self.n_p, np.float64)
        qc = np.empty(self.n_q, np.int8)
        b, im, kdr = C.c_double(), C.c_double(), C.c_double()
        _check(lib().refcpu_export_misc(self._h, _dp(mp), qc.ctypes.data_as(C.c_void_p), C.byref(b), C.byref(im),
                                        C.byref(kdr)))
        return dict(m_p_diag=mp, q_constrained=qc, biot_b=b.value, inv_m=im.value, k_dr=kdr.value)

    def assemble_rhs(self, t):
        u, q, p = np.empty(self.n_u), np.empty(self.n_q), np.empty(self.n_p)
        _check(lib().refcpu_assemble_rhs(self._h, C.c_double(t), _dp(u), _dp(q), _dp(p)))
        return u, q, p

    def set_test_fields(self, kind=1):
        """Install (1) or clear (0) the analytic, time-dependent VolumeData and boundary functions."""
        _check(lib().refcpu_set_test_fields(self._h, kind))

    def sample_rhs_data(self, t):
        """The installed fields at assemble_rhs's quadrature points at time t, as the dict
        paper_1801_04984_b200.solver.SpatialOperators.rhs_sampled takes."""
        nc, nb = self.n_p, 2 * (self.spec["nx"] + self.spec["ny"])
        out = dict(momentum=np.empty((nc, 36, 2)), darcy=np.empty((nc, 36, 2)), mass=np.empty((nc, 36)),
                   traction=np.empty((nb, 6, 2)), dirichlet=np.empty((nb, 6, 2)), flow=np.empty((nb, 6)))
        present = (C.c_int * 3)()
        _check(lib().refcpu_sample_rhs_data(self._h, C.c_double(t), _dp(out["momentum"]), _dp(out["darcy"]),
                                            _dp(out["mass"]), _dp(out["traction"]), _dp(out["dirichlet"]),
                                            _dp(out["flow"]), present))
        for k, name in enumerate(("momentum", "darcy", "mass")):
            if not present[k]:
                out[name] = None
        return out

    def sample_points3(self):
        """3D: the quadrature points of assemble_rhs3_sampled: cells (n_cells, 216, 3), boundary
        face ids, face points (n_bfaces, 36, 3)."""
        nx, ny, nz = self.spec["nx"], self.spec["ny"], self.spec["nz"]
        nb = 2 * (nx * ny + nx * nz + ny * nz)
        cxyz, ids, fxyz = np.empty((self.n_p, 216, 3)), np.empty(nb, np.int32), np.empty((nb, 36, 3))
        _check(lib().refcpu_rhs3_sample_points(self._h, _dp(cxyz), _ip(ids), _dp(fxyz)))
        return cxyz, ids, fxyz

    def rhs3_sampled(self, traction, dirichlet, flow, momentum=None, darcy=None, mass=None):
        """3D assemble_rhs with sampled volume sources and boundary data (fem3d.hpp)."""
        arrs = [None if a is None else np.ascontiguousarray(a, np.float64) for a in (momentum, darcy, mass, traction,
                                                                                      dirichlet, flow)]
        u, q, p = np.empty(self.n_u), np.empty(self.n_q), np.empty(self.n_p)
        _check(lib().refcpu_rhs3_sampled(self._h, *[None if a is None else _dp(a) for a in arrs], _dp(u), _dp(q), _dp(p)))
        return u, q, p

    def spacetime_csr(self, theta, tau):
        theta = np.ascontiguousarray(theta, dtype=np.float64)
        m = theta.shape[0]
        sp = C.c_void_p()
        rn = (C.c_longlong * 2)()
        _check(lib().refcpu_spacetime_build(self._h, m, _dp(theta), C.c_double(tau), C.byref(sp), rn))
        off = np.empty(rn[0] + 1, np.int32)
        idx = np.empty(rn[1], np.int32)
        val = np.empty(rn[1], np.float64)
        _check(lib().refcpu_spacetime_export(sp, _ip(off), _ip(idx), _dp(val)))
        lib().refcpu_spacetime_destroy(sp)
        return off, idx, val

    def apply_block(self, theta, tau, x):
        theta = np.ascontiguousarray(theta, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x)
        _check(lib().refcpu_apply_block(self._h, theta.shape[0], _dp(theta), C.c_double(tau), _dp(x), _dp(y)))
        return y

    def precondition(self, lam, tau, r, sweeps=1, stab=-1.0, backend=0):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.empty_like(r)
        _check(lib().refcpu_precondition(self._h, C.c_double(lam), C.c_double(tau), C.c_double(stab), sweeps, backend,
                                         _dp(r), _dp(z)))
        return z

    @staticmethod
    def _opts(tol, restart, max_iter, sweeps, stab, backend, flexible):
        o = _Opts()
        o.tol, o.restart, o.max_iter, o.sweeps, o.stab = tol, restart, max_iter, sweeps, stab
        o.backend, o.flexible = int(backend), int(flexible)
        return o

    def block_solve(self, r, tau, rhs, tol=1e-10, restart=50, max_iter=400, sweeps=1, stab=-1.0, backend=0,
                    flexible=False):
        ensure_schur(r)
        o = self._opts(tol, restart, max_iter, sweeps, stab, backend, flexible)
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        x = np.empty_like(rhs)
        rep = _Report()
        hist = np.empty(max_iter + 2, np.float64)
        _check(lib().refcpu_block_solve(self._h, r, C.c_double(tau), C.byref(o), _dp(rhs), _dp(x), C.byref(rep),
                                        _dp(hist), len(hist)))
        return x, dict(converged=bool(rep.converged), iterations=rep.iterations,
                       final_rel_res=rep.final_rel_res, history=hist[:rep.history_len].copy(),
                       setup_seconds=rep.setup_seconds, solve_seconds=rep.solve_seconds)

    def block_solve_theta(self, theta, tau, rhs, tol=1e-10, restart=50, max_iter=400, sweeps=1, stab=-1.0, backend=0,
                          flexible=False):
        """GMRES solve of one transformed diagonal block given its theta (m x m) directly."""
        theta = np.ascontiguousarray(np.atleast_2d(theta), dtype=np.float64)
        o = self._opts(tol, restart, max_iter, sweeps, stab, backend, flexible)
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        x = np.empty_like(rhs)
        rep = _Report()
        _check(lib().refcpu_block_solve_theta(self._h, theta.shape[0], _dp(theta), C.c_double(tau), C.byref(o),
                                              _dp(rhs), _dp(x), C.byref(rep)))
        return x, dict(converged=bool(rep.converged), iterations=rep.iterations, final_rel_res=rep.final_rel_res)

    def march(self, r, T, n_slabs, tol=1e-10, restart=50, max_iter=400, sweeps=1, stab=-1.0, backend=0,
              flexible=False, keep_states=False, max_slabs=0):
        ensure_schur(r)
        o = self._opts(tol, restart, max_iter, sweeps, stab, backend, flexible)
        its = np.zeros(n_slabs, np.int32)
        res = np.zeros(n_slabs)
        secs = np.zeros(n_slabs)
        setup = C.c_double()
        end = np.empty(self.n_total)
        run = n_slabs if max_slabs <= 0 else min(max_slabs, n_slabs)
        states = np.empty((run, r + 1, self.n_total)) if keep_states else None
        _check(lib().refcpu_march(self._h, r, C.c_double(T), n_slabs, C.byref(o), _ip(its), _dp(res), _dp(secs),
                                  C.byref(setup), _dp(end), _dp(states) if keep_states else None, max_slabs))
        return dict(iterations=its[:run], final_res=res[:run], solve_seconds=secs[:run],
                    setup_seconds=setup.value, end_state=end, states=states)

    def march_fs(self, r, T, n_slabs, tol=1e-10, max_sweeps=200, stab=-1.0, backend=0, keep_states=False,
                 max_slabs=0):
        """Fixed-stress march (march.hpp:80-108): per-slab sweep counts and final
        relative residuals (and all slab states)."""
        run = n_slabs if max_slabs <= 0 else min(max_slabs, n_slabs)
        sw = np.zeros(n_slabs, np.int32)
        res = np.zeros(n_slabs)
        secs = np.zeros(n_slabs)
        states = np.empty((run, r + 1, self.n_total)) if keep_states else None
        _check(lib().refcpu_march_fs(self._h, r, C.c_double(T), n_slabs, C.c_double(tol), max_sweeps,
                                     C.c_double(stab), backend, _ip(sw), _dp(res), _dp(secs),
                                     _dp(states) if keep_states else None, max_slabs))
        return dict(sweeps=sw[:run], final_res=res[:run], solve_seconds=secs[:run], states=states)

    def slab_rhs(self, r, t0, tau, u_prev, p_prev):
        out = np.empty((r + 1) * self.n_total)
        _check(lib().refcpu_slab_rhs(self._h, r, C.c_double(t0), C.c_double(tau),
                                     _dp(np.ascontiguousarray(u_prev, np.float64)),
                                     _dp(np.ascontiguousarray(p_prev, np.float64)), _dp(out)))
        return out

    def schur_forward(self, r, R):
        ensure_schur(r)
        R = np.ascontiguousarray(R, np.float64)
        out = np.empty_like(R)
        _check(lib().refcpu_schur_forward(self._h, r, _dp(R), _dp(out)))
        return out

    def mass_residual(self, r, tau, rhs, state):
        """local_mass_residual (slab.hpp:292-318): (|residual| per cell, scale)."""
        out = np.empty(self.n_p)
        sc = C.c_double()
        _check(lib().refcpu_mass_residual(self._h, r, C.c_double(tau), _dp(np.ascontiguousarray(rhs, np.float64)),
                                          _dp(np.ascontiguousarray(state, np.float64)), _dp(out), C.byref(sc)))
        return out, sc.value


_raw_schur_done = set()


def ensure_schur(r):
    """r >= 2: register the raw real Schur form of W = M_hat^{-1} G_hat, computed by LAPACK
    (scipy.linalg.schur), which the C++ restatement orders and standardizes as the reference
    does with Eigen::RealSchur's (solver.hpp real_schur)."""
    if r < 2 or r in _raw_schur_done:
        return
    import scipy.linalg as sl
    n = r + 1
    nodes, w, phi, G = np.empty(n), np.empty(n), np.empty(n), np.empty((n, n))
    _check(lib().refcpu_time_basis(r, _dp(nodes), _dp(w), _dp(phi), _dp(G)))
    T, Q = sl.schur(G / w[:, None], output="real")
    T, Q = np.ascontiguousarray(T), np.ascontiguousarray(Q)
    _check(lib().refcpu_set_raw_schur(r, _dp(T), _dp(Q)))
    _raw_schur_done.add(r)


def schur_blocks(r):
    ensure_schur(r)
    nb = C.c_int()
    sizes, starts = np.zeros(r + 1, np.int32), np.zeros(r + 1, np.int32)
    _check(lib().refcpu_schur_blocks(r, C.byref(nb), _ip(sizes), _ip(starts)))
    return sizes[:nb.value].copy(), starts[:nb.value].copy()


def time_constants(r):
    ensure_schur(r)
    n = r + 1
    nodes, w, phi = np.empty(n), np.empty(n), np.empty(n)
    G, T, Q = np.empty((n, n)), np.empty((n, n)), np.empty((n, n))
    _check(lib().refcpu_time_constants(r, _dp(nodes), _dp(w), _dp(phi), _dp(G), _dp(T), _dp(Q)))
    return dict(nodes=nodes, weights=w, phi_at0=phi, G_hat=G, T=T, Q=Q)


def gauss_points(n):
    pts, wts = np.empty(n), np.empty(n)
    _check(lib().refcpu_gauss(n, _dp(pts), _dp(wts)))
    return pts


def csr_apply(off, idx, val, x, threads=1):
    """SparseMatrix::apply (sparse.hpp:30-40) with 64-bit offsets."""
    off64 = np.ascontiguousarray(off, dtype=np.int64)
    y = np.empty(len(off64) - 1)
    _check(lib().refcpu_csr_apply(len(off64) - 1, off64.ctypes.data_as(C.POINTER(C.c_longlong)),
                                  _ip(np.ascontiguousarray(idx, np.int32)), _dp(np.ascontiguousarray(val, np.float64)),
                                  _dp(np.ascontiguousarray(x, np.float64)), _dp(y), threads))
    return y


def uniform(seed, n):
    out = np.empty(n)
    lib().refcpu_uniform(C.c_ulonglong(seed), C.c_longlong(n), _dp(out))
    return out


def lognormal(seed, n, sigma=1.0):
    out = np.empty(n)
    lib().refcpu_lognormal(C.c_ulonglong(seed), C.c_longlong(n), C.c_double(sigma), _dp(out))
    return out
