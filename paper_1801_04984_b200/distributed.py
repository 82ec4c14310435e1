"""Device path of the multi-GPU slab block solve (DESIGN.md section 6,
SURVEY.md 8(e)): one process per GPU, strips of cell rows per rank.

- operator: the strip-owned space-time SpMV with a neighbour halo exchange
  (parallel.DeviceStripSpMV, pdg_op_apply_strip_device);
- fixed-stress preconditioner (fixed_stress.hpp:109-139) with EXACT inner
  solves across the strips by substructuring (DeviceStripTri): every strip
  interior is solved by the library's block-tridiagonal sweep (pdg_tri_*),
  the separator system is assembled from precomputed spikes and solved
  redundantly after one all-gather per solve;
- GMRES (gmres.hpp:40-139) on owned rows with Gram-Schmidt coefficients and
  norms summed over ranks in rank order (bit-identical on every rank).

Communication goes through a `Comm` (torch.distributed): NCCL on device
tensors in production; gloo (staged through the host) lets several ranks share
one GPU in the tests without any kernel waiting on another rank's kernel.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from . import parallel as par
from ._lib import check, lib
from .solver import context


class Comm:
    """Rank-ordered collectives and point-to-point exchange on device tensors."""

    def __init__(self, dist, rank: int, nranks: int, stage_on_host: bool = False):
        self.dist, self.rank, self.nranks, self.host = dist, rank, nranks, stage_on_host

    def _out(self, t):
        return t.cpu() if self.host else t

    def ordered_sum(self, t):
        """Sum of t over ranks in rank order (all-gather then add): identical bits everywhere."""
        import torch

        if self.nranks == 1:
            return t.clone()
        src = self._out(t.contiguous())
        bufs = [torch.empty_like(src) for _ in range(self.nranks)]
        self.dist.all_gather(bufs, src)
        acc = bufs[0].clone()
        for b in bufs[1:]:
            acc += b
        return acc.to(t.device)

    def exchange(self, x, send: dict, recv: dict):
        """x[recv[k]] <- (x of rank k)[recv[k]] for the neighbour sets (global numbering)."""
        import torch

        if self.nranks == 1:
            return
        reqs, bufs = [], {}
        for k in sorted(send):
            reqs.append(self.dist.isend(self._out(x[send[k]].contiguous()), k))
        for k in sorted(recv):
            bufs[k] = torch.empty((len(recv[k]),) + tuple(x.shape[1:]), dtype=x.dtype,
                                  device="cpu" if self.host else x.device)
            reqs.append(self.dist.irecv(bufs[k], k))
        for r in reqs:
            r.wait()
        for k, idx in recv.items():
            x[idx] = bufs[k].to(x.device)


class TriSolver:
    """pdg_tri_*: exact block-tridiagonal solve of a host CSR on the device (SPD:
    twisted Cholesky; symmetric=False: twisted block LU)."""

    def __init__(self, A, block_sizes, perm=None, allow_local=True, device: int = 0, symmetric=True):
        import scipy.sparse as sp

        A = sp.csr_matrix(A)
        A.sort_indices()
        self.n = A.shape[0]
        off = np.ascontiguousarray(A.indptr, np.int32)
        idx = np.ascontiguousarray(A.indices, np.int32)
        val = np.ascontiguousarray(A.data, np.float64)
        csr = _lib.CSR(self.n, self.n, len(val), off.ctypes.data_as(C.POINTER(C.c_int)),
                       idx.ctypes.data_as(C.POINTER(C.c_int)), val.ctypes.data_as(_lib.DP))
        bs = np.ascontiguousarray(block_sizes, np.int32)
        pm = None if perm is None else np.ascontiguousarray(perm, np.int32)
        h = C.c_void_p()
        check(lib().pdg_tri_create(context(device), C.byref(csr), None if pm is None else pm.ctypes.data_as(_lib.IP),
                                   bs.ctypes.data_as(_lib.IP), len(bs),
                                   (1 if allow_local else 0) | (0 if symmetric else 2), C.byref(h)))
        self._h = h

    def solve(self, b):
        """b: (n,) or (n, k) device tensor (k <= 2 per library call)."""
        import torch

        b2 = b.reshape(self.n, -1)
        out = torch.empty_like(b2)
        for c0 in range(0, b2.shape[1], 2):
            cols = b2[:, c0:c0 + 2].t().contiguous()  # column-major: rhs after rhs
            x = torch.empty_like(cols)
            torch.cuda.synchronize()
            check(lib().pdg_tri_solve_device(self._h, cols.data_ptr(), x.data_ptr(), cols.shape[0]))
            out[:, c0:c0 + 2] = x.t()
        return out.reshape(b.shape)

    def __del__(self):
        if getattr(self, "_h", None) and _lib._lib is not None:
            _lib._lib.pdg_tri_destroy(self._h)
            self._h = None


class DeviceStripTri:
    """Rank `rank`'s part of the substructured exact solve of an SPD matrix A
    (scipy, global numbering) that is block tridiagonal under `perm` (new ->
    old) with blocks `bs`; `parts` = per-rank block ranges (parallel.block_partition
    semantics: the first block of every rank but rank 0 is its separator)."""

    def __init__(self, A, perm, bs, parts, rank, comm: Comm, device: int = 0):
        import scipy.sparse as sp
        import torch

        self.comm, self.rank, self.P = comm, rank, len(parts)
        bo = np.concatenate([[0], np.cumsum(bs)]).astype(np.int64)
        perm = np.arange(A.shape[0]) if perm is None else np.asarray(perm)
        Ap = sp.csr_matrix(A)[perm][:, perm].tocsr()
        j0, j1 = parts[rank]
        self.sep = j0 if rank > 0 else None
        self.interior = list(range(j0 + (1 if rank > 0 else 0), j1))
        rows_I = np.concatenate([np.arange(bo[j], bo[j + 1]) for j in self.interior])
        self.glob_I = perm[rows_I]
        self.glob_S = perm[bo[j0]:bo[j0 + 1]] if self.sep is not None else None
        AII = Ap[rows_I][:, rows_I]
        self.tri = TriSolver(AII, [int(bs[j]) for j in self.interior], None, True, device)
        dev = torch.device("cuda", device)
        self.dev = dev
        # spikes W = A_II^{-1} A_{I,s} for the own and the next separator
        self.W_top = self.W_bot = None
        seps = [parts[k][0] for k in range(1, self.P)]
        self.so = np.concatenate([[0], np.cumsum([bs[s] for s in seps])]).astype(np.int64)
        if self.sep is not None:
            cols = np.arange(bo[self.sep], bo[self.sep + 1])
            self.A_IS_top = Ap[rows_I][:, cols]
            self.W_top = self.tri.solve(torch.tensor(self.A_IS_top.toarray(), device=dev))
        if rank < self.P - 1:
            s2 = parts[rank + 1][0]
            cols = np.arange(bo[s2], bo[s2 + 1])
            self.A_IS_bot = Ap[rows_I][:, cols]
            self.W_bot = self.tri.solve(torch.tensor(self.A_IS_bot.toarray(), device=dev))
        # separator system S = A_SS - A_SI A_II^{-1} A_IS from the spikes, summed over ranks
        ns = int(self.so[-1])
        S = torch.zeros((ns, ns), dtype=torch.float64, device=dev)
        k = rank
        if self.sep is not None:
            a = slice(int(self.so[k - 1]), int(self.so[k]))
            cols = np.arange(bo[self.sep], bo[self.sep + 1])
            S[a, a] += torch.tensor(Ap[cols][:, cols].toarray(), device=dev)
            S[a, a] -= torch.tensor(self.A_IS_top.T.toarray(), device=dev) @ self.W_top
        if self.W_bot is not None:
            b_ = slice(int(self.so[k]), int(self.so[k + 1]))
            S[b_, b_] -= torch.tensor(self.A_IS_bot.T.toarray(), device=dev) @ self.W_bot
            if self.sep is not None:
                blk = -(torch.tensor(self.A_IS_top.T.toarray(), device=dev) @ self.W_bot)
                S[a, b_] += blk
                S[b_, a] += blk.T
        S = comm.ordered_sum(S)
        self.L = torch.linalg.cholesky(S) if ns else None
        self.ASI_top = None if self.sep is None else torch.tensor(self.A_IS_top.T.toarray(), device=dev)
        self.ASI_bot = None if self.W_bot is None else torch.tensor(self.A_IS_bot.T.toarray(), device=dev)

    def solve(self, b_glob):
        """b_glob: global-numbering device vector (n,) or right-hand sides (n, k)
        holding this rank's interior and separator entries; returns x in global
        numbering (own entries only)."""
        import torch

        B = b_glob.reshape(b_glob.shape[0], -1)
        y = self.tri.solve(B[self.glob_I])
        k = self.rank
        g = torch.zeros((int(self.so[-1]), B.shape[1]), dtype=torch.float64, device=self.dev)
        if self.sep is not None:
            g[int(self.so[k - 1]):int(self.so[k])] += B[self.glob_S] - self.ASI_top @ y
        if self.W_bot is not None:
            g[int(self.so[k]):int(self.so[k + 1])] -= self.ASI_bot @ y
        g = self.comm.ordered_sum(g)
        x = torch.zeros_like(B)
        xs = torch.cholesky_solve(g, self.L) if g.numel() else g
        xi = y
        if self.sep is not None:
            xk = xs[int(self.so[k - 1]):int(self.so[k])]
            xi = xi - self.W_top @ xk
            x[self.glob_S] = xk
        if self.W_bot is not None:
            xi = xi - self.W_bot @ xs[int(self.so[k]):int(self.so[k + 1])]
        x[self.glob_I] = xi
        return x.reshape(b_glob.shape)


class DeviceFixedStressPre:
    """One truncated fixed-stress sweep (fixed_stress.hpp:109-139) of one time
    component on this rank's strip, device tensors in global numbering."""

    def __init__(self, nx, ny, csr, misc, lam, tau, stab, rank, comm: Comm, device: int = 0):
        import scipy.sparse as sp
        import torch

        self.rank, self.comm, self.P = rank, comm, comm.nranks
        dev = torch.device("cuda", device)
        self.dev = dev
        npp = len(misc["m_p_diag"])
        nu, nq = 8 * npp, len(csr["M_q"][0]) - 1
        self.nu, self.nq, self.np = nu, nq, npp
        self.w, self.b = tau * 1.0, misc["biot_b"]
        strips = par.strip_partition(ny, self.P)
        cell_owner = np.repeat(np.arange(self.P), [r1 - r0 for r0, r1 in strips]).repeat(nx)
        face_owner = cell_owner.reshape(ny, nx)[:, 0][par.face_row(nx, ny)]
        u_owner = np.repeat(cell_owner, 8)

        def mat(name, shape):
            o, i, v = csr[name]
            return sp.csr_matrix((v, i, o), shape=shape)

        B, E, Mq, A = mat("B", (nq, npp)), mat("E", (nu, npp)), mat("M_q", (nq, nq)), mat("A", (nu, nu))
        Bt = B.T.tocsr()
        dinv = 1.0 / (-(lam * (misc["inv_m"] + stab)) * misc["m_p_diag"])

        def dplan(Mx, ro, co):
            plan = par.exchange_plans(Mx.indptr, Mx.indices, ro, co, self.P)[rank]
            return ({k: torch.as_tensor(v, device=dev) for k, v in plan["send"].items()},
                    {k: torch.as_tensor(v, device=dev) for k, v in plan["recv"].items()})

        self.plan_fp = dplan(B, face_owner, cell_owner)
        self.plan_q = dplan(Bt, cell_owner, face_owner)
        self.plan_p = dplan(E, u_owner, cell_owner)
        tsp = lambda M: torch.sparse_csr_tensor(torch.as_tensor(M.indptr, dtype=torch.int64),  # noqa: E731
                                                torch.as_tensor(M.indices, dtype=torch.int64),
                                                torch.as_tensor(M.data), size=M.shape, device=dev)
        self.B, self.Bt, self.E = tsp(B), tsp(Bt), tsp(E)
        self.dinv = torch.as_tensor(dinv, device=dev)
        self.own_c = torch.as_tensor(cell_owner == rank, device=dev)
        self.own_f = torch.as_tensor(face_owner == rank, device=dev)
        self.own_u = torch.as_tensor(u_owner == rank, device=dev)
        # flux Schur complement (face-row blocks) and displacement block (cell-row blocks)
        S = (self.w * Mq - (self.w ** 2) * (B @ sp.diags(dinv) @ Bt)).tocsr()
        perm, bs = [], []
        for j in range(ny + 1):
            before = len(perm)
            perm.extend(j * nx + i for i in range(nx))
            if j < ny:
                perm.extend(nx * (ny + 1) + i * ny + j for i in range(nx + 1))
            bs.append(len(perm) - before)
        fparts = [(r0, r1) for r0, r1 in strips]
        fparts[-1] = (fparts[-1][0], ny + 1)
        self.flow = DeviceStripTri(S, np.asarray(perm), np.asarray(bs), fparts, rank, comm, device)
        self.mech = DeviceStripTri(A, None, np.full(ny, 8 * nx), strips, rank, comm, device)

    def apply(self, r):
        """r: (nt, k) global-numbering components (owned entries valid), all k
        time components of the block at once (the inner solves batch them)."""
        import torch

        nu, nq, w = self.nu, self.nq, self.w
        oc, of, ou = self.own_c[:, None], self.own_f[:, None], self.own_u[:, None]
        fp = torch.where(oc, r[nu + nq:], torch.zeros_like(r[nu + nq:]))
        self.comm.exchange(fp, *self.plan_fp)
        rq = torch.where(of, r[nu:nu + nq] - w * (self.B @ (self.dinv[:, None] * fp)), torch.zeros_like(r[nu:nu + nq]))
        q = self.flow.solve(rq)
        self.comm.exchange(q, *self.plan_q)
        p = torch.where(oc, self.dinv[:, None] * (fp - w * (self.Bt @ q)), torch.zeros_like(fp))
        self.comm.exchange(p, *self.plan_p)
        mech = torch.where(ou, r[:nu] / w + self.b * (self.E @ p), torch.zeros_like(r[:nu]))
        u = self.mech.solve(mech)
        z = torch.zeros_like(r)
        z[:nu] = torch.where(ou, u, z[:nu])
        z[nu:nu + nq] = torch.where(of, q, z[nu:nu + nq])
        z[nu + nq:] = torch.where(oc, p, z[nu + nq:])
        return z


class DeviceDistributedBlock:
    """The transformed slab block (m components, Theta, tau; preconditioner
    lambda = Theta[0,0] per component, slab.hpp:220-227) solved by GMRES
    (gmres.hpp:40-139) across the ranks, everything on this rank's GPU. Vectors
    are this rank's owned rows of the m-component operator (parallel.row_owner)."""

    def __init__(self, spec, theta, tau, rank, comm: Comm, device: int = 0, tol=1e-10, restart=50, max_iter=400,
                 candidate="reference"):
        import torch

        from . import solver as S

        self.comm, self.rank, self.P = comm, rank, comm.nranks
        self.tol, self.restart, self.max_iter, self.candidate = tol, restart, max_iter, candidate
        theta = np.ascontiguousarray(np.atleast_2d(theta), np.float64)
        self.m = theta.shape[0]
        nx, ny = spec.nx, spec.ny
        self.dev = torch.device("cuda", device)
        ops = S.SpatialOperators.assemble(spec, device=device)
        self.ops = ops
        self.nt = ops.n_total
        csr = {k: ops.download(k) for k in ("A", "M_q", "B", "E")}
        misc = dict(m_p_diag=np.full(ops.n_p, (spec.lx / nx) * (spec.ly / ny)), biot_b=spec.biot_b,
                    inv_m=1.0 / spec.biot_m, k_dr=spec.lam + spec.mu)
        stab = misc["biot_b"] ** 2 / misc["k_dr"]
        self.op = S.SpaceTimeOperator(ops, theta, tau)
        strips = par.strip_partition(ny, self.P)
        r0, r1 = strips[rank]
        self.op.set_strip(nx, ny, r0, r1)
        send, recv = par.strip_exchange_sets(nx, ny, self.m, strips, rank)
        self.send = {k: torch.as_tensor(v, device=self.dev) for k, v in send.items()}
        self.recv = {k: torch.as_tensor(v, device=self.dev) for k, v in recv.items()}
        owner = par.row_owner(nx, ny, self.m, strips)
        self.owned = torch.as_tensor(np.flatnonzero(owner == rank), device=self.dev)
        own1 = np.flatnonzero(par.row_owner(nx, ny, 1, strips) == rank)
        self.owned_comp = torch.as_tensor(own1, device=self.dev)
        self.n_own1 = len(own1)
        self.pre = DeviceFixedStressPre(nx, ny, csr, misc, float(theta[0, 0]), tau, stab, rank, comm, device)

    def op_apply(self, v):
        import torch

        x = torch.zeros(self.m * self.nt, dtype=torch.float64, device=self.dev)
        x[self.owned] = v
        self.comm.exchange(x, self.send, self.recv)
        y = torch.zeros_like(x)
        torch.cuda.synchronize()
        self.op.apply_strip_device(x.data_ptr(), y.data_ptr())
        return y[self.owned]

    def prec(self, v):
        import torch

        R = torch.zeros((self.nt, self.m), dtype=torch.float64, device=self.dev)
        R[self.owned_comp] = v.reshape(self.m, self.n_own1).T
        return self.pre.apply(R)[self.owned_comp].T.reshape(-1)

    def nrm(self, v):
        return float(self.comm.ordered_sum((v @ v).reshape(1))[0].sqrt())

    def solve(self, b):
        """b: owned rows (device). Returns (x, report dict)."""
        import torch

        bnorm = self.nrm(b)
        hist = []
        if bnorm <= 1e-14:  # gmres.hpp:56-62
            return torch.zeros_like(b), dict(converged=True, iterations=0, history=[bnorm])
        x = torch.zeros_like(b)
        total, converged, true_res, x_zero = 0, False, bnorm, True
        hist.append(true_res)
        flexible = self.candidate == "flexible"
        while total < self.max_iter and not converged:
            r = b.clone() if x_zero else b - self.op_apply(x)
            beta = self.nrm(r)
            if beta / bnorm <= self.tol:
                converged = True
                break
            mm = min(self.restart, self.max_iter - total)
            V = torch.zeros((len(b), mm + 1), dtype=torch.float64, device=self.dev)
            Z = torch.zeros((len(b), mm), dtype=torch.float64, device=self.dev) if flexible else None
            H = np.zeros((mm + 1, mm))
            V[:, 0] = r / beta
            for k in range(mm):
                z = self.prec(V[:, k])
                if flexible:
                    Z[:, k] = z
                w = self.op_apply(z)
                for _ in range(2):  # classical Gram-Schmidt, two passes, rank-ordered sums
                    h = self.comm.ordered_sum(V[:, :k + 1].T @ w)
                    w = w - V[:, :k + 1] @ h
                    H[:k + 1, k] += h.cpu().numpy()
                H[k + 1, k] = self.nrm(w)
                breakdown = H[k + 1, k] <= 1e-14 * np.linalg.norm(H[:, k])
                if not breakdown:
                    V[:, k + 1] = w / H[k + 1, k]
                total += 1
                e1 = np.zeros(k + 2)
                e1[0] = beta
                y = torch.as_tensor(np.linalg.lstsq(H[:k + 2, :k + 1], e1, rcond=None)[0], device=self.dev)
                cand = x + (Z[:, :k + 1] @ y if flexible else self.prec(V[:, :k + 1] @ y))
                true_res = self.nrm(b - self.op_apply(cand))
                hist.append(true_res)
                if true_res / bnorm <= self.tol or breakdown or k == mm - 1 or total >= self.max_iter:
                    x, x_zero = cand, False
                    converged = true_res / bnorm <= self.tol
                    break
        return x, dict(converged=converged, iterations=total, history=hist, final_rel_res=true_res / bnorm)
