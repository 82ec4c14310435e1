"""Spatial row partitioning of the space-time slab operator across ranks
(SURVEY.md 8(e)).

Ranks own contiguous strips of cell rows. Cells are numbered row-major
(`mesh.hpp:58`), so a strip owns a contiguous range of cells and therefore of
displacement dofs (8c+k) and pressure dofs (c). Faces are numbered
horizontal-by-row then vertical-by-column (`mesh.hpp:59-60`), so a strip's
faces are not contiguous; a face is owned by the rank owning the cell row it
belongs to (horizontal face at level j -> row j, the top boundary level -> the
last row; vertical faces -> their row).

Operator application on P ranks: each rank computes its own rows entirely (so
every row is still summed in the canonical order: the distributed SpMV is
bit-identical to the single-device one); the x entries it needs from other
ranks form a one-cell-row halo, exchanged point-to-point (NCCL on GPUs, gloo in
the CPU tests). Krylov dot products are one all-reduce per Gram-Schmidt pass.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def strip_partition(ny: int, nranks: int):
    """Balanced contiguous cell-row ranges [r0, r1) per rank."""
    if nranks < 1 or nranks > ny:
        raise ValueError("strip_partition: need 1 <= nranks <= ny")
    base, extra = divmod(ny, nranks)
    out, r = [], 0
    for k in range(nranks):
        h = base + (1 if k < extra else 0)
        out.append((r, r + h))
        r += h
    return out


def face_row(nx: int, ny: int):
    """Cell row of every face (mesh.hpp:59-60 numbering)."""
    nh = nx * (ny + 1)
    f = np.arange(nh + (nx + 1) * ny)
    rows = np.empty(len(f), dtype=np.int64)
    rows[:nh] = np.minimum(f[:nh] // nx, ny - 1)
    rows[nh:] = (f[nh:] - nh) % ny
    return rows


def row_owner(nx: int, ny: int, m: int, strips):
    """Owner rank of every row of the m-component space-time operator,
    layout [u_0 q_0 p_0 | u_1 q_1 p_1 | ...]."""
    n_cells = nx * ny
    cell_row = np.arange(n_cells) // nx
    rank_of_row = np.empty(ny, dtype=np.int64)
    for k, (r0, r1) in enumerate(strips):
        rank_of_row[r0:r1] = k
    u = np.repeat(rank_of_row[cell_row], 8)
    q = rank_of_row[face_row(nx, ny)]
    p = rank_of_row[cell_row]
    one = np.concatenate([u, q, p])
    return np.tile(one, m)


@dataclass
class HaloPlan:
    rank: int
    rows: np.ndarray            # global rows owned by this rank (ascending)
    recv_from: dict             # src rank -> global column indices received (ascending)
    send_to: dict               # dst rank -> global indices this rank sends (ascending)
    local_off: np.ndarray       # CSR of the owned rows
    local_idx: np.ndarray       # columns in the extended local numbering
    local_val: np.ndarray
    ext_cols: np.ndarray        # extended numbering: owned rows then halo columns

    @property
    def halo_size(self):
        return sum(len(v) for v in self.recv_from.values())


def halo_plans(off, idx, val, owner, nranks):
    """Partition a square CSR by row owner; build every rank's halo plan."""
    off = np.asarray(off, dtype=np.int64)
    idx = np.asarray(idx)
    plans = []
    needs = []
    for k in range(nranks):
        rows = np.flatnonzero(owner == k)
        lo = off[rows]
        hi = off[rows + 1]
        cols = np.concatenate([idx[a:b] for a, b in zip(lo, hi)]) if len(rows) else np.zeros(0, np.int64)
        ext = np.unique(cols[owner[cols] != k])
        needs.append(ext)
        recv = {int(s): ext[owner[ext] == s] for s in np.unique(owner[ext])}
        ext_cols = np.concatenate([rows, ext])
        pos = {int(c): i for i, c in enumerate(ext_cols)}
        l_off = np.zeros(len(rows) + 1, dtype=np.int64)
        l_off[1:] = np.cumsum(hi - lo)
        l_idx = np.fromiter((pos[int(c)] for c in cols), dtype=np.int64, count=len(cols))
        l_val = np.concatenate([val[a:b] for a, b in zip(lo, hi)]) if len(rows) else np.zeros(0)
        plans.append(HaloPlan(k, rows, recv, {}, l_off, l_idx, l_val, ext_cols))
    for k in range(nranks):
        for src, cols in plans[k].recv_from.items():
            plans[src].send_to[k] = cols
    return plans


def local_spmv(plan: HaloPlan, x_ext: np.ndarray) -> np.ndarray:
    """Rows of this rank, each summed sequentially in stored (canonical) order
    (SparseMatrix::apply semantics, sparse.hpp:30-40)."""
    y = np.empty(len(plan.rows))
    for i in range(len(plan.rows)):
        s = 0.0
        for kk in range(plan.local_off[i], plan.local_off[i + 1]):
            s += plan.local_val[kk] * x_ext[plan.local_idx[kk]]
        y[i] = s
    return y


def _p2p(dist, sends, recvs):
    """All sends and receives of one exchange as ONE batch (dist.batch_isend_irecv): with NCCL the
    ops of a batch are grouped, so neighbours that both send first cannot block each other once a
    halo outgrows the p2p buffering. sends / recvs: lists of (tensor, peer)."""
    ops = [dist.P2POp(dist.isend, t, peer) for t, peer in sends]
    ops += [dist.P2POp(dist.irecv, t, peer) for t, peer in recvs]
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def exchange_halo(plan: HaloPlan, x_global_owned: dict, dist, device="cpu"):
    """Point-to-point halo exchange with torch.distributed: returns the halo
    values in plan.ext_cols order (after the owned rows)."""
    import torch

    sends, recvs = [], []
    bufs = {}
    for dst, cols in sorted(plan.send_to.items()):
        sends.append((torch.from_numpy(np.ascontiguousarray(x_global_owned["fn"](cols))).to(device), dst))
    for src, cols in sorted(plan.recv_from.items()):
        b = torch.empty(len(cols), dtype=torch.float64, device=device)
        bufs[src] = b
        recvs.append((b, src))
    _p2p(dist, sends, recvs)
    # the halo part of ext_cols is sorted by global index, which interleaves the
    # sources (vertical faces are numbered column-major): place by position
    ext = plan.ext_cols[len(plan.rows):]
    halo = np.zeros(len(ext))
    for src, cols in plan.recv_from.items():
        halo[np.searchsorted(ext, cols)] = bufs[src].cpu().numpy()
    return halo


def distributed_spmv(plan: HaloPlan, x_owned: np.ndarray, dist) -> np.ndarray:
    """y_owned = (A x)_owned with one halo exchange."""
    lookup = {int(r): i for i, r in enumerate(plan.rows)}

    def fn(cols):
        return np.array([x_owned[lookup[int(c)]] for c in cols], dtype=np.float64)

    halo = exchange_halo(plan, {"fn": fn}, dist)
    return local_spmv(plan, np.concatenate([x_owned, halo]))


def distributed_dots(V_owned: np.ndarray, w_owned: np.ndarray, dist) -> np.ndarray:
    """Classical Gram-Schmidt coefficients V^T w: local partial dots + one
    all-reduce (the batched form the GPU GMRES uses)."""
    import torch

    part = torch.from_numpy(np.ascontiguousarray(V_owned.T @ w_owned))
    dist.all_reduce(part)
    return part.numpy()


# ---------------------------------------------------------------------------
# Exact block-tridiagonal solve across strips (the inner solves of the
# fixed-stress preconditioner, fixed_stress.hpp:109-139, on P ranks).
#
# The matrix is block tridiagonal in the strip order (cell rows for the
# displacement block, face rows for the flow Schur complement). Rank k owns the
# consecutive blocks [J_k, J_{k+1}); for k >= 1 its first block J_k is a
# separator s_k, the others are its interior I_k. Substructuring (exact):
#   1. y_I = A_II^{-1} b_I                       (per rank: its strip interior)
#   2. g = b_S - A_SI y_I                          (couplings of the strip ends)
#   3. S x_S = g, S = A_SS - A_SI A_II^{-1} A_IS  (P-1 separator blocks; S is
#      block tridiagonal, assembled at setup from the spikes and factored
#      redundantly on every rank; g travels in ONE all-gather per solve)
#   4. x_I = y_I - W_top x_{s_k} - W_bot x_{s_{k+1}}  (the spikes
#      W = A_II^{-1} A_IS, precomputed)
# On the GPU step 1 is the persistent sweep kernel on a strip (nb/P blocks,
# nb/(2P) dependent steps per chain), steps 2 and 4 are GEMVs with the spikes,
# step 3 a (P-1) m dense solve after an NCCL all-gather.
# ---------------------------------------------------------------------------


def block_partition(nb: int, nranks: int):
    """Contiguous block ranges [J_k, J_{k+1}) with >= 2 blocks on every rank
    (a separator plus at least one interior block)."""
    if nranks < 1 or nb < 2 * nranks:
        raise ValueError("block_partition: need nb >= 2 * nranks")
    base, extra = divmod(nb, nranks)
    out, j = [], 0
    for k in range(nranks):
        h = base + (1 if k < extra else 0)
        out.append((j, j + h))
        j += h
    return out


class StripBlockTri:
    """Rank k's part of the substructured exact solve. D[j] are the diagonal
    blocks and C[j] = A_{j+1,j} the couplings of the SPD block-tridiagonal
    matrix (only the rank's own blocks and the couplings at its ends are
    read)."""

    def __init__(self, D, C, parts, rank, dist=None):
        self.rank, self.parts = rank, parts
        self.P = len(parts)
        self.sizes = [D[j].shape[0] for j in range(len(D))]
        j0, j1 = parts[rank]
        self.sep = j0 if rank > 0 else None
        self.interior = list(range(j0 + (1 if rank > 0 else 0), j1))
        self.off = {}
        o = 0
        for j in self.interior:
            self.off[j] = o
            o += self.sizes[j]
        self.n_int = o
        # dense interior matrix of the strip and its Cholesky factor
        A = np.zeros((o, o))
        for j in self.interior:
            a = self.off[j]
            A[a:a + self.sizes[j], a:a + self.sizes[j]] = D[j]
            if j + 1 in self.off:
                b = self.off[j + 1]
                A[b:b + self.sizes[j + 1], a:a + self.sizes[j]] = C[j]
                A[a:a + self.sizes[j], b:b + self.sizes[j + 1]] = C[j].T
        self.L = np.linalg.cholesky(A)
        first, last = self.interior[0], self.interior[-1]
        self.first, self.last = first, last
        # spikes: W_top = A_II^{-1} A_{I, s_k} (coupling at the first interior block),
        #         W_bot = A_II^{-1} A_{I, s_{k+1}} (coupling at the last interior block)
        self.W_top = self.W_bot = None
        if self.sep is not None:
            R = np.zeros((o, self.sizes[self.sep]))
            R[self.off[first]:self.off[first] + self.sizes[first]] = C[self.sep]  # A_{J_k+1, J_k}
            self.W_top = self._solve_int(R)
        if rank < self.P - 1:
            s_next = parts[rank + 1][0]
            R = np.zeros((o, self.sizes[s_next]))
            R[self.off[last]:self.off[last] + self.sizes[last]] = C[last].T  # A_{last, J_{k+1}}
            self.W_bot = self._solve_int(R)
        self.C_first = C[self.sep] if self.sep is not None else None          # A_{first, s_k}^T
        self.C_last = C[last] if rank < self.P - 1 else None                  # A_{s_{k+1}, last}
        self.D_sep = D[self.sep] if self.sep is not None else None
        self._assemble_schur(dist)

    def _solve_int(self, R):
        z = np.linalg.solve(self.L, R)
        return np.linalg.solve(self.L.T, z)

    def _int_block(self, v, j):
        return v[self.off[j]:self.off[j] + self.sizes[j]]

    def _assemble_schur(self, dist):
        """Every rank contributes its terms of S (blocks indexed by separator
        number 1..P-1); all-gathered and summed in rank order, then factored."""
        P = self.P
        ms = [self.sizes[self.parts[k][0]] for k in range(1, P)]
        so = np.concatenate([[0], np.cumsum(ms)]).astype(int)
        contrib = np.zeros((so[-1], so[-1]))
        k = self.rank
        if self.sep is not None:  # own separator: A_ss - A_{s,first} W_top[first]
            i = k - 1
            sl = slice(so[i], so[i + 1])
            contrib[sl, sl] += self.D_sep - self.C_first.T @ self._int_block(self.W_top, self.first)
        if self.W_bot is not None:  # next separator: - A_{s',last} W_bot[last]
            i = k
            sl = slice(so[i], so[i + 1])
            contrib[sl, sl] -= self.C_last @ self._int_block(self.W_bot, self.last)
        if self.sep is not None and self.W_bot is not None:  # S_{k,k+1} = - A_{s_k,first} W_bot[first]
            a, b = slice(so[k - 1], so[k]), slice(so[k], so[k + 1])
            blk = -self.C_first.T @ self._int_block(self.W_bot, self.first)
            contrib[a, b] += blk
            contrib[b, a] += blk.T
        self.so = so
        S = self._allreduce_ordered(contrib, dist)
        self.S_chol = np.linalg.cholesky(S) if S.size else None

    def _allreduce_ordered(self, a, dist):
        """Sum over ranks in rank order (deterministic): all-gather, then add."""
        if dist is None or self.P == 1:
            return a
        import torch

        t = torch.from_numpy(np.ascontiguousarray(a))
        bufs = [torch.empty_like(t) for _ in range(self.P)]
        dist.all_gather(bufs, t)
        out = np.zeros_like(a)
        for b in bufs:
            out += b.numpy()
        return out

    def solve(self, b_int, b_sep, dist=None):
        """b_int: this rank's interior rhs (concatenated blocks), b_sep: its
        separator rhs (None on rank 0). Returns (x_int, x_sep)."""
        y = self._solve_int(b_int)
        k = self.rank
        g = np.zeros(self.so[-1])
        if self.sep is not None:
            sl = slice(self.so[k - 1], self.so[k])
            g[sl] += b_sep - self.C_first.T @ self._int_block(y, self.first)
        if self.W_bot is not None:
            sl = slice(self.so[k], self.so[k + 1])
            g[sl] -= self.C_last @ self._int_block(y, self.last)
        g = self._allreduce_ordered(g, dist)
        xs = np.linalg.solve(self.S_chol.T, np.linalg.solve(self.S_chol, g)) if g.size else g
        x = y.copy()
        x_sep = None
        if self.sep is not None:
            x_sep = xs[self.so[k - 1]:self.so[k]]
            x -= self.W_top @ x_sep
        if self.W_bot is not None:
            x -= self.W_bot @ xs[self.so[k]:self.so[k + 1]]
        return x, x_sep


# ---------------------------------------------------------------------------
# Distributed preconditioned GMRES of one dG(0) slab block on P ranks (host
# reference of the multi-GPU design). Vectors are held in
# global numbering on every rank, only the owned entries (and, after an
# exchange, the halo entries a coupling needs) are meaningful.
# ---------------------------------------------------------------------------


def exchange_plans(off, idx, row_owner, col_owner, nranks):
    """Point-to-point plans of a rectangular coupling: rank k needs the columns
    of its owned rows that other ranks own."""
    off = np.asarray(off, dtype=np.int64)
    idx = np.asarray(idx, dtype=np.int64)
    plans = [dict(recv={}, send={}) for _ in range(nranks)]
    for k in range(nranks):
        rows = np.flatnonzero(row_owner == k)
        if not len(rows):
            continue
        cols = np.unique(np.concatenate([idx[off[r]:off[r + 1]] for r in rows]))
        ext = cols[col_owner[cols] != k]
        for s in np.unique(col_owner[ext]):
            sel = ext[col_owner[ext] == s]
            plans[k]["recv"][int(s)] = sel
            plans[int(s)]["send"][k] = sel
    return plans


def exchange(vec, plan, dist):
    """Fill the halo entries of vec (global numbering) from their owners."""
    import torch

    sends, recvs, bufs = [], [], {}
    for dst, sel in sorted(plan["send"].items()):
        sends.append((torch.from_numpy(np.ascontiguousarray(vec[sel])), dst))
    for src, sel in sorted(plan["recv"].items()):
        bufs[src] = torch.empty(len(sel), dtype=torch.float64)
        recvs.append((bufs[src], src))
    _p2p(dist, sends, recvs)
    for src, sel in plan["recv"].items():
        vec[sel] = bufs[src].numpy()


def ordered_allreduce(a, dist, nranks):
    """Deterministic sum over ranks (all-gather, then add in rank order): every
    rank gets bit-identical results."""
    import torch

    if nranks == 1:
        return np.array(a, dtype=np.float64)
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    bufs = [torch.empty_like(t) for _ in range(nranks)]
    dist.all_gather(bufs, t)
    out = np.zeros_like(t.numpy())
    for b in bufs:
        out += b.numpy()
    return out


def _csr_dense_blocks(off, idx, val, perm, sizes):
    """Dense block-tridiagonal pieces of a (small) CSR matrix under a symmetric
    permutation perm (new -> old)."""
    n = len(off) - 1
    inv = np.empty(n, dtype=np.int64)
    inv[perm] = np.arange(n)
    A = np.zeros((n, n))
    for r in range(n):
        A[inv[r], inv[np.asarray(idx[off[r]:off[r + 1]], dtype=np.int64)]] = val[off[r]:off[r + 1]]
    bo = np.concatenate([[0], np.cumsum(sizes)]).astype(int)
    D = [A[bo[j]:bo[j + 1], bo[j]:bo[j + 1]].copy() for j in range(len(sizes))]
    C = [A[bo[j + 1]:bo[j + 2], bo[j]:bo[j + 1]].copy() for j in range(len(sizes) - 1)]
    return D, C, bo


class DistFixedStressPre:
    """One truncated fixed-stress sweep (fixed_stress.hpp:109-139) for one time
    component (theta = lam, w = tau) on rank `rank` of P: the flow solve by
    pressure elimination + the flux Schur complement in face-row blocks, then
    the displacement solve in cell-row blocks, both by StripBlockTri; the
    couplings B, B^T, E read one halo cell/face row from the neighbours."""

    def __init__(self, nx, ny, csr, misc, lam, tau, stab, rank, nranks, dist):
        self.rank, self.P, self.dist = rank, nranks, dist
        nq, npp = len(csr["M_q"][0]) - 1, len(misc["m_p_diag"])
        nu = 8 * npp
        self.nu, self.nq, self.np = nu, nq, npp
        self.w = tau * 1.0
        self.b = misc["biot_b"]
        strips = strip_partition(ny, nranks)
        cell_owner = np.repeat(np.arange(nranks), [r1 - r0 for r0, r1 in strips]).repeat(nx)
        self.cell_owner = cell_owner
        self.face_owner = cell_owner.reshape(ny, nx)[:, 0][face_row(nx, ny)]
        self.u_owner = np.repeat(cell_owner, 8)
        self.dinv = 1.0 / (-(lam * (misc["inv_m"] + stab)) * misc["m_p_diag"])
        self.csr = csr
        import scipy.sparse as sp

        def mat(name, shape):
            o, i, v = csr[name]
            return sp.csr_matrix((v, i, o), shape=shape)

        B = mat("B", (nq, npp))
        E = mat("E", (nu, npp))
        Mq = mat("M_q", (nq, nq))
        A = mat("A", (nu, nu))
        self.B, self.Bt, self.E = B, B.T.tocsr(), E
        self.plan_fp = exchange_plans(B.indptr, B.indices, self.face_owner, cell_owner, nranks)[rank]
        self.plan_q = exchange_plans(self.Bt.indptr, self.Bt.indices, cell_owner, self.face_owner, nranks)[rank]
        self.plan_p = exchange_plans(E.indptr, E.indices, self.u_owner, cell_owner, nranks)[rank]
        # flux Schur complement S = w M_q - w^2 B diag(dinv) B^T in face-row blocks
        S = (self.w * Mq - (self.w ** 2) * (B @ sp.diags(self.dinv) @ self.Bt)).tocsr()
        perm, bs = [], []
        for j in range(ny + 1):
            before = len(perm)
            perm.extend(j * nx + i for i in range(nx))
            if j < ny:
                perm.extend(nx * (ny + 1) + i * ny + j for i in range(nx + 1))
            bs.append(len(perm) - before)
        self.fperm = np.asarray(perm)
        D, C, self.fbo = _csr_dense_blocks(S.indptr, S.indices, S.data, self.fperm, bs)
        fparts = [(r0, r1) for r0, r1 in strips]
        fparts[-1] = (fparts[-1][0], ny + 1)
        self.flow = StripBlockTri(D, C, fparts, rank, dist)
        self.fparts = fparts
        D, C, self.abo = _csr_dense_blocks(A.indptr, A.indices, A.data, np.arange(nu), [8 * nx] * ny)
        self.mech = StripBlockTri(D, C, strips, rank, dist)
        self.strips = strips

    def _strip_solve(self, solver, parts, bo, rhs_perm):
        """Solve with a StripBlockTri given the rank's rhs in permuted numbering."""
        j0, j1 = parts[self.rank]
        b_sep = rhs_perm[bo[j0]:bo[j0 + 1]] if self.rank > 0 else None
        b_int = np.concatenate([rhs_perm[bo[j]:bo[j + 1]] for j in solver.interior])
        x_int, x_sep = solver.solve(b_int, b_sep, self.dist)
        out = np.zeros_like(rhs_perm)
        o = 0
        for j in solver.interior:
            out[bo[j]:bo[j + 1]] = x_int[o:o + bo[j + 1] - bo[j]]
            o += bo[j + 1] - bo[j]
        if x_sep is not None:
            out[bo[j0]:bo[j0 + 1]] = x_sep
        return out

    def apply(self, r):
        """r, z: one component [u q p] in global numbering (owned entries valid)."""
        nu, nq, npp, w = self.nu, self.nq, self.np, self.w
        own_c = self.cell_owner == self.rank
        own_f = self.face_owner == self.rank
        own_u = self.u_owner == self.rank
        fp = np.zeros(npp)
        fp[own_c] = r[nu + nq:][own_c]
        exchange(fp, self.plan_fp, self.dist)
        rq = np.zeros(nq)
        rq[own_f] = r[nu:nu + nq][own_f] - (w * (self.B @ (self.dinv * fp)))[own_f]
        qp = self._strip_solve(self.flow, self.fparts, self.fbo, rq[self.fperm])
        q = np.zeros(nq)
        q[self.fperm] = qp
        exchange(q, self.plan_q, self.dist)
        p = np.zeros(npp)
        p[own_c] = (self.dinv * (fp - w * (self.Bt @ q)))[own_c]
        exchange(p, self.plan_p, self.dist)
        mech = np.zeros(nu)
        mech[own_u] = r[:nu][own_u] / w + self.b * (self.E @ p)[own_u]
        u = self._strip_solve(self.mech, self.strips, self.abo, mech)
        z = np.zeros(nu + nq + npp)
        z[:nu][own_u] = u[own_u]
        z[nu:nu + nq][own_f] = q[own_f]
        z[nu + nq:][own_c] = p[own_c]
        return z


def dist_gmres(op_plan, pre, b, dist, nranks, tol=1e-10, restart=50, max_iter=400):
    """gmres_impl (gmres.hpp:40-139) with the reference candidate x + P(V y) on
    P ranks: owned-row vectors, one halo exchange per operator, classical
    Gram-Schmidt with two passes of ordered all-reduces, identical
    least-squares on every rank. b: owned rows (op_plan.rows order)."""
    rows = op_plan.rows
    n_glob = pre.nu + pre.nq + pre.np

    def op(v):
        return distributed_spmv(op_plan, v, dist)

    def prec(v):
        g = np.zeros(n_glob)
        g[rows] = v
        return pre.apply(g)[rows]

    def dots(V, w):
        return ordered_allreduce(V.T @ w, dist, nranks)

    def nrm(v):
        return float(np.sqrt(ordered_allreduce(np.array([v @ v]), dist, nranks)[0]))

    bnorm = nrm(b)
    if bnorm <= 1e-14:
        return np.zeros_like(b), dict(converged=True, iterations=0)
    x = np.zeros_like(b)
    total, converged, true_res = 0, False, bnorm
    while total < max_iter and not converged:
        r = b - op(x) if total else b.copy()
        beta = nrm(r)
        if beta / bnorm <= tol:
            converged = True
            break
        m = min(restart, max_iter - total)
        V = np.zeros((len(b), m + 1))
        H = np.zeros((m + 1, m))
        V[:, 0] = r / beta
        for k in range(m):
            w = op(prec(V[:, k]))
            for _ in range(2):
                h = dots(V[:, :k + 1], w)
                w = w - V[:, :k + 1] @ h
                H[:k + 1, k] += h
            H[k + 1, k] = nrm(w)
            breakdown = H[k + 1, k] <= 1e-14 * np.linalg.norm(H[:, k])
            if not breakdown:
                V[:, k + 1] = w / H[k + 1, k]
            total += 1
            e1 = np.zeros(k + 2)
            e1[0] = beta
            y = np.linalg.lstsq(H[:k + 2, :k + 1], e1, rcond=None)[0]
            cand = x + prec(V[:, :k + 1] @ y)
            true_res = nrm(b - op(cand))
            if true_res / bnorm <= tol or breakdown or k == m - 1 or total >= max_iter:
                x = cand
                converged = true_res / bnorm <= tol
                break
    return x, dict(converged=converged, iterations=total, final_rel_res=true_res / bnorm)


# ---------------------------------------------------------------------------
# Device path of the distributed operator (pdg_op_set_strip /
# pdg_op_apply_strip_device): every rank keeps x in global numbering, computes
# its strip's rows with the same per-row arithmetic as the single-GPU SpMV, and
# exchanges a one-cell-row halo with its neighbours (NCCL send/recv through
# torch.distributed on the device).
# ---------------------------------------------------------------------------


def strip_boundary_dofs(nx: int, ny: int, m: int, row: int):
    """Global indices (m-component layout [u_0 q_0 p_0 | ...]) of the dofs a
    neighbour needs from cell row `row`: u and p of its cells and the faces of
    face row `row` (horizontal level `row`, plus the top level when row = ny-1,
    and the vertical faces of the row)."""
    n_u, nh = 8 * nx * ny, nx * (ny + 1)
    n_q = nh + (nx + 1) * ny
    n_p = nx * ny
    nt = n_u + n_q + n_p
    cells = row * nx + np.arange(nx)
    u = (8 * cells[:, None] + np.arange(8)[None, :]).ravel()
    levels = [row] + ([ny] if row == ny - 1 else [])
    qh = np.concatenate([lv * nx + np.arange(nx) for lv in levels])
    qv = nh + np.arange(nx + 1) * ny + row
    q = n_u + np.concatenate([qh, qv])
    p = n_u + n_q + cells
    one = np.sort(np.concatenate([u, q, p]))
    return np.concatenate([one + i * nt for i in range(m)])


def strip_exchange_sets(nx: int, ny: int, m: int, strips, rank: int):
    """send[k] / recv[k] global index sets between this rank and its neighbours."""
    r0, r1 = strips[rank]
    send, recv = {}, {}
    if rank > 0:
        send[rank - 1] = strip_boundary_dofs(nx, ny, m, r0)
        recv[rank - 1] = strip_boundary_dofs(nx, ny, m, strips[rank - 1][1] - 1)
    if rank < len(strips) - 1:
        send[rank + 1] = strip_boundary_dofs(nx, ny, m, r1 - 1)
        recv[rank + 1] = strip_boundary_dofs(nx, ny, m, strips[rank + 1][0])
    return send, recv


class StripHalo:
    """The neighbour exchange of the strip partition on `device` tensors in
    global numbering (point-to-point through torch.distributed: NCCL on GPUs,
    gloo on the CPU in the tests)."""

    def __init__(self, nx: int, ny: int, m: int, rank: int, nranks: int, dist=None, device="cuda"):
        import torch

        self.rank, self.nranks, self.dist = rank, nranks, dist
        self.strips = strip_partition(ny, nranks)
        send, recv = strip_exchange_sets(nx, ny, m, self.strips, rank)
        dev = torch.device(device)
        self.send = {k: torch.as_tensor(v, dtype=torch.int64, device=dev) for k, v in send.items()}
        self.recv = {k: torch.as_tensor(v, dtype=torch.int64, device=dev) for k, v in recv.items()}
        self.sbuf = {k: torch.empty(len(v), dtype=torch.float64, device=dev) for k, v in send.items()}
        self.rbuf = {k: torch.empty(len(v), dtype=torch.float64, device=dev) for k, v in recv.items()}
        self.halo_doubles = sum(len(v) for v in recv.values())

    def exchange(self, x):
        """Fill x's halo entries from the neighbours."""
        if self.dist is None or self.nranks == 1:
            return
        for k, idx in sorted(self.send.items()):
            torch_index_select(x, idx, self.sbuf[k])
        _p2p(self.dist, [(self.sbuf[k], k) for k in sorted(self.send)], [(self.rbuf[k], k) for k in sorted(self.recv)])
        for k, idx in self.recv.items():
            x.index_copy_(0, idx, self.rbuf[k])


class DeviceStripSpMV:
    """y_owned = (A x)_owned on this rank's GPU for the strip partition of the
    space-time operator `op` (solver.SpaceTimeOperator): halo exchange of the
    neighbour boundary rows (StripHalo), then the strip SpMV
    (pdg_op_apply_strip_device)."""

    def __init__(self, op, nx: int, ny: int, m: int, rank: int, nranks: int, dist=None, device="cuda"):
        self.op = op
        self.halo = StripHalo(nx, ny, m, rank, nranks, dist, device)
        r0, r1 = self.halo.strips[rank]
        op.set_strip(nx, ny, r0, r1)
        self.halo_doubles = self.halo.halo_doubles

    def exchange(self, x):
        self.halo.exchange(x)

    def apply(self, x, y, repeats=1, times=False):
        """Exchange, then the strip SpMV (y: owned rows written). The library runs
        on its own stream, so the exchange is completed on torch's stream first."""
        import torch

        self.exchange(x)
        torch.cuda.current_stream().synchronize()
        return self.op.apply_strip_device(x.data_ptr(), y.data_ptr(), repeats, times)


def torch_index_select(x, idx, out):
    import torch

    torch.index_select(x, 0, idx, out=out)
