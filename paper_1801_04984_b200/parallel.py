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


def exchange_halo(plan: HaloPlan, x_global_owned: dict, dist, device="cpu"):
    """Point-to-point halo exchange with torch.distributed: returns the halo
    values in plan.ext_cols order (after the owned rows)."""
    import torch

    reqs = []
    bufs = {}
    for dst, cols in sorted(plan.send_to.items()):
        t = torch.from_numpy(np.ascontiguousarray(x_global_owned["fn"](cols))).to(device)
        reqs.append(dist.isend(t, dst))
    for src, cols in sorted(plan.recv_from.items()):
        b = torch.empty(len(cols), dtype=torch.float64, device=device)
        bufs[src] = b
        reqs.append(dist.irecv(b, src))
    for r in reqs:
        r.wait()
    parts = [bufs[s].cpu().numpy() for s in sorted(plan.recv_from)]
    return np.concatenate(parts) if parts else np.zeros(0)


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
