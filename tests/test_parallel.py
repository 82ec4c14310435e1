"""Multi-rank host logic of the spatial partitioning,
world_size 2 over gloo on the CPU: the distributed order-fixed SpMV equals the
single-rank SparseMatrix::apply bit for bit; the batched Gram-Schmidt dots
equal the serial ones to roundoff."""
import os
import socket

import numpy as np
import pytest

from paper_1801_04984_b200 import parallel as par
from paper_1801_04984_b200 import problem as P


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_strip_partition_and_owner():
    strips = par.strip_partition(10, 3)
    assert strips == [(0, 4), (4, 7), (7, 10)]
    owner = par.row_owner(3, 10, 2, strips)
    n_u, n_q, n_p = P.ProblemSpec(nx=3, ny=10).sizes
    nt = n_u + n_q + n_p
    assert len(owner) == 2 * nt
    assert np.array_equal(owner[:nt], owner[nt:])
    # every rank owns 8 u dofs per owned cell and one p per owned cell
    for k, (r0, r1) in enumerate(strips):
        assert np.sum(owner[:n_u] == k) == 8 * 3 * (r1 - r0)
        assert np.sum(owner[n_u + n_q:nt] == k) == 3 * (r1 - r0)
    with pytest.raises(ValueError):
        par.strip_partition(2, 3)


def _worker(rank, world, port, n, r, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import refcpu
        spec = P.config1(n)
        rp = refcpu.RefProblem(spec.to_dict())
        T = refcpu.time_constants(r)["T"]
        off, idx, val = rp.spacetime_csr(T, 0.05)
        owner = par.row_owner(n, n, r + 1, par.strip_partition(n, world))
        plans = par.halo_plans(off, idx, val, owner, world)
        plan = plans[rank]
        x = P.uniform_vector(P.X_SEED, len(off) - 1)
        y_loc = par.distributed_spmv(plan, x[plan.rows], dist)
        y_ref = refcpu.csr_apply(off, idx, val, x)
        ok_spmv = np.array_equal(y_loc, y_ref[plan.rows])
        # halo is one cell row (u, p of the neighbour row) + the faces of that row
        halo = plan.halo_size
        rng = np.random.default_rng(5)
        V = rng.standard_normal((len(x), 4))
        w = rng.standard_normal(len(x))
        h = par.distributed_dots(V[plan.rows], w[plan.rows], dist)
        ok_dots = np.allclose(h, V.T @ w, rtol=1e-13, atol=1e-12)
        q.put((rank, ok_spmv, ok_dots, halo, len(plan.rows)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,r,world", [(6, 1, 2), (16, 0, 2), (12, 1, 3)])
def test_distributed_spmv_bit_identical_gloo(oracle, n, r, world):
    """world 3: the middle rank receives halo from both sides (interleaved in the
    global face numbering, mesh.hpp:60)."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, world, port, n, r, q)) for k in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    res = sorted(q.get(timeout=10) for _ in range(world))
    for rank, ok_spmv, ok_dots, halo, nrows in res:
        assert ok_spmv, f"rank {rank}: distributed SpMV differs"
        assert ok_dots, f"rank {rank}: distributed dots differ"
        # one-cell-row halo: 8 u + 1 p per cell of the neighbour row, plus its faces, per component
        assert 0 < halo <= 2 * (r + 1) * (8 * n + n + 2 * n + 1) * 2
    assert sum(x[4] for x in res) > 0


def _blocks_of(A, sizes):
    """Dense diagonal blocks and sub-diagonal couplings of a block-tridiagonal matrix."""
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(int)
    D = [A[off[j]:off[j + 1], off[j]:off[j + 1]].copy() for j in range(len(sizes))]
    C = [A[off[j + 1]:off[j + 2], off[j]:off[j + 1]].copy() for j in range(len(sizes) - 1)]
    return D, C, off


def _strip_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import refcpu
        # the displacement block A of config 1 at 8 x 8 in cell-row order (blocks of 8 nx)
        spec = P.config1(8)
        rp = refcpu.RefProblem(spec.to_dict())
        ro, ri, rv = rp.csr("A")
        n = len(ro) - 1
        A = np.zeros((n, n))
        for r in range(n):
            A[r, ri[ro[r]:ro[r + 1]]] = rv[ro[r]:ro[r + 1]]
        sizes = [8 * spec.nx] * spec.ny
        D, C, off = _blocks_of(A, sizes)
        parts = par.block_partition(len(sizes), world)
        solver = par.StripBlockTri(D, C, parts, rank, dist)
        b = P.uniform_vector(P.X_SEED, n)
        j0, j1 = parts[rank]
        b_sep = b[off[j0]:off[j0 + 1]] if rank > 0 else None
        b_int = np.concatenate([b[off[j]:off[j + 1]] for j in solver.interior])
        x_int, x_sep = solver.solve(b_int, b_sep, dist)
        x_ref = np.linalg.solve(A, b)
        ref_int = np.concatenate([x_ref[off[j]:off[j + 1]] for j in solver.interior])
        err = np.linalg.norm(x_int - ref_int) / np.linalg.norm(ref_int)
        if x_sep is not None:
            err = max(err, np.linalg.norm(x_sep - x_ref[off[j0]:off[j0 + 1]]) / np.linalg.norm(x_ref[off[j0]:off[j0 + 1]]))
        q.put((rank, float(err)))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_substructured_exact_solve_gloo(world):
    """The exact inner solve across strips (parallel.StripBlockTri: strip
    interiors, spikes, one all-gather of the separator right-hand sides per
    solve) equals the single-rank solve of the displacement block to 1e-12."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_strip_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, err in res:
        assert not isinstance(err, str), err
        assert err <= 1e-12, (rank, err)


def _gmres_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import refcpu
        spec = P.config0()
        rp = refcpu.RefProblem(spec.to_dict())
        tau = 0.1
        misc = rp.misc()
        csr = {k: rp.csr(k) for k in ("A", "M_q", "B", "E")}
        stab = misc["biot_b"] ** 2 / misc["k_dr"]
        off, idx, val = rp.spacetime_csr(np.array([[1.0]]), tau)
        strips = par.strip_partition(spec.ny, world)
        owner = par.row_owner(spec.nx, spec.ny, 1, strips)
        plan = par.halo_plans(off, idx, val, owner, world)[rank]
        pre = par.DistFixedStressPre(spec.nx, spec.ny, csr, misc, 1.0, tau, stab, rank, world, dist)
        R = rp.slab_rhs(0, 0.0, tau, np.zeros(rp.n_u), np.zeros(rp.n_p))
        x, rep = par.dist_gmres(plan, pre, R[plan.rows], dist, world, tol=1e-10, restart=50)
        x_ref, rep_ref = rp.block_solve(0, tau, R, tol=1e-10, restart=50, backend=0)
        err = float(np.linalg.norm(x - x_ref[plan.rows]) / np.linalg.norm(x_ref[plan.rows]))
        q.put((rank, rep["iterations"], rep_ref["iterations"], err))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc(), None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_gmres_matches_oracle_gloo(world):
    """The whole N > 1 path on the CPU: strip-partitioned operator (halo
    exchange), fixed-stress preconditioner with the substructured exact inner
    solves, GMRES with ordered all-reduces -- same iteration count as the
    single-rank oracle (gmres.hpp:40-139) and the slab solution within 1e-9."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gmres_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, its, its_ref, err in res:
        assert not isinstance(its, str), its
        assert abs(its - its_ref) <= 1 and err <= 1e-9, (rank, its, its_ref, err)


@pytest.mark.parametrize("world", [2, 3])
def test_strip_exchange_sets_cover_the_halo(oracle, world):
    """The device path's neighbour exchange (parallel.strip_exchange_sets) holds
    every column the owned rows of the space-time operator read that the rank
    does not own, and each rank sends only entries it owns."""
    n, m = 8, 2
    spec = P.config1(n)
    rp = oracle.RefProblem(spec.to_dict())
    off, idx, _ = rp.spacetime_csr(oracle.time_constants(1)["T"], 0.05)
    strips = par.strip_partition(n, world)
    owner = par.row_owner(n, n, m, strips)
    for k in range(world):
        rows = np.flatnonzero(owner == k)
        cols = np.unique(np.concatenate([idx[off[r]:off[r + 1]] for r in rows]))
        need = cols[owner[cols] != k]
        send, recv = par.strip_exchange_sets(n, n, m, strips, k)
        have = np.concatenate(list(recv.values())) if recv else np.zeros(0, np.int64)
        assert np.all(np.isin(need, have)), k
        for dst, s in send.items():
            assert np.all(owner[s] == k)
            assert np.array_equal(s, par.strip_exchange_sets(n, n, m, strips, dst)[1][k])


def _halo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, m = 8, 2
        strips = par.strip_partition(n, world)
        owner = par.row_owner(n, n, m, strips)
        truth = P.uniform_vector(P.X_SEED, len(owner))
        x = torch.from_numpy(np.where(owner == rank, truth, np.nan))
        halo = par.StripHalo(n, n, m, rank, world, dist, device="cpu")
        halo.exchange(x)
        _, recv = par.strip_exchange_sets(n, n, m, strips, rank)
        got = np.concatenate([x.numpy()[v] for v in recv.values()])
        ref = np.concatenate([truth[v] for v in recv.values()])
        q.put((rank, bool(np.array_equal(got, ref)), bool(np.array_equal(x.numpy()[owner == rank], truth[owner == rank]))))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc(), None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_strip_halo_exchange_gloo(world):
    """StripHalo (the exchange of the device distributed SpMV) delivers exactly
    the neighbours' boundary values and leaves the owned entries alone."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_halo, ok_own in res:
        assert ok_halo is True and ok_own is True, (rank, ok_halo)
