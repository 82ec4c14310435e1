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


@pytest.mark.parametrize("n,r", [(6, 1), (16, 0)])
def test_distributed_spmv_bit_identical_gloo(oracle, n, r):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, 2, port, n, r, q)) for k in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    res = sorted(q.get(timeout=10) for _ in range(2))
    for rank, ok_spmv, ok_dots, halo, nrows in res:
        assert ok_spmv, f"rank {rank}: distributed SpMV differs"
        assert ok_dots, f"rank {rank}: distributed dots differ"
        # one-cell-row halo: 8 u + 1 p per cell of the neighbour row, plus its faces, per component
        assert 0 < halo <= (r + 1) * (8 * n + n + 2 * n + 1) * 2
    assert sum(x[4] for x in res) > 0
