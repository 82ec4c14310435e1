"""The device path of the multi-GPU block solve (distributed.py) run as two
ranks sharing one GPU over gloo: no kernel waits on another rank's kernel
(every exchange is a host-level collective), so this exercises the real code
(strip SpMV + halo, substructured exact inner solves with the library's
sweeps, rank-ordered Krylov sums) without a second GPU. Bar: the single-GPU
solve's iteration count (+-1) and its solution within 1e-9."""
import os
import socket

import numpy as np
import pytest

from paper_1801_04984_b200 import problem as P

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, n, candidate, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1801_04984_b200 import distributed as D, solver as S

        torch.cuda.set_device(0)
        comm = D.Comm(dist, rank, world, stage_on_host=True)
        T = S.time_constants(1)["T"]
        blk = D.DeviceDistributedBlock(P.config1(n), T, 0.05, rank, comm, device=0, candidate=candidate)
        rhs = P.uniform_vector(P.X_SEED, 2 * blk.nt)
        owned = blk.owned.cpu().numpy()
        x, rep = blk.solve(torch.as_tensor(rhs[owned], device="cuda"))
        q.put((rank, owned, x.cpu().numpy(), rep["iterations"], rep["converged"]))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc(), None, None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("candidate", ["reference", "flexible"])
def test_distributed_block_solve_two_ranks_one_gpu(candidate):
    import multiprocessing as mp

    from paper_1801_04984_b200 import solver as S

    n, world = 16, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, n, candidate, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert not isinstance(r[1], str), r[1]
    ops = S.SpatialOperators.assemble(P.config1(n))
    blk = S.BlockSolver(ops, S.time_constants(1)["T"], 0.05,
                        opt=S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50), candidate=candidate))
    rhs = P.uniform_vector(P.X_SEED, blk.rows)
    x_ref, rep_ref = blk.solve(rhs)
    x = np.full(blk.rows, np.nan)
    for rank, owned, xo, its, conv in res:
        assert conv and abs(its - rep_ref.iterations) <= 1, (rank, its, rep_ref.iterations)
        x[owned] = xo
    assert not np.isnan(x).any()
    assert np.linalg.norm(x - x_ref) <= 1e-9 * np.linalg.norm(x_ref)
