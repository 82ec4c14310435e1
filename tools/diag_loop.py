"""Diagnostic: the GMRES loop variants on a 32^2 dG(1) block (histories)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1801_04984_b200 import problem as P, solver as S  # noqa: E402

ops = S.SpatialOperators.assemble(P.config1(32))
t = S.time_constants(1)
rhs = np.random.default_rng(11).standard_normal(2 * ops.n_total)
for tol in (1e-10, 1e-13):
    for env in ({}, {"PDG_SPMV_DOTS": "0"}, {"PDG_GMRES_HOST_LOOP": "1"}, {"PDG_GMRES_HOST_LOOP": "1", "PDG_SPMV_DOTS": "0"}):
        for k in ("PDG_SPMV_DOTS", "PDG_GMRES_HOST_LOOP"):
            os.environ.pop(k, None)
        os.environ.update(env)
        blk = S.BlockSolver(ops, t["T"], 0.05, opt=S.SolveOptions(gmres=S.GmresOptions(tol=tol, restart=50, max_iter=30),
                                                                  candidate="flexible"))
        try:
            x, rep = blk.solve(rhs)
            h = rep.residual_history / rep.residual_history[0]
            print(tol, env, rep.iterations, np.array2string(h, precision=3, max_line_width=250))
        except Exception as e:
            print(tol, env, "ERR", e)
