"""Diagnostic: GMRES(2) on a 16^2 dG(1) block through every loop variant."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_1801_04984_b200 import problem as P, solver as S  # noqa: E402

ops = S.SpatialOperators.assemble(P.config1(16))
t = S.time_constants(1)
rhs = np.random.default_rng(11).standard_normal(2 * ops.n_total)
for env in ({}, {"PDG_GMRES_DEVICE_LS": "1"}, {"PDG_GMRES_DEVICE_LS": "1", "PDG_GMRES_LOOKAHEAD": "1"},
            {"PDG_KRYLOV_UNFUSED": "1"}):
    for k in ("PDG_GMRES_DEVICE_LS", "PDG_GMRES_LOOKAHEAD", "PDG_KRYLOV_UNFUSED"):
        os.environ.pop(k, None)
    os.environ.update(env)
    for restart in (2, 50):
        blk = S.BlockSolver(ops, t["T"], 0.05, opt=S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=restart),
                                                                  candidate="flexible"))
        try:
            x, rep = blk.solve(rhs)
            h = rep.residual_history / rep.residual_history[0]
            print(env, restart, rep.iterations, rep.converged, np.array2string(h[:12], precision=2), h[-3:])
        except Exception as e:
            print(env, restart, "ERROR", e)
