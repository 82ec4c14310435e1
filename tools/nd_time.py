"""Timing of the config-1 preconditioner's inner solves (ND displacement and flow
solves, 2 right-hand sides): K preconditioner applications with the per-phase
event profiler; prints the mean and min device time per call of each solve."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_1801_04984_b200 import _lib, problem as P, solver as S  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 30
ops = S.SpatialOperators.assemble(P.config1(128))
blk = S.BlockSolver(ops, S.time_constants(1)["T"], 0.05)
r = P.uniform_vector(3, blk.rows)
z0 = blk.precondition(r)
for _ in range(3):
    blk.precondition(r)
per = {"a_solve": [], "flow_solve": []}
for _ in range(K):
    S.profile(enable=True, reset=True)
    z = blk.precondition(r)
    ph = S.profile(enable=False)
    for k in per:
        per[k].append(ph[k][0] / max(ph[k][1], 1))
print(" ".join(f"{k}: mean {1e3 * np.mean(v):7.1f} us  min {1e3 * np.min(v):7.1f} us" for k, v in per.items()),
      "| repeat identical:", bool(np.array_equal(z0, z)))
