"""Preconditioner applications of the config-1 dG(1) block (2 right-hand sides per
inner solve) with the nested-dissection solves, for ncu captures."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1801_04984_b200 import problem as P, solver as S  # noqa: E402

ops = S.SpatialOperators.assemble(P.config1(int(sys.argv[1]) if len(sys.argv) > 1 else 128))
blk = S.BlockSolver(ops, S.time_constants(1)["T"], 0.05)
r = np.random.default_rng(0).standard_normal(blk.rows)
for _ in range(3):
    blk.precondition(r)
print("ok")
