"""One preconditioner application of config 1 with the nested-dissection solves (for ncu)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1801_04984_b200 import problem as P, solver as S  # noqa: E402

os.environ.setdefault("PDG_A_SOLVER", "nd")
os.environ.setdefault("PDG_FLOW_SOLVER", "nd")
ops = S.SpatialOperators.assemble(P.config1(int(sys.argv[1]) if len(sys.argv) > 1 else 128))
blk = S.BlockSolver(ops, np.array([[1.7]]), 0.05)
r = np.random.default_rng(0).standard_normal(blk.rows)
for _ in range(2):
    blk.precondition(r)
print("ok")
