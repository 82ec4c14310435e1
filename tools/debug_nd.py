"""Per-phase timeline of the nested-dissection solves (PDG_ND_DEBUG) on config 1."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1801_04984_b200 import problem as P, solver as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
os.environ.setdefault("PDG_A_SOLVER", "nd")
os.environ.setdefault("PDG_FLOW_SOLVER", "nd")
ops = S.SpatialOperators.assemble(P.config1(n))
# PDG_DEBUG_M=2: the dG(1) block (2 right-hand sides per inner solve, as the bench)
theta = S.time_constants(1)["T"] if os.environ.get("PDG_DEBUG_M") == "2" else np.array([[1.7]])
blk = S.BlockSolver(ops, theta, 0.05)
r = np.random.default_rng(0).standard_normal(blk.rows)
z0 = blk.precondition(r)
os.environ["PDG_ND_DEBUG"] = "1"
z1 = blk.precondition(r)
del os.environ["PDG_ND_DEBUG"]
print("repeat identical:", bool(np.array_equal(z0, z1)))
