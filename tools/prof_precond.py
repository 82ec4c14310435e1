"""Profiling driver: config-1 block preconditioner applications (ncu traffic per solve)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1801_04984_b200 import problem as P, solver as S  # noqa: E402

ops = S.SpatialOperators.assemble(P.config1(128))
blk = S.BlockSolver(ops, S.time_constants(1)["T"], 0.05)
r = P.uniform_vector(3, blk.rows)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    z = blk.precondition(r)
print("ok", float(np.linalg.norm(z)))
