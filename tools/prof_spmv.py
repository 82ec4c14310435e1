"""Profiling driver: config-3 space-time SpMV at n x n (for ncu captures)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1801_04984_b200 import problem as P, solver as S  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    ops = S.SpatialOperators.assemble(P.config3(n))
    op = S.SpaceTimeOperator(ops, S.time_constants(1)["T"], 0.05)
    x = torch.from_numpy(P.uniform_vector(P.X_SEED, op.rows)).cuda()
    y = torch.empty_like(x)
    t = op.apply_device(x.data_ptr(), y.data_ptr(), reps, times=True)
    print("rows", op.rows, "nnz", op.nnz, "ms", [round(v, 4) for v in t])


if __name__ == "__main__":
    main()
