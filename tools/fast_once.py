"""One slab of config 2 at n^3 in fast or parity mode (for ncu captures of k_nd_stream).
usage: python tools/fast_once.py n mode"""
import sys

sys.path.insert(0, ".")
from paper_1801_04984_b200 import problem as P
from paper_1801_04984_b200 import solver as S

n, mode = int(sys.argv[1]), sys.argv[2]
ops = S.SpatialOperators.assemble(P.config2(n))
opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50), candidate="flexible", mode=mode)
reps, _ = S.march(ops, 0, 0.1, 1, opt)
print(mode, [r.iterations for r in reps], [round(r.device_ms, 2) for r in reps])
