"""Setup stage timers (pdg_setup_read) of the config-1 slab solver, built several times in one process."""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1801_04984_b200 import problem as P
from paper_1801_04984_b200 import solver as S

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
names = ("assemble", "a_analysis", "a_factor", "a_schedule", "f_analysis", "f_factor", "f_schedule", "operator", "total")
for rep in range(3):
    S.lib().pdg_setup_reset()
    t = time.perf_counter()
    ops = S.SpatialOperators.assemble(P.config1(n))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    slab = S.SlabSolver(ops, 1, 0.05, S.SolveOptions(gmres=S.GmresOptions(restart=50), candidate="flexible"))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    buf = (C.c_double * 9)()
    S.lib().pdg_setup_read(buf, 9)
    print(f"rep {rep}: assemble wall {t1 - t:.3f} s, slab solver wall {t2 - t1:.3f} s | " +
          " ".join(f"{k} {v:.3f}" for k, v in zip(names, buf)), flush=True)
    del slab, ops
