"""Slab solve at larger meshes (config-1 material): setup, one slab, iterations."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1801_04984_b200 import problem as P, solver as S  # noqa: E402

for n in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "192,256").split(",")]:
    try:
        t0 = time.time()
        ops = S.SpatialOperators.assemble(P.config3(n))
        opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50), candidate="flexible")
        reps, _ = S.march(ops, 1, 0.1, 2, opt, mass_check=True)
        print(f"n={n} ok: {time.time() - t0:.1f} s incl. setup, iterations {[r.iterations for r in reps]}, "
              f"device ms {[round(r.device_ms, 2) for r in reps]}, mass {[f'{r.mass_rel:.1e}' for r in reps]}", flush=True)
    except Exception as e:
        print(f"n={n} FAILED: {e}", flush=True)
    torch.cuda.empty_cache()
