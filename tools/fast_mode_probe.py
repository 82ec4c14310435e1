"""Fast mode (pdg_gmres_opts.mode 1: fp32-stored streaming factor) against parity mode on config 2 at n^3:
iterations, device time per slab, relative difference of the marched states.
usage: python tools/fast_mode_probe.py n [n_slabs] [r]"""
import gc
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1801_04984_b200 import problem as P
from paper_1801_04984_b200 import solver as S

n = int(sys.argv[1])
n_slabs = int(sys.argv[2]) if len(sys.argv) > 2 else 3
r = int(sys.argv[3]) if len(sys.argv) > 3 else 0
spec = P.config2(n) if r == 0 else P.config4(n)
out = {}
for mode in ("parity", "fast"):
    ops = S.SpatialOperators.assemble(spec)
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50), candidate="flexible", mode=mode)
    reps, state = S.march(ops, r, n_slabs / 10.0, n_slabs, opt, mass_check=True, keep_states=True)
    free, total = torch.cuda.mem_get_info()
    print(f"{mode:7s} n={n} r={r}: iterations {[q.iterations for q in reps]} ms/slab {[round(q.device_ms, 2) for q in reps]} "
          f"rel res {max(q.final_relative_residual for q in reps):.2e} mass {max(q.mass_rel for q in reps):.2e} "
          f"memory {(total - free) / 2**30:.1f} GiB", flush=True)
    out[mode] = state[-1]
    del ops, reps, state
    gc.collect()
    torch.cuda.empty_cache()
d = np.linalg.norm(out["fast"] - out["parity"]) / np.linalg.norm(out["parity"])
print(f"relative l2 difference of the final states (fast vs parity): {d:.3e}")
