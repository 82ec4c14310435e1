"""Config 2 (3D) size probe: setup time, device memory and slab time at n^3.
usage: python tools/config2_probe.py n [n_slabs]"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1801_04984_b200 import problem as P
from paper_1801_04984_b200 import solver as S

n = int(sys.argv[1])
n_slabs = int(sys.argv[2]) if len(sys.argv) > 2 else 2
spec = P.config2(n)
t = time.time()
ops = S.SpatialOperators.assemble(spec)
torch.cuda.synchronize()
print(f"n={n} n_u={ops.n_u} n_q={ops.n_q} n_p={ops.n_p} nnzA={ops.nnz['A']} assemble {time.time() - t:.2f}s", flush=True)
opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50), candidate="flexible")
S.lib().pdg_setup_reset()
t = time.time()
slab = S.SlabSolver(ops, 0, 1.0 / 10, opt)
torch.cuda.synchronize()
free, total = torch.cuda.mem_get_info()
print(f"slab solver setup {time.time() - t:.2f}s, device memory used {(total - free) / 2**30:.2f} GiB", flush=True)
import ctypes as C
buf = (C.c_double * 9)()
S.lib().pdg_setup_read(buf, 9)
print("setup stages", [round(v, 3) for v in buf], flush=True)
del slab
reps, _ = S.march(ops, 0, n_slabs / 10.0, n_slabs, opt, mass_check=True)
for r in reps:
    print(f"  iterations {r.iterations} rel res {r.final_relative_residual:.2e} mass {r.mass_rel:.2e} device {r.device_ms:.3f} ms launches {r.kernel_launches}", flush=True)
