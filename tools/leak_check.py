"""Repeated slab steps: device memory must not grow, results stay bit-identical per slab index."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1801_04984_b200 import problem as P
from paper_1801_04984_b200 import solver as S

ops = S.SpatialOperators.assemble(P.config1(64))
opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50), candidate="flexible")
for r in (1, 2):
    slab = S.SlabSolver(ops, r, 0.05, opt)
    nt = ops.n_total
    outs = [torch.empty((r + 1) * nt, dtype=torch.float64, device="cuda") for _ in range(2)]
    torch.cuda.synchronize()
    first = None
    marks = []
    for rep_ in range(4):
        prev = None
        for k in range(100):
            o = outs[k % 2]
            slab.step_device(0.05 * k, prev, o.data_ptr())
            prev = o.data_ptr() + 8 * r * nt
        torch.cuda.synchronize()
        end = outs[99 % 2].clone()
        if first is None:
            first = end
        assert torch.equal(first, end)
        del end
        marks.append(torch.cuda.mem_get_info()[0])
    # the first passes allocate lazily created buffers (library work buffers, torch's cache, the
    # driver's module / local-memory pools); after them nothing may grow
    growth = (marks[1] - marks[-1]) / 2**20
    print(f"r={r}: 400 slab steps, free memory after each 100: {[round(m / 2**20, 1) for m in marks]} MiB, "
          f"growth after the first 200: {growth:.1f} MiB, repeats bit-identical")
    assert growth < 8.0
