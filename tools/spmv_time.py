"""Order-fixed space-time SpMV timing: config 1 (128^2, GMRES operator) and the
config-3 sizes given; median of 50 applications (CUDA events per launch)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1801_04984_b200 import problem as P, solver as S  # noqa: E402

T = S.time_constants(1)["T"]
peak = 6549.4
for n in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "128,256,1024").split(",")]:
    op = S.SpaceTimeOperator(S.SpatialOperators.assemble(P.config1(n) if n == 128 else P.config3(n)), T, 0.05)
    x = torch.from_numpy(P.uniform_vector(P.X_SEED, op.rows)).cuda()
    y = torch.empty_like(x)
    op.apply_device(x.data_ptr(), y.data_ptr(), 3)
    t = sorted(op.apply_device(x.data_ptr(), y.data_ptr(), 50, times=True))
    med = t[len(t) // 2] * 1e-3
    ba = 8.0 * (op.nnz + 2 * op.rows)
    print(f"n={n:5d} rows={op.rows:9d} median {med * 1e6:8.1f} us  {ba / med / 1e9:7.0f} GB/s  frac {ba / med / 1e9 / peak:.3f}"
          f"  checksum {float(y.sum()):.12e}")
    del op, x, y
    torch.cuda.empty_cache()
