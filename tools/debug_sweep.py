"""Per-step timeline of the displacement solve's sweep kernel (config 1): for each
step and chain, min/max over CTAs of step start, then the max over CTAs of: all
warps' inputs polled, all warps' Sinv rows in shared memory, all warps' partial
products done (us from the
first stamp)."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1801_04984_b200 import _lib, problem as P, solver as S  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    ops = S.SpatialOperators.assemble(P.config1(n))
    blk = S.BlockSolver(ops, S.time_constants(1)["T"], 0.05)
    blk.precondition(np.ones(blk.rows))
    cap = 4_000_000
    buf = (C.c_ulonglong * cap)()
    g, ns = C.c_int(), C.c_int()
    _lib.check(_lib.lib().pdg_debug_recurrence_timing(blk._h, 0, buf, cap, C.byref(g), C.byref(ns)))
    g, ns = g.value, ns.value
    a = np.frombuffer(buf, dtype=np.uint64, count=g * ns * 4).reshape(g, ns, 4).astype(np.int64)
    a = (a - a[:, :, 0].min()) / 1e3
    h = g // 2
    print(f"ctas={g} steps={ns} total={a[:, -1, 3].max():.1f} us")
    print("step | top: start min/max  polled  rows-ready  partials | bottom: same")
    for s in list(range(min(steps, ns))) + list(range(max(steps, ns - 4), ns)):
        row = []
        for c in (slice(0, h), slice(h, g)):
            x = a[c, s]
            row.append(f"{x[:, 0].min():7.2f}/{x[:, 0].max():7.2f} {x[:, 1].max():7.2f} {x[:, 2].max():7.2f} "
                       f"{x[:, 3].max():7.2f}")
        print(f"{s:4d} | " + " | ".join(row))


if __name__ == "__main__":
    main()
