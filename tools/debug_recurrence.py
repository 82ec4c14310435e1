"""Per-step timing breakdown of the block-tridiagonal recurrence (config 1)."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1801_04984_b200 import _lib, problem as P, solver as S  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    ops = S.SpatialOperators.assemble(P.config1(n))
    blk = S.BlockSolver(ops, S.time_constants(1)["T"], 0.05)
    blk.precondition(np.ones(blk.rows))
    for which in (0, 1):
        cap = 4_000_000
        buf = (C.c_ulonglong * cap)()
        g, ns = C.c_int(), C.c_int()
        _lib.check(_lib.lib().pdg_debug_recurrence_timing(blk._h, which, buf, cap, C.byref(g), C.byref(ns)))
        g, ns = g.value, ns.value
        a = np.frombuffer(buf, dtype=np.uint64, count=g * ns * 4).reshape(g, ns, 4).astype(np.int64)
        t0 = a[:, :, 0].min()
        has_wait = bool(a[:, :, 3].any())
        a = a - t0
        total = a[:, -1, 2].max()
        gather = np.median(a[:, 1:, 1] - a[:, 1:, 0], axis=0)
        comp = np.median(a[:, 1:, 2] - a[:, 1:, 1], axis=0)
        # step period: consecutive step starts of CTA 0
        period = np.diff(a[0, :, 0])
        # latency: consumer gather end - last producer store of previous step (all CTAs approx)
        lat = [np.median(a[:, s, 1]) - np.max(a[:, s - 1, 2]) for s in range(2, ns)]
        print(f"{'A' if which == 0 else 'flow'}: ctas={g} steps={ns} total={total/1e3:.1f} us "
              f"period median={np.median(period)/1e3:.2f} us; gather median={np.median(gather)/1e3:.2f} us; "
              f"compute+store median={np.median(comp)/1e3:.2f} us; latency(prev store->gather end) median="
              f"{np.median(lat)/1e3:.2f} us")
        if has_wait:  # phase 3 = ring data ready (sweep kernel)
            wait = np.median(a[:, 1:, 3] - a[:, 1:, 1], axis=0)
            rest = np.median(a[:, 1:, 2] - a[:, 1:, 3], axis=0)
            print(f"   data wait after gather median={np.median(wait)/1e3:.2f} us; "
                  f"GEMV+reduce+publish median={np.median(rest)/1e3:.2f} us")
        print("   first steps period (us):", np.round(period[:8] / 1e3, 2))
        print("   step start spread across CTAs (us) at step 10:", (a[:, 10, 0].max() - a[:, 10, 0].min()) / 1e3)


if __name__ == "__main__":
    main()
