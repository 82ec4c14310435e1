"""Timeline of the flow solve's dense sweep (config 1): per chain, the times at
which its steps end (us from the first stamp), to see the phases (strip sweeps,
separator, correction) of the substructured solve."""
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
    cap = 4_000_000
    buf = (C.c_ulonglong * cap)()
    g, ns = C.c_int(), C.c_int()
    _lib.check(_lib.lib().pdg_debug_recurrence_timing(blk._h, 1, buf, cap, C.byref(g), C.byref(ns)))
    g, ns = g.value, ns.value
    a = np.frombuffer(buf, dtype=np.uint64, count=g * ns * 4).reshape(g, ns, 4).astype(np.int64)
    t0 = a[:, :, 0][a[:, :, 0] > 0].min()
    end = np.where(a[:, :, 2] > 0, (a[:, :, 2] - t0) / 1e3, np.nan)
    start = np.where(a[:, :, 0] > 0, (a[:, :, 0] - t0) / 1e3, np.nan)
    per = int(os.environ.get("CTAS_PER_CHAIN", "33"))
    nch = g // per
    print(f"ctas={g} steps={ns} chains={nch} total={np.nanmax(end):.1f} us")
    for c in range(nch):
        e = np.nanmax(end[c * per:(c + 1) * per], axis=0)
        st = np.nanmin(start[c * per:(c + 1) * per], axis=0)
        marks = [f"{s}:{st[s]:.0f}-{e[s]:.0f}" for s in range(0, ns, max(1, ns // 12))]
        print(f"chain {c}: " + " ".join(marks) + f" | last {e[-1]:.1f}")


if __name__ == "__main__":
    main()
