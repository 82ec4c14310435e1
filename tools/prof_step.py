"""Profiling driver: a few slabs of config 1 (for ncu launch lists / captures)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1801_04984_b200 import problem as P, solver as S  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    slabs = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    cand = sys.argv[3] if len(sys.argv) > 3 else "reference"
    ops = S.SpatialOperators.assemble(P.config1(n))
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50), candidate=cand)
    phases = os.environ.get("PROF_PHASES") == "1"
    if phases:
        S.march(ops, 1, 0.05, 1, opt)  # warm-up
        S.profile(enable=True, reset=True)
    reps, _ = S.march(ops, 1, 0.05 * slabs, slabs, opt)
    torch.cuda.synchronize()
    if phases:
        for nm, (ms, calls, by) in S.profile(enable=False).items():
            print(f"  {nm:16s} {ms / slabs:8.3f} ms/slab {calls / slabs:6.1f} calls/slab "
                  f"{(by / (ms * 1e-3) / 1e9 if ms else 0):8.1f} GB/s")
    print("iterations", [r.iterations for r in reps], "device_ms", [round(r.device_ms, 3) for r in reps])


if __name__ == "__main__":
    main()
