"""Regenerates the committed golden fixtures (run in the build container).

reference_iterations.json  -- the reference's own recorded run
                              (/root/reference/proj/out/iterations.csv),
                              parsed into numbers plus its raw lines (the
                              iteration-log schema, csv.hpp:56-71); the oracle
                              must reproduce it.
config1_k_perm.npy         -- per-cell permeability of config 1 (seed 1801),
                              from the oracle's generator.
config0_oracle.npz         -- oracle march of config 0 (dense inner solves):
                              iterations, final residuals, all slab states.
terzaghi_oracle.npz        -- oracle march of the recorded Terzaghi run.
config2_small_oracle.npz   -- 3D extension (no reference counterpart; oracle/refcpu/fem3d.hpp):
                              oracle march of config 2 at 4^3 (3 slabs) with the sums of the
                              operator values and of the right-hand side, pinning the 3D
                              restatement against accidental edits.
highorder_oracle.npz       -- oracle marches of config 0 at 6^2 with dG(2) and dG(3)
                              (multi-block Schur back-substitution): iterations and states.
"""
import csv
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import refcpu  # noqa: E402
from paper_1801_04984_b200 import problem as P  # noqa: E402


def main():
    ref_csv = "/root/reference/proj/out/iterations.csv"
    if os.path.exists(ref_csv):
        rows = list(csv.DictReader(open(ref_csv)))
        out = dict(source="proj/out/iterations.csv", columns=list(rows[0].keys()),
                   slab_index=[int(r["slab_index"]) for r in rows], t_n=[float(r["t_n"]) for r in rows],
                   gmres_iterations=[int(r["gmres_iterations"]) for r in rows],
                   fs_sweeps=[int(r["fs_sweeps"]) for r in rows],
                   final_residual=[float(r["final_residual"]) for r in rows],
                   lines=open(ref_csv).read().splitlines())
        json.dump(out, open(os.path.join(HERE, "reference_iterations.json"), "w"), indent=1)
    k = refcpu.lognormal(P.K_SEED, 128 * 128, 1.0)
    np.save(os.path.join(HERE, "config1_k_perm.npy"), k)
    for name, spec in (("config0", P.config0()), ("terzaghi", P.terzaghi_recorded())):
        run = P.RUNS["config0" if name == "config0" else "terzaghi_recorded"]
        rp = refcpu.RefProblem(spec.to_dict())
        res = rp.march(run["r"], run["T"], run["n_slabs"], tol=run["tol"], restart=run["restart"], backend=0,
                       keep_states=True)
        np.savez_compressed(os.path.join(HERE, f"{name}_oracle.npz"), iterations=res["iterations"],
                            final_res=res["final_res"], states=res["states"])


    spec = P.config2(4)
    rp = refcpu.RefProblem(spec.to_dict())
    res = rp.march(0, 0.3, 3, tol=1e-10, restart=50, backend=0, keep_states=True)
    sums = {nm: np.array([rp.csr(nm)[2].sum(), np.abs(rp.csr(nm)[2]).sum()]) for nm in ("A", "M_q", "B", "E")}
    ru, rq, rpp = rp.assemble_rhs(0.0)
    np.savez_compressed(os.path.join(HERE, "config2_small_oracle.npz"), iterations=res["iterations"],
                        final_res=res["final_res"], states=res["states"], k_perm=spec.k_perm_cells,
                        rhs_sums=np.array([ru.sum(), rq.sum(), rpp.sum()]), **{f"sum_{k}": v for k, v in sums.items()})
    spec = P.config0()
    spec.nx = spec.ny = 6
    rp = refcpu.RefProblem(spec.to_dict())
    out = {}
    for r in (2, 3):
        res = rp.march(r, 0.3, 2, tol=1e-10, restart=50, backend=0, keep_states=True)
        out[f"iterations_r{r}"] = res["iterations"]
        out[f"states_r{r}"] = res["states"]
    np.savez_compressed(os.path.join(HERE, "highorder_oracle.npz"), **out)


if __name__ == "__main__":
    main()
