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


if __name__ == "__main__":
    main()
