"""Run output in the reference's formats, for diffing GPU runs against the
reference's (or the oracle's) on the schema:

- the per-block iteration log ``iterations.csv`` (write_iteration_log,
  csv.hpp:56-71): ``slab_index,t_n,block_index,block_type,gmres_iterations,
  fs_sweeps,final_residual`` with t_n = t_end(n) as ``%.12g`` and the final
  relative residual as ``%.6e``;
- the driver's per-slab stdout line (driver.hpp:38-47):
  ``slab %4d  t_n=%-12.6g method=%s iters=%d res=%.3e``.

For dG(r), r <= 1, the spectral method has exactly one transformed block per
slab (block 0, size r + 1: "1x1" or "2x2", slab.hpp:194-207); its fs_sweeps is
the truncation sweep count (slab.hpp:233).
"""
from __future__ import annotations

HEADER = "slab_index,t_n,block_index,block_type,gmres_iterations,fs_sweeps,final_residual"


def _block_rows(r: int, report, sweeps: int):
    """BlockReports of one slab (r <= 1: one block)."""
    return [dict(block_index=0, block_size=r + 1, gmres_iterations=report.iterations, fs_sweeps=sweeps,
                 final_residual=report.final_relative_residual)]


def iteration_log_lines(reports, t_points, r: int, sweeps: int = 1):
    """Lines of iterations.csv (csv.hpp:56-71) for a march's per-slab reports."""
    lines = [HEADER]
    for n, rep in enumerate(reports):
        for b in _block_rows(r, rep, sweeps):
            lines.append("%d,%s,%d,%dx%d,%d,%d,%s" % (n, "%.12g" % t_points[n + 1], b["block_index"], b["block_size"],
                                                      b["block_size"], b["gmres_iterations"], b["fs_sweeps"],
                                                      "%.6e" % b["final_residual"]))
    return lines


def write_iteration_log(path: str, reports, t_points, r: int, sweeps: int = 1):
    """write_iteration_log (csv.hpp:56-71)."""
    with open(path, "w") as f:
        for line in iteration_log_lines(reports, t_points, r, sweeps):
            f.write(line + "\n")


def slab_line(n: int, t_n: float, report, r: int, sweeps: int = 1, method: str = "monolithic-spectral"):
    """The driver's per-slab line (driver.hpp:38-47): iters = max over blocks of
    max(gmres_iterations, fs_sweeps), res = max final relative residual."""
    rows = _block_rows(r, report, sweeps)
    iters = max(max(b["gmres_iterations"], b["fs_sweeps"]) for b in rows)
    res = max(b["final_residual"] for b in rows)
    return "slab %4d  t_n=%-12.6g method=%s iters=%d res=%.3e" % (n, t_n, method, iters, res)
