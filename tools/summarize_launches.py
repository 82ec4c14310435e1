"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel
totals, solve-phase kernels only (setup factorisation / assembly launches excluded)."""
import collections
import csv
import re
import sys

SETUP = re.compile(r"cusolver|cublas|potrf|trsm|syrk|gemm|getrf|Kernel<|k_nd_pack|k_nd_extend_add|k_nd_identity|"
                   r"k_nd_scatter|k_nd_tile_pack|trtri|copy_info|k_nd_factor_batch|k_nd_top_scatter|k_nd_top_sym|k_uk_|k_pk_|k_qk_|k_slice_max|k_assemble|k_row_lengths|k_cell|k_face|k_csr|DeviceScan|DeviceRadix|DeviceReduce|"
                   r"k_u_count|k_u_fill|k_s_len|k_s_slice_width|k_s_fill|k_flux|k_qc|k_mp|k_dinv|k_flow_schur|"
                   r"elementwise|at::|xxtrf|trsv|k_sort_rows|k_count_cols|k_blk|k_fill|k_step|k_sweep_setup|k_pack|k_transpose|k_copy_tri|k_scatter",
                   re.I)


def main(path, header):
    rows = [l for l in open(path) if l.startswith('"')]
    r = list(csv.reader(rows))
    h = r[0]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    tot, cnt = collections.Counter(), collections.Counter()
    n_all = 0
    for row in r[1:]:
        n_all += 1
        name = re.sub(r"\(.*", "", row[ik]).replace("pdg::<unnamed>::", "").replace("pdg::", "")
        if SETUP.search(row[ik]):
            continue
        tot[name] += float(row[iv]) / 1e3
        cnt[name] += 1
    s = sum(tot.values())
    print(header)
    print(f"# {n_all} launches in the capture; cold-cache serialised per-launch times (shares, not absolutes, are meaningful)")
    print(f"{'kernel':40s} {'launches':>9s} {'total us':>10s} {'avg us':>9s} {'share':>6s}")
    for k, v in tot.most_common():
        print(f"{k[:40]:40s} {cnt[k]:9d} {v:10.1f} {v / cnt[k]:9.2f} {100 * v / s:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
