// Canonical assembled space-time operator of one transformed slab block and
// its order-fixed SpMV (DESIGN.md section "Space-time operator").
#pragma once

#include "common.cuh"

namespace pdg {

struct SpatialOps;  // defined in ops.cuh

// Cell-blocked sliced layout:
//  U class : one group per (component i, cell c) = the 8 displacement rows of
//            the cell, which share one column list (A columns of the cell and
//            its face neighbours, then their E columns). Values are stored
//            [group][entry k][row l] (8 doubles per k), so the 8 lanes that
//            own a group read 64 contiguous bytes per step and share one
//            column index.
//  S class : q- and p-rows, SELL-32: slice of 32 consecutive rows,
//            [slice][entry k][lane], per-entry column index.
// Every row is summed sequentially in ascending global column order with
// __dmul_rn/__dadd_rn: bit-identical to SparseMatrix::apply
// (sparse.hpp:30-40) on the canonical CSR.
struct SpaceTimeOp {
    int m = 1;           // time components in the block
    int nt = 0;          // n_u + n_q + n_p
    int n_u = 0, n_q = 0, n_p = 0, n_cells = 0;
    int n_ug = 0;        // U groups per component (n_u / 8: one per 2D cell, three per 3D cell)
    long long rows = 0, nnz = 0;
    // U class
    long long u_groups = 0, u_entries = 0;  // entries counted per group (x8 values)
    DBuf<long long> u_off;                  // u_groups + 1 (entry offset per group)
    DBuf<int> u_col;                        // u_entries
    DBuf<double> u_val;                     // 8 * u_entries
    // S class
    long long s_rows = 0, s_slices = 0, s_slots = 0;
    DBuf<long long> s_off;  // s_slices + 1 (slot offset per slice, slots of 32)
    DBuf<int> s_len;        // s_rows
    DBuf<int> s_col;        // 32 * s_slots
    DBuf<double> s_val;     // 32 * s_slots

    // Kronecker-paired layout (the default when the structure allows it; `kp` true):
    // the M = m rows that share one spatial row pattern are kept together, one
    // thread per pattern, so a column list and the x reuse serve all M rows and the
    // M values of an entry are one 16-byte load (m = 2). Column lists keep one index
    // per run of 8 consecutive displacement columns (cell blocks of A and of E^T).
    //  UK : one pattern per cell (its 8 displacement rows x M components); per cell
    //       a header [A run starts..., E columns...], values [cell][entry k][row l][i].
    //  PK : one pattern per cell (its M pressure rows), SELL-32 over cells; header
    //       per lane [counts, E^T run starts..., B^T faces...], slots of M values:
    //       for j: E^T u_j entries (row i: theta_ij*((-b)*e)), B^T q_j pairs of
    //       consecutive entries of row j only (w_j*bv), the p_j entry of every row.
    //  QK : one pattern per face (its M flux rows), SELL-32 over faces; one int32
    //       column (offset within [q p]) and one slot of M values per entry.
    // Each row is still summed alone in ascending column order with
    // __dmul_rn/__dadd_rn: the same bits as the SELL layout and as
    // SparseMatrix::apply (sparse.hpp:30-40) on the canonical CSR.
    bool kp = false;
    long long kp_u_entries = 0, kp_u_hdr = 0;  // per-cell entries / header ints (sums)
    DBuf<long long> uk_voff;                   // n_cells + 1 (entry offset per cell)
    DBuf<long long> uk_hoff;                   // n_cells + 1 (header offset per cell)
    DBuf<int> uk_na;                           // n_cells: A runs (entries 8 * na), then E columns
    DBuf<int> uk_hdr;
    DBuf<double> uk_val;                       // 8 * M * kp_u_entries
    long long pk_slices = 0, pk_slots = 0, pk_hslots = 0;
    DBuf<long long> pk_voff, pk_hoff;          // pk_slices + 1
    DBuf<int> pk_hdr;                          // 32 * pk_hslots
    DBuf<double> pk_val;                       // 32 * M * pk_slots
    long long qk_slices = 0, qk_slots = 0;
    DBuf<long long> qk_off;                    // qk_slices + 1
    DBuf<int> qk_len;                          // n_q
    DBuf<int> qk_col;                          // 32 * qk_slots
    DBuf<double> qk_val;                       // 32 * M * qk_slots
    DBuf<long long> strip_qslices;             // kp strips: QK slices holding an owned face
    bool build_kp(const SpatialOps& ops, const double* theta, const double* w, cudaStream_t st);
    void kp_launch(const double* x, double* y, double* y2, const double* V, int ncols, double* partial, bool strip,
                   cudaStream_t st) const;
    int kp_grid(bool strip) const;
    void kp_to_csr(std::vector<long long>& off, std::vector<int>& idx, std::vector<double>& val, cudaStream_t st) const;

    // kappa: per-component stationary weights (w_i = tau kappa_i, fixed_stress.hpp:50);
    // null = 1 (the slab solver, slab.hpp:162)
    void build(const SpatialOps& ops, int m, const double* theta, double tau, cudaStream_t st,
               const double* kappa = nullptr);
    void apply(const double* x, double* y, cudaStream_t st) const;
    // y = A x (the same bits as apply), y2 = y, and per-block partials of V_j . y for
    // j < ncols <= 8 into partial[dots_grid()][ncols] (the first Gram-Schmidt pass of the
    // Arnoldi step, fused into the SpMV epilogue: gmres.hpp:95-97 after fixed_stress.hpp:38-60)
    void apply_dots(const double* x, double* y, double* y2, const double* V, int ncols, double* partial,
                    cudaStream_t st) const;
    int dots_grid() const;
    // when set, apply() is skipped on the device once *guard != 0 (speculative GMRES steps)
    const int* guard = nullptr;
    // Rows owned by the strip of cell rows [r0, r1) of an nx x ny mesh (multi-GPU
    // row partitioning): displacement and pressure rows of its
    // cells, flux rows of its face rows. Only owned y entries are written; x must
    // hold the owned entries and the one-cell-row halo. Same per-row arithmetic as
    // apply(): the union over strips is bit-identical to it.
    int strip_nx = 0, strip_ny = 0, strip_r0 = 0, strip_r1 = 0;
    DBuf<long long> strip_slices;  // S-class slices holding at least one owned row
    void set_strip(int nx, int ny, int r0, int r1, cudaStream_t st);
    void apply_strip(const double* x, double* y, cudaStream_t st) const;
    // canonical CSR download (tests / CPU bitwise check)
    void to_csr(std::vector<long long>& off, std::vector<int>& idx, std::vector<double>& val, cudaStream_t st) const;
};

// exclusive prefix sum of in[0..n) into out[0..n] (out[n] = total, returned)
long long scan_ll(const long long* in, long long* out, long long n, cudaStream_t st);

void spmv_csr_device(int rows, const long long* off, const int* idx, const double* val, const double* x, double* y,
                     cudaStream_t st);

}  // namespace pdg
