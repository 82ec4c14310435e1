// Exact SPD solver for matrices that are block tridiagonal in a given
// symmetric permutation (the displacement block A in cell-row order, the
// flow Schur complement in face-row order). Replaces the reference's dense
// partial-pivot LU (dense.hpp:14-45, used at slab.hpp:155 and
// fixed_stress.hpp:184-201) with the same exact solve at O(n * w^2) memory.
#pragma once

#include <cublas_v2.h>
#include <cusolverDn.h>

#include "common.cuh"

namespace pdg {

// A = L L^T with L block lower bidiagonal: diag L_j, subdiag K_j = L_{j+1,j}.
// Stored for the solve:
//   Linv_j = L_j^{-1}                      (col-major, lower)      -- c_j = Linv_j b_j,  e_j = Linv_j^T y_j
//   M_j    = Linv_j K_{j-1}  (row-major)   -- forward  y_j = c_j - M_j y_{j-1}
//   N_j    = Linv_j^T K_j^T  (row-major)   -- backward x_j = e_j - N_j x_{j+1}
// The two recurrences run in one persistent cooperative kernel each.
struct BlockTriChol {
    int n = 0, nb = 0, max_b = 0;
    std::vector<int> bsz, boff;            // block sizes / offsets (permuted order)
    std::vector<long long> o_linv, o_m, o_n;  // offsets into store
    DBuf<double> store;
    DBuf<int> d_bsz, d_boff;
    DBuf<long long> d_olinv, d_om, d_on;
    DBuf<int> perm;  // new -> old (empty = identity)
    DBuf<unsigned int> bar;  // grid barrier state
    int coop_blocks = 0;
    void* rec_fn = nullptr;  // register-prefetch recurrence (fallback) for max_b
    bool use_tma = false;    // TMA-pipelined recurrence available
    int tma_blocks = 0, tma_stages = 0, maxld = 0;
    size_t tma_smem = 0;
    std::vector<long long> o_linvr;
    std::vector<int> ld_m, ld_n, ld_l;
    DBuf<long long> d_olinvr;
    DBuf<int> d_ldm, d_ldn, d_ldl;
    DBuf<unsigned int> counter;
    DBuf<uint4> ll;  // LL lines (value + flag) of the dataflow recurrence, n * max_rhs
    unsigned long long tag_call = 0;
    int prof_phase = PROF_A_SOLVE;
    // algorithmic bytes of one solve: L read by the forward and the backward
    // substitution (stored as Linv lower + M + N = 3 m^2/block) + b in, x out
    double alg_bytes(int nrhs) const;
    // work vectors (n * max_rhs)
    int max_rhs = 0;
    DBuf<double> wb, wc, wy, we, wx;

    // Factor the SPD matrix given as device CSR rows (natural numbering) with
    // permutation perm_host (new -> old, empty = identity) and block sizes.
    void factor(int n_, const int* off, const int* idx, const double* val, const std::vector<int>& perm_host,
                const std::vector<int>& block_sizes, int max_rhs_, cudaStream_t st);
    // Factor from dense blocks already scattered (used by the flow Schur complement builder).
    void factor_dense(double* D, double* C, cudaStream_t st);
    // x = A^{-1} b for nrhs right-hand sides; b/x columns at stride ldb/ldx (natural numbering).
    void solve(const double* b, long long ldb, double* x, long long ldx, int nrhs, cudaStream_t st);
    void recurrence(int dir, const double* in, double* out, int nrhs, cudaStream_t st);

    // helpers exposed to builders
    void layout(int n_, const std::vector<int>& perm_host, const std::vector<int>& block_sizes);
    long long dense_d_offset(int j) const { return dD_[j]; }
    long long dense_c_offset(int j) const { return dC_[j]; }
    long long dense_total() const { return dtot_; }
    DBuf<int> inv_perm;  // old -> new
    DBuf<int> blk_of;    // new index -> block
    DBuf<int> loc_of;    // new index -> local index

private:
    std::vector<long long> dD_, dC_;
    long long dtot_ = 0;
};

// cuBLAS / cuSOLVER handles bound to a stream (setup only).
struct LaHandles {
    cublasHandle_t blas = nullptr;
    cusolverDnHandle_t solver = nullptr;
    LaHandles(cudaStream_t st);
    ~LaHandles();
};

}  // namespace pdg
