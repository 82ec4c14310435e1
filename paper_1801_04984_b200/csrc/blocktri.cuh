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

struct LaHandles;

// One step of the dense sweep for one chain (see blocktri_dense.cu): output
// rows [0, mout) of the step = M * [seg0; seg1], M row-major at store + moff
// (row stride ld). seg0: n0 values at LL offset in0 (or from b at b0 when
// in0 < 0); seg1: n1 values at LL offset in1. Outputs go to LL offset out_ll
// and/or x offset out_x (-1 = none); moff < 0 = idle.
struct DenseTask {
    long long moff, in0, in1, b0, out_ll, out_x;
    int n0, n1, mout, ld;
    long long base;  // b offset added to the outputs (-1 none)
    int acc, pad_;   // acc: x[out_x] += outputs
};

// One step of the local-coupling sweep for one chain (see BlockTriChol::local).
enum SweepKind { SW_IDLE = 0, SW_FIRST = 1, SW_FWD = 2, SW_TWIST = 3, SW_BWD = 4 };
struct SweepTask {
    int blk, kind;
};

// Twisted ("burn at both ends") block Cholesky A = P P^T with twist block t:
// blocks 0..t-1 are eliminated from the top (L_j, K_j = L_{j+1,j}), blocks
// nb-1..t+1 from the bottom (L'_j, K'_j = L_{j-1,j}), and
// L_t L_t^T = A_tt - K_{t-1} K_{t-1}^T - K'_{t+1} K'_{t+1}^T.
// A solve is ONE persistent cooperative kernel in which a top and a bottom
// chain run concurrently as a barrier-free dataflow (LL lines between CTAs,
// TMA-streamed matrix rows), about nb dependent steps in all:
//   local mode  (chunk-local couplings, the displacement block): k_sweep,
//               blocktri_local.cu, stores Sinv_j of the twisted Schur complements;
//   dense mode  (any coupling, the flow block): k_sweep_dense,
//               blocktri_dense.cu, stores [Linv | -Linv K]-type step matrices.
struct BlockTriChol {
    int n = 0, nb = 0, max_b = 0, twist = 0;
    std::vector<int> bsz, boff;
    DBuf<int> d_bsz, d_boff;
    DBuf<int> perm;                 // new -> old (empty = identity)
    DBuf<int> inv_perm, blk_of, loc_of;
    DBuf<double> store;              // the solve matrices
    double factor_bytes = 0.0;       // bytes of the stored solve matrices read per solve
    DBuf<uint4> ll;                  // LL lines (value + flag)
    unsigned long long call = 0;
    int prof_phase = PROF_A_SOLVE;
    int max_rhs = 0;
    bool debug_timing = false;       // per-step %globaltimer stamps of the last recurrence into dbg
    DBuf<unsigned long long> dbg;
    DBuf<double> wb, wx;             // permuted right-hand sides / solutions (dense mode)
    int dbg_steps = 0;               // steps recorded in dbg by the last solve

    // ---- local-coupling mode (the displacement block A) -------------------------------
    // When all blocks have one size m (multiple of 8), no permutation is used and
    // every coupling block C_j = A_{j+1,j} only couples an 8-row chunk (a cell) to
    // the same chunk of the neighbour block, the solve keeps the inverse twisted
    // Schur complements Sinv_j (full, row-major) and the 8x8 coupling chunks and
    // runs ONE persistent kernel (k_sweep):
    //   forward   v_j = Sinv_j w_j,   w_{j+1} = b_{j+1} - C_j v_j         (top chain)
    //             v_j = Sinv_j w_j,   w_{j-1} = b_{j-1} - C_{j-1}^T v_j   (bottom chain)
    //   twist     x_t = Sinv_t (b_t - C_{t-1} v_{t-1} - C_t^T v_{t+1})
    //   backward  x_j = Sinv_j (w_j - C_j^T x_{j+1}) / Sinv_j (w_j - C_{j-1} x_{j-1})
    // The chunk-local products are formed by the CTA that owns the chunk, so each
    // step streams one Sinv_j: 2 m^2 doubles per block per solve (the general
    // path reads 3 m^2: Linv twice, F/G and N).
    bool allow_local = false;        // set by the owner before factor()
    bool symmetric = true;           // false: non-symmetric matrix, twisted block LU (set before layout/factor)
    bool local = false;              // chosen by factor()
    DBuf<double> cloc;               // [nb-1][m/8][8][8]: chunk (r, q) of C_j, row-major
    DBuf<double> wsave;              // w_j of the forward sweep, read back by the backward sweep
    long long sinv_stride = 0;       // Sinv_j at store + j * sinv_stride, row stride ld_s
    int ld_s = 0, sw_rpc = 0, sw_g = 0, sw_stages = 0;
    size_t sw_smem = 0;
    std::vector<SweepTask> sweep;    // steps x 2 chains
    DBuf<SweepTask> d_sweep;

    // ---- dense-sweep mode (any coupling pattern: the flow solve) -------------------------
    std::vector<DenseTask> dsched;   // steps x nchains
    int nchains = 2;
    DBuf<DenseTask> d_dsched;
    long long d_lln = 0;
    int d_ldmax = 0, d_g = 0, d_stages = 0;
    size_t d_smem = 0;

    // Factor the SPD matrix given as device CSR rows (natural numbering) with
    // permutation perm_host (new -> old, empty = identity) and block sizes.
    void factor(int n_, const int* off, const int* idx, const double* val, const std::vector<int>& perm_host,
                const std::vector<int>& block_sizes, int max_rhs_, cudaStream_t st);
    // Factor from dense blocks already scattered by a builder (layout()/dense offsets).
    void factor_dense(double* dense, cudaStream_t st);
    // x = A^{-1} b for nrhs <= 2 right-hand sides; columns at stride ldb/ldx (natural numbering).
    void solve(const double* b, long long ldb, double* x, long long ldx, int nrhs, cudaStream_t st);
    // algorithmic bytes of one solve: the factor read by both substitutions + b in, x out
    double alg_bytes(int nrhs) const { return factor_bytes + 16.0 * n * nrhs; }

    // builder helpers: dense diagonal blocks D_j (m_j x m_j col-major) and
    // sub-diagonal blocks C_j = A_{j+1,j} (m_{j+1} x m_j col-major)
    void layout(int n_, const std::vector<int>& perm_host, const std::vector<int>& block_sizes);
    long long dense_d_offset(int j) const { return dD_[j]; }
    long long dense_c_offset(int j) const { return dC_[j]; }
    long long dense_u_offset(int j) const { return dU_[j]; }  // non-symmetric: A_{j,j+1}
    long long dense_total() const { return dtot_; }

private:
    std::vector<long long> dD_, dC_, dU_;
    long long dtot_ = 0;
    bool local_prepare(double* dense, cudaStream_t st);   // structure check + coupling chunks
    void local_finish(double* dense, cudaStream_t st);    // Sinv_j from the Cholesky factors, schedule, kernel config
    void solve_local(const double* b, long long ldb, double* x, long long ldx, int nrhs, cudaStream_t st);
    void dense_setup(double* dense, cudaStream_t st);
    void solve_dense(const double* b, double* x, int nrhs, cudaStream_t st);
};

// cuBLAS / cuSOLVER handles bound to a stream (setup only).
struct LaHandles {
    cublasHandle_t blas = nullptr;
    cusolverDnHandle_t solver = nullptr;
    LaHandles(cudaStream_t st);
    ~LaHandles();
};

}  // namespace pdg
