// Stand-ins for the reference types the GPU binding touches (member names and
// shapes as in proj/include/porodg: sparse.hpp:20-27, material.hpp:25-33,
// assembly.hpp:18-20 and :38-52, time_basis.hpp:104-114, slab.hpp:22-56 and
// :113-127, gmres.hpp:15-28, fixed_stress.hpp:17-22). The reference itself
// cannot be compiled here (Eigen3 is absent), so the binding is compiled and run
// against these; Eigen::VectorXd is replaced by a vector with data()/size().
#pragma once

#include <vector>

namespace porodg {

struct VectorXd {
    std::vector<double> v;
    VectorXd() = default;
    explicit VectorXd(int n) : v(static_cast<size_t>(n), 0.0) {}
    double* data() { return v.data(); }
    const double* data() const { return v.data(); }
    long size() const { return static_cast<long>(v.size()); }
};
struct SparseMatrix {
    int rows = 0, cols = 0;
    std::vector<int> row_offsets, col_indices;
    std::vector<double> values;
    int nnz() const { return static_cast<int>(values.size()); }
};
struct MaterialParameters {
    double lambda_lame = 1.0, mu_lame = 1.0, k_perm = 1.0, eta = 1.0, biot_b = 0.8, biot_m = 10.0, k_dr = 2.0;
};
struct FieldVecs {
    VectorXd u, q, p;
};
struct SpatialOperators {
    SparseMatrix A, M_q, B, E, M_p;
    VectorXd m_p_diag;
    double penalty = 0.0;
    MaterialParameters mat;
    std::vector<char> q_constrained;
    int n_u = 0, n_q = 0, n_p = 0;
    int n_total() const { return n_u + n_q + n_p; }
};
struct TimeBasis {
    int r = 0;
    int n_nodes() const { return r + 1; }
};
struct SlabState {
    std::vector<FieldVecs> comps;
};
struct SlabSystem {
    const SpatialOperators* ops = nullptr;
    double tau = 0.0;
    std::vector<VectorXd> rhs;
};
struct SolverReport {
    bool converged = false;
    int iterations = 0;
    std::vector<double> residual_history;
    double final_relative_residual = 0.0;
};
struct BlockReport {
    int block_index = 0, block_size = 1, gmres_iterations = 0, fs_sweeps = 0;
    SolverReport report;
};
struct GmresOptions {
    double tol = 1e-10;
    int restart = 100, max_iter = 400;
};
struct FixedStressConfig {
    double stab = -1.0;
    int truncation_sweeps = 1;
};
struct SolveOptions {
    GmresOptions gmres;
    FixedStressConfig fs;
};
inline FieldVecs unstack_fields(const SpatialOperators& ops, const VectorXd& x) {
    FieldVecs f;
    f.u.v.assign(x.v.begin(), x.v.begin() + ops.n_u);
    f.q.v.assign(x.v.begin() + ops.n_u, x.v.begin() + ops.n_u + ops.n_q);
    f.p.v.assign(x.v.begin() + ops.n_u + ops.n_q, x.v.end());
    return f;
}

}  // namespace porodg
