// Header-only C++ host layer over the porodg_b200 C ABI (porodg_b200.h).
//
// Mirrors the reference's slab-solve interface (paths relative to
// /root/reference/proj/include/porodg/):
//   porodg_b200::Context            device + stream (new; the reference is CPU-only)
//   porodg_b200::SpatialOperators   SpatialOperators (assembly.hpp:38-52) on the device
//   porodg_b200::SlabSolver         SlabSolver (slab.hpp:133-274), gmres_fs on the GPU
//   porodg_b200::SolverError        SolverError (errors.hpp:10-13), same message texts
// Vectors are any contiguous double container with data()/size() (std::vector,
// Eigen::VectorXd), so the reference can call it with its own types
// (INTEGRATION.md). No Eigen dependency here.
#pragma once

#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "porodg_b200.h"

namespace porodg_b200 {

class SolverError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

inline void check(int rc) {
    if (rc == PDG_OK) return;
    const std::string msg = pdg_last_error();
    if (rc == PDG_NOT_CONVERGED) throw SolverError(msg);
    if (rc == PDG_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

struct GmresOptions {  // gmres.hpp:24-28
    double tol = 1e-10;
    int restart = 100;
    int max_iter = 400;
};
struct SolveOptions {  // slab.hpp:123-127 (+ fixed_stress.hpp:17-22)
    GmresOptions gmres;
    int truncation_sweeps = 1;
    double stab = -1.0;      // < 0: b^2 / K_dr
    bool flexible = false;   // candidate x + Z y (gmres_flexible) instead of x + P(V y)
    bool fast = false;       // pdg_gmres_opts.mode 1: fp32-stored displacement factor on 3D meshes
    pdg_gmres_opts c() const {
        pdg_gmres_opts o{};
        o.tol = gmres.tol;
        o.restart = gmres.restart;
        o.max_iter = gmres.max_iter;
        o.sweeps = truncation_sweeps;
        o.stab = stab;
        o.candidate = flexible ? 1 : 0;
        o.mode = fast ? 1 : 0;
        return o;
    }
};
struct SolverReport {  // gmres.hpp:15-20
    bool converged = false;
    int iterations = 0;
    std::vector<double> residual_history;
    double final_relative_residual = 0.0;
    double device_ms = 0.0;
};

class Context {
public:
    explicit Context(int device = 0) { check(pdg_ctx_create(device, &h_)); }
    ~Context() { pdg_ctx_destroy(h_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    pdg_ctx* get() const { return h_; }

private:
    pdg_ctx* h_ = nullptr;
};

// CSR view of a reference SparseMatrix (sparse.hpp:20-27).
template <class Sparse>
pdg_csr csr_view(const Sparse& s) {
    return pdg_csr{s.rows, s.cols, static_cast<int>(s.values.size()), s.row_offsets.data(), s.col_indices.data(),
                   s.values.data()};
}

class SpatialOperators {
public:
    // Upload operators assembled by the reference (assemble_operators).
    template <class Ops>
    SpatialOperators(Context& ctx, int nx, int ny, const Ops& ops) {
        const pdg_csr A = csr_view(ops.A), Mq = csr_view(ops.M_q), B = csr_view(ops.B), E = csr_view(ops.E);
        std::vector<signed char> qc(ops.q_constrained.begin(), ops.q_constrained.end());
        check(pdg_ops_upload(ctx.get(), nx, ny, &A, &Mq, &B, &E, ops.m_p_diag.data(), qc.data(), ops.mat.biot_b,
                             1.0 / ops.mat.biot_m, ops.mat.k_dr, &h_));
    }
    // Assemble on the device from a structured-mesh problem description.
    SpatialOperators(Context& ctx, const pdg_problem& p) { check(pdg_ops_assemble(ctx.get(), &p, &h_)); }
    // 3D extension (BASELINE config 2; no reference counterpart): nx x ny x nz hexahedra.
    SpatialOperators(Context& ctx, const pdg_problem3& p) { check(pdg_ops_assemble3(ctx.get(), &p, &h_)); }
    ~SpatialOperators() { pdg_ops_destroy(h_); }
    SpatialOperators(const SpatialOperators&) = delete;
    SpatialOperators& operator=(const SpatialOperators&) = delete;
    pdg_ops* get() const { return h_; }
    long long n_total() const {
        long long s[7];
        check(pdg_ops_sizes(h_, s));
        return s[0] + s[1] + s[2];
    }

private:
    pdg_ops* h_ = nullptr;
};

// SlabSolver for dG(r), r in {0, 1}: solve(rhs) takes the stacked SlabSystem
// rhs ((r+1) * n_total, per Radau node) and returns the (r+1) solution
// components in the same layout (slab.hpp:179-255).
class SlabSolver {
public:
    SlabSolver(SpatialOperators& ops, int r, double tau, const SolveOptions& opt) : r_(r), n_(ops.n_total()) {
        const pdg_gmres_opts o = opt.c();
        check(pdg_slab_create(ops.get(), r, tau, &o, &h_));
        cap_ = opt.gmres.max_iter + 2;
    }
    ~SlabSolver() { pdg_slab_destroy(h_); }
    SlabSolver(const SlabSolver&) = delete;
    SlabSolver& operator=(const SlabSolver&) = delete;

    template <class Vec>
    std::pair<std::vector<double>, SolverReport> solve(const Vec& rhs) const {
        if (static_cast<long long>(rhs.size()) != (r_ + 1) * n_)
            throw std::invalid_argument("SlabSolver::solve: rhs dimension mismatch");
        std::vector<double> out(rhs.size()), hist(cap_);
        pdg_report rep{};
        rep.history = hist.data();
        rep.history_cap = cap_;
        check(pdg_slab_solve(h_, rhs.data(), out.data(), &rep));
        SolverReport sr;
        sr.converged = rep.converged != 0;
        sr.iterations = rep.iterations;
        sr.final_relative_residual = rep.final_rel_res;
        sr.residual_history.assign(hist.begin(), hist.begin() + std::min(rep.history_len, cap_));
        sr.device_ms = rep.device_ms;
        return {std::move(out), std::move(sr)};
    }

private:
    pdg_slab* h_ = nullptr;
    int r_ = 0, cap_ = 0;
    long long n_ = 0;
};

// FixedStressSolver of the fixed-stress march (fixed_stress.hpp:144-172 as built
// at march.hpp:83-84): solve(rhs, x0) sweeps from x0 (empty = zero) until the
// true residual drops below tol; report.iterations = fs_sweeps. Device path: dG(0).
class FixedStressSolver {
public:
    FixedStressSolver(SpatialOperators& ops, int r, double tau, double tol = 1e-10, int max_sweeps = 200,
                      double stab = -1.0)
        : r_(r), n_(ops.n_total()), cap_(max_sweeps + 2) {
        const pdg_fs_opts o{tol, max_sweeps, stab};
        check(pdg_fs_create(ops.get(), r, tau, &o, &h_));
    }
    ~FixedStressSolver() { pdg_fs_destroy(h_); }
    FixedStressSolver(const FixedStressSolver&) = delete;
    FixedStressSolver& operator=(const FixedStressSolver&) = delete;

    template <class Vec>
    std::pair<std::vector<double>, SolverReport> solve(const Vec& rhs, const Vec* x0 = nullptr) const {
        if (static_cast<long long>(rhs.size()) != (r_ + 1) * n_ ||
            (x0 && static_cast<long long>(x0->size()) != (r_ + 1) * n_))
            throw std::invalid_argument("fixed-stress: bad initial guess size");
        std::vector<double> out(rhs.size()), hist(cap_);
        pdg_report rep{};
        rep.history = hist.data();
        rep.history_cap = cap_;
        check(pdg_fs_solve(h_, rhs.data(), x0 ? x0->data() : nullptr, out.data(), &rep));
        SolverReport sr;
        sr.converged = rep.converged != 0;
        sr.iterations = rep.iterations;
        sr.final_relative_residual = rep.final_rel_res;
        sr.residual_history.assign(hist.begin(), hist.begin() + std::min(rep.history_len, cap_));
        sr.device_ms = rep.device_ms;
        return {std::move(out), std::move(sr)};
    }

private:
    pdg_fs* h_ = nullptr;
    int r_ = 0;
    long long n_ = 0;
    int cap_ = 0;
};

// local_mass_residual (slab.hpp:292-318): |residual| per cell and the scale, from
// the stacked slab rhs and state ((r+1) * n_total each).
template <class Vec>
std::pair<std::vector<double>, double> mass_residual(SpatialOperators& ops, int r, double tau, const Vec& rhs,
                                                     const Vec& state) {
    long long s[7];
    check(pdg_ops_sizes(ops.get(), s));
    if (static_cast<long long>(rhs.size()) != (r + 1) * ops.n_total() ||
        static_cast<long long>(state.size()) != (r + 1) * ops.n_total())
        throw std::invalid_argument("mass_residual: rhs/state dimension mismatch");
    std::vector<double> res(s[2]);
    double scale = 0.0;
    check(pdg_mass_residual(ops.get(), r, tau, rhs.data(), state.data(), res.data(), &scale));
    return {std::move(res), scale};
}

}  // namespace porodg_b200
