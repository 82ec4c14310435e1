// ORACLE / TEST INFRASTRUCTURE ONLY. Not part of the product.
//
// Eigen-free restatement of the dense / Krylov pieces the reference takes from
// Eigen >= 3.3 (absent from /root/reference and from this image; the version
// is not pinned by the reference, proj/CMakeLists.txt:13):
//   - PartialPivLU          (dense.hpp:14-45)          -> DenseLu
//   - ColPivHouseholderQR   (gmres.hpp:111)            -> colpiv_qr_solve
//   - dot / norm reductions (gmres.hpp:54,69,97,102)   -> sequential sums
// plus an exact sparse-direct backend (banded Cholesky) that replaces the
// reference's dense LU where the dense matrix cannot be formed (config 1:
// 137 GB for A at 128^2, slab.hpp:155). Same math, roundoff-level changes.
#pragma once

#include <cmath>
#include <cstring>
#include <functional>
#include <memory>

#include "fem.hpp"

namespace refcpu {

inline double dot(const double* a, const double* b, int n) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}
inline double norm(const double* a, int n) { return std::sqrt(dot(a, a, n)); }
inline double norm(const Vec& a) { return norm(a.data(), static_cast<int>(a.size())); }

// Interface of an exact inner solve (DenseLu::solve, dense.hpp:32-36).
struct InnerSolver {
    virtual ~InnerSolver() = default;
    virtual int size() const = 0;
    virtual void solve(const double* b, double* x) const = 0;
};

// dense.hpp:14-45 : partial-pivoting LU with the 1e-14 pivot-ratio check.
class DenseLu : public InnerSolver {
public:
    explicit DenseLu(std::vector<double> a_rowmajor, int n) : n_(n), lu_(std::move(a_rowmajor)), perm_(n) {
        for (int i = 0; i < n; ++i) perm_[i] = i;
        for (int k = 0; k < n; ++k) {
            int piv = k;
            double best = std::abs(lu_[static_cast<size_t>(k) * n + k]);
            for (int i = k + 1; i < n; ++i) {
                const double v = std::abs(lu_[static_cast<size_t>(i) * n + k]);
                if (v > best) {
                    best = v;
                    piv = i;
                }
            }
            if (piv != k) {
                std::swap_ranges(lu_.begin() + static_cast<size_t>(k) * n, lu_.begin() + static_cast<size_t>(k + 1) * n,
                                 lu_.begin() + static_cast<size_t>(piv) * n);
                std::swap(perm_[k], perm_[piv]);
            }
            const double dkk = lu_[static_cast<size_t>(k) * n + k];
            if (dkk == 0.0) continue;
            const double* rk = &lu_[static_cast<size_t>(k) * n];
#pragma omp parallel for schedule(static) if (n - k > 256)
            for (int i = k + 1; i < n; ++i) {
                double* ri = &lu_[static_cast<size_t>(i) * n];
                const double l = ri[k] / dkk;
                ri[k] = l;
                if (l != 0.0)
                    for (int j = k + 1; j < n; ++j) ri[j] -= l * rk[j];
            }
        }
        double dmax = 0.0, dmin = std::numeric_limits<double>::infinity();
        for (int i = 0; i < n; ++i) {
            const double d = std::abs(lu_[static_cast<size_t>(i) * n + i]);
            dmax = std::max(dmax, d);
            dmin = std::min(dmin, d);
        }
        if (n > 0 && (dmax == 0.0 || dmin <= 1e-14 * dmax))
            throw SolverError("dense LU: matrix is singular to working precision");
    }
    int size() const override { return n_; }
    void solve(const double* b, double* x) const override {
        const int n = n_;
        std::vector<double> y(n);
        for (int i = 0; i < n; ++i) y[i] = b[perm_[i]];
        for (int i = 0; i < n; ++i) {
            const double* ri = &lu_[static_cast<size_t>(i) * n];
            double s = y[i];
            for (int j = 0; j < i; ++j) s -= ri[j] * y[j];
            y[i] = s;
        }
        for (int i = n - 1; i >= 0; --i) {
            const double* ri = &lu_[static_cast<size_t>(i) * n];
            double s = y[i];
            for (int j = i + 1; j < n; ++j) s -= ri[j] * y[j];
            y[i] = s / ri[i];
        }
        std::memcpy(x, y.data(), sizeof(double) * n);
    }

private:
    int n_;
    std::vector<double> lu_;
    std::vector<int> perm_;
};

// Exact sparse-direct replacement for DenseLu on an SPD matrix: symmetric
// permutation `perm` (new -> old) followed by a banded Cholesky factorization
// (lower band stored by columns). Used for A (cell-row order is already
// banded, bandwidth 8 nx + 7) and for the flow Schur complement.
class BandCholesky : public InnerSolver {
public:
    BandCholesky(const SparseMatrix& a, std::vector<int> perm) : n_(a.rows), perm_(std::move(perm)) {
        if (a.rows != a.cols) throw std::invalid_argument("BandCholesky: matrix must be square");
        if (perm_.empty()) {
            perm_.resize(n_);
            for (int i = 0; i < n_; ++i) perm_[i] = i;
        }
        inv_.assign(n_, 0);
        for (int i = 0; i < n_; ++i) inv_[perm_[i]] = i;
        bw_ = 0;
        for (int i = 0; i < n_; ++i)
            for (int k = a.row_offsets[i]; k < a.row_offsets[i + 1]; ++k)
                bw_ = std::max(bw_, std::abs(inv_[i] - inv_[a.col_indices[k]]));
        const size_t ld = static_cast<size_t>(bw_) + 1;
        band_.assign(static_cast<size_t>(n_) * ld, 0.0);
        for (int i = 0; i < n_; ++i)
            for (int k = a.row_offsets[i]; k < a.row_offsets[i + 1]; ++k) {
                const int r = inv_[i], c = inv_[a.col_indices[k]];
                if (r >= c) band_[static_cast<size_t>(c) * ld + (r - c)] = a.values[k];
            }
        double dmax = 0.0;
        for (int k = 0; k < n_; ++k) dmax = std::max(dmax, std::abs(band_[static_cast<size_t>(k) * ld]));
        for (int k = 0; k < n_; ++k) {
            double* ck = &band_[static_cast<size_t>(k) * ld];
            const double d = ck[0];
            if (!(d > 1e-14 * dmax)) throw SolverError("dense LU: matrix is singular to working precision");
            const double lkk = std::sqrt(d);
            ck[0] = lkk;
            const int len = std::min(bw_, n_ - 1 - k);
            for (int i = 1; i <= len; ++i) ck[i] /= lkk;
#pragma omp parallel for schedule(static) if (len > 128)
            for (int j = 1; j <= len; ++j) {
                const double ljk = ck[j];
                if (ljk == 0.0) continue;
                double* cj = &band_[static_cast<size_t>(k + j) * ld];
                for (int i = j; i <= len; ++i) cj[i - j] -= ck[i] * ljk;
            }
        }
    }
    int size() const override { return n_; }
    int bandwidth() const { return bw_; }
    void solve(const double* b, double* x) const override {
        const size_t ld = static_cast<size_t>(bw_) + 1;
        std::vector<double> y(n_);
        for (int i = 0; i < n_; ++i) y[i] = b[perm_[i]];
        for (int k = 0; k < n_; ++k) {
            const double* ck = &band_[static_cast<size_t>(k) * ld];
            const double yk = y[k] / ck[0];
            y[k] = yk;
            const int len = std::min(bw_, n_ - 1 - k);
            for (int i = 1; i <= len; ++i) y[k + i] -= ck[i] * yk;
        }
        for (int k = n_ - 1; k >= 0; --k) {
            const double* ck = &band_[static_cast<size_t>(k) * ld];
            const int len = std::min(bw_, n_ - 1 - k);
            double s = y[k];
            for (int i = 1; i <= len; ++i) s -= ck[i] * y[k + i];
            y[k] = s / ck[0];
        }
        for (int i = 0; i < n_; ++i) x[perm_[i]] = y[i];
    }

private:
    int n_, bw_ = 0;
    std::vector<int> perm_, inv_;
    std::vector<double> band_;
};

// ---------------------------------------------------------------------------
// ColPivHouseholderQR least-squares solve (Eigen's algorithm as called at
// gmres.hpp:111): Householder vectors as in Eigen's makeHouseholder, column
// pivoting on the largest updated column norm with LAPACK-style downdating,
// numerical rank from the nonzero-pivot threshold, and the solve
// y = P R11^{-1} (Q^T b)[0:rank].
// `a` is column-major rows x cols.
// ---------------------------------------------------------------------------
inline std::vector<double> colpiv_qr_solve(std::vector<double> a, int rows, int cols, std::vector<double> b) {
    auto A = [&](int i, int j) -> double& { return a[static_cast<size_t>(j) * rows + i]; };
    const int size = std::min(rows, cols);
    std::vector<double> hcoeffs(size), norms_upd(cols), norms_dir(cols);
    std::vector<int> transp(size);
    const double eps = std::numeric_limits<double>::epsilon();
    double max_col_norm = 0.0;
    for (int j = 0; j < cols; ++j) {
        norms_dir[j] = norm(&A(0, j), rows);
        norms_upd[j] = norms_dir[j];
        max_col_norm = std::max(max_col_norm, norms_dir[j]);
    }
    const double threshold_helper = (max_col_norm * eps) * (max_col_norm * eps) / rows;
    const double norm_downdate_threshold = std::sqrt(eps);
    int nonzero_pivots = size;
    for (int k = 0; k < size; ++k) {
        int biggest = k;
        for (int j = k + 1; j < cols; ++j)
            if (norms_upd[j] > norms_upd[biggest]) biggest = j;
        const double biggest_sq = norms_upd[biggest] * norms_upd[biggest];
        if (nonzero_pivots == size && biggest_sq < threshold_helper * (rows - k)) nonzero_pivots = k;
        transp[k] = biggest;
        if (k != biggest) {
            for (int i = 0; i < rows; ++i) std::swap(A(i, k), A(i, biggest));
            std::swap(norms_upd[k], norms_upd[biggest]);
            std::swap(norms_dir[k], norms_dir[biggest]);
        }
        // makeHouseholderInPlace on column k, rows k..rows-1
        const int len = rows - k;
        double tail_sq = 0.0;
        for (int i = 1; i < len; ++i) tail_sq += A(k + i, k) * A(k + i, k);
        const double c0 = A(k, k);
        double tau, beta;
        if (tail_sq <= std::numeric_limits<double>::min()) {
            tau = 0.0;
            beta = c0;
            for (int i = 1; i < len; ++i) A(k + i, k) = 0.0;
        } else {
            beta = std::sqrt(c0 * c0 + tail_sq);
            if (c0 >= 0.0) beta = -beta;
            for (int i = 1; i < len; ++i) A(k + i, k) = A(k + i, k) / (c0 - beta);
            tau = (beta - c0) / beta;
        }
        hcoeffs[k] = tau;
        A(k, k) = beta;
        // applyHouseholderOnTheLeft to columns k+1..cols-1, rows k..rows-1
        if (tau != 0.0)
            for (int j = k + 1; j < cols; ++j) {
                double tmp = A(k, j);
                for (int i = 1; i < len; ++i) tmp += A(k + i, k) * A(k + i, j);
                A(k, j) -= tau * tmp;
                for (int i = 1; i < len; ++i) A(k + i, j) -= tau * A(k + i, k) * tmp;
            }
        for (int j = k + 1; j < cols; ++j) {
            if (norms_upd[j] != 0.0) {
                double temp = std::abs(A(k, j)) / norms_upd[j];
                temp = (1.0 + temp) * (1.0 - temp);
                temp = temp < 0.0 ? 0.0 : temp;
                const double r = norms_upd[j] / norms_dir[j];
                const double temp2 = temp * r * r;
                if (temp2 <= norm_downdate_threshold) {
                    norms_dir[j] = k + 1 < rows ? norm(&A(k + 1, j), rows - k - 1) : 0.0;
                    norms_upd[j] = norms_dir[j];
                } else {
                    norms_upd[j] *= std::sqrt(temp);
                }
            }
        }
    }
    // c = Q^T b restricted to the nonzero pivots
    std::vector<double> y(cols, 0.0);
    if (nonzero_pivots == 0) return y;
    for (int k = 0; k < nonzero_pivots; ++k) {
        const double tau = hcoeffs[k];
        if (tau == 0.0) continue;
        double tmp = b[k];
        for (int i = k + 1; i < rows; ++i) tmp += A(i, k) * b[i];
        b[k] -= tau * tmp;
        for (int i = k + 1; i < rows; ++i) b[i] -= tau * A(i, k) * tmp;
    }
    for (int i = nonzero_pivots - 1; i >= 0; --i) {
        double s = b[i];
        for (int j = i + 1; j < nonzero_pivots; ++j) s -= A(i, j) * b[j];
        b[i] = s / A(i, i);
    }
    // column permutation: apply the transpositions to recover indices
    std::vector<int> perm(cols);
    for (int j = 0; j < cols; ++j) perm[j] = j;
    for (int k = 0; k < size; ++k) std::swap(perm[k], perm[transp[k]]);
    for (int i = 0; i < nonzero_pivots; ++i) y[perm[i]] = b[i];
    return y;
}

// ---------------------------------------------------------------------------
// gmres.hpp:15-158
// ---------------------------------------------------------------------------
struct SolverReport {
    bool converged = false;
    int iterations = 0;
    std::vector<double> residual_history;
    double final_relative_residual = std::numeric_limits<double>::quiet_NaN();
};
struct GmresOptions {
    double tol = 1e-10;
    int restart = 100;
    int max_iter = 400;
};
using LinOp = std::function<void(const double*, double*)>;  // y = op(x), sizes n

inline Vec gmres_impl(const LinOp& apply_op, const LinOp& apply_precond, const Vec& b, const GmresOptions& opt,
                      bool flexible, SolverReport& rep) {
    if (!(opt.tol > 0.0 && opt.tol < 1.0)) throw std::invalid_argument("gmres: tol must be in (0,1)");
    if (opt.restart < 1 || opt.max_iter < 1) throw std::invalid_argument("gmres: bad iteration limits");
    const int n = static_cast<int>(b.size());
    rep = SolverReport{};
    const double bnorm = norm(b);
    if (bnorm <= 1e-14) {  // gmres.hpp:56-62
        rep.converged = true;
        rep.iterations = 0;
        rep.residual_history = {bnorm};
        rep.final_relative_residual = 0.0;
        return Vec(n, 0.0);
    }
    Vec x(n, 0.0), tmp(n), tmp2(n);
    double true_res = bnorm;
    rep.residual_history.push_back(true_res);
    auto record = [&](const Vec& cand) {  // gmres.hpp:68-72
        apply_op(cand.data(), tmp.data());
        for (int i = 0; i < n; ++i) tmp[i] = b[i] - tmp[i];
        true_res = norm(tmp);
        rep.residual_history.push_back(true_res);
        return true_res / bnorm <= opt.tol;
    };
    int total_iters = 0;
    while (total_iters < opt.max_iter) {
        Vec r(n);
        apply_op(x.data(), tmp.data());
        for (int i = 0; i < n; ++i) r[i] = b[i] - tmp[i];
        const double beta = norm(r);
        if (beta / bnorm <= opt.tol) break;
        const int m = std::min(opt.restart, opt.max_iter - total_iters);
        std::vector<double> V(static_cast<size_t>(n) * (m + 1)), Z;
        if (flexible) Z.resize(static_cast<size_t>(n) * m);
        std::vector<double> H(static_cast<size_t>(m + 1) * m, 0.0);  // column-major (m+1) x m
        auto h = [&](int i, int j) -> double& { return H[static_cast<size_t>(j) * (m + 1) + i]; };
        for (int i = 0; i < n; ++i) V[i] = r[i] / beta;
        bool done = false;
        Vec zk(n), w(n);
        for (int k = 0; k < m && !done; ++k) {
            apply_precond(&V[static_cast<size_t>(k) * n], zk.data());
            if (flexible) std::copy(zk.begin(), zk.end(), Z.begin() + static_cast<size_t>(k) * n);
            apply_op(zk.data(), w.data());
            for (int pass = 0; pass < 2; ++pass)  // gmres.hpp:94-101
                for (int i = 0; i <= k; ++i) {
                    const double* vi = &V[static_cast<size_t>(i) * n];
                    const double c = dot(vi, w.data(), n);
                    h(i, k) += c;
                    for (int t = 0; t < n; ++t) w[t] -= c * vi[t];
                }
            h(k + 1, k) = norm(w);
            const bool breakdown = h(k + 1, k) <= 1e-14 * norm(&h(0, k), m + 1);
            if (!breakdown)
                for (int t = 0; t < n; ++t) V[static_cast<size_t>(k + 1) * n + t] = w[t] / h(k + 1, k);
            ++total_iters;
            // least squares on the leading (k+2) x (k+1) block
            std::vector<double> hk(static_cast<size_t>(k + 2) * (k + 1));
            for (int j = 0; j <= k; ++j)
                for (int i = 0; i < k + 2; ++i) hk[static_cast<size_t>(j) * (k + 2) + i] = h(i, j);
            std::vector<double> e1(k + 2, 0.0);
            e1[0] = beta;
            const std::vector<double> y = colpiv_qr_solve(hk, k + 2, k + 1, e1);
            Vec cand(n);
            if (flexible) {
                std::fill(tmp2.begin(), tmp2.end(), 0.0);
                for (int j = 0; j <= k; ++j) {
                    const double* zj = &Z[static_cast<size_t>(j) * n];
                    for (int t = 0; t < n; ++t) tmp2[t] += zj[t] * y[j];
                }
                for (int t = 0; t < n; ++t) cand[t] = x[t] + tmp2[t];
            } else {
                std::fill(tmp2.begin(), tmp2.end(), 0.0);
                for (int j = 0; j <= k; ++j) {
                    const double* vj = &V[static_cast<size_t>(j) * n];
                    for (int t = 0; t < n; ++t) tmp2[t] += vj[t] * y[j];
                }
                Vec pz(n);
                apply_precond(tmp2.data(), pz.data());
                for (int t = 0; t < n; ++t) cand[t] = x[t] + pz[t];
            }
            if (record(cand)) {
                x = cand;
                rep.converged = true;
                done = true;
            } else if (breakdown) {
                x = cand;
                done = true;
            } else if (k == m - 1 || total_iters >= opt.max_iter) {
                x = cand;
                done = true;
            }
        }
        if (rep.converged) break;
    }
    rep.iterations = total_iters;
    rep.final_relative_residual = true_res / bnorm;
    if (!rep.converged) rep.converged = rep.final_relative_residual <= opt.tol;
    return x;
}

}  // namespace refcpu
