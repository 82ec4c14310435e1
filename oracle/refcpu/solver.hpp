// ORACLE / TEST INFRASTRUCTURE ONLY. Not part of the product.
//
// Restatement of the reference's time discretisation (time_basis.hpp,
// schur.hpp for r <= 1), the fixed-stress preconditioner / block operator
// (fixed_stress.hpp), the slab solver (slab.hpp) and the monolithic march
// (march.hpp:45-79,109-117), plus the canonical assembled space-time operator
// of SURVEY.md section 8(a) row a9.
#pragma once

#include <complex>
#include <map>

#include "linalg.hpp"

namespace refcpu {

// time_basis.hpp:33-40
struct TimePartition {
    std::vector<double> t_points;
    int n_slabs() const { return static_cast<int>(t_points.size()) - 1; }
    double slab_length(int n) const { return t_points[n + 1] - t_points[n]; }
    double t_begin(int n) const { return t_points[n]; }
    double t_end(int n) const { return t_points[n + 1]; }
};
inline TimePartition uniform_partition(double T, int n_slabs) {
    if (!(T > 0.0) || n_slabs < 1) throw std::invalid_argument("uniform_partition: bad arguments");
    TimePartition p;
    p.t_points.resize(n_slabs + 1);
    for (int n = 0; n <= n_slabs; ++n) p.t_points[n] = T * n / n_slabs;
    p.t_points.back() = T;
    return p;
}

// time_basis.hpp:47-97
inline std::vector<double> radau_points(int r) {
    if (r < 0 || r > 10) throw std::invalid_argument("radau_points: r out of range [0, 10]");
    std::vector<double> s;
    if (r > 0) {
        auto g = [&](double x) { return (legendre(r, x).first + legendre(r + 1, x).first) / (1.0 + x); };
        auto gprime = [&](double x) {
            const auto a = legendre(r, x), b = legendre(r + 1, x);
            const double f = a.first + b.first, df = a.second + b.second;
            return (df * (1.0 + x) - f) / ((1.0 + x) * (1.0 + x));
        };
        const int grid = 200 * (r + 1);
        double xa = -1.0 + 1e-12;
        double ga = g(xa);
        for (int k = 1; k <= grid; ++k) {
            const double xb = -1.0 + 2.0 * k / grid - (k == grid ? 1e-12 : 0.0);
            const double gb = g(xb);
            if (ga == 0.0) s.push_back(0.5 * (1.0 - xa));
            if (ga * gb < 0.0) {
                double lo = xa, hi = xb;
                for (int it = 0; it < 60; ++it) {
                    const double mid = 0.5 * (lo + hi);
                    (g(lo) * g(mid) <= 0.0 ? hi : lo) = mid;
                }
                double x = 0.5 * (lo + hi);
                for (int it = 0; it < 50; ++it) {
                    const double dx = g(x) / gprime(x);
                    x -= dx;
                    if (std::abs(dx) < 1e-16) break;
                }
                s.push_back(0.5 * (1.0 - x));
            }
            xa = xb;
            ga = gb;
        }
        if (static_cast<int>(s.size()) != r) throw std::runtime_error("radau_points: root search failed");
    }
    s.push_back(1.0);
    std::sort(s.begin(), s.end());
    return s;
}

// time_basis.hpp:104-182 ; small matrices row-major n x n
struct TimeBasis {
    int r = 0;
    std::vector<double> nodes, weights, bary, phi_at0, deriv, G_hat, M_hat;
    int n_nodes() const { return r + 1; }
    std::vector<double> eval(double s) const {
        const int n = n_nodes();
        std::vector<double> v(n, 0.0);
        for (int j = 0; j < n; ++j)
            if (std::abs(s - nodes[j]) < 1e-14) {
                v[j] = 1.0;
                return v;
            }
        double denom = 0.0;
        for (int j = 0; j < n; ++j) {
            v[j] = bary[j] / (s - nodes[j]);
            denom += v[j];
        }
        for (int j = 0; j < n; ++j) v[j] = v[j] / denom;
        return v;
    }
};
inline TimeBasis time_matrices(int r) {
    TimeBasis b;
    b.r = r;
    b.nodes = radau_points(r);
    const int n = r + 1;
    b.bary.resize(n);
    for (int j = 0; j < n; ++j) {
        double w = 1.0;
        for (int k = 0; k < n; ++k)
            if (k != j) w /= (b.nodes[j] - b.nodes[k]);
        b.bary[j] = w;
    }
    if (r == 0) {
        b.weights = {1.0};
    } else {
        const QuadratureRule gl = gauss_legendre(n + 1);
        b.weights.assign(n, 0.0);
        for (size_t k = 0; k < gl.points.size(); ++k) {
            const auto e = b.eval(gl.points[k]);
            for (int j = 0; j < n; ++j) b.weights[j] += gl.weights[k] * e[j];
        }
    }
    b.M_hat.assign(n * n, 0.0);
    for (int i = 0; i < n; ++i) b.M_hat[i * n + i] = b.weights[i];
    b.deriv.assign(n * n, 0.0);
    for (int i = 0; i < n; ++i) {
        double diag = 0.0;
        for (int j = 0; j < n; ++j) {
            if (i == j) continue;
            b.deriv[i * n + j] = (b.bary[j] / b.bary[i]) / (b.nodes[i] - b.nodes[j]);
            diag -= b.deriv[i * n + j];
        }
        b.deriv[i * n + i] = diag;
    }
    b.phi_at0 = b.eval(0.0);
    b.G_hat.assign(n * n, 0.0);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) b.G_hat[i * n + j] = b.weights[i] * b.deriv[i * n + j] + b.phi_at0[i] * b.phi_at0[j];
    return b;
}

// schur.hpp:101-173, restricted to r <= 1 (1x1, or one 2x2 block with a
// complex pair). For a 2x2 input Eigen's RealSchur reduces W/scale to
// Hessenberg with an identity transform, finds il == iu-1 and calls
// splitOffTwoRows, which leaves a complex-pair block untouched; the result is
// T = (W/scale)*scale, U = I. standardize_block (schur.hpp:87-97) follows.
struct SchurForm {
    int n = 1;
    std::vector<double> W, Q, T;  // row-major n x n
    std::vector<int> block_sizes, block_starts;
    int n_blocks() const { return static_cast<int>(block_sizes.size()); }
    double t(int i, int j) const { return T[i * n + j]; }
    double q(int i, int j) const { return Q[i * n + j]; }
    std::complex<double> block_eigenvalue(int g) const {
        const int i = block_starts[g];
        if (block_sizes[g] == 1) return {t(i, i), 0.0};
        const double a = t(i, i), b = t(i, i + 1), c = t(i + 1, i), d = t(i + 1, i + 1);
        const double re = 0.5 * (a + d);
        const double disc = 0.25 * (a - d) * (a - d) + b * c;
        return {re, std::sqrt(std::max(0.0, -disc))};
    }
};
// r >= 2: the reference calls Eigen::RealSchur (schur.hpp:108-114), an unvendored dependency
// (Eigen >= 3.3, version unpinned). Its published algorithm is the Hessenberg + Francis
// double-shift QR iteration of LAPACK dhseqr / EISPACK hqr2, so the oracle takes the RAW real
// Schur form from LAPACK (scipy.linalg.schur in oracle/refcpu.py, registered per matrix size
// through refcpu_set_raw_schur) and restates everything the reference does with it: block
// detection, ordering by ascending (Re, |Im|) with direct adjacent swaps (schur.hpp:47-85),
// standardization of the 2x2 blocks (schur.hpp:87-97), cleaning and the sanity checks
// (schur.hpp:163-170). A real Schur form is unique only up to rotations of its invariant
// subspaces, so T and Q are compared through their invariants, the slab solution directly.
struct RawSchur {
    std::vector<double> T, Q;  // row-major n x n
};
inline std::map<int, RawSchur>& raw_schur_registry() {
    static std::map<int, RawSchur> reg;
    return reg;
}

namespace schur_detail {
// schur.hpp:47-85 (direct swap): A11 X - X A22 = -A12 by PartialPivLU, [X; I] = QR by
// HouseholderQR (full Q), window rotated by Q, new strictly-lower part set to zero
inline void swap_adjacent_blocks(int n, std::vector<double>& t, std::vector<double>& q, int i, int p, int pq) {
    const int qs = pq - p, ns = p * qs;
    std::vector<double> sys(static_cast<size_t>(ns) * ns, 0.0), rhs(ns);
    for (int cc = 0; cc < qs; ++cc)
        for (int rr = 0; rr < p; ++rr) {
            const int eq = cc * p + rr;
            for (int k = 0; k < p; ++k) sys[eq * ns + cc * p + k] += t[(i + rr) * n + i + k];
            for (int k = 0; k < qs; ++k) sys[eq * ns + k * p + rr] -= t[(i + p + k) * n + i + p + cc];
            rhs[eq] = -t[(i + rr) * n + i + p + cc];
        }
    std::vector<double> xv(ns);
    DenseLu(sys, ns).solve(rhs.data(), xv.data());
    // Householder QR of stack = [X; I] (pq x qs), Q_full = H_0 ... H_{qs-1} (makeHouseholder:
    // beta = -sign(c0) ||x||, v = x / (c0 - beta) with v_0 = 1, tau = (beta - c0) / beta)
    std::vector<double> st(static_cast<size_t>(pq) * qs, 0.0), qr(static_cast<size_t>(pq) * pq, 0.0);
    for (int cc = 0; cc < qs; ++cc) {
        for (int rr = 0; rr < p; ++rr) st[rr * qs + cc] = xv[cc * p + rr];
        st[(p + cc) * qs + cc] = 1.0;
    }
    for (int k = 0; k < pq; ++k) qr[k * pq + k] = 1.0;
    for (int k = 0; k < qs; ++k) {
        double tail = 0.0;
        for (int r2 = k + 1; r2 < pq; ++r2) tail += st[r2 * qs + k] * st[r2 * qs + k];
        const double c0 = st[k * qs + k];
        if (tail == 0.0) continue;
        double beta = std::sqrt(c0 * c0 + tail);
        if (c0 >= 0.0) beta = -beta;
        std::vector<double> v(pq, 0.0);
        v[k] = 1.0;
        for (int r2 = k + 1; r2 < pq; ++r2) v[r2] = st[r2 * qs + k] / (c0 - beta);
        const double tau = (beta - c0) / beta;
        for (int c2 = 0; c2 < qs; ++c2) {  // st <- (I - tau v v^T) st
            double d = 0.0;
            for (int r2 = k; r2 < pq; ++r2) d += v[r2] * st[r2 * qs + c2];
            for (int r2 = k; r2 < pq; ++r2) st[r2 * qs + c2] -= tau * d * v[r2];
        }
        for (int r2 = 0; r2 < pq; ++r2) {  // qr <- qr (I - tau v v^T)
            double d = 0.0;
            for (int c2 = k; c2 < pq; ++c2) d += qr[r2 * pq + c2] * v[c2];
            for (int c2 = k; c2 < pq; ++c2) qr[r2 * pq + c2] -= tau * d * v[c2];
        }
    }
    auto right = [&](std::vector<double>& m) {
        for (int r2 = 0; r2 < n; ++r2) {
            std::vector<double> o(pq, 0.0);
            for (int c2 = 0; c2 < pq; ++c2)
                for (int k = 0; k < pq; ++k) o[c2] += m[r2 * n + i + k] * qr[k * pq + c2];
            for (int c2 = 0; c2 < pq; ++c2) m[r2 * n + i + c2] = o[c2];
        }
    };
    right(t);
    for (int c2 = 0; c2 < n; ++c2) {
        std::vector<double> o(pq, 0.0);
        for (int r2 = 0; r2 < pq; ++r2)
            for (int k = 0; k < pq; ++k) o[r2] += qr[k * pq + r2] * t[(i + k) * n + c2];
        for (int r2 = 0; r2 < pq; ++r2) t[(i + r2) * n + c2] = o[r2];
    }
    right(q);
    for (int rr = qs; rr < pq; ++rr)
        for (int cc = 0; cc < qs; ++cc) t[(i + rr) * n + i + cc] = 0.0;
    if (qs == 2 && std::abs(t[(i + 1) * n + i]) < 1e-13) t[(i + 1) * n + i] = 0.0;
    if (p == 2) {
        const int j = i + qs;
        if (std::abs(t[(j + 1) * n + j]) < 1e-13) t[(j + 1) * n + j] = 0.0;
    }
}
// schur.hpp:87-97
inline void standardize_block(int n, std::vector<double>& t, std::vector<double>& q, int i) {
    const double a = t[i * n + i], b = t[i * n + i + 1], c = t[(i + 1) * n + i], d = t[(i + 1) * n + i + 1];
    if (a == d) return;
    const double theta = 0.5 * std::atan2(a - d, b + c);
    const double cs = std::cos(theta), sn = std::sin(theta);
    auto right = [&](std::vector<double>& m) {  // m.middleCols(i, 2) = m.middleCols(i, 2) * [cs sn; -sn cs]
        for (int r2 = 0; r2 < n; ++r2) {
            const double x = m[r2 * n + i], y = m[r2 * n + i + 1];
            m[r2 * n + i] = x * cs - y * sn;
            m[r2 * n + i + 1] = x * sn + y * cs;
        }
    };
    right(t);
    for (int c2 = 0; c2 < n; ++c2) {  // rows <- g^T rows
        const double x = t[i * n + c2], y = t[(i + 1) * n + c2];
        t[i * n + c2] = cs * x - sn * y;
        t[(i + 1) * n + c2] = sn * x + cs * y;
    }
    right(q);
}
}  // namespace schur_detail

inline SchurForm real_schur(const TimeBasis& basis) {
    const int n = basis.n_nodes();
    SchurForm s;
    s.n = n;
    s.W.assign(n * n, 0.0);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) s.W[i * n + j] = (1.0 / basis.weights[i]) * basis.G_hat[i * n + j];
    s.Q.assign(n * n, 0.0);
    for (int i = 0; i < n; ++i) s.Q[i * n + i] = 1.0;
    if (n > 2) {
        const auto it = raw_schur_registry().find(n);
        if (it == raw_schur_registry().end())
            throw std::invalid_argument("real_schur: no raw Schur form registered for r = " + std::to_string(n - 1) +
                                        " (refcpu_set_raw_schur)");
        s.T = it->second.T;
        s.Q = it->second.Q;
        auto detect = [&]() {  // schur.hpp:117-129
            s.block_sizes.clear();
            s.block_starts.clear();
            int i = 0;
            while (i < n) {
                const bool two = (i + 1 < n) && std::abs(s.t(i + 1, i)) > 1e-12 * (std::abs(s.t(i, i)) + std::abs(s.t(i + 1, i + 1)));
                s.block_starts.push_back(i);
                s.block_sizes.push_back(two ? 2 : 1);
                i += two ? 2 : 1;
            }
        };
        detect();
        auto key_less = [&](int g1, int g2) {  // schur.hpp:133-137
            const auto e1 = s.block_eigenvalue(g1), e2 = s.block_eigenvalue(g2);
            if (std::abs(e1.real() - e2.real()) > 1e-12 * (1.0 + std::abs(e1.real()))) return e1.real() < e2.real();
            return std::abs(e1.imag()) < std::abs(e2.imag());
        };
        bool swapped = true;
        while (swapped) {
            swapped = false;
            for (int g = 0; g + 1 < s.n_blocks(); ++g)
                if (key_less(g + 1, g)) {
                    const int i = s.block_starts[g], p = s.block_sizes[g];
                    schur_detail::swap_adjacent_blocks(n, s.T, s.Q, i, p, p + s.block_sizes[g + 1]);
                    detect();
                    swapped = true;
                    break;
                }
        }
        for (int g = 0; g < s.n_blocks(); ++g)
            if (s.block_sizes[g] == 2) schur_detail::standardize_block(n, s.T, s.Q, s.block_starts[g]);
        for (int g = 0; g < s.n_blocks(); ++g) {
            const int i = s.block_starts[g], bs = s.block_sizes[g];
            for (int rr = i; rr < i + bs; ++rr)
                for (int cc = 0; cc < i; ++cc) s.T[rr * n + cc] = 0.0;
            if (bs == 1 && i + 1 < n) s.T[(i + 1) * n + i] = 0.0;
        }
        double orth = 0.0, resid = 0.0, wmax = 0.0;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                double qq = 0.0, rec = 0.0;
                for (int k = 0; k < n; ++k) {
                    qq += s.q(k, i) * s.q(k, j);
                    double tq = 0.0;
                    for (int l = 0; l < n; ++l) tq += s.t(k, l) * s.q(j, l);
                    rec += s.q(i, k) * tq;
                }
                orth = std::max(orth, std::abs(qq - (i == j ? 1.0 : 0.0)));
                resid = std::max(resid, std::abs(rec - s.W[i * n + j]));
                wmax = std::max(wmax, std::abs(s.W[i * n + j]));
            }
        if (orth > 1e-12) throw SolverError("real_schur: Q lost orthogonality");
        if (resid > 1e-10 * (1.0 + wmax)) throw SolverError("real_schur: factorization residual too large");
    } else if (n == 1) {
        s.T = s.W;
        s.block_sizes = {1};
        s.block_starts = {0};
    } else {
        double scale = 0.0;
        for (double v : s.W) scale = std::max(scale, std::abs(v));
        s.T.resize(4);
        for (int k = 0; k < 4; ++k) s.T[k] = s.W[k] / scale;
        const double p = 0.5 * (s.T[0] - s.T[3]);
        const double qd = p * p + s.T[2] * s.T[1];
        if (qd >= 0.0) throw SolverError("real_schur: dG(1) time operator must have a complex pair");
        for (int k = 0; k < 4; ++k) s.T[k] *= scale;
        s.block_sizes = {2};
        s.block_starts = {0};
        // standardize_block (schur.hpp:87-97)
        const double a = s.T[0], b = s.T[1], c = s.T[2], d = s.T[3];
        if (a != d) {
            const double theta = 0.5 * std::atan2(a - d, b + c);
            const double cs = std::cos(theta), sn = std::sin(theta);
            const double g[4] = {cs, sn, -sn, cs};
            auto rmul = [&](std::vector<double>& m) {  // m.middleCols(0,2) = m * g
                std::vector<double> o(4);
                for (int r = 0; r < 2; ++r)
                    for (int cc = 0; cc < 2; ++cc) o[r * 2 + cc] = m[r * 2 + 0] * g[0 * 2 + cc] + m[r * 2 + 1] * g[1 * 2 + cc];
                m = o;
            };
            auto lmul_t = [&](std::vector<double>& m) {  // m = g^T * m
                std::vector<double> o(4);
                for (int r = 0; r < 2; ++r)
                    for (int cc = 0; cc < 2; ++cc) o[r * 2 + cc] = g[0 * 2 + r] * m[0 * 2 + cc] + g[1 * 2 + r] * m[1 * 2 + cc];
                m = o;
            };
            rmul(s.T);
            lmul_t(s.T);
            rmul(s.Q);
        }
    }
    for (int g = 0; g < s.n_blocks(); ++g)
        if (s.block_eigenvalue(g).real() <= 0.0)
            throw SolverError("real_schur: nonpositive real part in a diagonal block");
    return s;
}

// ---------------------------------------------------------------------------
// fixed_stress.hpp:17-212
// ---------------------------------------------------------------------------
enum class InnerBackend { dense = 0, banded = 1 };

struct FixedStressConfig {
    double stab = -1.0;
    double tol = 1e-10;
    int max_sweeps = 200;
    int truncation_sweeps = 1;
    double resolve_stab(const MaterialParameters& m) const {
        const double s = stab < 0.0 ? m.biot_b * m.biot_b / m.k_dr : stab;
        if (!(s >= 0.0)) throw std::invalid_argument("fixed-stress: stabilization must be nonnegative");
        return s;
    }
};

// fixed_stress.hpp:38-60 (kappa empty = all ones, as in the slab solver, slab.hpp:162)
inline void apply_block_operator(const SpatialOperators& ops, const std::vector<double>& theta, int m, double tau,
                                 const double* x, double* y, const std::vector<double>& kappa = {}) {
    const int nt = ops.n_total(), nu = ops.n_u, nq = ops.n_q, np = ops.n_p;
    const double b = ops.mat.biot_b;
    std::vector<Vec> dp(m);
    for (int j = 0; j < m; ++j) dp[j] = apply_time_derivative_p(ops, x + j * nt, x + j * nt + nu + nq);
    Vec au(nu), ep(nu), mq(nq), bp(nq);
    for (int i = 0; i < m; ++i) {
        const double* u = x + i * nt;
        const double* q = x + i * nt + nu;
        const double* p = x + i * nt + nu + nq;
        const double w = tau * (kappa.empty() ? 1.0 : kappa[i]);
        ops.A.apply(u, au.data());
        ops.E.apply(p, ep.data());
        for (int k = 0; k < nu; ++k) y[i * nt + k] = w * (au[k] - b * ep[k]);
        ops.M_q.apply(q, mq.data());
        ops.B.apply(p, bp.data());
        for (int k = 0; k < nq; ++k) y[i * nt + nu + k] = w * (mq[k] + bp[k]);
        Vec qv(q, q + nq);
        Vec bt = ops.B.apply_transpose(qv);
        for (int k = 0; k < np; ++k) bt[k] = w * bt[k];
        for (int j = 0; j < m; ++j)
            if (theta[i * m + j] != 0.0)
                for (int k = 0; k < np; ++k) bt[k] += theta[i * m + j] * dp[j][k];
        for (int k = 0; k < np; ++k) y[i * nt + nu + nq + k] = bt[k];
    }
}

// Flow solve for one time component (m == 1) by exact elimination of the
// diagonal pressure block: S q = f_q - w B D^{-1} f_p with
// S = w M_q - w^2 B D^{-1} B^T (SPD), then p = D^{-1}(f_p - w B^T q), where
// D = -theta (1/M + stab) M_p. Faces are permuted into cell-row groups so S
// is banded. Exact replacement of the dense flow LU of
// fixed_stress.hpp:184-201 at sizes where the dense matrix cannot be formed.
class FlowSchurSolver : public InnerSolver {
public:
    FlowSchurSolver(const SpatialOperators& ops, int nx, int ny, double w, double theta, double inv_m, double stab)
        : nq_(ops.n_q), np_(ops.n_p), w_(w), B_(&ops.B) {
        dinv_.resize(np_);
        for (int c = 0; c < np_; ++c) dinv_[c] = 1.0 / (-(theta * (inv_m + stab)) * ops.m_p_diag[c]);
        std::vector<Triplet> ts;
        for (int i = 0; i < nq_; ++i)
            for (int k = ops.M_q.row_offsets[i]; k < ops.M_q.row_offsets[i + 1]; ++k)
                ts.push_back({i, ops.M_q.col_indices[k], w * ops.M_q.values[k]});
        // B^T by cells: list faces of each cell from B's rows
        std::vector<std::vector<std::pair<int, double>>> cell_faces(np_);
        for (int f = 0; f < nq_; ++f)
            for (int k = ops.B.row_offsets[f]; k < ops.B.row_offsets[f + 1]; ++k)
                cell_faces[ops.B.col_indices[k]].push_back({f, ops.B.values[k]});
        for (int c = 0; c < np_; ++c)
            for (auto& a : cell_faces[c])
                for (auto& bb : cell_faces[c]) ts.push_back({a.first, bb.first, -(w * a.second) * (w * bb.second) * dinv_[c]});
        const SparseMatrix S = csr_from_triplets(nq_, nq_, ts);
        std::vector<int> perm = ops.face_band_perm;
        if (perm.empty()) {
            perm.reserve(nq_);
            for (int j = 0; j <= ny; ++j) {
                for (int i = 0; i < nx; ++i) perm.push_back(j * nx + i);
                if (j < ny)
                    for (int i = 0; i <= nx; ++i) perm.push_back(nx * (ny + 1) + i * ny + j);
            }
        }
        chol_ = std::make_unique<BandCholesky>(S, perm);
    }
    int size() const override { return nq_ + np_; }
    void solve(const double* f, double* x) const override {
        Vec rq(f, f + nq_);
        for (int fi = 0; fi < nq_; ++fi)
            for (int k = B_->row_offsets[fi]; k < B_->row_offsets[fi + 1]; ++k)
                rq[fi] -= w_ * B_->values[k] * (dinv_[B_->col_indices[k]] * f[nq_ + B_->col_indices[k]]);
        chol_->solve(rq.data(), x);
        Vec btq(np_, 0.0);
        for (int fi = 0; fi < nq_; ++fi)
            for (int k = B_->row_offsets[fi]; k < B_->row_offsets[fi + 1]; ++k)
                btq[B_->col_indices[k]] += B_->values[k] * x[fi];
        for (int c = 0; c < np_; ++c) x[nq_ + c] = dinv_[c] * (f[nq_ + c] - w_ * btq[c]);
    }

private:
    int nq_, np_;
    double w_;
    const SparseMatrix* B_;
    Vec dinv_;
    std::unique_ptr<BandCholesky> chol_;
};

inline std::vector<double> dense_of(const SparseMatrix& s) {
    std::vector<double> d(static_cast<size_t>(s.rows) * s.cols, 0.0);
    for (int i = 0; i < s.rows; ++i)
        for (int k = s.row_offsets[i]; k < s.row_offsets[i + 1]; ++k) d[static_cast<size_t>(i) * s.cols + s.col_indices[k]] = s.values[k];
    return d;
}

// Shared exact A solve (DenseLu(ops.A.to_dense()) at slab.hpp:155).
inline std::shared_ptr<InnerSolver> make_a_solver(const SpatialOperators& ops, InnerBackend be) {
    if (be == InnerBackend::dense) return std::make_shared<DenseLu>(dense_of(ops.A), ops.n_u);
    return std::make_shared<BandCholesky>(ops.A, std::vector<int>{});
}

class FixedStressSolver {
public:
    FixedStressSolver(const SpatialOperators& ops, std::vector<double> theta, int m, double tau, double stab,
                      std::shared_ptr<InnerSolver> a_solver, InnerBackend be, int nx, int ny,
                      std::vector<double> kappa = {})
        : ops_(&ops), theta_(std::move(theta)), m_(m), tau_(tau), stab_(stab), a_(std::move(a_solver)), be_(be),
          nx_(nx), ny_(ny), kappa_(kappa.empty() ? std::vector<double>(m, 1.0) : std::move(kappa)) {
        if (static_cast<int>(kappa_.size()) != m_ || static_cast<int>(theta_.size()) != m_ * m_)
            throw std::invalid_argument("FixedStressSolver: weight dimensions mismatch");
        if (!(tau_ > 0.0)) throw std::invalid_argument("FixedStressSolver: tau must be positive");
    }
    int block_size() const { return m_ * ops_->n_total(); }
    void apply_block(const double* x, double* y) const { apply_block_operator(*ops_, theta_, m_, tau_, x, y, kappa_); }

    // fixed_stress.hpp:109-139
    Vec sweep(const Vec& x, const double* rhs) const {
        ensure_flow();
        const int nt = ops_->n_total(), nu = ops_->n_u, nq = ops_->n_q, np = ops_->n_p;
        const double b = ops_->mat.biot_b;
        Vec fr(static_cast<size_t>(m_) * (nq + np));
        for (int i = 0; i < m_; ++i) {
            for (int k = 0; k < nq; ++k) fr[i * nq + k] = rhs[i * nt + nu + k];
            Vec pr(rhs + i * nt + nu + nq, rhs + i * nt + nu + nq + np);
            for (int j = 0; j < m_; ++j) {
                const double th = theta_[i * m_ + j];
                if (th == 0.0) continue;
                Vec uj(x.begin() + j * nt, x.begin() + j * nt + nu);
                const Vec et = ops_->E.apply_transpose(uj);
                for (int k = 0; k < np; ++k)
                    pr[k] += th * (b * et[k] - stab_ * (ops_->m_p_diag[k] * x[j * nt + nu + nq + k]));
            }
            for (int k = 0; k < np; ++k) fr[m_ * nq + i * np + k] = pr[k];
        }
        Vec fsol(fr.size());
        flow_->solve(fr.data(), fsol.data());
        Vec xn(static_cast<size_t>(m_) * nt);
        Vec ep(nu), mech(nu);
        for (int i = 0; i < m_; ++i) {
            const double* p_new = &fsol[m_ * nq + i * np];
            const double* q_new = &fsol[i * nq];
            const double w = tau_ * kappa_[i];
            ops_->E.apply(p_new, ep.data());
            for (int k = 0; k < nu; ++k) mech[k] = rhs[i * nt + k] / w + b * ep[k];
            a_->solve(mech.data(), &xn[i * nt]);
            for (int k = 0; k < nq; ++k) xn[i * nt + nu + k] = q_new[k];
            for (int k = 0; k < np; ++k) xn[i * nt + nu + nq + k] = p_new[k];
        }
        return xn;
    }
    // fixed_stress.hpp:177-181
    void precondition(const double* residual, double* out, int sweeps) const {
        Vec x(block_size(), 0.0);
        for (int k = 0; k < sweeps; ++k) x = sweep(x, residual);
        std::copy(x.begin(), x.end(), out);
    }
    // fixed_stress.hpp:144-172
    Vec solve(const Vec& rhs, const FixedStressConfig& cfg, const Vec& x0, SolverReport& rep) const {
        rep = SolverReport{};
        const double rnorm = norm(rhs);
        Vec x = x0.empty() ? Vec(block_size(), 0.0) : x0;
        Vec ax(block_size()), r(block_size());
        auto resid = [&]() {
            apply_block(x.data(), ax.data());
            for (int i = 0; i < block_size(); ++i) r[i] = rhs[i] - ax[i];
            return norm(r);
        };
        if (rnorm <= 1e-14) {
            rep.converged = true;
            rep.residual_history = {resid()};
            rep.final_relative_residual = 0.0;
            return Vec(block_size(), 0.0);
        }
        double res = resid();
        rep.residual_history.push_back(res);
        for (int k = 0; k < cfg.max_sweeps; ++k) {
            x = sweep(x, rhs.data());
            ++rep.iterations;
            res = resid();
            rep.residual_history.push_back(res);
            if (res / rnorm <= cfg.tol) {
                rep.converged = true;
                break;
            }
        }
        rep.final_relative_residual = res / rnorm;
        return x;
    }

private:
    // fixed_stress.hpp:184-201, built lazily (only sweeps need it).
    void ensure_flow() const {
        if (flow_) return;
        const int nq = ops_->n_q, np = ops_->n_p;
        const double inv_m = 1.0 / ops_->mat.biot_m;
        if (be_ == InnerBackend::banded && m_ == 1) {
            flow_ = std::make_shared<FlowSchurSolver>(*ops_, nx_, ny_, tau_ * kappa_[0], theta_[0], inv_m, stab_);
            return;
        }
        const int nf = m_ * (nq + np);
        std::vector<double> f(static_cast<size_t>(nf) * nf, 0.0);
        auto F = [&](int i, int j) -> double& { return f[static_cast<size_t>(i) * nf + j]; };
        for (int i = 0; i < m_; ++i) {
            const double w = tau_ * kappa_[i];
            for (int r = 0; r < nq; ++r)
                for (int k = ops_->M_q.row_offsets[r]; k < ops_->M_q.row_offsets[r + 1]; ++k)
                    F(i * nq + r, i * nq + ops_->M_q.col_indices[k]) = w * ops_->M_q.values[k];
            for (int r = 0; r < nq; ++r)
                for (int k = ops_->B.row_offsets[r]; k < ops_->B.row_offsets[r + 1]; ++k) {
                    const int c = ops_->B.col_indices[k];
                    F(i * nq + r, m_ * nq + i * np + c) = w * ops_->B.values[k];
                    F(m_ * nq + i * np + c, i * nq + r) = w * ops_->B.values[k];
                }
            for (int j = 0; j < m_; ++j)
                if (theta_[i * m_ + j] != 0.0)
                    for (int c = 0; c < np; ++c)
                        F(m_ * nq + i * np + c, m_ * nq + j * np + c) -= theta_[i * m_ + j] * (inv_m + stab_) * ops_->m_p_diag[c];
        }
        flow_ = std::make_shared<DenseLu>(std::move(f), nf);
    }

    const SpatialOperators* ops_;
    std::vector<double> theta_;
    int m_;
    double tau_, stab_;
    std::shared_ptr<InnerSolver> a_;
    InnerBackend be_;
    int nx_, ny_;
    std::vector<double> kappa_;
    mutable std::shared_ptr<InnerSolver> flow_;
};

// ---------------------------------------------------------------------------
// slab.hpp:31-274
// ---------------------------------------------------------------------------
struct SlabSystem {
    double tau = 0.0;
    std::vector<Vec> rhs;  // stacked (u,q,p) per time index
};

inline Vec stack_fields(const SpatialOperators& ops, const FieldVecs& f) {
    Vec x(ops.n_total());
    std::copy(f.u.begin(), f.u.end(), x.begin());
    std::copy(f.q.begin(), f.q.end(), x.begin() + ops.n_u);
    std::copy(f.p.begin(), f.p.end(), x.begin() + ops.n_u + ops.n_q);
    return x;
}

// slab.hpp:58-87
inline SlabSystem build_slab_system(const SpatialOperators& ops, const TimeBasis& basis, double tau,
                                    const std::vector<FieldVecs>& nodal_rhs, const Vec& jump_u, const Vec& jump_p) {
    if (!(tau > 0.0)) throw std::invalid_argument("build_slab_system: tau must be positive");
    SlabSystem sys;
    sys.tau = tau;
    const Vec djump = apply_time_derivative_p(ops, jump_u.data(), jump_p.data());
    sys.rhs.resize(basis.n_nodes());
    for (int i = 0; i < basis.n_nodes(); ++i) {
        Vec r = stack_fields(ops, nodal_rhs[i]);
        const double s = tau * basis.weights[i];
        for (double& v : r) v = s * v;
        for (int c = 0; c < ops.n_p; ++c) r[ops.n_u + ops.n_q + c] += basis.phi_at0[i] * djump[c];
        sys.rhs[i] = std::move(r);
    }
    return sys;
}

// slab.hpp:283-318 : discrete local mass balance of a converged slab. For
// each cell: sum over the time test functions i of
//   storage_i = sum_j G_hat(i,j) D(u_j, p_j)   (j ascending, zero entries skipped)
//   flux_i    = (tau w_i) B^T q_i
//   src_i     = p-rows of rhs_i
// residual += (storage + flux) - src, scale += (|storage| + |flux|) + |src|;
// returns |residual| per cell and scale = max over cells.
struct MassResidual {
    Vec residual;
    double scale = 0.0;
};
inline MassResidual local_mass_residual(const SpatialOperators& ops, const TimeBasis& basis, double tau,
                                        const std::vector<Vec>& rhs, const std::vector<const double*>& comps) {
    const int n = basis.n_nodes(), np = ops.n_p, nu = ops.n_u, nq = ops.n_q;
    std::vector<Vec> dp(n), kp(n);
    for (int j = 0; j < n; ++j) {
        dp[j] = apply_time_derivative_p(ops, comps[j], comps[j] + nu + nq);
        kp[j] = ops.B.apply_transpose(Vec(comps[j] + nu, comps[j] + nu + nq));
    }
    MassResidual out;
    out.residual.assign(np, 0.0);
    Vec scale(np, 0.0);
    for (int i = 0; i < n; ++i) {
        Vec storage(np, 0.0);
        for (int j = 0; j < n; ++j) {
            const double g = basis.G_hat[i * n + j];
            if (g != 0.0)
                for (int c = 0; c < np; ++c) storage[c] += g * dp[j][c];
        }
        const double s = tau * basis.weights[i];
        for (int c = 0; c < np; ++c) {
            const double flux = s * kp[i][c];
            const double src = rhs[i][nu + nq + c];
            out.residual[c] += (storage[c] + flux) - src;
            scale[c] += (std::fabs(storage[c]) + std::fabs(flux)) + std::fabs(src);
        }
    }
    for (double& v : out.residual) v = std::fabs(v);
    for (double v : scale) out.scale = std::max(out.scale, v);
    return out;
}

struct BlockReport {
    int block_index = 0, block_size = 1, gmres_iterations = 0, fs_sweeps = 0;
    SolverReport report;
};

struct SolveOptions {
    GmresOptions gmres;
    FixedStressConfig fs;
    InnerBackend backend = InnerBackend::dense;
    bool flexible = false;  // gmres (false, as slab.hpp:227) or gmres_flexible
};

class SlabSolver {  // slab.hpp:133-274, BlockSolverKind::gmres_fs
public:
    SlabSolver(const SpatialOperators& ops, const TimeBasis& basis, const SchurForm& schur, double tau,
               SolveOptions opt, int nx, int ny, std::shared_ptr<InnerSolver> a_solver = nullptr)
        : ops_(&ops), basis_(&basis), schur_(&schur), tau_(tau), opt_(opt) {
        a_ = a_solver ? a_solver : make_a_solver(ops, opt.backend);
        const double stab = opt_.fs.resolve_stab(ops.mat);
        for (int g = 0; g < schur.n_blocks(); ++g) {
            const int m = schur.block_sizes[g], i0 = schur.block_starts[g];
            std::vector<double> theta(m * m);
            for (int a = 0; a < m; ++a)
                for (int c = 0; c < m; ++c) theta[a * m + c] = schur.t(i0 + a, i0 + c);
            fs_block_.push_back(std::make_unique<FixedStressSolver>(ops, theta, m, tau, stab, a_, opt.backend, nx, ny));
            fs_pre_.push_back(std::make_unique<FixedStressSolver>(ops, std::vector<double>{theta[0]}, 1, tau, stab, a_,
                                                                  opt.backend, nx, ny));
        }
    }

    // Solve of one transformed diagonal block g with right-hand side rhs
    // (slab.hpp:456-473). Throws SolverError on non-convergence.
    Vec solve_block(int g, const Vec& rhs, BlockReport& br) const {
        const int m = schur_->block_sizes[g], nt = ops_->n_total();
        const FixedStressSolver& fsb = *fs_block_[g];
        const FixedStressSolver& fsp = *fs_pre_[g];
        const int sweeps = opt_.fs.truncation_sweeps;
        LinOp op = [&](const double* v, double* out) { fsb.apply_block(v, out); };
        LinOp pre = [&](const double* v, double* out) {
            for (int bi = 0; bi < m; ++bi) fsp.precondition(v + bi * nt, out + bi * nt, sweeps);
        };
        SolverReport rep;
        Vec x = gmres_impl(op, pre, rhs, opt_.gmres, opt_.flexible, rep);
        if (!rep.converged) {
            char buf[64];
            std::snprintf(buf, sizeof(buf), "%f", rep.final_relative_residual);
            throw SolverError("slab block " + std::to_string(g) + ": GMRES did not converge (rel res " + buf + ")");
        }
        br.block_index = g;
        br.block_size = m;
        br.gmres_iterations = rep.iterations;
        br.fs_sweeps = sweeps;
        br.report = rep;
        return x;
    }

    // slab.hpp:179-255
    std::vector<FieldVecs> solve(const SlabSystem& sys, std::vector<BlockReport>& reports) const {
        const SchurForm& s = *schur_;
        const int n = basis_->n_nodes(), nt = ops_->n_total();
        const int nu = ops_->n_u, nq = ops_->n_q, np = ops_->n_p;
        std::vector<Vec> shat(n, Vec(nt, 0.0));
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                const double qji = s.q(j, i), wj = basis_->weights[j];
                for (int k = 0; k < nt; ++k) shat[i][k] += qji * (sys.rhs[j][k] / wj);
            }
        std::vector<Vec> y(n), dp(n);
        reports.clear();
        for (int g = s.n_blocks() - 1; g >= 0; --g) {
            const int m = s.block_sizes[g], i0 = s.block_starts[g];
            Vec rhs(static_cast<size_t>(m) * nt);
            for (int bi = 0; bi < m; ++bi) {
                Vec r = shat[i0 + bi];
                for (int j = i0 + m; j < n; ++j)
                    if (s.t(i0 + bi, j) != 0.0)
                        for (int c = 0; c < np; ++c) r[nu + nq + c] -= s.t(i0 + bi, j) * dp[j][c];
                std::copy(r.begin(), r.end(), rhs.begin() + bi * nt);
            }
            BlockReport br;
            const Vec sol = solve_block(g, rhs, br);
            for (int bi = 0; bi < m; ++bi) {
                y[i0 + bi] = Vec(sol.begin() + bi * nt, sol.begin() + (bi + 1) * nt);
                dp[i0 + bi] = apply_time_derivative_p(*ops_, y[i0 + bi].data(), y[i0 + bi].data() + nu + nq);
            }
            reports.push_back(br);
        }
        std::vector<FieldVecs> out(n);
        for (int i = 0; i < n; ++i) {
            Vec xi(nt, 0.0);
            for (int j = 0; j < n; ++j)
                for (int k = 0; k < nt; ++k) xi[k] += s.q(i, j) * y[j][k];
            out[i].u.assign(xi.begin(), xi.begin() + nu);
            out[i].q.assign(xi.begin() + nu, xi.begin() + nu + nq);
            out[i].p.assign(xi.begin() + nu + nq, xi.end());
        }
        std::reverse(reports.begin(), reports.end());
        return out;
    }

    const FixedStressSolver& block(int g) const { return *fs_block_[g]; }
    const FixedStressSolver& pre(int g) const { return *fs_pre_[g]; }

private:
    const SpatialOperators* ops_;
    const TimeBasis* basis_;
    const SchurForm* schur_;
    double tau_;
    SolveOptions opt_;
    std::shared_ptr<InnerSolver> a_;
    std::vector<std::unique_ptr<FixedStressSolver>> fs_block_, fs_pre_;
};

// Canonical assembled space-time operator of one transformed block: the
// matrix the reference's own direct block path forms densely at
// slab.hpp:146-153,  mat(bi,bj) = T(bi,bj) * D  [+ tau * K if bi == bj],
// with D = dense_time_derivative (slab.hpp:106-111) and
// K = dense_stationary (slab.hpp:92-103), held as CSR over the stored entries
// of the spatial blocks (stored zeros included). Layout
// [u_0 q_0 p_0 | u_1 q_1 p_1 | ...]; entry values (no entry has both a D and
// a K part, so each is one product chain, bit-defined):
//   u-rows of component i : tau*a on u_i,  tau*((-b)*e) on p_i
//   q-rows               : tau*mq on q_i, tau*bv on p_i
//   p-rows               : tau*bv on q_i (B^T),
//                          T_ij*((-b)*e) on u_j, T_ij*((-(1/M))*m_p) on p_j  (T_ij != 0)
inline SparseMatrix build_spacetime_csr(const SpatialOperators& ops, const std::vector<double>& theta, int m,
                                        double tau) {
    const int nt = ops.n_total(), nu = ops.n_u, nq = ops.n_q;
    const double mb = -ops.mat.biot_b, minv = -(1.0 / ops.mat.biot_m);
    std::vector<Triplet> t;
    t.reserve(static_cast<size_t>(m) * (ops.A.nnz() + 2 * ops.E.nnz() + ops.M_q.nnz() + 2 * ops.B.nnz()) +
              static_cast<size_t>(m) * m * (ops.E.nnz() + ops.n_p));
    for (int i = 0; i < m; ++i) {
        const int r0 = i * nt;
        for (int r = 0; r < nu; ++r) {
            for (int k = ops.A.row_offsets[r]; k < ops.A.row_offsets[r + 1]; ++k)
                t.push_back({r0 + r, r0 + ops.A.col_indices[k], tau * ops.A.values[k]});
            for (int k = ops.E.row_offsets[r]; k < ops.E.row_offsets[r + 1]; ++k)
                t.push_back({r0 + r, r0 + nu + nq + ops.E.col_indices[k], tau * (mb * ops.E.values[k])});
        }
        for (int r = 0; r < nq; ++r) {
            for (int k = ops.M_q.row_offsets[r]; k < ops.M_q.row_offsets[r + 1]; ++k)
                t.push_back({r0 + nu + r, r0 + nu + ops.M_q.col_indices[k], tau * ops.M_q.values[k]});
            for (int k = ops.B.row_offsets[r]; k < ops.B.row_offsets[r + 1]; ++k) {
                t.push_back({r0 + nu + r, r0 + nu + nq + ops.B.col_indices[k], tau * ops.B.values[k]});
                t.push_back({r0 + nu + nq + ops.B.col_indices[k], r0 + nu + r, tau * ops.B.values[k]});
            }
        }
        for (int j = 0; j < m; ++j) {
            const double th = theta[i * m + j];
            if (th == 0.0) continue;
            for (int r = 0; r < nu; ++r)
                for (int k = ops.E.row_offsets[r]; k < ops.E.row_offsets[r + 1]; ++k)
                    t.push_back({r0 + nu + nq + ops.E.col_indices[k], j * nt + r, th * (mb * ops.E.values[k])});
            for (int c = 0; c < ops.n_p; ++c)
                t.push_back({r0 + nu + nq + c, j * nt + nu + nq + c, th * (minv * ops.m_p_diag[c])});
        }
    }
    return csr_from_triplets(m * nt, m * nt, t);
}

}  // namespace refcpu
