// Host-side dG(r) time constants (time_basis.hpp:47-182) and the ordered real Schur form
// of W = M_hat^{-1} G_hat (schur.hpp:101-173). These are a handful of scalars computed once
// per run. r <= 1 follows the reference's numerical route exactly (Radau roots by bisection
// + Newton, weights by Gauss quadrature of the barycentric basis; for a 2x2 W with a complex
// pair Eigen's RealSchur returns W itself, then standardize_block), so that T, Q and the
// weights agree bit-for-bit with it. r >= 2 (kMaxTimeDegree below) uses a Hessenberg
// reduction + Francis double-shift QR iteration here where the reference calls
// Eigen::RealSchur, followed by the reference's own post-processing: blocks ordered by
// ascending (Re, |Im|) with direct adjacent swaps (schur.hpp:47-85), 2x2 blocks rotated to
// equal diagonal entries (schur.hpp:87-97), the strictly lower part cleaned, and the same
// sanity checks (schur.hpp:163-170). A real Schur form is unique only up to the signs /
// rotations of its invariant subspaces; the slab solution does not depend on that choice.
#pragma once

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <utility>
#include <vector>

namespace pdg {

constexpr int kMaxTimeDegree = 5;  // the reference allows 10 (time_basis.hpp:42); device buffers are sized for 6 nodes

struct TimeConsts {
    int r = 0, n = 1;
    std::vector<double> nodes, weights, phi0, G, T, Q;  // n, n, n, n*n (row-major)
    std::vector<int> block_sizes, block_starts;         // diagonal blocks of T (1x1 real, 2x2 complex pair)
    int n_blocks() const { return static_cast<int>(block_sizes.size()); }
};

namespace schur_detail {

using Mat = std::vector<double>;  // row-major n x n

// Hessenberg reduction by Householder reflectors, H = Z^T A Z (Z accumulated)
inline void hessenberg(int n, Mat& a, Mat& z) {
    for (int k = 0; k + 2 < n; ++k) {
        double alpha = 0.0;
        for (int i = k + 1; i < n; ++i) alpha += a[i * n + k] * a[i * n + k];
        alpha = std::sqrt(alpha);
        if (alpha == 0.0) continue;
        std::vector<double> v(n, 0.0);
        const double x0 = a[(k + 1) * n + k];
        const double beta = x0 >= 0.0 ? -alpha : alpha;
        v[k + 1] = x0 - beta;
        for (int i = k + 2; i < n; ++i) v[i] = a[i * n + k];
        double vn = 0.0;
        for (int i = k + 1; i < n; ++i) vn += v[i] * v[i];
        if (vn == 0.0) continue;
        // A <- (I - 2 v v^T / vn) A (I - 2 v v^T / vn)
        for (int j = 0; j < n; ++j) {
            double d = 0.0;
            for (int i = k + 1; i < n; ++i) d += v[i] * a[i * n + j];
            d = 2.0 * d / vn;
            for (int i = k + 1; i < n; ++i) a[i * n + j] -= d * v[i];
        }
        for (int i = 0; i < n; ++i) {
            double d = 0.0;
            for (int j = k + 1; j < n; ++j) d += a[i * n + j] * v[j];
            d = 2.0 * d / vn;
            for (int j = k + 1; j < n; ++j) a[i * n + j] -= d * v[j];
            double e = 0.0;
            for (int j = k + 1; j < n; ++j) e += z[i * n + j] * v[j];
            e = 2.0 * e / vn;
            for (int j = k + 1; j < n; ++j) z[i * n + j] -= e * v[j];
        }
        for (int i = k + 2; i < n; ++i) a[i * n + k] = 0.0;
    }
}

// apply the reflector I - 2 v v^T / (v^T v) on rows / columns [k, k + nv) of H (both sides) and Z
inline void reflect(int n, Mat& h, Mat& z, int k, int nv, const double* v) {
    double vn = 0.0;
    for (int i = 0; i < nv; ++i) vn += v[i] * v[i];
    if (vn == 0.0) return;
    for (int j = 0; j < n; ++j) {
        double d = 0.0;
        for (int i = 0; i < nv; ++i) d += v[i] * h[(k + i) * n + j];
        d = 2.0 * d / vn;
        for (int i = 0; i < nv; ++i) h[(k + i) * n + j] -= d * v[i];
    }
    for (int i = 0; i < n; ++i) {
        double d = 0.0, e = 0.0;
        for (int j = 0; j < nv; ++j) {
            d += h[i * n + k + j] * v[j];
            e += z[i * n + k + j] * v[j];
        }
        d = 2.0 * d / vn;
        e = 2.0 * e / vn;
        for (int j = 0; j < nv; ++j) {
            h[i * n + k + j] -= d * v[j];
            z[i * n + k + j] -= e * v[j];
        }
    }
}

// Real Schur form of a (n x n): on return a = T quasi-upper-triangular, z = Q, Q T Q^T = input.
// Francis implicit double-shift QR on the Hessenberg form with deflation from the bottom;
// a deflated 2x2 block with real eigenvalues is split by a rotation.
inline bool real_schur_qr(int n, Mat& a, Mat& z, int max_iter) {
    z.assign(n * n, 0.0);
    for (int i = 0; i < n; ++i) z[i * n + i] = 1.0;
    hessenberg(n, a, z);
    double norm = 0.0;
    for (double v : a) norm = std::max(norm, std::abs(v));
    if (norm == 0.0) return true;
    const double eps = 2.220446049250313e-16;
    int hi = n - 1, iter = 0, total = 0;
    while (hi >= 0) {
        // the active unreduced block [lo, hi]
        int lo = hi;
        while (lo > 0) {
            double sc = std::abs(a[(lo - 1) * n + lo - 1]) + std::abs(a[lo * n + lo]);
            if (sc == 0.0) sc = norm;
            if (std::abs(a[lo * n + lo - 1]) <= eps * sc) {
                a[lo * n + lo - 1] = 0.0;
                break;
            }
            --lo;
        }
        if (lo == hi) {  // 1x1 block
            --hi;
            iter = 0;
            continue;
        }
        if (lo == hi - 1) {  // 2x2 block: split it if its eigenvalues are real
            const double p = 0.5 * (a[lo * n + lo] - a[hi * n + hi]);
            const double q = p * p + a[hi * n + lo] * a[lo * n + hi];
            if (q >= 0.0) {
                // rotation that makes the block upper triangular: first column = eigenvector of
                // the eigenvalue nearer to a(hi,hi)
                const double zr = p >= 0.0 ? p + std::sqrt(q) : p - std::sqrt(q);
                // eigenvector direction (zr, a(hi,lo)) of the block [a b; c d] for the eigenvalue d + zr
                double c0 = zr, s0 = a[hi * n + lo];
                const double nr = std::hypot(c0, s0);
                if (nr > 0.0) {
                    c0 /= nr;
                    s0 /= nr;
                    // G = [c0 -s0; s0 c0]: columns lo, hi <- [lo hi] G, rows <- G^T [lo; hi]
                    for (int j = 0; j < n; ++j) {
                        const double x = a[lo * n + j], y = a[hi * n + j];
                        a[lo * n + j] = c0 * x + s0 * y;
                        a[hi * n + j] = -s0 * x + c0 * y;
                    }
                    for (int i = 0; i < n; ++i) {
                        const double x = a[i * n + lo], y = a[i * n + hi];
                        a[i * n + lo] = c0 * x + s0 * y;
                        a[i * n + hi] = -s0 * x + c0 * y;
                        const double u = z[i * n + lo], w = z[i * n + hi];
                        z[i * n + lo] = c0 * u + s0 * w;
                        z[i * n + hi] = -s0 * u + c0 * w;
                    }
                }
                a[hi * n + lo] = 0.0;
            }
            hi -= 2;
            iter = 0;
            continue;
        }
        if (++total > max_iter) return false;
        ++iter;
        // shifts from the trailing 2x2 block (exceptional shifts every 10 stalled iterations)
        double s = a[(hi - 1) * n + hi - 1] + a[hi * n + hi];
        double t = a[(hi - 1) * n + hi - 1] * a[hi * n + hi] - a[(hi - 1) * n + hi] * a[hi * n + hi - 1];
        if (iter % 10 == 0) {
            const double w = std::abs(a[hi * n + hi - 1]) + std::abs(a[(hi - 1) * n + hi - 2]);
            s = 1.5 * w;
            t = w * w;
        }
        double x = a[lo * n + lo] * a[lo * n + lo] + a[lo * n + lo + 1] * a[(lo + 1) * n + lo] - s * a[lo * n + lo] + t;
        double y = a[(lo + 1) * n + lo] * (a[lo * n + lo] + a[(lo + 1) * n + lo + 1] - s);
        double zz = a[(lo + 1) * n + lo] * a[(lo + 2) * n + lo + 1];
        for (int k = lo; k <= hi - 2; ++k) {
            // reflector that maps (x, y, zz) to a multiple of e1
            const double al = std::sqrt(x * x + y * y + zz * zz);
            if (al != 0.0) {
                double v[3] = {x + (x >= 0.0 ? al : -al), y, zz};
                reflect(n, a, z, k, 3, v);
            }
            if (k > lo) {
                a[(k + 1) * n + k - 1] = 0.0;
                a[(k + 2) * n + k - 1] = 0.0;
            }
            x = a[(k + 1) * n + k];
            y = a[(k + 2) * n + k];
            if (k < hi - 2) zz = a[(k + 3) * n + k];
        }
        {
            const double al = std::sqrt(x * x + y * y);
            if (al != 0.0) {
                double v[2] = {x + (x >= 0.0 ? al : -al), y};
                reflect(n, a, z, hi - 1, 2, v);
            }
            if (hi - 1 > lo) a[hi * n + hi - 2] = 0.0;
        }
    }
    return true;
}

// dense solve of a small system by Gaussian elimination with partial pivoting
inline std::vector<double> small_solve(int n, Mat a, std::vector<double> b) {
    for (int k = 0; k < n; ++k) {
        int piv = k;
        for (int i = k + 1; i < n; ++i)
            if (std::abs(a[i * n + k]) > std::abs(a[piv * n + k])) piv = i;
        if (piv != k) {
            for (int j = 0; j < n; ++j) std::swap(a[k * n + j], a[piv * n + j]);
            std::swap(b[k], b[piv]);
        }
        for (int i = k + 1; i < n; ++i) {
            const double f = a[i * n + k] / a[k * n + k];
            for (int j = k; j < n; ++j) a[i * n + j] -= f * a[k * n + j];
            b[i] -= f * b[k];
        }
    }
    for (int i = n - 1; i >= 0; --i) {
        for (int j = i + 1; j < n; ++j) b[i] -= a[i * n + j] * b[j];
        b[i] /= a[i * n + i];
    }
    return b;
}

// schur.hpp:47-85: swap the adjacent diagonal blocks at i (sizes p, then pq - p) by the direct
// method: A11 X - X A22 = -A12, orthonormal basis of [X; I] completed to a rotation of the window
inline void swap_adjacent_blocks(int n, Mat& t, Mat& q, int i, int p, int pq) {
    const int qs = pq - p;
    Mat sys(p * qs * p * qs, 0.0);
    std::vector<double> rhs(p * qs);
    const int ns = p * qs;
    for (int cc = 0; cc < qs; ++cc)
        for (int rr = 0; rr < p; ++rr) {
            const int eq = cc * p + rr;
            for (int k = 0; k < p; ++k) sys[eq * ns + cc * p + k] += t[(i + rr) * n + i + k];
            for (int k = 0; k < qs; ++k) sys[eq * ns + k * p + rr] -= t[(i + p + k) * n + i + p + cc];
            rhs[eq] = -t[(i + rr) * n + i + p + cc];
        }
    const std::vector<double> xv = small_solve(ns, sys, rhs);
    // full QR of the (pq x qs) matrix [X; I] by Householder reflectors; qr = H_0 H_1 ... (pq x pq)
    Mat st(pq * qs, 0.0), qr(pq * pq, 0.0);
    for (int cc = 0; cc < qs; ++cc) {
        for (int rr = 0; rr < p; ++rr) st[rr * qs + cc] = xv[cc * p + rr];
        st[(p + cc) * qs + cc] = 1.0;
    }
    for (int k = 0; k < pq; ++k) qr[k * pq + k] = 1.0;
    for (int k = 0; k < qs; ++k) {
        double al = 0.0;
        for (int r2 = k; r2 < pq; ++r2) al += st[r2 * qs + k] * st[r2 * qs + k];
        al = std::sqrt(al);
        if (al == 0.0) continue;
        std::vector<double> v(pq, 0.0);
        v[k] = st[k * qs + k] + (st[k * qs + k] >= 0.0 ? al : -al);
        for (int r2 = k + 1; r2 < pq; ++r2) v[r2] = st[r2 * qs + k];
        double vn = 0.0;
        for (int r2 = k; r2 < pq; ++r2) vn += v[r2] * v[r2];
        for (int c2 = 0; c2 < qs; ++c2) {
            double d = 0.0;
            for (int r2 = k; r2 < pq; ++r2) d += v[r2] * st[r2 * qs + c2];
            d = 2.0 * d / vn;
            for (int r2 = k; r2 < pq; ++r2) st[r2 * qs + c2] -= d * v[r2];
        }
        for (int r2 = 0; r2 < pq; ++r2) {  // qr <- qr H_k
            double d = 0.0;
            for (int c2 = k; c2 < pq; ++c2) d += qr[r2 * pq + c2] * v[c2];
            d = 2.0 * d / vn;
            for (int c2 = k; c2 < pq; ++c2) qr[r2 * pq + c2] -= d * v[c2];
        }
    }
    auto cols_times = [&](Mat& m) {  // m.middleCols(i, pq) = m.middleCols(i, pq) * qr
        for (int r2 = 0; r2 < n; ++r2) {
            std::vector<double> o(pq, 0.0);
            for (int c2 = 0; c2 < pq; ++c2)
                for (int k = 0; k < pq; ++k) o[c2] += m[r2 * n + i + k] * qr[k * pq + c2];
            for (int c2 = 0; c2 < pq; ++c2) m[r2 * n + i + c2] = o[c2];
        }
    };
    cols_times(t);
    for (int c2 = 0; c2 < n; ++c2) {  // t.middleRows(i, pq) = qr^T * t.middleRows(i, pq)
        std::vector<double> o(pq, 0.0);
        for (int r2 = 0; r2 < pq; ++r2)
            for (int k = 0; k < pq; ++k) o[r2] += qr[k * pq + r2] * t[(i + k) * n + c2];
        for (int r2 = 0; r2 < pq; ++r2) t[(i + r2) * n + c2] = o[r2];
    }
    cols_times(q);
    for (int rr = qs; rr < pq; ++rr)
        for (int cc = 0; cc < qs; ++cc) t[(i + rr) * n + i + cc] = 0.0;
    if (qs == 2 && std::abs(t[(i + 1) * n + i]) < 1e-13) t[(i + 1) * n + i] = 0.0;
    if (p == 2) {
        const int j = i + qs;
        if (std::abs(t[(j + 1) * n + j]) < 1e-13) t[(j + 1) * n + j] = 0.0;
    }
}

// schur.hpp:87-97: rotate the 2x2 block at i to equal diagonal entries
inline void standardize_block(int n, Mat& t, Mat& q, int i) {
    const double a = t[i * n + i], b = t[i * n + i + 1], c = t[(i + 1) * n + i], d = t[(i + 1) * n + i + 1];
    if (a == d) return;
    const double th = 0.5 * std::atan2(a - d, b + c);
    const double cs = std::cos(th), sn = std::sin(th);
    const double g[4] = {cs, sn, -sn, cs};
    auto cols = [&](Mat& m) {
        for (int r2 = 0; r2 < n; ++r2) {
            const double x = m[r2 * n + i], y = m[r2 * n + i + 1];
            m[r2 * n + i] = x * g[0] + y * g[2];
            m[r2 * n + i + 1] = x * g[1] + y * g[3];
        }
    };
    cols(t);
    for (int c2 = 0; c2 < n; ++c2) {
        const double x = t[i * n + c2], y = t[(i + 1) * n + c2];
        t[i * n + c2] = g[0] * x + g[2] * y;
        t[(i + 1) * n + c2] = g[1] * x + g[3] * y;
    }
    cols(q);
}

}  // namespace schur_detail

inline std::pair<double, double> tc_legendre(int n, double x) {
    if (n == 0) return {1.0, 0.0};
    double pm = 1.0, p = x;
    for (int k = 2; k <= n; ++k) {
        const double pn = ((2.0 * k - 1.0) * x * p - (k - 1.0) * pm) / k;
        pm = p;
        p = pn;
    }
    return {p, n * (x * p - pm) / (x * x - 1.0)};
}

inline void tc_gauss(int n, std::vector<double>& pts, std::vector<double>& wts) {
    pts.assign(n, 0.0);
    wts.assign(n, 0.0);
    for (int i = 0; i < n; ++i) {
        double x = std::cos(M_PI * (i + 0.75) / (n + 0.5));
        for (int it = 0; it < 100; ++it) {
            const auto pd = tc_legendre(n, x);
            const double dx = pd.first / pd.second;
            x -= dx;
            if (std::abs(dx) < 1e-15) break;
        }
        const auto pd = tc_legendre(n, x);
        pts[n - 1 - i] = 0.5 * (x + 1.0);
        wts[n - 1 - i] = 0.5 * (2.0 / ((1.0 - x * x) * pd.second * pd.second));
    }
}

inline TimeConsts time_consts(int r) {
    if (r < 0 || r > kMaxTimeDegree) throw std::invalid_argument("radau_points: r out of range [0, 5]");
    TimeConsts tc;
    tc.r = r;
    tc.n = r + 1;
    const int n = tc.n;
    if (r >= 1) {
        auto g = [r](double x) { return (tc_legendre(r, x).first + tc_legendre(r + 1, x).first) / (1.0 + x); };
        auto gp = [r](double x) {
            const auto a = tc_legendre(r, x), b = tc_legendre(r + 1, x);
            const double f = a.first + b.first, df = a.second + b.second;
            return (df * (1.0 + x) - f) / ((1.0 + x) * (1.0 + x));
        };
        const int grid = 200 * (r + 1);
        double xa = -1.0 + 1e-12, ga = g(xa);
        for (int k = 1; k <= grid; ++k) {
            const double xb = -1.0 + 2.0 * k / grid - (k == grid ? 1e-12 : 0.0);
            const double gb = g(xb);
            if (ga == 0.0) tc.nodes.push_back(0.5 * (1.0 - xa));
            if (ga * gb < 0.0) {
                double lo = xa, hi = xb;
                for (int it = 0; it < 60; ++it) {
                    const double mid = 0.5 * (lo + hi);
                    (g(lo) * g(mid) <= 0.0 ? hi : lo) = mid;
                }
                double x = 0.5 * (lo + hi);
                for (int it = 0; it < 50; ++it) {
                    const double dx = g(x) / gp(x);
                    x -= dx;
                    if (std::abs(dx) < 1e-16) break;
                }
                tc.nodes.push_back(0.5 * (1.0 - x));
            }
            xa = xb;
            ga = gb;
        }
        if (static_cast<int>(tc.nodes.size()) != r) throw std::runtime_error("radau_points: root search failed");
    }
    tc.nodes.push_back(1.0);
    std::sort(tc.nodes.begin(), tc.nodes.end());
    std::vector<double> bary(n);
    for (int j = 0; j < n; ++j) {
        double w = 1.0;
        for (int k = 0; k < n; ++k)
            if (k != j) w /= (tc.nodes[j] - tc.nodes[k]);
        bary[j] = w;
    }
    auto eval = [&](double s) {
        std::vector<double> v(n, 0.0);
        for (int j = 0; j < n; ++j)
            if (std::abs(s - tc.nodes[j]) < 1e-14) {
                v[j] = 1.0;
                return v;
            }
        double den = 0.0;
        for (int j = 0; j < n; ++j) {
            v[j] = bary[j] / (s - tc.nodes[j]);
            den += v[j];
        }
        for (int j = 0; j < n; ++j) v[j] = v[j] / den;
        return v;
    };
    if (r == 0) {
        tc.weights = {1.0};
    } else {
        std::vector<double> p, w;
        tc_gauss(n + 1, p, w);
        tc.weights.assign(n, 0.0);
        for (size_t k = 0; k < p.size(); ++k) {
            const auto e = eval(p[k]);
            for (int j = 0; j < n; ++j) tc.weights[j] += w[k] * e[j];
        }
    }
    std::vector<double> D(n * n, 0.0);
    for (int i = 0; i < n; ++i) {
        double diag = 0.0;
        for (int j = 0; j < n; ++j) {
            if (i == j) continue;
            D[i * n + j] = (bary[j] / bary[i]) / (tc.nodes[i] - tc.nodes[j]);
            diag -= D[i * n + j];
        }
        D[i * n + i] = diag;
    }
    tc.phi0 = eval(0.0);
    tc.G.assign(n * n, 0.0);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) tc.G[i * n + j] = tc.weights[i] * D[i * n + j] + tc.phi0[i] * tc.phi0[j];
    std::vector<double> W(n * n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) W[i * n + j] = (1.0 / tc.weights[i]) * tc.G[i * n + j];
    tc.Q.assign(n * n, 0.0);
    for (int i = 0; i < n; ++i) tc.Q[i * n + i] = 1.0;
    if (n == 1) {
        tc.T = W;
        tc.block_sizes = {1};
        tc.block_starts = {0};
        return tc;
    }
    if (n > 2) {  // real_schur (schur.hpp:101-173) with the QR iteration above in place of Eigen::RealSchur
        using namespace schur_detail;
        tc.T = W;
        if (!real_schur_qr(n, tc.T, tc.Q, 60 * n))
            throw std::runtime_error("real_schur: QR iteration did not converge within the sweep budget");
        auto detect = [&]() {
            tc.block_sizes.clear();
            tc.block_starts.clear();
            int i = 0;
            while (i < n) {
                const bool two = (i + 1 < n) && std::abs(tc.T[(i + 1) * n + i]) >
                                                    1e-12 * (std::abs(tc.T[i * n + i]) + std::abs(tc.T[(i + 1) * n + i + 1]));
                tc.block_starts.push_back(i);
                tc.block_sizes.push_back(two ? 2 : 1);
                i += two ? 2 : 1;
            }
        };
        auto eig = [&](int gb, double& re, double& im) {
            const int i = tc.block_starts[gb];
            if (tc.block_sizes[gb] == 1) {
                re = tc.T[i * n + i];
                im = 0.0;
                return;
            }
            const double a = tc.T[i * n + i], b = tc.T[i * n + i + 1], c = tc.T[(i + 1) * n + i], d = tc.T[(i + 1) * n + i + 1];
            re = 0.5 * (a + d);
            im = std::sqrt(std::max(0.0, -(0.25 * (a - d) * (a - d) + b * c)));
        };
        auto key_less = [&](int g1, int g2) {
            double r1, i1, r2, i2;
            eig(g1, r1, i1);
            eig(g2, r2, i2);
            if (std::abs(r1 - r2) > 1e-12 * (1.0 + std::abs(r1))) return r1 < r2;
            return std::abs(i1) < std::abs(i2);
        };
        detect();
        bool swapped = true;
        while (swapped) {
            swapped = false;
            for (int gb = 0; gb + 1 < tc.n_blocks(); ++gb)
                if (key_less(gb + 1, gb)) {
                    const int i = tc.block_starts[gb], p = tc.block_sizes[gb];
                    swap_adjacent_blocks(n, tc.T, tc.Q, i, p, p + tc.block_sizes[gb + 1]);
                    detect();
                    swapped = true;
                    break;
                }
        }
        for (int gb = 0; gb < tc.n_blocks(); ++gb)
            if (tc.block_sizes[gb] == 2) standardize_block(n, tc.T, tc.Q, tc.block_starts[gb]);
        for (int gb = 0; gb < tc.n_blocks(); ++gb) {
            const int i = tc.block_starts[gb], bs = tc.block_sizes[gb];
            for (int rr = i; rr < i + bs; ++rr)
                for (int cc = 0; cc < i; ++cc) tc.T[rr * n + cc] = 0.0;
            if (bs == 1 && i + 1 < n) tc.T[(i + 1) * n + i] = 0.0;
        }
        // sanity (schur.hpp:163-170)
        double orth = 0.0, resid = 0.0, wmax = 0.0;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                double qq = 0.0, qtq = 0.0;
                for (int k = 0; k < n; ++k) {
                    qq += tc.Q[k * n + i] * tc.Q[k * n + j];
                    double tq = 0.0;
                    for (int l = 0; l < n; ++l) tq += tc.T[k * n + l] * tc.Q[j * n + l];
                    qtq += tc.Q[i * n + k] * tq;
                }
                orth = std::max(orth, std::abs(qq - (i == j ? 1.0 : 0.0)));
                resid = std::max(resid, std::abs(qtq - W[i * n + j]));
                wmax = std::max(wmax, std::abs(W[i * n + j]));
            }
        if (orth > 1e-12) throw std::runtime_error("real_schur: Q lost orthogonality");
        if (resid > 1e-10 * (1.0 + wmax)) throw std::runtime_error("real_schur: factorization residual too large");
        for (int gb = 0; gb < tc.n_blocks(); ++gb) {
            double re, im;
            eig(gb, re, im);
            if (re <= 0.0) throw std::runtime_error("real_schur: nonpositive real part in a diagonal block");
        }
        return tc;
    }
    tc.block_sizes = {2};
    tc.block_starts = {0};
    double scale = 0.0;
    for (double v : W) scale = std::max(scale, std::abs(v));
    tc.T.resize(4);
    for (int k = 0; k < 4; ++k) tc.T[k] = W[k] / scale;
    const double p = 0.5 * (tc.T[0] - tc.T[3]);
    if (p * p + tc.T[2] * tc.T[1] >= 0.0) throw std::runtime_error("real_schur: expected a complex pair for r = 1");
    for (int k = 0; k < 4; ++k) tc.T[k] *= scale;
    const double a = tc.T[0], b = tc.T[1], c = tc.T[2], d = tc.T[3];
    if (a != d) {
        const double th = 0.5 * std::atan2(a - d, b + c);
        const double cs = std::cos(th), sn = std::sin(th);
        const double g[4] = {cs, sn, -sn, cs};
        auto rmul = [&](std::vector<double>& m) {
            std::vector<double> o(4);
            for (int i = 0; i < 2; ++i)
                for (int j = 0; j < 2; ++j) o[i * 2 + j] = m[i * 2 + 0] * g[0 * 2 + j] + m[i * 2 + 1] * g[1 * 2 + j];
            m = o;
        };
        auto lmul_t = [&](std::vector<double>& m) {
            std::vector<double> o(4);
            for (int i = 0; i < 2; ++i)
                for (int j = 0; j < 2; ++j) o[i * 2 + j] = g[0 * 2 + i] * m[0 * 2 + j] + g[1 * 2 + i] * m[1 * 2 + j];
            m = o;
        };
        rmul(tc.T);
        lmul_t(tc.T);
        rmul(tc.Q);
    }
    return tc;
}

}  // namespace pdg
