// Host-side dG(r) time constants for r <= 1 (time_basis.hpp:47-182 and the
// 2x2 branch of real_schur, schur.hpp:87-97,101-173). These are a handful of
// scalars computed once per run; they follow the reference's numerical route
// (Radau roots by bisection + Newton, weights by Gauss quadrature of the
// barycentric basis) so that T, Q and the weights agree bit-for-bit with it.
#pragma once

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <utility>
#include <vector>

namespace pdg {

struct TimeConsts {
    int r = 0, n = 1;
    std::vector<double> nodes, weights, phi0, G, T, Q;  // n, n, n, n*n (row-major)
};

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
    if (r < 0 || r > 1) throw std::invalid_argument("time constants: r must be 0 or 1");
    TimeConsts tc;
    tc.r = r;
    tc.n = r + 1;
    const int n = tc.n;
    if (r == 1) {
        auto g = [](double x) { return (tc_legendre(1, x).first + tc_legendre(2, x).first) / (1.0 + x); };
        auto gp = [](double x) {
            const auto a = tc_legendre(1, x), b = tc_legendre(2, x);
            const double f = a.first + b.first, df = a.second + b.second;
            return (df * (1.0 + x) - f) / ((1.0 + x) * (1.0 + x));
        };
        const int grid = 400;
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
        return tc;
    }
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
