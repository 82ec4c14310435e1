// Host check of the library's real Schur iteration (csrc/timebasis.hpp, schur_detail::real_schur_qr)
// on seeded random matrices with real and complex eigenvalues: Q orthogonal, Q T Q^T = A, T quasi-
// upper-triangular with 2x2 blocks only for complex pairs. Prints the worst defects.
#include <cstdio>
#include <random>

#include "timebasis.hpp"

int main() {
    using namespace pdg::schur_detail;
    std::mt19937_64 gen(1801);
    std::uniform_real_distribution<double> U(-1.0, 1.0);
    double worst_orth = 0.0, worst_res = 0.0, worst_low = 0.0;
    int bad_blocks = 0, cases = 0;
    for (int n = 2; n <= 7; ++n)
        for (int rep = 0; rep < 60; ++rep) {
            Mat a(n * n);
            for (double& v : a) v = U(gen);
            if (rep % 3 == 0)  // symmetric: all eigenvalues real, every 2x2 block must split
                for (int i = 0; i < n; ++i)
                    for (int j = 0; j < i; ++j) a[i * n + j] = a[j * n + i];
            const Mat a0 = a;
            Mat q;
            if (!real_schur_qr(n, a, q, 60 * n)) {
                std::printf("no convergence n=%d rep=%d\n", n, rep);
                return 1;
            }
            ++cases;
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) {
                    double qq = 0.0, rec = 0.0;
                    for (int k = 0; k < n; ++k) {
                        qq += q[k * n + i] * q[k * n + j];
                        double tq = 0.0;
                        for (int l = 0; l < n; ++l) tq += a[k * n + l] * q[j * n + l];
                        rec += q[i * n + k] * tq;
                    }
                    worst_orth = std::max(worst_orth, std::abs(qq - (i == j ? 1.0 : 0.0)));
                    worst_res = std::max(worst_res, std::abs(rec - a0[i * n + j]));
                    if (i > j + 1) worst_low = std::max(worst_low, std::abs(a[i * n + j]));
                }
            for (int i = 0; i + 1 < n; ++i)
                if (a[(i + 1) * n + i] != 0.0) {
                    // a 2x2 block: must carry a complex pair, and no two blocks may overlap
                    const double p = 0.5 * (a[i * n + i] - a[(i + 1) * n + i + 1]);
                    if (p * p + a[(i + 1) * n + i] * a[i * n + i + 1] >= 0.0) ++bad_blocks;
                    if (i + 2 < n && a[(i + 2) * n + i + 1] != 0.0) ++bad_blocks;
                }
        }
    std::printf("cases %d orth %.3e resid %.3e lower %.3e bad_blocks %d\n", cases, worst_orth, worst_res, worst_low, bad_blocks);
    return (worst_orth < 1e-12 && worst_res < 1e-12 && worst_low == 0.0 && bad_blocks == 0) ? 0 : 2;
}
