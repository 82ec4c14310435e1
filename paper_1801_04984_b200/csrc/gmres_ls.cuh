// GMRES least squares min || beta e1 - H y || by Householder QR with column
// pivoting (the reference's ColPivHouseholderQR solve, gmres.hpp:111; Eigen's
// published algorithm: column norms, pivot = largest remaining norm, Householder
// vectors as makeHouseholder, numerical rank from the threshold eps * max norm).
//
// Host implementation (block.cu): x86-64 code without -mfma (no contraction), IEEE
// sqrt and division.
#pragma once

#include <cfloat>

namespace pdg {

// a: rows x cols column-major (overwritten), rhs: rows (overwritten),
// scratch tau[cols], nrm[cols], piv[cols]; y: cols.
__host__ __device__ inline void ls_colpiv_raw(double* a, int rows, int cols, double* rhs, double* tau, double* nrm,
                                              int* piv, double* y) {
#define PDG_A(i, j) a[(long long)(j) * rows + (i)]
    const int size = rows < cols ? rows : cols;
    for (int j = 0; j < cols; ++j) {
        piv[j] = j;
        tau[j] = 0.0;
    }
    double maxn = 0.0;
    for (int j = 0; j < cols; ++j) {
        double s = 0.0;
        for (int i = 0; i < rows; ++i) s += PDG_A(i, j) * PDG_A(i, j);
        nrm[j] = sqrt(s);
        maxn = maxn > nrm[j] ? maxn : nrm[j];
    }
    const double eps = DBL_EPSILON;
    const double thr = (maxn * eps) * (maxn * eps) / rows;
    int rank = size;
    for (int k = 0; k < size; ++k) {
        // exact remaining column norms (rows k..)
        int best = k;
        double bestv = -1.0;
        for (int j = k; j < cols; ++j) {
            double s = 0.0;
            for (int i = k; i < rows; ++i) s += PDG_A(i, j) * PDG_A(i, j);
            nrm[j] = s;
            if (s > bestv) {
                bestv = s;
                best = j;
            }
        }
        if (rank == size && bestv < thr * (rows - k)) rank = k;
        if (best != k) {
            for (int i = 0; i < rows; ++i) {
                const double t = PDG_A(i, k);
                PDG_A(i, k) = PDG_A(i, best);
                PDG_A(i, best) = t;
            }
            const int t = piv[k];
            piv[k] = piv[best];
            piv[best] = t;
        }
        double tail = 0.0;
        for (int i = k + 1; i < rows; ++i) tail += PDG_A(i, k) * PDG_A(i, k);
        const double c0 = PDG_A(k, k);
        double beta;
        if (tail <= DBL_MIN) {
            tau[k] = 0.0;
            beta = c0;
            for (int i = k + 1; i < rows; ++i) PDG_A(i, k) = 0.0;
        } else {
            beta = sqrt(c0 * c0 + tail);
            if (c0 >= 0.0) beta = -beta;
            for (int i = k + 1; i < rows; ++i) PDG_A(i, k) /= (c0 - beta);
            tau[k] = (beta - c0) / beta;
        }
        PDG_A(k, k) = beta;
        if (tau[k] != 0.0)
            for (int j = k + 1; j < cols; ++j) {
                double t = PDG_A(k, j);
                for (int i = k + 1; i < rows; ++i) t += PDG_A(i, k) * PDG_A(i, j);
                PDG_A(k, j) -= tau[k] * t;
                for (int i = k + 1; i < rows; ++i) PDG_A(i, j) -= tau[k] * PDG_A(i, k) * t;
            }
    }
    for (int j = 0; j < cols; ++j) y[j] = 0.0;
    if (rank == 0) return;
    for (int k = 0; k < rank; ++k) {
        if (tau[k] == 0.0) continue;
        double t = rhs[k];
        for (int i = k + 1; i < rows; ++i) t += PDG_A(i, k) * rhs[i];
        rhs[k] -= tau[k] * t;
        for (int i = k + 1; i < rows; ++i) rhs[i] -= tau[k] * PDG_A(i, k) * t;
    }
    for (int i = rank - 1; i >= 0; --i) {
        double s = rhs[i];
        for (int j = i + 1; j < rank; ++j) s -= PDG_A(i, j) * rhs[j];
        rhs[i] = s / PDG_A(i, i);
    }
    for (int i = 0; i < rank; ++i) y[piv[i]] = rhs[i];
#undef PDG_A
}

}  // namespace pdg
