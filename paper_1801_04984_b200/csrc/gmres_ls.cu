// Device-side GMRES step decisions (compiled with --fmad=false: the same bits as
// the host least squares in block.cu, see gmres_ls.cuh).
#include <cmath>

#include "common.cuh"
#include "gmres_ls.cuh"

namespace pdg {

namespace {
constexpr int kLsThreads = 64;  // one thread per least-squares column (restart <= 63 for the parallel path)

// ls_colpiv_raw (gmres_ls.cuh) in shared memory with one thread per column: every
// column's sums run in the same sequential order as the serial version, and the
// pivot, rank and Householder decisions stay serial, so the bits are identical.
__device__ void ls_colpiv_par(double* a, int rows, int cols, double* rhs, double* tau, double* nrm, int* piv, double* y,
                              double* shd, int* shi) {
#define PDG_A(i, j) a[(j) * rows + (i)]
    const int t = threadIdx.x;
    const int size = rows < cols ? rows : cols;
    if (t < cols) {
        piv[t] = t;
        tau[t] = 0.0;
        double s = 0.0;
        for (int i = 0; i < rows; ++i) s += PDG_A(i, t) * PDG_A(i, t);
        nrm[t] = sqrt(s);
    }
    __syncthreads();
    if (t == 0) {
        double maxn = 0.0;
        for (int j = 0; j < cols; ++j) maxn = maxn > nrm[j] ? maxn : nrm[j];
        shd[0] = (maxn * DBL_EPSILON) * (maxn * DBL_EPSILON) / rows;  // thr
        shi[0] = size;                                                // rank
    }
    __syncthreads();
    const double thr = shd[0];
    for (int k = 0; k < size; ++k) {
        if (t >= k && t < cols) {
            double s = 0.0;
            for (int i = k; i < rows; ++i) s += PDG_A(i, t) * PDG_A(i, t);
            nrm[t] = s;
        }
        __syncthreads();
        if (t == 0) {
            int best = k;
            double bestv = -1.0;
            for (int j = k; j < cols; ++j)
                if (nrm[j] > bestv) {
                    bestv = nrm[j];
                    best = j;
                }
            if (shi[0] == size && bestv < thr * (rows - k)) shi[0] = k;
            shi[1] = best;
            if (best != k) {
                const int tp = piv[k];
                piv[k] = piv[best];
                piv[best] = tp;
            }
        }
        __syncthreads();
        const int best = shi[1];
        if (best != k && t < rows) {
            const double tv = PDG_A(t, k);
            PDG_A(t, k) = PDG_A(t, best);
            PDG_A(t, best) = tv;
        }
        __syncthreads();
        if (t == 0) {
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
        }
        __syncthreads();
        if (tau[k] != 0.0 && t > k && t < cols) {
            const int j = t;
            double tt = PDG_A(k, j);
            for (int i = k + 1; i < rows; ++i) tt += PDG_A(i, k) * PDG_A(i, j);
            PDG_A(k, j) -= tau[k] * tt;
            for (int i = k + 1; i < rows; ++i) PDG_A(i, j) -= tau[k] * PDG_A(i, k) * tt;
        }
        __syncthreads();
    }
    if (t == 0) {
        const int rank = shi[0];
        for (int j = 0; j < cols; ++j) y[j] = 0.0;
        if (rank > 0) {
            for (int k = 0; k < rank; ++k) {
                if (tau[k] == 0.0) continue;
                double tt = rhs[k];
                for (int i = k + 1; i < rows; ++i) tt += PDG_A(i, k) * rhs[i];
                rhs[k] -= tau[k] * tt;
                for (int i = k + 1; i < rows; ++i) rhs[i] -= tau[k] * PDG_A(i, k) * tt;
            }
            for (int i = rank - 1; i >= 0; --i) {
                double s = rhs[i];
                for (int j = i + 1; j < rank; ++j) s -= PDG_A(i, j) * rhs[j];
                rhs[i] = s / PDG_A(i, i);
            }
            for (int i = 0; i < rank; ++i) y[piv[i]] = rhs[i];
        }
    }
#undef PDG_A
}

__global__ void __launch_bounds__(kLsThreads) k_gmres_ls(int k, int mm, double beta, const double* __restrict__ hd,
                                                         double* __restrict__ H, double* __restrict__ hk,
                                                         double* __restrict__ rhs, double* __restrict__ tau,
                                                         double* __restrict__ nrm, int* __restrict__ piv,
                                                         double* __restrict__ y, GmresDevState* gs) {
    if (gs->stop) return;  // the previous step already ended the cycle (speculative launch)
    const int ld = mm + 1, rows = k + 2, cols = k + 1, t = threadIdx.x;
    // column k: (0 + pass 0) + pass 1 as the host accumulates it, h(k+1,k) = the norm; the
    // column's entries below k+1 are zero and add exactly nothing to its squared norm
    __shared__ double scol[kLsThreads + 1];
    for (int i = t; i <= k + 1; i += blockDim.x) {
        const double v = i <= k ? (H[(long long)k * ld + i] + hd[i]) + hd[(long long)(k + 1) + i] : hd[2 * (k + 1)];
        H[(long long)k * ld + i] = v;
        scol[i < kLsThreads + 1 ? i : 0] = v;
    }
    __syncthreads();
    if (t == 0) {
        double cn = 0.0;
        if (k + 1 < kLsThreads + 1)
            for (int i = 0; i <= k + 1; ++i) cn += scol[i] * scol[i];
        else
            for (int i = 0; i <= k + 1; ++i) cn += H[(long long)k * ld + i] * H[(long long)k * ld + i];
        gs->brk = H[(long long)k * ld + k + 1] <= 1e-14 * sqrt(cn);
    }
    if (rows > kLsThreads) {  // long cycles: the serial version in global memory
        if (t == 0) {
            for (int j = 0; j < cols; ++j)
                for (int i = 0; i < rows; ++i) hk[(long long)j * rows + i] = H[(long long)j * ld + i];
            rhs[0] = beta;
            for (int i = 1; i < rows; ++i) rhs[i] = 0.0;
            ls_colpiv_raw(hk, rows, cols, rhs, tau, nrm, piv, y);
        }
        return;
    }
    __shared__ double sa[(kLsThreads + 1) * kLsThreads];
    __shared__ double srhs[kLsThreads + 1], stau[kLsThreads], snrm[kLsThreads], sy[kLsThreads], shd[2];
    __shared__ int spiv[kLsThreads], shi[2];
    __syncthreads();  // column k of H written
    for (int e = t; e < rows * cols; e += blockDim.x) {
        const int j = e / rows, i = e - j * rows;
        sa[e] = H[(long long)j * ld + i];
    }
    for (int i = t; i < rows; i += blockDim.x) srhs[i] = i == 0 ? beta : 0.0;
    __syncthreads();
    ls_colpiv_par(sa, rows, cols, srhs, stau, snrm, spiv, sy, shd, shi);
    __syncthreads();
    for (int j = t; j < cols; j += blockDim.x) y[j] = sy[j];
}
}  // namespace

void gmres_ls_launch(int k, int mm, double beta, const double* hd, double* H, double* hk, double* rhs, double* tau,
                     double* nrm, int* piv, double* y, GmresDevState* gs, cudaStream_t st) {
    k_gmres_ls<<<1, kLsThreads, 0, st>>>(k, mm, beta, hd, H, hk, rhs, tau, nrm, piv, y, gs);
    count_launch();
    PDG_CHECK_LAUNCH();
}

}  // namespace pdg
