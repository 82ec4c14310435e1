// Fixed-stress preconditioner, deterministic Krylov kernels and the GMRES
// driver of one slab block.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>

#include "block.cuh"
#include "gmres_ls.cuh"  // ls_colpiv_raw (host least squares)
#include "timebasis.hpp"

namespace pdg {

namespace {

constexpr int kRedBlocks = 256;  // fixed => reductions are bit-reproducible on any GPU (148 and 592 measured slower)
constexpr int kRedThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];
    return s;  // valid on thread 0
}

// Deterministic Krylov reductions: kRedBlocks fixed-size blocks write one
// partial per (block, column) (grid-stride rows, fixed order), and every
// consumer re-sums the kRedBlocks partials of a column with the same fixed
// tree, so results are bit-reproducible on any GPU and no separate
// "finish the reduction" launch is needed.

// partial[b * ncols + j] = sum over this block's rows of V_j . w (8 columns per pass)
__global__ void __launch_bounds__(kRedThreads) k_multidot1(long long n, int ncols, const double* __restrict__ V,
                                                           const double* __restrict__ w, double* __restrict__ partial) {
    __shared__ double sh[8][kRedThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int j0 = 0; j0 < ncols; j0 += 8) {
        double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
            const double wr = w[r];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (j0 + q < ncols) a[q] += V[(long long)(j0 + q) * n + r] * wr;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
            for (int o = 16; o; o >>= 1) a[q] += __shfl_xor_sync(0xffffffffu, a[q], o);
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < 8; ++q) sh[q][warp] = a[q];
        __syncthreads();
        if (threadIdx.x < 8 && j0 + threadIdx.x < ncols) {
            double s = 0.0;
            for (int i = 0; i < kRedThreads / 32; ++i) s += sh[threadIdx.x][i];
            partial[(long long)blockIdx.x * ncols + j0 + threadIdx.x] = s;
        }
        __syncthreads();
    }
}

// Sum of the kRedBlocks partials of column j (fixed tree); valid on thread 0.
__device__ __forceinline__ double sum_partials(const double* __restrict__ partial, int ncols, int j, double* sh) {
    double v = 0.0;
    for (int b = threadIdx.x; b < kRedBlocks; b += blockDim.x) v += partial[(long long)b * ncols + j];
    return block_sum(v, sh);
}

// h = column sums of the partials (block 0 writes them to h_out), then
// w -= sum_j h_j V_j, subtracting column by column in j order
__global__ void __launch_bounds__(kRedThreads) k_red_multiaxpy(long long n, int ncols, const double* __restrict__ partial,
                                                               const double* __restrict__ V, double* __restrict__ w,
                                                               double* __restrict__ h_out) {
    __shared__ double sh[32];
    extern __shared__ double hs[];  // [ncols]
    for (int j = 0; j < ncols; ++j) {
        const double s = sum_partials(partial, ncols, j, sh);
        if (threadIdx.x == 0) hs[j] = s;
    }
    __syncthreads();
    if (blockIdx.x == 0)
        for (int j = threadIdx.x; j < ncols; j += blockDim.x) h_out[j] = hs[j];
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
        double v = w[r];
        for (int j = 0; j < ncols; ++j) v -= hs[j] * V[(long long)j * n + r];
        w[r] = v;
    }
}

// nrm = sqrt(sum of the partials); dst = src / nrm (dst may be null); block 0 writes nrm
__global__ void __launch_bounds__(kRedThreads) k_red_norm_scale(long long n, const double* __restrict__ partial,
                                                                const double* __restrict__ src, double* __restrict__ dst,
                                                                double* __restrict__ nrm_out) {
    __shared__ double sh[32];
    __shared__ double nv;
    const double s = sum_partials(partial, 1, 0, sh);
    if (threadIdx.x == 0) nv = sqrt(s);
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) *nrm_out = nv;
    if (!dst) return;
    const double d = nv;
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x)
        dst[r] = src[r] / d;
}

// out = a - b, and the partial sums of out . out (same layout as k_multidot1 with one column)
__global__ void __launch_bounds__(kRedThreads) k_sub_dot(long long n, const double* __restrict__ a,
                                                         const double* __restrict__ b, double* __restrict__ out,
                                                         double* __restrict__ partial) {
    __shared__ double sh[kRedThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double acc = 0.0;
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
        const double v = a[r] - b[r];
        out[r] = v;
        acc += v * v;
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) sh[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < kRedThreads / 32; ++i) s += sh[i];
        partial[blockIdx.x] = s;
    }
}

// out = base + sum_j y_j V_j (base may be null => 0), summed in j order from 0.0
__global__ void k_combine(long long n, int ncols, const double* __restrict__ V, const double* __restrict__ y,
                          const double* __restrict__ base, double* __restrict__ out) {
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int j = 0; j < ncols; ++j) s += V[(long long)j * n + r] * y[j];
        out[r] = base ? base[r] + s : s;
    }
}

// ---- fused Arnoldi kernels (one cooperative launch each, grid = kRedBlocks) ----
// Same arithmetic, in the same order, as the unfused launch sequences they
// replace (k_multidot1 / k_red_multiaxpy / k_red_norm_scale / k_combine /
// k_sub_dot): the grid-stride row order, the per-block partials and the fixed
// partial-sum tree are unchanged, so results are bit-identical to them. The
// grid barriers replace kernel boundaries.

// block partials of V_j . w for j < ncols (the k_multidot1 body)
__device__ __forceinline__ void block_multidot(long long n, int ncols, const double* __restrict__ V,
                                               const double* w, double* __restrict__ partial) {
    __shared__ double sh[8][kRedThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int j0 = 0; j0 < ncols; j0 += 8) {
        double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
            const double wr = __ldcg(w + r);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (j0 + q < ncols) a[q] += V[(long long)(j0 + q) * n + r] * wr;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
            for (int o = 16; o; o >>= 1) a[q] += __shfl_xor_sync(0xffffffffu, a[q], o);
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < 8; ++q) sh[q][warp] = a[q];
        __syncthreads();
        if (threadIdx.x < 8 && j0 + threadIdx.x < ncols) {
            double s = 0.0;
            for (int i = 0; i < kRedThreads / 32; ++i) s += sh[threadIdx.x][i];
            partial[(long long)blockIdx.x * ncols + j0 + threadIdx.x] = s;
        }
        __syncthreads();
    }
}

// column sums of the partials into hs[ncols] (smem, every block), block 0 copies them to h_out
__device__ __forceinline__ void block_column_sums(const double* partial, int ncols, double* hs, double* h_out,
                                                  int nblocks = kRedBlocks) {
    __shared__ double sh[32];
    for (int j = 0; j < ncols; ++j) {
        double v = 0.0;
        for (int b = threadIdx.x; b < nblocks; b += blockDim.x) v += __ldcg(partial + (long long)b * ncols + j);
        const double s = block_sum(v, sh);
        if (threadIdx.x == 0) hs[j] = s;
    }
    __syncthreads();
    if (blockIdx.x == 0 && h_out)
        for (int j = threadIdx.x; j < ncols; j += blockDim.x) h_out[j] = hs[j];
}

// Two classical Gram-Schmidt passes of w against V_0..V_{ncols-1}, then
// h_out[2 ncols] = ||w|| and vnext = w / ||w||. h_out[0..ncols) pass 1, [ncols..2 ncols) pass 2.
// partial: 3 regions of kRedBlocks * ncols (a region is never rewritten while another block may read it).
// pre1 != null: the first pass's partials were formed by the SpMV epilogue (k_spmv<true>,
// nb1 blocks); the kernel starts at their column sums
// Device-driven GMRES steps (LoopState, flexible candidate): after the norm, block 0 stores
// the Hessenberg column H(0..k+1, k) = (0 + pass 1) + pass 2, ||w|| (as the host assembles
// it) into Hcol, runs the breakdown test of gmres.hpp:103, applies the cycle's Givens
// rotations and forms the next one; |g_{k+1}| = || beta e1 - H y || is the step's residual
// estimate. stop = estimate <= tol ||b|| || breakdown || last step of the cycle.
struct LoopState {
    int stop, brk;
    double res;
};
__device__ __forceinline__ void givens_step(int k, int mm, const double* h1, const double* h2, double nv,
                                            double* Hcol, double* cs, double* sn, double* g, double tolb,
                                            LoopState* ls) {
    double cn = 0.0;
    for (int i = 0; i <= k; ++i) {
        const double v = (0.0 + h1[i]) + h2[i];
        Hcol[i] = v;
        cn += v * v;
    }
    Hcol[k + 1] = nv;
    cn += nv * nv;
    const int brk = nv <= 1e-14 * sqrt(cn);
    // rotate the column by the previous rotations, then annihilate H(k+1, k)
    double hk = Hcol[0];
    for (int i = 0; i < k; ++i) {
        const double hn = Hcol[i + 1];
        const double t = cs[i] * hk + sn[i] * hn;
        hk = -sn[i] * hk + cs[i] * hn;
        (void)t;
    }
    // (the rotated entries above the diagonal are not needed: only the residual estimate is)
    const double r = hypot(hk, nv);
    const double c = r == 0.0 ? 1.0 : hk / r, sg = r == 0.0 ? 0.0 : nv / r;
    cs[k] = c;
    sn[k] = sg;
    g[k + 1] = -sg * g[k];
    g[k] = c * g[k];
    const double res = fabs(g[k + 1]);
    ls->res = res;
    ls->brk = brk;
    ls->stop = (res <= tolb) || brk || (k == mm - 1);
}

__global__ void __launch_bounds__(kRedThreads) k_arnoldi_gs(long long n, int ncols, const double* __restrict__ V,
                                                            double* w, double* partial, double* h_out,
                                                            double* __restrict__ vnext, LoopState* ls,
                                                            const double* pre1, int nb1, double* Hcol, double* cs,
                                                            double* sn, double* g, int mm, double tolb) {
    if (ls && ls->stop) return;  // speculative step after the cycle ended
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double hs[];  // [ncols]
    double* p1 = partial;
    double* p2 = partial + (size_t)kRedBlocks * ncols;
    double* p3 = partial + (size_t)2 * kRedBlocks * ncols;
    if (!pre1) block_multidot(n, ncols, V, w, p1);
    if (ncols <= 8) {
        // Fused passes (up to 8 basis vectors): a thread updates its rows of w and accumulates the
        // next pass's partial dots from the values it just formed, in the same row order and with
        // the same partial-sum tree as the separate loops, so the bits are those of the unfused
        // sequence; only the partials cross blocks: two grid barriers fewer, half the sweeps.
        __shared__ double shd[8][kRedThreads / 32];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        for (int pass = 0; pass < 2; ++pass) {
            if (pass > 0 || !pre1) grid.sync();
            if (pass == 0 && pre1)
                block_column_sums(pre1, ncols, hs, h_out, nb1);
            else
                block_column_sums(pass == 0 ? p1 : p2, ncols, hs, h_out + (size_t)pass * ncols);
            double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            // two rows per trip: both rows' loads are issued before either is used (a thread has ~6
            // rows at config 1, each a round trip to L2); the rows are then processed in order, so
            // the sums are those of the one-row loop
            const long long stride = (long long)gridDim.x * blockDim.x;
            for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += 2 * stride) {
                const long long r2 = r + stride;
                const bool two = r2 < n;
                double v = __ldcg(w + r), v2 = two ? __ldcg(w + r2) : 0.0;
                double vj[8], vk[8];
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j < ncols) {
                        vj[j] = V[(long long)j * n + r];
                        vk[j] = two ? V[(long long)j * n + r2] : 0.0;
                    }
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j < ncols) v -= hs[j] * vj[j];
                w[r] = v;
                if (pass == 0) {
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        if (q < ncols) a[q] += vj[q] * v;
                } else {
                    a[0] += v * v;
                }
                if (two) {
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (j < ncols) v2 -= hs[j] * vk[j];
                    w[r2] = v2;
                    if (pass == 0) {
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            if (q < ncols) a[q] += vk[q] * v2;
                    } else {
                        a[0] += v2 * v2;
                    }
                }
            }
            const int nq = pass == 0 ? ncols : 1;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                for (int o = 16; o; o >>= 1) a[q] += __shfl_xor_sync(0xffffffffu, a[q], o);
            if (lane == 0)
#pragma unroll
                for (int q = 0; q < 8; ++q) shd[q][warp] = a[q];
            __syncthreads();
            if (threadIdx.x < 8 && threadIdx.x < nq) {
                double sacc = 0.0;
                for (int i = 0; i < kRedThreads / 32; ++i) sacc += shd[threadIdx.x][i];
                (pass == 0 ? p2 : p3)[(long long)blockIdx.x * nq + threadIdx.x] = sacc;
            }
            __syncthreads();
        }
    } else {
    for (int pass = 0; pass < 2; ++pass) {
        if (pass > 0 || !pre1) grid.sync();
        if (pass == 0 && pre1)
            block_column_sums(pre1, ncols, hs, h_out, nb1);
        else
            block_column_sums(pass == 0 ? p1 : p2, ncols, hs, h_out + (size_t)pass * ncols);
        for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
            double v = __ldcg(w + r);
            for (int j = 0; j < ncols; ++j) v -= hs[j] * V[(long long)j * n + r];
            w[r] = v;
        }
        __syncthreads();
        grid.sync();  // w complete before the next pass reads it
        if (pass == 0)
            block_multidot(n, ncols, V, w, p2);
        else
            block_multidot(n, 1, w, w, p3);
    }
    }
    grid.sync();
    {
        __shared__ double sh[32];
        __shared__ double nv;
        double v = 0.0;
        for (int b = threadIdx.x; b < kRedBlocks; b += blockDim.x) v += __ldcg(p3 + b);
        const double s = block_sum(v, sh);
        if (threadIdx.x == 0) nv = sqrt(s);
        __syncthreads();
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            h_out[2 * ncols] = nv;
            if (ls) givens_step(ncols - 1, mm, h_out, h_out + ncols, nv, Hcol, cs, sn, g, tolb, ls);
        }
        const double d = nv;
        const long long stride = (long long)gridDim.x * blockDim.x;
        for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += 2 * stride) {
            const long long r2 = r + stride;
            const double x0 = __ldcg(w + r), x1 = r2 < n ? __ldcg(w + r2) : 0.0;
            vnext[r] = x0 / d;
            if (r2 < n) vnext[r2] = x1 / d;
        }
    }
}

// r = r0 - sum_j y_j AZ_j (sum from 0.0 in j order), ||r|| into nrm_out
__global__ void __launch_bounds__(kRedThreads) k_arnoldi_residual(long long n, int ncols, const double* __restrict__ AZ,
                                                                  const double* __restrict__ y,
                                                                  const double* __restrict__ r0, double* r,
                                                                  double* partial, double* nrm_out) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ double sh[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double acc = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int j = 0; j < ncols; ++j) s += AZ[(long long)j * n + i] * y[j];
        const double v = r0[i] - s;
        r[i] = v;
        acc += v * v;
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) sh[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < kRedThreads / 32; ++i) s += sh[i];
        partial[blockIdx.x] = s;
    }
    grid.sync();
    double v = 0.0;
    if (blockIdx.x == 0) {
        for (int b = threadIdx.x; b < kRedBlocks; b += blockDim.x) v += __ldcg(partial + b);
        const double s = block_sum(v, sh);
        if (threadIdx.x == 0) *nrm_out = sqrt(s);
    }
}

__global__ void k_add(long long n, const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out) {
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x)
        out[r] = a[r] + b[r];
}

// ---- fixed-stress sweep kernels (fixed_stress.hpp:109-139) ------------------
// fp_i = r_p_i [+ lambda (b E^T u_i - stab m_p p_i) for sweeps after the first]
__global__ void k_flow_fp(int m, int np, int nt, int nu, int nq, int lag, double lambda, double b, double stab,
                          const double* __restrict__ r, const double* __restrict__ xold, const int* et_off,
                          const int* et_idx, const double* et_val, const double* m_p, double* __restrict__ fp, const int* __restrict__ stop) {
    if (stop && *stop) return;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * np; t += (long long)gridDim.x * blockDim.x) {
        const int i = static_cast<int>(t / np), c = static_cast<int>(t % np);
        double pr = r[(long long)i * nt + nu + nq + c];
        if (lag) {
            double et = 0.0;
            for (int k = et_off[c]; k < et_off[c + 1]; ++k) et += et_val[k] * xold[(long long)i * nt + et_idx[k]];
            pr += lambda * (b * et - stab * (m_p[c] * xold[(long long)i * nt + nu + nq + c]));
        }
        fp[t] = pr;
    }
}
// rq_i[f] = r_q_i[f] - sum_{B row f} (w bv) (dinv_c fp_c)
__global__ void k_flow_rq(int m, int nq, int np, int nt, int nu, double w, const double* __restrict__ r,
                          const double* __restrict__ fp, long long fps, const int* b_off, const int* b_idx,
                          const double* b_val, const double* __restrict__ dinv, double* __restrict__ rq,
                          const int* __restrict__ stop) {
    if (stop && *stop) return;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * nq; t += (long long)gridDim.x * blockDim.x) {
        const int i = static_cast<int>(t / nq), f = static_cast<int>(t % nq);
        double v = r[(long long)i * nt + nu + f];
        for (int k = b_off[f]; k < b_off[f + 1]; ++k) {
            const int c = b_idx[k];
            v -= w * b_val[k] * (dinv[c] * fp[(long long)i * fps + c]);
        }
        rq[t] = v;
    }
}
// p_i[c] = dinv_c (fp_c - w sum_{B^T row c} bv q_f)   (q already in z)
__global__ void k_flow_p(int m, int np, int nt, int nu, int nq, double w, const double* __restrict__ fp, long long fps,
                         const int* bt_off, const int* bt_idx, const double* bt_val, const double* __restrict__ dinv,
                         double* __restrict__ z, const int* __restrict__ stop) {
    if (stop && *stop) return;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * np; t += (long long)gridDim.x * blockDim.x) {
        const int i = static_cast<int>(t / np), c = static_cast<int>(t % np);
        double btq = 0.0;
        for (int k = bt_off[c]; k < bt_off[c + 1]; ++k) btq += bt_val[k] * z[(long long)i * nt + nu + bt_idx[k]];
        z[(long long)i * nt + nu + nq + c] = dinv[c] * (fp[(long long)i * fps + c] - w * btq);
    }
}
// mech_i = r_u_i / w + b (E p_i)
__global__ void k_mech_rhs(int m, int nu, int nt, int nq, double w, double b, const double* __restrict__ r,
                           const double* __restrict__ z, const int* e_off, const int* e_idx, const double* e_val,
                           double* __restrict__ mech, const int* __restrict__ stop) {
    if (stop && *stop) return;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * nu; t += (long long)gridDim.x * blockDim.x) {
        const int i = static_cast<int>(t / nu), k0 = static_cast<int>(t % nu);
        double ep = 0.0;
        for (int k = e_off[k0]; k < e_off[k0 + 1]; ++k) ep += e_val[k] * z[(long long)i * nt + nu + nq + e_idx[k]];
        mech[t] = r[(long long)i * nt + k0] / w + b * ep;
    }
}

// S_q dense blocks (face-row order), one thread per face row: no write conflicts.
__global__ void k_flow_schur_blocks(int nq, double w, const int* mq_off, const int* mq_idx, const double* mq_val,
                                    const int* b_off, const int* b_idx, const double* b_val, const int* bt_off,
                                    const int* bt_idx, const double* bt_val, const double* dinv, const int* inv_perm,
                                    const int* blk_of, const int* loc_of, const int* bsz, const long long* dD,
                                    const long long* dC, double* dense, int* err) {
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nq; f += gridDim.x * blockDim.x) {
        const int nr = inv_perm[f], jr = blk_of[nr], lr = loc_of[nr];
        auto add = [&](int f2, double v) {
            const int nc = inv_perm[f2], jc = blk_of[nc], lc = loc_of[nc];
            if (jc == jr)
                dense[dD[jr] + lr + (long long)lc * bsz[jr]] += v;
            else if (jr == jc + 1)
                dense[dC[jc] + lr + (long long)lc * bsz[jr]] += v;
            else if (jc != jr + 1)
                atomicOr(err, 1);
        };
        for (int k = mq_off[f]; k < mq_off[f + 1]; ++k) add(mq_idx[k], w * mq_val[k]);
        for (int k = b_off[f]; k < b_off[f + 1]; ++k) {
            const int c = b_idx[k];
            const double wa = w * b_val[k];
            for (int q = bt_off[c]; q < bt_off[c + 1]; ++q) add(bt_idx[q], -(wa * (w * bt_val[q])) * dinv[c]);
        }
    }
}

__global__ void k_dinv(int np, double coef, const double* m_p, double* dinv) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < np; c += gridDim.x * blockDim.x) dinv[c] = 1.0 / (-coef * m_p[c]);
}

// ---- host least squares: Householder QR with column pivoting ---------------
// min || beta e1 - H y ||, H (rows x cols) column-major; numerical rank as in
// a column-pivoted QR with threshold eps * max column norm.
std::vector<double> ls_colpiv(std::vector<double> a, int rows, int cols, std::vector<double> rhs) {
    std::vector<double> tau(cols), nrm(cols), y(cols);
    std::vector<int> piv(cols);
    ls_colpiv_raw(a.data(), rows, cols, rhs.data(), tau.data(), nrm.data(), piv.data(), y.data());
    return y;
}

}  // namespace

// ---------------------------------------------------------------------------
HCsr csr_download(const DCsr& a, cudaStream_t st) {
    HCsr h;
    h.rows = a.rows;
    h.cols = a.cols;
    h.off = a.off.download(st);
    h.idx = a.idx.download(st);
    h.val = a.val.download(st);
    return h;
}

HCsr flow_schur_host(const SpatialOps& o, double w, const std::vector<double>& di, cudaStream_t st) {
    // S_q = w M_q - w^2 B D^{-1} B^T, rows in face order, columns ascending; each entry summed
    // in the order of k_flow_schur_blocks (M_q term, then the B D^{-1} B^T products)
    const HCsr mq = csr_download(o.M_q, st), bb = csr_download(o.B, st), bt = csr_download(o.Bt, st);
    HCsr h;
    h.rows = h.cols = o.n_q;
    h.off.assign(o.n_q + 1, 0);
    for (int f = 0; f < o.n_q; ++f) {
        std::vector<std::pair<int, double>> row;
        for (int k = mq.off[f]; k < mq.off[f + 1]; ++k) row.push_back({mq.idx[k], w * mq.val[k]});
        for (int k = bb.off[f]; k < bb.off[f + 1]; ++k) {
            const int c = bb.idx[k];
            const double wa = w * bb.val[k];
            for (int q = bt.off[c]; q < bt.off[c + 1]; ++q) row.push_back({bt.idx[q], -(wa * (w * bt.val[q])) * di[c]});
        }
        std::stable_sort(row.begin(), row.end(), [](auto& a, auto& b) { return a.first < b.first; });
        for (size_t k = 0; k < row.size();) {
            double v = 0.0;
            const int col = row[k].first;
            for (; k < row.size() && row[k].first == col; ++k) v += row[k].second;
            h.idx.push_back(col);
            h.val.push_back(v);
        }
        h.off[f + 1] = static_cast<int>(h.idx.size());
    }
    return h;
}

void face_coords(int nx, int ny, std::vector<double>& cx, std::vector<double>& cy) {
    const int nq = nx * (ny + 1) + (nx + 1) * ny;
    cx.assign(nq, 0.0);
    cy.assign(nq, 0.0);
    for (int f = 0; f < nq; ++f) {
        if (f < nx * (ny + 1)) {
            cx[f] = f % nx + 0.5;
            cy[f] = f / nx;
        } else {
            const int g = f - nx * (ny + 1);
            cx[f] = g / ny;
            cy[f] = g % ny + 0.5;
        }
    }
}

int nd_leaf_dofs(int dflt, const char* var) {
    const char* e = std::getenv(var);
    return e ? std::max(1, std::atoi(e)) : dflt;
}

// 3D face centres (assembly3d.cu numbering): z-normal (i + 1/2, j + 1/2, k), y-normal
// (i + 1/2, j, k + 1/2), x-normal (i, j + 1/2, k + 1/2)
void face_coords3(int nx, int ny, int nz, std::vector<double>& cx, std::vector<double>& cy, std::vector<double>& cz) {
    const int nzf = nx * ny * (nz + 1), nyf = nx * (ny + 1) * nz, nq = nzf + nyf + (nx + 1) * ny * nz;
    cx.assign(nq, 0.0);
    cy.assign(nq, 0.0);
    cz.assign(nq, 0.0);
    for (int f = 0; f < nq; ++f) {
        if (f < nzf) {
            cx[f] = f % nx + 0.5;
            cy[f] = (f / nx) % ny + 0.5;
            cz[f] = f / (nx * ny);
        } else if (f < nzf + nyf) {
            const int g = f - nzf;
            cx[f] = g % nx + 0.5;
            cz[f] = (g / nx) % nz + 0.5;
            cy[f] = g / (nx * nz);
        } else {
            const int g = f - nzf - nyf;
            cy[f] = g % ny + 0.5;
            cz[f] = (g / ny) % nz + 0.5;
            cx[f] = g / (ny * nz);
        }
    }
}

std::shared_ptr<ASolver> make_a_solver(const SpatialOps& ops, int max_rhs, cudaStream_t st, bool fp32_factor) {
    auto a = std::make_shared<ASolver>();
    if (ops.nz > 0) {
        // 3D: nested dissection over cells (24 dofs each, centres (i + 1/2, j + 1/2, k + 1/2))
        const long long nc = (long long)ops.nx * ops.ny * ops.nz;
        require(ops.nx > 0 && ops.ny > 0 && ops.n_u == 24 * nc, "A solver: mesh dimensions do not match n_u");
        const HCsr h = csr_download(ops.A, st);
        std::vector<int> node_of(ops.n_u);
        for (int d = 0; d < ops.n_u; ++d) node_of[d] = d / 24;
        std::vector<double> cx(nc), cy(nc), cz(nc);
        for (int c = 0; c < nc; ++c) {
            cx[c] = c % ops.nx + 0.5;
            cy[c] = (c / ops.nx) % ops.ny + 0.5;
            cz[c] = c / (ops.nx * ops.ny) + 0.5;
        }
        a->use_nd = true;
        a->nd.prof_phase = PROF_A_SOLVE;
        a->nd.fp32_req = fp32_factor;
        a->nd.factor(ops.n_u, h.off, h.idx, h.val, node_of, cx, cy, nd_leaf_dofs(192), max_rhs, st, &cz);
        return a;
    }
    // cell-row order: block j = displacement dofs of cell row j (8 nx each)
    require(ops.nx > 0 && ops.ny > 0 && ops.n_u == 8 * ops.nx * ops.ny, "A solver: mesh dimensions do not match n_u");
    // nd (default): nested dissection; local: twisted block-tridiagonal inverse-Schur sweep;
    // general: the block-tridiagonal three-matrix recurrence
    const char* mode = std::getenv("PDG_A_SOLVER");
    if (!mode || std::string(mode) == "nd") {
        // nested dissection over cells (row-major, 8 dofs each, centres (i + 1/2, j + 1/2))
        const HCsr h = csr_download(ops.A, st);
        const int nc = ops.nx * ops.ny;
        std::vector<int> node_of(ops.n_u);
        for (int d = 0; d < ops.n_u; ++d) node_of[d] = d / 8;
        std::vector<double> cx(nc), cy(nc);
        for (int c = 0; c < nc; ++c) {
            cx[c] = c % ops.nx + 0.5;
            cy[c] = c / ops.nx + 0.5;
        }
        a->use_nd = true;
        a->nd.prof_phase = PROF_A_SOLVE;
        a->nd.factor(ops.n_u, h.off, h.idx, h.val, node_of, cx, cy, nd_leaf_dofs(128), max_rhs, st);
        return a;
    }
    std::vector<int> bs(ops.ny, 8 * ops.nx);
    a->chol.allow_local = !(mode && std::string(mode) == "general");
    a->chol.factor(ops.n_u, ops.A.off.p, ops.A.idx.p, ops.A.val.p, {}, bs, max_rhs, st);
    return a;
}

// ---- coupled fixed-stress sweep (fixed_stress.hpp:109-139 with a full Theta) ----
constexpr int kMaxC = 2;
struct Mat2 {
    double a[4];
};
// 1 / ((1/M + stab) m_p)
__global__ void k_dinvc(int np, double s, const double* m_p, double* d) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < np; c += gridDim.x * blockDim.x) d[c] = 1.0 / (s * m_p[c]);
}
// S[(i,f),(i2,f2)] = [i==i2] w_i M_q[f,f2] + Gamma_{i,i2} sum_c B[f,c] B[f2,c] / d_c   (Gamma = W Theta^{-1} W)
__global__ void k_flowc_schur_blocks(int m, int nq, Mat2 w, Mat2 gam, const int* mq_off, const int* mq_idx,
                                     const double* mq_val, const int* b_off, const int* b_idx, const double* b_val,
                                     const int* bt_off, const int* bt_idx, const double* bt_val, const double* dinvc,
                                     const int* inv_perm, const int* blk_of, const int* loc_of, const int* bsz,
                                     const long long* dD, const long long* dC, const long long* dU, double* dense,
                                     int* err) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < m * nq; t += gridDim.x * blockDim.x) {
        const int i = t / nq, f = t % nq;
        const int nr = inv_perm[t], jr = blk_of[nr], lr = loc_of[nr];
        auto add = [&](int i2, int f2, double v) {
            const int nc = inv_perm[i2 * nq + f2], jc = blk_of[nc], lc = loc_of[nc];
            if (jc == jr)
                dense[dD[jr] + lr + (long long)lc * bsz[jr]] += v;
            else if (jr == jc + 1)
                dense[dC[jc] + lr + (long long)lc * bsz[jr]] += v;
            else if (jc == jr + 1)
                dense[dU[jr] + lr + (long long)lc * bsz[jr]] += v;
            else
                atomicOr(err, 1);
        };
        for (int k = mq_off[f]; k < mq_off[f + 1]; ++k) add(i, mq_idx[k], w.a[i] * mq_val[k]);
        for (int k = b_off[f]; k < b_off[f + 1]; ++k) {
            const int c = b_idx[k];
            for (int q = bt_off[c]; q < bt_off[c + 1]; ++q)
                for (int i2 = 0; i2 < m; ++i2) add(i2, bt_idx[q], gam.a[i * m + i2] * (b_val[k] * bt_val[q]) * dinvc[c]);
        }
    }
}
// fp_i = r_p_i [+ sum_j Theta_ij (b E^T u_j - stab m_p p_j) from the previous iterate]
__global__ void k_fsc_fp(int m, int np, int nt, int nu, int nq, const double* __restrict__ xold, Mat2 th, double b,
                         double stab, const double* __restrict__ r, const int* et_off, const int* et_idx,
                         const double* et_val, const double* m_p, double* __restrict__ fp) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * np;
         t += (long long)gridDim.x * blockDim.x) {
        const int i = static_cast<int>(t / np), c = static_cast<int>(t % np);
        double pr = r[(long long)i * nt + nu + nq + c];
        if (xold)
            for (int j = 0; j < m; ++j) {
                const double tij = th.a[i * m + j];
                if (tij == 0.0) continue;
                double et = 0.0;
                for (int k = et_off[c]; k < et_off[c + 1]; ++k) et += et_val[k] * xold[(long long)j * nt + et_idx[k]];
                pr += tij * (b * et - stab * (m_p[c] * xold[(long long)j * nt + nu + nq + c]));
            }
        fp[t] = pr;
    }
}
// rq_i[f] = r_q_i[f] + w_i sum_j Thinv_ij sum_{B row f} bv fp_j[c] / d_c
__global__ void k_fsc_rq(int m, int nq, int np, int nt, int nu, Mat2 w, Mat2 thinv, const double* __restrict__ r,
                         const double* __restrict__ fp, const int* b_off, const int* b_idx, const double* b_val,
                         const double* __restrict__ dinvc, double* __restrict__ rq) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * nq;
         t += (long long)gridDim.x * blockDim.x) {
        const int i = static_cast<int>(t / nq), f = static_cast<int>(t % nq);
        double v = r[(long long)i * nt + nu + f];
        for (int k = b_off[f]; k < b_off[f + 1]; ++k) {
            const int c = b_idx[k];
            double s = 0.0;
            for (int j = 0; j < m; ++j) s += thinv.a[i * m + j] * fp[(long long)j * np + c];
            v += w.a[i] * b_val[k] * s * dinvc[c];
        }
        rq[t] = v;
    }
}
// q into z, then p_i[c] = -(1/d_c) sum_j Thinv_ij (fp_j[c] - w_j (B^T q_j)[c])
__global__ void k_fsc_qp(int m, int np, int nq, int nt, int nu, Mat2 w, Mat2 thinv, const double* __restrict__ fp,
                         const double* __restrict__ q, const int* bt_off, const int* bt_idx, const double* bt_val,
                         const double* __restrict__ dinvc, double* __restrict__ z) {
    const long long nqq = (long long)m * nq;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nqq + (long long)m * np;
         t += (long long)gridDim.x * blockDim.x) {
        if (t < nqq) {
            const int i = static_cast<int>(t / nq), f = static_cast<int>(t % nq);
            z[(long long)i * nt + nu + f] = q[t];
            continue;
        }
        const long long u = t - nqq;
        const int i = static_cast<int>(u / np), c = static_cast<int>(u % np);
        double s = 0.0;
        for (int j = 0; j < m; ++j) {
            double btq = 0.0;
            for (int k = bt_off[c]; k < bt_off[c + 1]; ++k) btq += bt_val[k] * q[(long long)j * nq + bt_idx[k]];
            s += thinv.a[i * m + j] * (fp[(long long)j * np + c] - w.a[j] * btq);
        }
        z[(long long)i * nt + nu + nq + c] = -dinvc[c] * s;
    }
}
// mech_i = r_u_i / w_i + b (E p_i)
__global__ void k_fsc_mech(int m, int nu, int nt, int nq, Mat2 w, double b, const double* __restrict__ r,
                           const double* __restrict__ z, const int* e_off, const int* e_idx, const double* e_val,
                           double* __restrict__ mech) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * nu;
         t += (long long)gridDim.x * blockDim.x) {
        const int i = static_cast<int>(t / nu), k0 = static_cast<int>(t % nu);
        double ep = 0.0;
        for (int k = e_off[k0]; k < e_off[k0 + 1]; ++k) ep += e_val[k] * z[(long long)i * nt + nu + nq + e_idx[k]];
        mech[t] = r[(long long)i * nt + k0] / w.a[i] + b * ep;
    }
}

void FixedStressPre::setup(const SpatialOps& o, int m_, double tau_, double lambda_, double stab_, int sweeps_,
                           std::shared_ptr<ASolver> a_, cudaStream_t st) {
    ops = &o;
    m = m_;
    tau = tau_;
    lambda = lambda_;
    stab = stab_;
    sweeps = sweeps_;
    w = tau * 1.0;
    a = std::move(a_);
    require(sweeps >= 1, "fixed-stress: sweep counts must be >= 1");
    require(lambda * (o.inv_m + stab) > 0.0, "fixed-stress: flow storage block must be negative definite");
    dinv.alloc(o.n_p);
    k_dinv<<<grid_for(o.n_p, 256), 256, 0, st>>>(o.n_p, lambda * (o.inv_m + stab), o.m_p.p, dinv.p);
    PDG_CHECK_LAUNCH();
    // face-row permutation: level j horizontal faces, then row j vertical faces
    const int nx = o.nx, ny = o.ny;
    if (o.nz > 0)
        require(o.n_q == nx * ny * (o.nz + 1) + nx * (ny + 1) * o.nz + (nx + 1) * ny * o.nz,
                "fixed-stress: face count does not match the mesh");
    else
        require(o.n_q == nx * (ny + 1) + (nx + 1) * ny, "fixed-stress: face count does not match the mesh");
    rq.alloc((size_t)m * o.n_q);
    fp.alloc((size_t)m * o.n_p);
    mech.alloc((size_t)m * o.n_u);
    if (sweeps > 1) xold.alloc((size_t)m * o.n_total());
    const char* fmode = std::getenv("PDG_FLOW_SOLVER");  // nd (default) | blocktri
    if (o.nz > 0 || ((!fmode || std::string(fmode) == "nd") && !std::getenv("PDG_FLOW_STRIPS"))) {
        // S_q assembled on the host (the entries of k_flow_schur_blocks), nested dissection over
        // faces: horizontal j*nx+i at (i + 1/2, j), vertical nx(ny+1) + i*ny + j at (i, j + 1/2)
        const HCsr sq = flow_schur_host(o, w, dinv.download(st), st);
        const std::vector<int>& off = sq.off;
        const std::vector<int>& idx = sq.idx;
        const std::vector<double>& val = sq.val;
        std::vector<int> node_of(o.n_q);
        std::vector<double> cx, cy, cz;
        if (o.nz > 0)
            face_coords3(nx, ny, o.nz, cx, cy, cz);
        else
            face_coords(nx, ny, cx, cy);
        for (int f = 0; f < o.n_q; ++f) node_of[f] = f;
        flow_use_nd = true;
        flow_nd.prof_phase = PROF_FLOW_SOLVE;
        flow_nd.factor(o.n_q, off, idx, val, node_of, cx, cy, nd_leaf_dofs(128, "PDG_ND_FLOW_LEAF"), m, st,
                       o.nz > 0 ? &cz : nullptr);
        return;
    }
    std::vector<int> perm;
    std::vector<int> bs;
    perm.reserve(o.n_q);
    for (int j = 0; j <= ny; ++j) {
        const size_t before = perm.size();
        for (int i = 0; i < nx; ++i) perm.push_back(j * nx + i);
        if (j < ny)
            for (int i = 0; i <= nx; ++i) perm.push_back(nx * (ny + 1) + i * ny + j);
        bs.push_back(static_cast<int>(perm.size() - before));
    }
    flow.prof_phase = PROF_FLOW_SOLVE;
    flow.layout(o.n_q, perm, bs);
    flow.max_rhs = m;
    DBuf<double> dense(flow.dense_total());
    dense.zero(st);
    std::vector<long long> dD(flow.nb), dC(flow.nb);
    for (int j = 0; j < flow.nb; ++j) {
        dD[j] = flow.dense_d_offset(j);
        dC[j] = flow.dense_c_offset(j);
    }
    DBuf<long long> ddD, ddC;
    ddD.upload(dD, st);
    ddC.upload(dC, st);
    DBuf<int> err(1);
    err.zero(st);
    k_flow_schur_blocks<<<grid_for(o.n_q, 256), 256, 0, st>>>(o.n_q, w, o.M_q.off.p, o.M_q.idx.p, o.M_q.val.p, o.B.off.p,
                                                               o.B.idx.p, o.B.val.p, o.Bt.off.p, o.Bt.idx.p, o.Bt.val.p,
                                                               dinv.p, flow.inv_perm.p, flow.blk_of.p, flow.loc_of.p,
                                                               flow.d_bsz.p, ddD.p, ddC.p, dense.p, err.p);
    PDG_CHECK_LAUNCH();
    int herr = 0;
    PDG_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    require(herr == 0, "fixed-stress: flow Schur complement is not block tridiagonal in face-row order");
    flow.factor_dense(dense.p, st);
}

void FixedStressPre::setup_coupled(const SpatialOps& o, int m_, double tau_, const double* theta, const double* kappa,
                                   double stab_, std::shared_ptr<ASolver> a_, cudaStream_t st) {
    require(m_ >= 1 && m_ <= kMaxC, "fixed-stress: coupled sweep supports up to 2 time components");
    ops = &o;
    m = m_;
    tau = tau_;
    stab = stab_;
    sweeps = 1;
    coupled = true;
    a = std::move(a_);
    for (int k = 0; k < m * m; ++k) th[k] = theta[k];
    for (int i = 0; i < m; ++i) wc[i] = tau * kappa[i];
    if (m == 1) {
        require(th[0] != 0.0, "fixed-stress: singular time weight");
        thinv[0] = 1.0 / th[0];
    } else {
        const double det = th[0] * th[3] - th[1] * th[2];
        require(det != 0.0, "fixed-stress: singular time weight");
        thinv[0] = th[3] / det;
        thinv[1] = -th[1] / det;
        thinv[2] = -th[2] / det;
        thinv[3] = th[0] / det;
    }
    require(o.inv_m + stab > 0.0, "fixed-stress: flow storage block must be negative definite");
    dinvc.alloc(o.n_p);
    k_dinvc<<<grid_for(o.n_p, 256), 256, 0, st>>>(o.n_p, o.inv_m + stab, o.m_p.p, dinvc.p);
    PDG_CHECK_LAUNCH();
    // face-row blocks holding both components: block j = [comp 0 faces of face row j, comp 1 ...]
    const int nx = o.nx, ny = o.ny;
    require(o.nz == 0, "fixed-stress march with coupled components: 2D meshes only");
    require(o.n_q == nx * (ny + 1) + (nx + 1) * ny, "fixed-stress: face count does not match the mesh");
    std::vector<int> perm, bs;
    for (int j = 0; j <= ny; ++j) {
        std::vector<int> faces;
        for (int i = 0; i < nx; ++i) faces.push_back(j * nx + i);
        if (j < ny)
            for (int i = 0; i <= nx; ++i) faces.push_back(nx * (ny + 1) + i * ny + j);
        for (int c = 0; c < m; ++c)
            for (int f : faces) perm.push_back(c * o.n_q + f);
        bs.push_back(static_cast<int>(m * faces.size()));
    }
    flow.prof_phase = PROF_FLOW_SOLVE;
    flow.symmetric = false;
    flow.layout(m * o.n_q, perm, bs);
    flow.max_rhs = 1;
    DBuf<double> dense(flow.dense_total());
    dense.zero(st);
    std::vector<long long> dD(flow.nb), dC(flow.nb), dU(flow.nb);
    for (int j = 0; j < flow.nb; ++j) {
        dD[j] = flow.dense_d_offset(j);
        dC[j] = flow.dense_c_offset(j);
        dU[j] = flow.dense_u_offset(j);
    }
    DBuf<long long> ddD, ddC, ddU;
    ddD.upload(dD, st);
    ddC.upload(dC, st);
    ddU.upload(dU, st);
    Mat2 wm{}, gam{};
    for (int i = 0; i < m; ++i) wm.a[i] = wc[i];
    for (int i = 0; i < m; ++i)
        for (int k = 0; k < m; ++k) gam.a[i * m + k] = wc[i] * thinv[i * m + k] * wc[k];
    DBuf<int> err(1);
    err.zero(st);
    k_flowc_schur_blocks<<<grid_for((long long)m * o.n_q, 256), 256, 0, st>>>(
        m, o.n_q, wm, gam, o.M_q.off.p, o.M_q.idx.p, o.M_q.val.p, o.B.off.p, o.B.idx.p, o.B.val.p, o.Bt.off.p,
        o.Bt.idx.p, o.Bt.val.p, dinvc.p, flow.inv_perm.p, flow.blk_of.p, flow.loc_of.p, flow.d_bsz.p, ddD.p, ddC.p,
        ddU.p, dense.p, err.p);
    PDG_CHECK_LAUNCH();
    int herr = 0;
    PDG_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    require(herr == 0, "fixed-stress: coupled flow Schur complement is not block tridiagonal in face-row order");
    flow.factor_dense(dense.p, st);
    rq.alloc((size_t)m * o.n_q);
    qtmp.alloc((size_t)m * o.n_q);
    fp.alloc((size_t)m * o.n_p);
    mech.alloc((size_t)m * o.n_u);
}

void FixedStressPre::apply(const double* r, double* z, cudaStream_t st) {
    const size_t len = (size_t)m * ops->n_total();
    for (int s = 0; s < sweeps; ++s) {
        if (s > 0) PDG_CUDA(cudaMemcpyAsync(xold.p, z, sizeof(double) * len, cudaMemcpyDeviceToDevice, st));
        sweep_once(s > 0 ? xold.p : nullptr, r, z, st);
    }
}

// One flow-then-mechanics sweep (fixed_stress.hpp:109-139) from iterate xprev
// (null = the zero iterate) into z (z must not alias xprev or r).
void FixedStressPre::sweep_once(const double* xprev, const double* r, double* z, cudaStream_t st) {
    const SpatialOps& o = *ops;
    const int nt = o.n_total(), nu = o.n_u, nq = o.n_q, np = o.n_p;
    if (coupled) {
        Mat2 wm{}, tm{}, ti{};
        for (int i = 0; i < m; ++i) wm.a[i] = wc[i];
        for (int k = 0; k < m * m; ++k) {
            tm.a[k] = th[k];
            ti.a[k] = thinv[k];
        }
        {
            ProfScope prof(PROF_PRE_OTHER, st, 0.0);
            k_fsc_fp<<<grid_for((long long)m * np, 256), 256, 0, st>>>(m, np, nt, nu, nq, xprev, tm, o.biot_b, stab, r,
                                                                       o.Et.off.p, o.Et.idx.p, o.Et.val.p, o.m_p.p, fp.p);
            k_fsc_rq<<<grid_for((long long)m * nq, 256), 256, 0, st>>>(m, nq, np, nt, nu, wm, ti, r, fp.p, o.B.off.p,
                                                                       o.B.idx.p, o.B.val.p, dinvc.p, rq.p);
            count_launch(2);
            PDG_CHECK_LAUNCH();
        }
        flow.solve(rq.p, (long long)m * nq, qtmp.p, (long long)m * nq, 1, st);
        {
            ProfScope prof(PROF_PRE_OTHER, st, 0.0);
            k_fsc_qp<<<grid_for((long long)m * (nq + np), 256), 256, 0, st>>>(m, np, nq, nt, nu, wm, ti, fp.p, qtmp.p,
                                                                              o.Bt.off.p, o.Bt.idx.p, o.Bt.val.p,
                                                                              dinvc.p, z);
            k_fsc_mech<<<grid_for((long long)m * nu, 256), 256, 0, st>>>(m, nu, nt, nq, wm, o.biot_b, r, z, o.E.off.p,
                                                                         o.E.idx.p, o.E.val.p, mech.p);
            count_launch(2);
            PDG_CHECK_LAUNCH();
        }
        a->solve(mech.p, nu, z, nt, m, st);
        return;
    }
    const int lag = xprev != nullptr;
    // first sweep (lag = 0): fp is r_p itself, read in place (no copy kernel)
    const double* fpb = r + nu + nq;
    long long fps = nt;
    {
        ProfScope prof(PROF_PRE_OTHER, st, 8.0 * m * (2.0 * np + 2.0 * nq + 3.0 * o.B.nnz));
        if (lag) {
            k_flow_fp<<<grid_for((long long)m * np, 256), 256, 0, st>>>(m, np, nt, nu, nq, lag, lambda, o.biot_b, stab, r,
                                                                        xprev, o.Et.off.p, o.Et.idx.p, o.Et.val.p, o.m_p.p,
                                                                        fp.p, guard);
            count_launch();
            fpb = fp.p;
            fps = np;
        }
        k_flow_rq<<<grid_for((long long)m * nq, 256), 256, 0, st>>>(m, nq, np, nt, nu, w, r, fpb, fps, o.B.off.p, o.B.idx.p,
                                                                    o.B.val.p, dinv.p, rq.p, guard);
        count_launch();
        PDG_CHECK_LAUNCH();
    }
    if (flow_use_nd)
        flow_nd.solve(rq.p, nq, z + nu, nt, m, st);
    else
        flow.solve(rq.p, nq, z + nu, nt, m, st);
    {
        ProfScope prof(PROF_PRE_OTHER, st, 8.0 * m * (3.0 * np + 2.0 * o.Bt.nnz + 2.0 * nu + 2.0 * o.E.nnz));
        k_flow_p<<<grid_for((long long)m * np, 256), 256, 0, st>>>(m, np, nt, nu, nq, w, fpb, fps, o.Bt.off.p, o.Bt.idx.p,
                                                                   o.Bt.val.p, dinv.p, z, guard);
        k_mech_rhs<<<grid_for((long long)m * nu, 256), 256, 0, st>>>(m, nu, nt, nq, w, o.biot_b, r, z, o.E.off.p,
                                                                     o.E.idx.p, o.E.val.p, mech.p, guard);
        count_launch(2);
        PDG_CHECK_LAUNCH();
    }
    a->solve(mech.p, nu, z, nt, m, st);
}

void Gmres::setup(long long n_, int restart_, bool keep_z, cudaStream_t st) {
    n = n_;
    restart = restart_;
    V.alloc((size_t)n * (restart + 1));
    if (keep_z) {
        Z.alloc((size_t)n * restart);
        AZ.alloc((size_t)n * restart);
        r0.alloc(n);
    }
    w.alloc(n);
    x.alloc(n);
    r.alloc(n);
    cand.alloc(n);
    t.alloc(n);
    y_dev.alloc(restart + 2);
    h_dev.alloc(2 * (restart + 2));
    partial.alloc((size_t)3 * kRedBlocks * (restart + 2));  // three regions for the fused Arnoldi kernel
    norm_dev.alloc(4);
    if (!h_host) PDG_CUDA(cudaMallocHost(&h_host, sizeof(double) * (2 * restart + 8)));
    if (keep_z) {
        Hd.alloc((size_t)(restart + 1) * restart);
        lstate.alloc(2);  // one LoopState
        givens.alloc((size_t)3 * (restart + 1));  // cs, sn, g
        if (!h_slots) PDG_CUDA(cudaMallocHost(&h_slots, sizeof(LoopState) * (restart + 1)));
        for (auto& e : evs)
            if (!e) PDG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    (void)st;
}
Gmres::~Gmres() {
    if (h_host) cudaFreeHost(h_host);
    if (h_slots) cudaFreeHost(h_slots);
    for (auto& e : evs)
        if (e) cudaEventDestroy(e);
}

void Block::create(const SpatialOps& o, int m_, const double* th, double tau_, double lambda_, const pdg_gmres_opts& op_,
                   std::shared_ptr<ASolver> a) {
    ops = &o;
    ctx = o.ctx;
    m = m_;
    tau = tau_;
    lambda = lambda_;
    theta.assign(th, th + m * m);
    opts = op_;
    require(opts.tol > 0.0 && opts.tol < 1.0, "gmres: tol must be in (0,1)");
    require(opts.restart >= 1 && opts.max_iter >= 1, "gmres: bad iteration limits");
    require(tau > 0.0, "FixedStressSolver: tau must be positive");
    cudaStream_t st = ctx->stream;
    SetupTimer total(SETUP_SOLVER_TOTAL, st);
    {
        SetupTimer t(SETUP_OPERATOR, st);
        op.build(o, m, th, tau, st);
    }
    const double stab = opts.stab < 0.0 ? o.biot_b * o.biot_b / o.k_dr : opts.stab;
    require(stab >= 0.0, "fixed-stress: stabilization must be nonnegative");
    if (!a) a = make_a_solver(o, 2, st);
    pre.setup(o, m, tau, lambda, stab, opts.sweeps, a, st);
    kr.setup(rows(), opts.restart, opts.candidate == 1, st);
    kr.spmv_blocks = op.dots_grid();
    kr.spmv_part.alloc((size_t)kr.spmv_blocks * 8);
    PDG_CUDA(cudaEventCreate(&ev0));
    PDG_CUDA(cudaEventCreate(&ev1));
    PDG_CUDA(cudaStreamSynchronize(st));
}

Block::~Block() {
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
}

namespace {
struct KrylovOps {
    cudaStream_t st;
    Gmres& g;
    unsigned gr;  // elementwise grid (a few blocks per SM)
    // partials of V_j . w for j < ncols
    void dots(const double* V, int ncols, const double* w) {
        ProfScope prof(PROF_KRYLOV, st, 8.0 * (double)g.n * (ncols + 1));
        k_multidot1<<<kRedBlocks, kRedThreads, 0, st>>>(g.n, ncols, V, w, g.partial.p);
        count_launch();
        PDG_CHECK_LAUNCH();
    }
    // one Gram-Schmidt pass: h_out = V^T w (device), w -= V h
    void gs_pass(const double* V, int ncols, double* w, double* h_out) {
        dots(V, ncols, w);
        ProfScope prof(PROF_KRYLOV, st, 8.0 * (double)g.n * (ncols + 2));
        k_red_multiaxpy<<<gr, kRedThreads, sizeof(double) * ncols, st>>>(g.n, ncols, g.partial.p, V, w, h_out);
        count_launch();
        PDG_CHECK_LAUNCH();
    }
    // norm of v into g.norm_dev (device); dst = v / norm when dst != null
    void norm_dev(const double* v, double* dst) {
        dots(v, 1, v);
        ProfScope prof(PROF_KRYLOV, st, dst ? 16.0 * (double)g.n : 0.0);
        k_red_norm_scale<<<dst ? gr : 1, kRedThreads, 0, st>>>(g.n, g.partial.p, v, dst, g.norm_dev.p);
        count_launch();
        PDG_CHECK_LAUNCH();
    }
    // r = b - t and ||r|| on the host
    double sub_norm(const double* b, const double* t, double* r) {
        {
            ProfScope prof(PROF_KRYLOV, st, 24.0 * (double)g.n);
            k_sub_dot<<<kRedBlocks, kRedThreads, 0, st>>>(g.n, b, t, r, g.partial.p);
            k_red_norm_scale<<<1, kRedThreads, 0, st>>>(g.n, g.partial.p, r, nullptr, g.norm_dev.p);
            count_launch(2);
            PDG_CHECK_LAUNCH();
        }
        return fetch_norm();
    }
    double norm(const double* v) {
        norm_dev(v, nullptr);
        return fetch_norm();
    }
    // both Gram-Schmidt passes + the norm + v_{k+1} = w / ||w|| in ONE cooperative launch
    // (bit-identical to gs_pass x 2 + norm_dev); h_out[0 .. 2 ncols] as the unfused sequence
    void gs_fused(const double* V, int ncols, double* w, double* h_out, double* vnext, LoopState* ls = nullptr,
                  const double* pre1 = nullptr, int nb1 = 0, double* Hcol = nullptr, double* cs = nullptr,
                  double* sn = nullptr, double* gv = nullptr, int mm = 0, double tolb = 0.0) {
        ProfScope prof(PROF_KRYLOV, st, 8.0 * (double)g.n * (3.0 * ncols + 6.0 - (pre1 ? ncols + 1.0 : 0.0)));
        long long n = g.n;
        double* part = g.partial.p;
        void* args[] = {&n,   &ncols,       (void*)&V, &w,  &part, &h_out, &vnext, (void*)&ls,
                        (void*)&pre1, &nb1, &Hcol,     &cs, &sn,   &gv,    &mm,    &tolb};
        PDG_CUDA(cudaLaunchCooperativeKernel((void*)k_arnoldi_gs, kRedBlocks, kRedThreads, args, sizeof(double) * ncols, st));
        count_launch();
        PDG_CHECK_LAUNCH();
    }
    // r = r0 - AZ y and ||r|| (bit-identical to k_combine + sub_norm), on the host
    void residual_launch(const double* AZ, int ncols, const double* y, const double* r0, double* r) {
        ProfScope prof(PROF_KRYLOV, st, 8.0 * (double)g.n * (ncols + 2.0));
        long long n = g.n;
        double* part = g.partial.p;
        double* nrm = g.norm_dev.p;
        void* args[] = {&n, &ncols, (void*)&AZ, (void*)&y, (void*)&r0, &r, &part, &nrm};
        PDG_CUDA(cudaLaunchCooperativeKernel((void*)k_arnoldi_residual, kRedBlocks, kRedThreads, args, 0, st));
        count_launch();
        PDG_CHECK_LAUNCH();
    }
    double residual_fused(const double* AZ, int ncols, const double* y, const double* r0, double* r) {
        residual_launch(AZ, ncols, y, r0, r);
        return fetch_norm();
    }
    double fetch_norm() {
        PDG_CUDA(cudaMemcpyAsync(g.h_host, g.norm_dev.p, sizeof(double), cudaMemcpyDeviceToHost, st));
        PDG_CUDA(cudaStreamSynchronize(st));
        return g.h_host[0];
    }
};
}  // namespace

void Block::solve(const double* b, double* x_out, pdg_report* rep, int block_index) {
    cudaStream_t st = ctx->stream;
    const long long n = rows();
    const unsigned gr = grid_for(n, 256);
    const long long launches0 = g_launches;
    KrylovOps K{st, kr, static_cast<unsigned>(2 * num_sms())};
    PDG_CUDA(cudaEventRecord(ev0, st));
    std::vector<double> hist;
    const double bnorm = K.norm(b);
    bool converged = false;
    int total = 0;
    double true_res = bnorm;
    auto finish = [&](double final_rel) {
        PDG_CUDA(cudaEventRecord(ev1, st));
        PDG_CUDA(cudaEventSynchronize(ev1));
        float ms = 0.f;
        PDG_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
        if (rep) {
            rep->converged = converged;
            rep->iterations = total;
            rep->final_rel_res = final_rel;
            rep->history_len = static_cast<int>(hist.size());
            if (rep->history)
                for (int i = 0; i < std::min<int>(rep->history_cap, (int)hist.size()); ++i) rep->history[i] = hist[i];
            rep->device_ms = ms;
            rep->kernel_launches = static_cast<int>(g_launches - launches0);
        }
    };
    if (bnorm <= 1e-14) {  // gmres.hpp:56-62
        PDG_CUDA(cudaMemsetAsync(x_out, 0, sizeof(double) * n, st));
        converged = true;
        hist.push_back(bnorm);
        finish(0.0);
        return;
    }
    PDG_CUDA(cudaMemsetAsync(kr.x.p, 0, sizeof(double) * n, st));
    hist.push_back(true_res);
    const int restart = opts.restart, max_iter = opts.max_iter;
    const bool flexible = opts.candidate == 1;
    // flexible: the true residual of x + Z y is r0 - (A Z) y, from the op(z_j) products the
    // Arnoldi step already formed (A linear): no second operator application per iteration
    const bool arnoldi_res = flexible && !std::getenv("PDG_GMRES_EXPLICIT_RESIDUAL");
    // fused cooperative Arnoldi kernels (default); PDG_KRYLOV_UNFUSED=1 selects the launch-per-step
    // sequence they replace (bit-identical results, kept for the A/B test)
    const bool fused = !std::getenv("PDG_KRYLOV_UNFUSED");
    const bool spmv_dots = fused && !(std::getenv("PDG_SPMV_DOTS") && std::atoi(std::getenv("PDG_SPMV_DOTS")) == 0);
    // flexible candidate (default): device-driven steps with the Givens residual estimate
    // (below); PDG_GMRES_HOST_LOOP=1 selects the host-driven loop (Arnoldi-relation residual
    // per step, two host round trips per step), also used by the reference candidate
    const bool devloop = flexible && fused && !(std::getenv("PDG_GMRES_HOST_LOOP") && std::atoi(std::getenv("PDG_GMRES_HOST_LOOP")) > 0);
    std::vector<double> H;
    bool x_is_zero = true;
    while (total < max_iter) {
        double beta;
        if (x_is_zero) {  // r = b - op(0) = b exactly, so ||r|| is ||b|| (same kernels, same bits)
            PDG_CUDA(cudaMemcpyAsync(kr.r.p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
            beta = bnorm;
        } else {
            op.apply(kr.x.p, kr.t.p, st);
            beta = K.sub_norm(b, kr.t.p, kr.r.p);
        }
        if (beta / bnorm <= opts.tol) break;
        const int mm = std::min(restart, max_iter - total);
        H.assign((size_t)(mm + 1) * mm, 0.0);
        auto h = [&](int i, int j) -> double& { return H[(size_t)j * (mm + 1) + i]; };
        // v_0 = r / beta (beta recomputed on the device by the same fixed tree)
        K.norm_dev(kr.r.p, kr.V.p);
        if (arnoldi_res && !devloop) PDG_CUDA(cudaMemcpyAsync(kr.r0.p, kr.r.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
        if (devloop) {
            // Device-driven steps: step k (preconditioner, SpMV + first-pass dots, Gram-Schmidt
            // with the Givens residual estimate) is queued before step k - 1's stop flag is read,
            // so the GPU never waits for the host inside a cycle; a step queued after the cycle
            // ended exits at entry on the device (guard). At the stop, the host solves the
            // least squares (ColPivHouseholderQR, gmres.hpp:111) on the downloaded Hessenberg
            // columns and confirms on the explicit true residual (gmres.hpp:68-72); if that
            // fails before the cycle's end, the cycle goes on (gmres.hpp:118-131).
            LoopState* lsd = reinterpret_cast<LoopState*>(kr.lstate.p);
            LoopState* slots = static_cast<LoopState*>(kr.h_slots);
            double* cs = kr.givens.p;
            double* sn = cs + (restart + 1);
            double* gv = sn + (restart + 1);
            PDG_CUDA(cudaMemsetAsync(kr.lstate.p, 0, sizeof(LoopState), st));
            // the columns are written down to the subdiagonal only: the rest of H is zero
            PDG_CUDA(cudaMemsetAsync(kr.Hd.p, 0, sizeof(double) * (size_t)(mm + 1) * mm, st));
            kr.h_host[0] = beta;
            PDG_CUDA(cudaMemcpyAsync(gv, kr.h_host, sizeof(double), cudaMemcpyHostToDevice, st));
            auto set_guard = [&](const int* gp) {
                op.guard = gp;
                pre.guard = gp;
                pre.flow_nd.guard = gp;
                if (pre.a) pre.a->nd.guard = gp;
            };
            set_guard(&lsd->stop);
            const double tolb = opts.tol * bnorm;
            const bool no_lookahead = std::getenv("PDG_GMRES_NO_LOOKAHEAD") != nullptr;
            static const bool predict = !(std::getenv("PDG_GMRES_PREDICT") && std::atoi(std::getenv("PDG_GMRES_PREDICT")) == 0);
            auto step = [&](int k) {
                double* vk = kr.V.p + (size_t)k * n;
                double* zk = kr.Z.p + (size_t)k * n;
                pre.apply(vk, zk, st);
                double* Hcol = kr.Hd.p + (size_t)k * (mm + 1);
                if (spmv_dots && k + 1 <= 8) {  // w and the first Gram-Schmidt pass's partials in the SpMV
                    op.apply_dots(zk, kr.w.p, nullptr, kr.V.p, k + 1, kr.spmv_part.p, st);
                    K.gs_fused(kr.V.p, k + 1, kr.w.p, kr.h_dev.p, kr.V.p + (size_t)(k + 1) * n, lsd, kr.spmv_part.p,
                               kr.spmv_blocks, Hcol, cs, sn, gv, mm, tolb);
                } else {
                    op.apply(zk, kr.w.p, st);
                    K.gs_fused(kr.V.p, k + 1, kr.w.p, kr.h_dev.p, kr.V.p + (size_t)(k + 1) * n, lsd, nullptr, 0, Hcol,
                               cs, sn, gv, mm, tolb);
                }
                PDG_CUDA(cudaMemcpyAsync(slots + k, lsd, sizeof(LoopState), cudaMemcpyDeviceToHost, st));
                PDG_CUDA(cudaEventRecord(kr.evs[k & 1], st));
            };
            const int left = max_iter - total;  // == mm unless the iteration limit cuts the cycle
            int k0 = 0;
            for (;;) {
                int kend = -1;
                const double beta_k0 = k0 > 0 ? slots[k0 - 1].res : beta;  // residual estimate before step k0
                for (int k = k0; k < mm; ++k) {
                    step(k);  // queued behind step k - 1: skipped on the device if k - 1 ended the cycle
                    if (no_lookahead) {
                        PDG_CUDA(cudaEventSynchronize(kr.evs[k & 1]));
                        if (slots[k].stop) {
                            kend = k;
                            break;
                        }
                    } else if (k > k0) {
                        PDG_CUDA(cudaEventSynchronize(kr.evs[(k - 1) & 1]));
                        if (slots[k - 1].stop) {
                            kend = k - 1;
                            break;
                        }
                        // predicted stop: when the residual estimate extrapolated from the last two
                        // steps reaches the tolerance at step k, wait for step k instead of queuing
                        // step k + 1 speculatively (a skipped step still costs its launches on the
                        // GPU; a wrong prediction costs one host round trip). Same iterates either way.
                        if (predict && k + 1 < mm) {
                            const double r1 = slots[k - 1].res, r0 = k - 1 > k0 ? slots[k - 2].res : beta_k0;
                            if (r0 > 0.0 && r1 * (r1 / r0) <= 4.0 * tolb) {
                                PDG_CUDA(cudaEventSynchronize(kr.evs[k & 1]));
                                if (slots[k].stop) {
                                    kend = k;
                                    break;
                                }
                            }
                        }
                    }
                }
                if (kend < 0) {
                    PDG_CUDA(cudaEventSynchronize(kr.evs[(mm - 1) & 1]));
                    for (int k = k0; k < mm; ++k)
                        if (slots[k].stop) {
                            kend = k;
                            break;
                        }
                    if (kend < 0) kend = mm - 1;
                }
                set_guard(nullptr);  // the explicit check below must run with the stop flag set
                for (int k = k0; k < kend; ++k) hist.push_back(slots[k].res);
                total += kend + 1 - k0;
                // least squares on the Hessenberg columns 0..kend (host, as gmres.hpp:110-111)
                const int kk = kend + 1;
                std::vector<double> hk((size_t)(kk + 1) * kk);
                PDG_CUDA(cudaMemcpy2DAsync(hk.data(), sizeof(double) * (kk + 1), kr.Hd.p, sizeof(double) * (mm + 1),
                                           sizeof(double) * (kk + 1), kk, cudaMemcpyDeviceToHost, st));
                PDG_CUDA(cudaStreamSynchronize(st));
                std::vector<double> e1(kk + 1, 0.0);
                e1[0] = beta;
                const std::vector<double> y = ls_colpiv(hk, kk + 1, kk, e1);
                PDG_CUDA(cudaMemcpyAsync(kr.y_dev.p, y.data(), sizeof(double) * kk, cudaMemcpyHostToDevice, st));
                { ProfScope prof_(PROF_KRYLOV, st, 0.0); k_combine<<<gr, 256, 0, st>>>(n, kk, kr.Z.p, kr.y_dev.p, kr.x.p, kr.cand.p); }
                count_launch();
                op.apply(kr.cand.p, kr.t.p, st);
                true_res = K.sub_norm(b, kr.t.p, kr.r.p);
                converged = true_res / bnorm <= opts.tol;
                hist.push_back(true_res);
                const bool cycle_end = slots[kend].brk || kend == mm - 1 || kend + 1 >= left;
                if (std::getenv("PDG_GMRES_TRACE")) {
                    std::fprintf(stderr, "gmres devloop: k0 %d kend %d mm %d beta %.6e bnorm %.6e |", k0, kend, mm, beta, bnorm);
                    for (int k = k0; k <= kend; ++k) std::fprintf(stderr, " %.3e", slots[k].res / bnorm);
                    std::fprintf(stderr, " | explicit %.3e brk %d", true_res / bnorm, slots[kend].brk);
                    std::fprintf(stderr, "\n");
                }
                if (converged || cycle_end) break;
                // the estimate passed but the explicit residual did not: the cycle goes on
                PDG_CUDA(cudaMemsetAsync(&lsd->stop, 0, sizeof(int), st));
                set_guard(&lsd->stop);
                k0 = kend + 1;
            }
            PDG_CUDA(cudaMemcpyAsync(kr.x.p, kr.cand.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
            x_is_zero = false;
            if (converged) break;
            continue;
        }
        bool done = false;
        for (int k = 0; k < mm && !done; ++k) {
            double* vk = kr.V.p + (size_t)k * n;
            double* zk = flexible ? kr.Z.p + (size_t)k * n : kr.cand.p;
            pre.apply(vk, zk, st);
            // fused (default, up to 8 basis vectors): the SpMV epilogue forms w and the first
            // Gram-Schmidt pass's partial dots (PDG_SPMV_DOTS=0: separate passes)
            const bool dots = fused && spmv_dots && k + 1 <= 8;
            if (arnoldi_res) {
                double* azk = kr.AZ.p + (size_t)k * n;
                if (dots) {
                    op.apply_dots(zk, azk, kr.w.p, kr.V.p, k + 1, kr.spmv_part.p, st);
                } else {
                    op.apply(zk, azk, st);
                    PDG_CUDA(cudaMemcpyAsync(kr.w.p, azk, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
                }
            } else if (dots) {
                op.apply_dots(zk, kr.w.p, nullptr, kr.V.p, k + 1, kr.spmv_part.p, st);
            } else {
                op.apply(zk, kr.w.p, st);
            }
            // classical Gram-Schmidt, two passes, and the new norm, all on the device;
            // the Hessenberg column comes back in ONE transfer
            // h(k+1,k) = ||w|| and v_{k+1} = w / h(k+1,k) (unused when the column breaks down)
            if (fused) {
                K.gs_fused(kr.V.p, k + 1, kr.w.p, kr.h_dev.p, kr.V.p + (size_t)(k + 1) * n, nullptr,
                           dots ? kr.spmv_part.p : nullptr, kr.spmv_blocks);
                PDG_CUDA(cudaMemcpyAsync(kr.h_host, kr.h_dev.p, sizeof(double) * (2 * (k + 1) + 1), cudaMemcpyDeviceToHost, st));
            } else {
                for (int pass = 0; pass < 2; ++pass) K.gs_pass(kr.V.p, k + 1, kr.w.p, kr.h_dev.p + (size_t)pass * (k + 1));
                K.norm_dev(kr.w.p, kr.V.p + (size_t)(k + 1) * n);
                PDG_CUDA(cudaMemcpyAsync(kr.h_host, kr.h_dev.p, sizeof(double) * 2 * (k + 1), cudaMemcpyDeviceToHost, st));
                PDG_CUDA(cudaMemcpyAsync(kr.h_host + 2 * (k + 1), kr.norm_dev.p, sizeof(double), cudaMemcpyDeviceToHost, st));
            }
            PDG_CUDA(cudaStreamSynchronize(st));
            for (int pass = 0; pass < 2; ++pass)
                for (int i = 0; i <= k; ++i) h(i, k) += kr.h_host[(size_t)pass * (k + 1) + i];
            h(k + 1, k) = kr.h_host[2 * (k + 1)];
            double cn = 0.0;
            for (int i = 0; i <= mm; ++i) cn += h(i, k) * h(i, k);
            const bool breakdown = h(k + 1, k) <= 1e-14 * std::sqrt(cn);
            ++total;
            std::vector<double> hk((size_t)(k + 2) * (k + 1));
            for (int j = 0; j <= k; ++j)
                for (int i = 0; i < k + 2; ++i) hk[(size_t)j * (k + 2) + i] = h(i, j);
            std::vector<double> e1(k + 2, 0.0);
            e1[0] = beta;
            const std::vector<double> y = ls_colpiv(hk, k + 2, k + 1, e1);
            PDG_CUDA(cudaMemcpyAsync(kr.y_dev.p, y.data(), sizeof(double) * (k + 1), cudaMemcpyHostToDevice, st));
            if (flexible) {  // cand = x + Z y (with the Arnoldi residual: formed when the cycle ends)
                if (!arnoldi_res) {
                    { ProfScope prof_(PROF_KRYLOV, st, 0.0); k_combine<<<gr, 256, 0, st>>>(n, k + 1, kr.Z.p, kr.y_dev.p, kr.x.p, kr.cand.p); }
                    count_launch();
                }
            } else {  // cand = x + P(V y)   (gmres.hpp:116)
                { ProfScope prof_(PROF_KRYLOV, st, 0.0); k_combine<<<gr, 256, 0, st>>>(n, k + 1, kr.V.p, kr.y_dev.p, nullptr, kr.t.p); }
                count_launch();
                pre.apply(kr.t.p, kr.r.p, st);
                { ProfScope prof_(PROF_KRYLOV, st, 0.0); k_add<<<gr, 256, 0, st>>>(n, kr.x.p, kr.r.p, kr.cand.p); }
                count_launch();
            }
            // true residual (gmres.hpp:68-72)
            if (arnoldi_res && fused) {
                true_res = K.residual_fused(kr.AZ.p, k + 1, kr.y_dev.p, kr.r0.p, kr.r.p);
            } else if (arnoldi_res) {
                { ProfScope prof_(PROF_KRYLOV, st, 0.0); k_combine<<<gr, 256, 0, st>>>(n, k + 1, kr.AZ.p, kr.y_dev.p, nullptr, kr.t.p); }
                count_launch();
                true_res = K.sub_norm(kr.r0.p, kr.t.p, kr.r.p);
            } else {
                op.apply(kr.cand.p, kr.t.p, st);
                true_res = K.sub_norm(b, kr.t.p, kr.r.p);
            }
            bool ok = true_res / bnorm <= opts.tol;
            const bool cycle_end = breakdown || k == mm - 1 || total >= max_iter;
            if (ok && arnoldi_res) {
                // the Arnoldi-relation residual passed: the stop is decided on the explicit
                // true residual b - op(x + Z y), as gmres.hpp:68-72
                { ProfScope prof_(PROF_KRYLOV, st, 0.0); k_combine<<<gr, 256, 0, st>>>(n, k + 1, kr.Z.p, kr.y_dev.p, kr.x.p, kr.cand.p); }
                count_launch();
                op.apply(kr.cand.p, kr.t.p, st);
                true_res = K.sub_norm(b, kr.t.p, kr.r.p);
                ok = true_res / bnorm <= opts.tol;
            } else if (!ok && cycle_end && arnoldi_res) {
                // breakdown / full cycle / iteration limit: x = cand (gmres.hpp:123-130) and the
                // recorded residual is the explicit one
                { ProfScope prof_(PROF_KRYLOV, st, 0.0); k_combine<<<gr, 256, 0, st>>>(n, k + 1, kr.Z.p, kr.y_dev.p, kr.x.p, kr.cand.p); }
                count_launch();
                op.apply(kr.cand.p, kr.t.p, st);
                true_res = K.sub_norm(b, kr.t.p, kr.r.p);
                ok = true_res / bnorm <= opts.tol;
            }
            // gmres.hpp:118-131: accept on the true residual; otherwise the cycle goes on
            // unless it broke down, is full or hit the iteration limit
            if (ok || cycle_end) {
                PDG_CUDA(cudaMemcpyAsync(kr.x.p, kr.cand.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
                x_is_zero = false;
                done = true;
                converged = ok;
            }
            hist.push_back(true_res);
        }
        if (converged) break;
    }
    const double final_rel = true_res / bnorm;
    if (!converged) converged = final_rel <= opts.tol;
    PDG_CUDA(cudaMemcpyAsync(x_out, kr.x.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    finish(final_rel);
    if (!converged) {
        char buf[64];
        std::snprintf(buf, sizeof(buf), "%f", final_rel);
        throw Error(PDG_NOT_CONVERGED,
                    "slab block " + std::to_string(block_index) + ": GMRES did not converge (rel res " + buf + ")");
    }
}

void FsSolver::create(const SpatialOps& o, int r, double tau_, double stab, std::shared_ptr<ASolver> a) {
    require(r == 0 || r == 1, "fixed-stress solver: dG(r) with r <= 1 on the device");
    require(tau_ > 0.0, "FixedStressSolver: tau must be positive");
    stab = stab < 0.0 ? o.biot_b * o.biot_b / o.k_dr : stab;  // FixedStressConfig::resolve_stab
    require(stab >= 0.0, "fixed-stress: stabilization must be nonnegative");
    ctx = o.ctx;
    ops = &o;
    m = r + 1;
    tau = tau_;
    cudaStream_t st = ctx->stream;
    SetupTimer total(SETUP_SOLVER_TOTAL, st);
    const TimeConsts tc = time_consts(r);  // Theta = G_hat, kappa = weights (both [1] for r = 0)
    {
        SetupTimer t(SETUP_OPERATOR, st);
        op.build(o, m, tc.G.data(), tau, st, tc.weights.data());
    }
    if (!a) a = make_a_solver(o, 2, st);
    if (m == 1)
        pre.setup(o, m, tau, tc.G[0], stab, 1, a, st);
    else
        pre.setup_coupled(o, m, tau, tc.G.data(), tc.weights.data(), stab, a, st);
    const long long n = (long long)m * o.n_total();
    red.setup(n, 1, false, st);
    xa.alloc(n);
    xb.alloc(n);
    t.alloc(n);
    this->r.alloc(n);
    PDG_CUDA(cudaEventCreate(&ev0));
    PDG_CUDA(cudaEventCreate(&ev1));
    PDG_CUDA(cudaStreamSynchronize(st));
}

FsSolver::~FsSolver() {
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
}

void FsSolver::solve(const double* rhs, const double* x0, double* x_out, double tol, int max_sweeps, pdg_report* rep) {
    require(tol > 0.0 && tol < 1.0, "fixed-stress: tol must be in (0,1)");
    require(max_sweeps >= 1, "fixed-stress: sweep counts must be >= 1");
    cudaStream_t st = ctx->stream;
    const long long n = (long long)m * ops->n_total();
    const long long launches0 = g_launches;
    KrylovOps K{st, red, static_cast<unsigned>(2 * num_sms())};
    PDG_CUDA(cudaEventRecord(ev0, st));
    std::vector<double> hist;
    double* x = xa.p;
    double* xn = xb.p;
    if (x0)
        PDG_CUDA(cudaMemcpyAsync(x, x0, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    else
        PDG_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, st));
    auto residual = [&](const double* v) {
        op.apply(v, t.p, st);
        return K.sub_norm(rhs, t.p, r.p);
    };
    const double rnorm = K.norm(rhs);
    bool converged = false;
    int iters = 0;
    double final_rel = 0.0;
    if (rnorm <= 1e-14) {  // fixed_stress.hpp:154-159
        hist.push_back(residual(x));
        converged = true;
        PDG_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, st));
    } else {
        double res = residual(x);
        hist.push_back(res);
        for (int k = 0; k < max_sweeps; ++k) {
            pre.sweep_once(x, rhs, xn, st);
            std::swap(x, xn);
            ++iters;
            res = residual(x);
            hist.push_back(res);
            if (res / rnorm <= tol) {
                converged = true;
                break;
            }
        }
        final_rel = res / rnorm;
    }
    PDG_CUDA(cudaMemcpyAsync(x_out, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    PDG_CUDA(cudaEventRecord(ev1, st));
    PDG_CUDA(cudaEventSynchronize(ev1));
    float ms = 0.f;
    PDG_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    if (rep) {
        rep->converged = converged;
        rep->iterations = iters;
        rep->final_rel_res = final_rel;
        rep->history_len = static_cast<int>(hist.size());
        if (rep->history)
            for (int i = 0; i < std::min<int>(rep->history_cap, (int)hist.size()); ++i) rep->history[i] = hist[i];
        rep->device_ms = ms;
        rep->kernel_launches = static_cast<int>(g_launches - launches0);
    }
    if (!converged) {
        char buf[64];
        std::snprintf(buf, sizeof(buf), "%f", final_rel);
        throw Error(PDG_NOT_CONVERGED, std::string("fixed-stress did not converge (rel res ") + buf + ")");
    }
}

}  // namespace pdg
