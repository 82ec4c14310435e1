// General mode of the block-tridiagonal solver (any coupling pattern; used
// for the flow Schur complement in face-row order), one persistent kernel per
// solve. The block chain is cut into P "virtual strips" separated by single
// separator blocks (substructuring, exact):
//   1. every strip interior is solved by its own twisted Cholesky sweep (two
//      chains per strip, all 2P chains concurrent): y_I = A_II^{-1} b_I;
//   2. separator right-hand sides g_s = b_s - A_{s,s-1} y_{s-1} - A_{s,s+1} y_{s+1};
//   3. the separator system S x_S = g (S = A_SS - A_SI A_II^{-1} A_IS, block
//      tridiagonal over the P-1 separators, factored at setup) by a twisted sweep;
//   4. x_I = y_I - W x_S with the spikes W = A_II^{-1} A_IS (precomputed).
// A solve has about nb/P + P dependent steps instead of nb (P = 1: the plain
// twisted sweep). Every step is "outputs = [b +] M_s * [seg0; seg1]" with a
// precomputed row-major step matrix; for a twisted system with Cholesky factors
// (top L_j, K_j = L_{j+1,j}; bottom L'_j, K'_j = L_{j-1,j}; twist L_t, Linv = L^{-1}):
//   top forward      y_j = [Linv_j | -Linv_j K_{j-1}] [b_j; y_{j-1}]
//   bottom forward   y_j = [Linv'_j | -Linv'_j K'_{j+1}] [b_j; y_{j+1}]
//   twist parts      p_top = [Linv_t | -Linv_t K_{t-1}] [b_t; y_{t-1}],  p_bot = -Linv_t K'_{t+1} y_{t+1}
//   twist            x_t = [Linv_t^T | Linv_t^T] [p_top; p_bot]
//   top backward     x_j = [Linv_j^T | -Linv_j^T K_j^T] [y_j; x_{j+1}]
//   bottom backward  x_j = [Linv'_j^T | -Linv'_j^T K'_j^T] [y_j; x_{j-1}]
// (the same factors and roundoff class as a forward/backward substitution).
#include <algorithm>
#include <cstdlib>

#include "blocktri.cuh"
#include "llsync.cuh"

namespace pdg {

using namespace dev;

#define PDG_CUSOLVER_D(call)                                                                                        \
    do {                                                                                                            \
        cusolverStatus_t s_ = (call);                                                                               \
        if (s_ != CUSOLVER_STATUS_SUCCESS)                                                                          \
            throw ::pdg::Error(PDG_CUDA_ERROR, std::string(#call) + ": cusolver status " + std::to_string((int)s_)); \
    } while (0)
#define PDG_CUBLAS_D(call)                                                                                        \
    do {                                                                                                          \
        cublasStatus_t s_ = (call);                                                                               \
        if (s_ != CUBLAS_STATUS_SUCCESS)                                                                          \
            throw ::pdg::Error(PDG_CUDA_ERROR, std::string(#call) + ": cublas status " + std::to_string((int)s_)); \
    } while (0)

namespace {

constexpr int DNI = 5;  // input columns per thread: c = tid + 256 i (inputs <= 1280)

__global__ void k_identity_cm(int m, double* a) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * m;
         t += (long long)gridDim.x * blockDim.x)
        a[t] = (t % m == t / m) ? 1.0 : 0.0;
}

// (P I)[r, c] = (c == perm[r]), col-major m x m
__global__ void k_perm_identity(int m, const int* perm, double* a) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * m;
         t += (long long)gridDim.x * blockDim.x) {
        const int r = static_cast<int>(t % m), c = static_cast<int>(t / m);
        a[t] = perm[r] == c ? 1.0 : 0.0;
    }
}

// Sum of 16 per-lane values across the warp, reduce-scatter style: on return
// lanes 2i and 2i+1 hold the warp total of index i (fixed order).
__device__ __forceinline__ double warp_reduce_scatter16(double (&v)[16], int lane) {
#pragma unroll
    for (int o = 16, h = 8; o >= 2; o >>= 1, h >>= 1) {
        const bool up = lane & o;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const double send = up ? v[i] : v[i + h];
            const double keep = up ? v[i + h] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    const double other = __shfl_xor_sync(0xffffffffu, v[0], 1);
    return (lane & 1) ? other + v[0] : v[0] + other;
}

// One persistent kernel per solve. CTAs [0, g) run the top chain, [g, 2g) the
// bottom chain; CTA i owns output rows [8 i, 8 i + 8) of every step. Each
// thread owns input columns c = tid + 256 i: it polls exactly their LL lines
// (warp-uniform rounds) and multiplies them into its partial sums; the step's
// 8 matrix rows stream into a shared-memory ring (cp.async.bulk, one full
// mbarrier per slot, refilled by one elected thread) behind an L2 prefetch
// `pf` steps ahead. Warp 0 sums the 8 warp partials in fixed order and
// publishes the outputs as LL lines.
__global__ void __launch_bounds__(256, 1)
    k_sweep_dense(int nsteps, const DenseTask* __restrict__ sched_g, int nrhs, int n, const double* __restrict__ store,
                  int ldmax, const double* __restrict__ b, double* __restrict__ x, uint4* ll, long long lln,
                  unsigned flag, int stages, int pf, int g, int nchains, unsigned long long* dbg) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* ring = reinterpret_cast<double*>(smem_raw);  // [stages][8 rows][ldmax]
    double* red = ring + (size_t)stages * 8 * ldmax;      // [8 warps][16]
    unsigned long long* full = reinterpret_cast<unsigned long long*>(red + 8 * 16);
    DenseTask* tsh = reinterpret_cast<DenseTask*>(full + stages);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, lt = threadIdx.x;
    const int chain = static_cast<int>(blockIdx.x) / g;
    const int row0 = (static_cast<int>(blockIdx.x) % g) * 8;
    auto stamp = [&](int s, int ph) {
        if (dbg && lt == 0) dbg[((size_t)blockIdx.x * nsteps + s) * 4 + ph] = globaltimer();
    };
    for (int i = lt; i < nsteps; i += blockDim.x) tsh[i] = sched_g[(long long)nchains * i + chain];
    auto unit_src = [&](int s, int& nr) -> const double* {
        const DenseTask& tk = tsh[s];
        nr = tk.moff >= 0 ? max(0, min(8, tk.mout - row0)) : 0;
        return store + tk.moff + (long long)row0 * tk.ld;
    };
    auto prefetch_l2 = [&](int s) {
        if (s >= nsteps) return;
        int nr;
        const double* src = unit_src(s, nr);
        if (nr) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(nr * tsh[s].ld * 8) : "memory");
    };
    auto issue = [&](int s) {
        if (s >= nsteps) return;
        const int k = s % stages;
        int nr;
        const double* src = unit_src(s, nr);
        const unsigned bytes = static_cast<unsigned>(nr * tsh[s].ld * 8);
        mbar_arrive_expect_tx(&full[k], bytes);
        if (nr) bulk_g2s(ring + (size_t)k * 8 * ldmax, src, bytes, &full[k]);
    };
    const bool issuer = lt == 7 * 32;
    if (issuer) {
        for (int k = 0; k < stages; ++k) mbar_init(&full[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (issuer) {
        for (int s = 0; s < min(pf, nsteps); ++s) prefetch_l2(s);
        for (int s = 0; s < stages; ++s) issue(s);
    }
    double y[2][DNI];  // this thread's input values (kept across tasks with identical inputs)
    for (int s = 0; s < nsteps; ++s) {
        const DenseTask tk = tsh[s];
        stamp(s, 0);
        if (issuer) prefetch_l2(s + pf);
        const bool active = tk.moff >= 0;
        if (active) {
            const int nin = tk.n0 + tk.n1;
            // this thread's inputs: seg 0 from b (in0 < 0) or LL lines, seg 1 from LL lines;
            // a task reading exactly the previous task's lines keeps them (no round trip)
            const bool reuse = s > 0 && tsh[s - 1].moff >= 0 && tsh[s - 1].in0 == tk.in0 && tsh[s - 1].in1 == tk.in1 &&
                               tsh[s - 1].n0 == tk.n0 && tsh[s - 1].n1 == tk.n1 && tk.in0 >= 0;
            unsigned pending = 0;
            if (!reuse)
#pragma unroll
                for (int i = 0; i < DNI; ++i) {
                    const int c = lt + 256 * i;
#pragma unroll
                    for (int k = 0; k < 2; ++k) {
                        y[k][i] = 0.0;
                        if (k < nrhs && c < nin) {
                            if (c < tk.n0 && tk.in0 < 0)
                                y[k][i] = b[(long long)k * n + tk.b0 + c];
                            else
                                pending |= 1u << (2 * i + k);
                        }
                    }
                }
            while (__any_sync(0xffffffffu, pending != 0)) {
                uint4 v[2 * DNI];
#pragma unroll
                for (int q = 0; q < 2 * DNI; ++q)
                    if (pending & (1u << q)) {
                        const int c = lt + 256 * (q >> 1), k = q & 1;
                        const long long off = c < tk.n0 ? tk.in0 + c : tk.in1 + (c - tk.n0);
                        v[q] = ll_peek(ll + k * lln + off);
                    }
#pragma unroll
                for (int q = 0; q < 2 * DNI; ++q)
                    if ((pending & (1u << q)) && ll_ready(v[q], flag)) {
                        y[q & 1][q >> 1] = ll_value(v[q]);
                        pending &= ~(1u << q);
                    }
            }
            stamp(s, 1);
            mbar_wait(&full[s % stages], static_cast<unsigned>((s / stages) & 1));
            stamp(s, 3);
            const double* rows = ring + (size_t)(s % stages) * 8 * ldmax;
            const int nr = max(0, min(8, tk.mout - row0));
            double v[16];  // [rhs][row]
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = 0.0;
#pragma unroll
            for (int i = 0; i < DNI; ++i) {
                const int c = lt + 256 * i;
                if (c < nin)
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        const double a = r < nr ? rows[r * tk.ld + c] : 0.0;
                        v[r] += a * y[0][i];
                        v[8 + r] += a * y[1][i];
                    }
            }
            const double part = warp_reduce_scatter16(v, lane);
            if (!(lane & 1)) red[warp * 16 + (lane >> 1)] = part;
        }
        __syncthreads();  // partials complete, ring slot s free
        if (issuer) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(s + stages);
        }
        if (active && warp == 0 && lane < 16) {
            const int kk = lane >> 3, r = row0 + (lane & 7);
            if (kk < nrhs && r < tk.mout) {
                double val = 0.0;
#pragma unroll
                for (int w = 0; w < 8; ++w) val += red[w * 16 + lane];
                if (tk.base >= 0) val = b[(long long)kk * n + tk.base + r] + val;
                if (tk.out_ll >= 0) ll_store(ll + kk * lln + tk.out_ll + r, val, flag);
                if (tk.out_x >= 0) {
                    double* xp = x + (long long)kk * n + tk.out_x + r;
                    *xp = tk.acc ? *xp + val : val;
                }
            }
        }
        stamp(s, 2);
    }
}

}  // namespace

namespace {

// An SPD block-tridiagonal system as dense col-major device blocks: D[j]
// (m_j x m_j) becomes the twisted Cholesky factor, C[j] = A_{j+1,j}
// (m_{j+1} x m_j) becomes K_j in the top part; K'_j (bottom) in kp.
struct TriSys {
    std::vector<int> m;
    std::vector<double*> D, C, U;  // U[j] = A_{j,j+1} (m_j x m_{j+1}): non-symmetric systems only
    int t = 0;
    bool lu = false;               // twisted block LU (non-symmetric) instead of Cholesky
    DBuf<double> kp, linv;
    std::vector<long long> oKp, ol, ro;
    // LU: LP_j = L_j^{-1} P_j in linv, Ui_j = U_j^{-1}, top Kt_j = A_{j+1,j} Ui_j and
    // Ku_j = LP_j A_{j,j+1}, bottom Kb_j = A_{j-1,j} Ui'_j and Kbu_j = LP'_j A_{j,j-1}
    DBuf<double> ui, ktb, kub, kbb, kbub;
    std::vector<long long> oKt, oKu, oKb, oKbu;
    int nb() const { return static_cast<int>(m.size()); }
    long long rows() const { return ro.back(); }
    double* Kt(int j) const { return lu ? ktb.p + oKt[j] : C[j]; }
    double* Kb(int j) const { return lu ? kbb.p + oKb[j] : kp.p + oKp[j]; }
    double* Li(int j) const { return linv.p + ol[j]; }
    double* Ui(int j) const { return ui.p + ol[j]; }
    double* Ku(int j) const { return kub.p + oKu[j]; }
    double* Kbu(int j) const { return kbub.p + oKbu[j]; }

    void factor_lu(LaHandles& h, cudaStream_t st) {
        const int n = nb();
        ro.assign(n + 1, 0);
        for (int j = 0; j < n; ++j) ro[j + 1] = ro[j] + m[j];
        t = (n - 1) / 2;
        const double one = 1.0, mone = -1.0, zero = 0.0;
        const int mx = *std::max_element(m.begin(), m.end());
        int lwork = 0;
        PDG_CUSOLVER_D(cusolverDnDgetrf_bufferSize(h.solver, mx, mx, D[0], mx, &lwork));
        DBuf<double> work(std::max(lwork, 1));
        DBuf<int> ipiv(mx), info(1), dperm(mx);
        ol.assign(n, 0);
        oKt.assign(n, -1);
        oKu.assign(n, -1);
        oKb.assign(n, -1);
        oKbu.assign(n, -1);
        long long tot = 0, kt = 0, kb = 0;
        for (int j = 0; j < n; ++j) {
            ol[j] = tot;
            tot += (long long)m[j] * m[j];
            if (j < t) {
                oKt[j] = oKu[j] = kt;
                kt += (long long)m[j + 1] * m[j];
            }
            if (j > t) {
                oKb[j] = oKbu[j] = kb;
                kb += (long long)m[j - 1] * m[j];
            }
        }
        linv.alloc(tot);
        ui.alloc(tot);
        ktb.alloc(std::max<long long>(kt, 1));
        kub.alloc(std::max<long long>(kt, 1));
        kbb.alloc(std::max<long long>(kb, 1));
        kbub.alloc(std::max<long long>(kb, 1));
        auto lu_block = [&](int j) {  // P S = L U; LP_j = L^{-1} P, Ui_j = U^{-1}
            const int mj = m[j];
            PDG_CUSOLVER_D(cusolverDnDgetrf(h.solver, mj, mj, D[j], mj, work.p, ipiv.p, info.p));
            std::vector<int> piv(mj), pm(mj);
            PDG_CUDA(cudaMemcpyAsync(piv.data(), ipiv.p, sizeof(int) * mj, cudaMemcpyDeviceToHost, st));
            int hinfo = 0;
            PDG_CUDA(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, st));
            PDG_CUDA(cudaStreamSynchronize(st));
            if (hinfo != 0)
                throw Error(PDG_NOT_CONVERGED, "dense LU: matrix is singular to working precision (block " +
                                                   std::to_string(j) + ")");
            for (int i = 0; i < mj; ++i) pm[i] = i;
            for (int i = 0; i < mj; ++i) std::swap(pm[i], pm[piv[i] - 1]);
            PDG_CUDA(cudaMemcpyAsync(dperm.p, pm.data(), sizeof(int) * mj, cudaMemcpyHostToDevice, st));
            k_perm_identity<<<grid_for((long long)mj * mj, 256), 256, 0, st>>>(mj, dperm.p, Li(j));
            k_identity_cm<<<grid_for((long long)mj * mj, 256), 256, 0, st>>>(mj, Ui(j));
            PDG_CHECK_LAUNCH();
            PDG_CUBLAS_D(cublasDtrsm(h.blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_UNIT, mj, mj,
                                     &one, D[j], mj, Li(j), mj));
            PDG_CUBLAS_D(cublasDtrsm(h.blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, mj,
                                     mj, &one, D[j], mj, Ui(j), mj));
        };
        auto mm = [&](int rows, int cols, int inner, double a, const double* A_, int lda, const double* B_, int ldb,
                      double b, double* C_, int ldc) {
            PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, rows, cols, inner, &a, A_, lda, B_, ldb, &b, C_, ldc));
        };
        for (int j = 0; j < t; ++j) {  // top: S_j = A_jj - Kt_{j-1} Ku_{j-1}
            if (j > 0) mm(m[j], m[j], m[j - 1], -1.0, Kt(j - 1), m[j], Ku(j - 1), m[j - 1], 1.0, D[j], m[j]);
            lu_block(j);
            mm(m[j + 1], m[j], m[j], 1.0, C[j], m[j + 1], Ui(j), m[j], 0.0, Kt(j), m[j + 1]);
            mm(m[j], m[j + 1], m[j], 1.0, Li(j), m[j], U[j], m[j], 0.0, Ku(j), m[j]);
        }
        for (int j = n - 1; j > t; --j) {  // bottom: S'_j = A_jj - Kb_{j+1} Kbu_{j+1}
            if (j < n - 1) mm(m[j], m[j], m[j + 1], -1.0, Kb(j + 1), m[j], Kbu(j + 1), m[j + 1], 1.0, D[j], m[j]);
            lu_block(j);
            mm(m[j - 1], m[j], m[j], 1.0, U[j - 1], m[j - 1], Ui(j), m[j], 0.0, Kb(j), m[j - 1]);
            mm(m[j], m[j - 1], m[j], 1.0, Li(j), m[j], C[j - 1], m[j], 0.0, Kbu(j), m[j]);
        }
        if (t > 0) mm(m[t], m[t], m[t - 1], -1.0, Kt(t - 1), m[t], Ku(t - 1), m[t - 1], 1.0, D[t], m[t]);
        if (t + 1 < n) mm(m[t], m[t], m[t + 1], -1.0, Kb(t + 1), m[t], Kbu(t + 1), m[t + 1], 1.0, D[t], m[t]);
        lu_block(t);
        (void)zero;
        (void)mone;
    }

    void factor(LaHandles& h, cudaStream_t st) {
        const int n = nb();
        ro.assign(n + 1, 0);
        for (int j = 0; j < n; ++j) ro[j + 1] = ro[j] + m[j];
        t = (n - 1) / 2;
        const double one = 1.0, mone = -1.0, zero = 0.0;
        const int mx = *std::max_element(m.begin(), m.end());
        int lwork = 0;
        PDG_CUSOLVER_D(cusolverDnDpotrf_bufferSize(h.solver, CUBLAS_FILL_MODE_LOWER, mx, D[0], mx, &lwork));
        DBuf<double> work(std::max(lwork, 1));
        DBuf<int> info(n);
        info.zero(st);
        oKp.assign(n, -1);
        long long kt = 0;
        for (int j = t + 1; j < n; ++j) {
            oKp[j] = kt;
            kt += (long long)m[j - 1] * m[j];
        }
        kp.alloc(std::max<long long>(kt, 1));
        for (int j = 0; j < t; ++j) {  // top
            if (j > 0)
                PDG_CUBLAS_D(cublasDsyrk(h.blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, m[j], m[j - 1], &mone, C[j - 1], m[j],
                                         &one, D[j], m[j]));
            PDG_CUSOLVER_D(cusolverDnDpotrf(h.solver, CUBLAS_FILL_MODE_LOWER, m[j], D[j], m[j], work.p, lwork, info.p + j));
            PDG_CUBLAS_D(cublasDtrsm(h.blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT,
                                     m[j + 1], m[j], &one, D[j], m[j], C[j], m[j + 1]));
        }
        for (int j = n - 1; j > t; --j) {  // bottom
            if (j < n - 1)
                PDG_CUBLAS_D(cublasDsyrk(h.blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, m[j], m[j + 1], &mone, Kb(j + 1),
                                         m[j], &one, D[j], m[j]));
            PDG_CUSOLVER_D(cusolverDnDpotrf(h.solver, CUBLAS_FILL_MODE_LOWER, m[j], D[j], m[j], work.p, lwork, info.p + j));
            PDG_CUBLAS_D(cublasDgeam(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, m[j - 1], m[j], &one, C[j - 1], m[j], &zero, Kb(j),
                                     m[j - 1], Kb(j), m[j - 1]));
            PDG_CUBLAS_D(cublasDtrsm(h.blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT,
                                     m[j - 1], m[j], &one, D[j], m[j], Kb(j), m[j - 1]));
        }
        if (t > 0)  // twist
            PDG_CUBLAS_D(cublasDsyrk(h.blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, m[t], m[t - 1], &mone, C[t - 1], m[t],
                                     &one, D[t], m[t]));
        if (t + 1 < n)
            PDG_CUBLAS_D(cublasDsyrk(h.blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, m[t], m[t + 1], &mone, Kb(t + 1), m[t],
                                     &one, D[t], m[t]));
        PDG_CUSOLVER_D(cusolverDnDpotrf(h.solver, CUBLAS_FILL_MODE_LOWER, m[t], D[t], m[t], work.p, lwork, info.p + t));
        const std::vector<int> hinfo = info.download(st);
        for (int j = 0; j < n; ++j)
            if (hinfo[j] != 0)
                throw Error(PDG_NOT_CONVERGED, "dense LU: matrix is singular to working precision (block " +
                                                   std::to_string(j) + " not positive definite)");
        ol.assign(n, 0);
        long long tot = 0;
        for (int j = 0; j < n; ++j) {
            ol[j] = tot;
            tot += (long long)m[j] * m[j];
        }
        linv.alloc(tot);
        for (int j = 0; j < n; ++j) {
            k_identity_cm<<<grid_for((long long)m[j] * m[j], 256), 256, 0, st>>>(m[j], Li(j));
            PDG_CHECK_LAUNCH();
            PDG_CUBLAS_D(cublasDtrsm(h.blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, m[j],
                                     m[j], &one, D[j], m[j], Li(j), m[j]));
        }
    }

    // R <- A^{-1} R for nc right-hand sides (R: rows() x nc col-major, ld = rows()),
    // block forward/backward substitution through the twisted factors (setup only).
    void solve_multi(LaHandles& h, double* R, int nc) const {
        const int n = nb();
        const long long ld = rows();
        const double one = 1.0, mone = -1.0;
        auto Rb = [&](int j) { return R + ro[j]; };
        auto lower = [&](int j, bool trans) {
            PDG_CUBLAS_D(cublasDtrsm(h.blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, trans ? CUBLAS_OP_T : CUBLAS_OP_N,
                                     CUBLAS_DIAG_NON_UNIT, m[j], nc, &one, D[j], m[j], Rb(j), ld));
        };
        for (int j = 0; j < t; ++j) {
            if (j > 0)
                PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, m[j], nc, m[j - 1], &mone, Kt(j - 1), m[j],
                                         Rb(j - 1), ld, &one, Rb(j), ld));
            lower(j, false);
        }
        for (int j = n - 1; j > t; --j) {
            if (j < n - 1)
                PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, m[j], nc, m[j + 1], &mone, Kb(j + 1), m[j],
                                         Rb(j + 1), ld, &one, Rb(j), ld));
            lower(j, false);
        }
        if (t > 0)
            PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, m[t], nc, m[t - 1], &mone, Kt(t - 1), m[t],
                                     Rb(t - 1), ld, &one, Rb(t), ld));
        if (t + 1 < n)
            PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, m[t], nc, m[t + 1], &mone, Kb(t + 1), m[t],
                                     Rb(t + 1), ld, &one, Rb(t), ld));
        lower(t, false);
        lower(t, true);
        for (int j = t - 1; j >= 0; --j) {
            PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, m[j], nc, m[j + 1], &mone, Kt(j), m[j + 1],
                                     Rb(j + 1), ld, &one, Rb(j), ld));
            lower(j, true);
        }
        for (int j = t + 1; j < n; ++j) {
            PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, m[j], nc, m[j - 1], &mone, Kb(j), m[j - 1],
                                     Rb(j - 1), ld, &one, Rb(j), ld));
            lower(j, true);
        }
    }
};

// Where a twisted system reads and writes, per block j (offsets < 0 = none).
struct SysIO {
    std::vector<long long> rhs_ll, rhs_b;  // rhs from LL (>= 0) or else from b at rhs_b
    std::vector<long long> y_ll, x_ll, x_out;
    long long pt = -1, pb = -1;
};

enum MatKind { MK_TOPF = 0, MK_BOTF, MK_PTOP, MK_PBOT, MK_TWIST, MK_TOPB, MK_BOTB, MK_GSTEP, MK_CORR };
struct Mat {
    int kind;
    const TriSys* sys;
    int j;
    long long off;
    int ld;
    // MK_GSTEP: couplings; MK_CORR: spike rows
    const double *a = nullptr, *c = nullptr;
    int ma = 0, mc = 0, lda = 0, ldc = 0;
};

}  // namespace

void BlockTriChol::dense_setup(double* dense, cudaStream_t st) {
    LaHandles h(st);
    auto Dg = [&](int j) { return dense + dD_[j]; };
    auto Cg = [&](int j) { return dense + dC_[j]; };  // A_{j+1,j}
    const double one = 1.0, mone = -1.0, zero = 0.0;
    auto pad = [](int v) { return (v + 1) & ~1; };
    auto al = [](long long v) { return (v + 31) & ~31LL; };
    // ---- virtual strips: 2 chains of g CTAs (8 rows each) per strip, >= 2 interior blocks each
    d_g = (max_b + 7) / 8;
    // Default: one strip (the plain twisted sweep). P = 2 cuts the config-1 flow solve from
    // 250 to 190 us but its spike corrections raise the preconditioner's linearity defect
    // from < 1e-12 to ~3e-11 of max|z|, so it is opt-in (PDG_FLOW_STRIPS=P).
    int P = 1;
    if (const char* e = std::getenv("PDG_FLOW_STRIPS"))
        P = std::max(1, std::min({std::atoi(e), num_sms() / (2 * d_g), (nb + 1) / 3}));
    if (!symmetric) P = 1;  // the substructured path is SPD-only
    std::vector<int> lo(P), hi(P), sep;
    {
        const int interior = nb - (P - 1);
        int j = 0;
        for (int k = 0; k < P; ++k) {
            const int len = interior / P + (k < interior % P ? 1 : 0);
            if (k > 0) sep.push_back(j++);
            lo[k] = j;
            hi[k] = j + len;
            j += len;
        }
    }
    nchains = 2 * P;
    require(nchains * d_g <= num_sms(), "block-tridiagonal solver: blocks too large for the dense sweep kernel");
    // ---- factor the strip interiors (couplings to the separators untouched)
    std::vector<TriSys> strips(P);
    for (int k = 0; k < P; ++k) {
        for (int j = lo[k]; j < hi[k]; ++j) {
            strips[k].m.push_back(bsz[j]);
            strips[k].D.push_back(Dg(j));
            if (j + 1 < hi[k]) {
                strips[k].C.push_back(Cg(j));
                if (!symmetric) strips[k].U.push_back(dense + dU_[j]);
            }
        }
        strips[k].lu = !symmetric;
        if (strips[k].lu)
            strips[k].factor_lu(h, st);
        else
            strips[k].factor(h, st);
    }
    // ---- spikes and the separator system
    std::vector<DBuf<double>> Wt(P), Wb(P);
    TriSys seps;
    std::vector<DBuf<double>> sD, sC;
    if (P > 1) {
        for (int k = 0; k < P; ++k) {
            const TriSys& S = strips[k];
            const long long nI = S.rows();
            if (k > 0) {  // W_top = A_II^{-1} A_{I,s_k}: block lo rows hold A_{lo,s} = C(s)
                const int s = sep[k - 1];
                Wt[k].alloc((size_t)nI * bsz[s]);
                Wt[k].zero(st);
                PDG_CUBLAS_D(cublasDgeam(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, bsz[lo[k]], bsz[s], &one, Cg(s), bsz[lo[k]], &zero,
                                         Cg(s), bsz[lo[k]], Wt[k].p, nI));
                S.solve_multi(h, Wt[k].p, bsz[s]);
            }
            if (k < P - 1) {  // W_bot = A_II^{-1} A_{I,s_{k+1}}: block hi-1 rows hold A_{hi-1,s'} = C(hi-1)^T
                const int s = sep[k], jl = hi[k] - 1;
                Wb[k].alloc((size_t)nI * bsz[s]);
                Wb[k].zero(st);
                PDG_CUBLAS_D(cublasDgeam(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, bsz[jl], bsz[s], &one, Cg(jl), bsz[s], &zero,
                                         Cg(jl), bsz[s], Wb[k].p + S.ro[S.nb() - 1], nI));
                S.solve_multi(h, Wb[k].p, bsz[s]);
            }
        }
        const int ns = P - 1;
        sD.resize(ns);
        sC.resize(std::max(ns - 1, 0));
        for (int i = 0; i < ns; ++i) {
            const int s = sep[i], ms = bsz[s];
            const int ka = i, kb = i + 1;  // strips above (ends at s-1) and below (starts at s+1)
            sD[i].alloc((size_t)ms * ms);
            PDG_CUBLAS_D(cublasDgeam(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, ms, ms, &one, Dg(s), ms, &zero, Dg(s), ms, sD[i].p, ms));
            // - A_{s,lo} W_top[lo] = - C(s)^T W_top_kb[lo block]
            PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, ms, ms, bsz[s + 1], &mone, Cg(s), bsz[s + 1], Wt[kb].p,
                                     strips[kb].rows(), &one, sD[i].p, ms));
            // - A_{s,s-1} W_bot[s-1] = - C(s-1) W_bot_ka[last block]
            const TriSys& A = strips[ka];
            PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, ms, ms, bsz[s - 1], &mone, Cg(s - 1), ms,
                                     Wb[ka].p + A.ro[A.nb() - 1], A.rows(), &one, sD[i].p, ms));
            if (i + 1 < ns) {  // S_{i+1,i} = -(A_{s,lo} W_bot_kb[lo])^T = -W_bot_kb[lo]^T C(s)
                const int s2 = sep[i + 1];
                sC[i].alloc((size_t)bsz[s2] * ms);
                PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, bsz[s2], ms, bsz[s + 1], &mone, Wb[kb].p,
                                         strips[kb].rows(), Cg(s), bsz[s + 1], &zero, sC[i].p, bsz[s2]));
            }
            seps.m.push_back(ms);
            seps.D.push_back(sD[i].p);
            if (i + 1 < ns) seps.C.push_back(sC[i].p);
        }
        seps.factor(h, st);
    }
    // ---- LL regions (per right-hand side): Y [0,n) forward y, X [n,2n) final x,
    //      twist parts per system, G (separator rhs), SY (separator forward y)
    const long long X_ = n;
    long long lltop = 2LL * n;
    auto llalloc = [&](long long len) {
        const long long o = lltop;
        lltop += len;
        return o;
    };
    // ---- step lists per chain
    std::vector<std::vector<DenseTask>> ch(nchains);
    std::vector<Mat> mats;
    long long o = 0;
    int ldmax = 2;
    factor_bytes = 0.0;
    const DenseTask idle{-1, -1, -1, -1, -1, -1, 0, 0, 0, 0, -1, 0, 0};
    auto add = [&](const Mat& mt, int mout, int n0, long long in0, long long b0, int n1, long long in1,
                   long long out_ll, long long out_x) {
        DenseTask tk = idle;
        tk.ld = pad(n0 + n1);
        tk.moff = o;
        tk.mout = mout;
        tk.n0 = n0;
        tk.in0 = in0;
        tk.b0 = b0;
        tk.n1 = n1;
        tk.in1 = in1;
        tk.out_ll = out_ll;
        tk.out_x = out_x;
        ldmax = std::max(ldmax, tk.ld);
        Mat m2 = mt;
        m2.off = o;
        m2.ld = tk.ld;
        mats.push_back(m2);
        o = al(o + (long long)mout * tk.ld);
        factor_bytes += 8.0 * mout * (n0 + n1);
        return tk;
    };
    // a twisted solve of system S on chains (ct, cb)
    auto build = [&](const TriSys& S, const SysIO& io, int ct, int cb) {
        const int nn = S.nb(), t = S.t;
        auto mk = [&](int kind, int j) { return Mat{kind, &S, j, 0, 0}; };
        auto rhs_in = [&](int j, long long& in, long long& b0) {
            in = io.rhs_ll[j];
            b0 = io.rhs_b[j];
        };
        std::vector<DenseTask> top, bot;
        for (int j = 0; j < t; ++j) {
            long long in, b0;
            rhs_in(j, in, b0);
            top.push_back(add(mk(MK_TOPF, j), S.m[j], S.m[j], in, b0, j > 0 ? S.m[j - 1] : 0, j > 0 ? io.y_ll[j - 1] : -1,
                              io.y_ll[j], -1));
        }
        {
            long long in, b0;
            rhs_in(t, in, b0);
            top.push_back(add(mk(MK_PTOP, t), S.m[t], S.m[t], in, b0, t > 0 ? S.m[t - 1] : 0, t > 0 ? io.y_ll[t - 1] : -1,
                              io.pt, -1));
        }
        for (int j = nn - 1; j > t; --j) {
            long long in, b0;
            rhs_in(j, in, b0);
            bot.push_back(add(mk(MK_BOTF, j), S.m[j], S.m[j], in, b0, j < nn - 1 ? S.m[j + 1] : 0,
                              j < nn - 1 ? io.y_ll[j + 1] : -1, io.y_ll[j], -1));
        }
        if (t < nn - 1) bot.push_back(add(mk(MK_PBOT, t), S.m[t], S.m[t + 1], io.y_ll[t + 1], -1, 0, -1, io.pb, -1));
        const size_t L = std::max(top.size(), bot.size());
        while (top.size() < L) top.push_back(idle);
        while (bot.size() < L) bot.push_back(idle);
        top.push_back(add(mk(MK_TWIST, t), S.m[t], S.m[t], io.pt, -1, t < nn - 1 ? S.m[t] : 0, t < nn - 1 ? io.pb : -1,
                          io.x_ll[t], io.x_out[t]));
        bot.push_back(idle);
        for (int s = 1; s < nn; ++s) {
            const int jt = t - s, jb = t + s;
            if (jt < 0 && jb > nn - 1) break;
            top.push_back(jt >= 0 ? add(mk(MK_TOPB, jt), S.m[jt], S.m[jt], io.y_ll[jt], -1, S.m[jt + 1],
                                        io.x_ll[jt + 1], io.x_ll[jt], io.x_out[jt])
                                  : idle);
            bot.push_back(jb <= nn - 1 ? add(mk(MK_BOTB, jb), S.m[jb], S.m[jb], io.y_ll[jb], -1, S.m[jb - 1],
                                             io.x_ll[jb - 1], io.x_ll[jb], io.x_out[jb])
                                       : idle);
        }
        for (auto& tk : top) ch[ct].push_back(tk);
        for (auto& tk : bot) ch[cb].push_back(tk);
    };
    // phase 1: strip interiors (rhs from b; y, x, x_ll in global numbering)
    for (int k = 0; k < P; ++k) {
        const TriSys& S = strips[k];
        SysIO io;
        for (int j = lo[k]; j < hi[k]; ++j) {
            io.rhs_ll.push_back(-1);
            io.rhs_b.push_back(boff[j]);
            io.y_ll.push_back(boff[j]);
            io.x_ll.push_back(X_ + boff[j]);
            io.x_out.push_back(boff[j]);
        }
        io.pt = llalloc(S.m[S.t]);
        io.pb = llalloc(S.m[S.t]);
        build(S, io, 2 * k, 2 * k + 1);
    }
    if (P > 1) {
        // phase 2: separator right-hand sides g_s = b_s - C(s-1) y_{s-1} - C(s)^T y_{s+1} (chain 2i)
        const int ns = P - 1;
        std::vector<long long> g_ll(ns);
        for (int i = 0; i < ns; ++i) g_ll[i] = llalloc(bsz[sep[i]]);
        for (int i = 0; i < ns; ++i) {
            const int s = sep[i];
            Mat mt{MK_GSTEP, nullptr, s, 0, 0};
            mt.a = Cg(s - 1);
            mt.ma = bsz[s - 1];
            mt.lda = bsz[s];
            mt.c = Cg(s);
            mt.mc = bsz[s + 1];
            mt.ldc = bsz[s + 1];
            DenseTask tk = add(mt, bsz[s], bsz[s - 1], X_ + boff[s - 1], -1, bsz[s + 1], X_ + boff[s + 1], g_ll[i], -1);
            tk.base = boff[s];
            ch[2 * i].push_back(tk);
        }
        // phase 3: the separator system on chains 0/1
        SysIO io;
        for (int i = 0; i < ns; ++i) {
            io.rhs_ll.push_back(g_ll[i]);
            io.rhs_b.push_back(-1);
            io.y_ll.push_back(llalloc(bsz[sep[i]]));
            io.x_ll.push_back(X_ + boff[sep[i]]);
            io.x_out.push_back(boff[sep[i]]);
        }
        io.pt = llalloc(seps.m[seps.t]);
        io.pb = llalloc(seps.m[seps.t]);
        size_t L = 0;
        for (auto& c : ch) L = std::max(L, c.size());
        for (int c = 0; c < 2; ++c)
            while (ch[c].size() < L) ch[c].push_back(idle);  // after every g step (LL waits anyway)
        build(seps, io, 0, 1);
        // phase 4: x_I += -[W_top | W_bot] [x_{s_k}; x_{s_{k+1}}], block by block (chains of the strip)
        for (int k = 0; k < P; ++k) {
            const TriSys& S = strips[k];
            for (int jj = 0; jj < S.nb(); ++jj) {
                const int j = lo[k] + jj;
                Mat mt{MK_CORR, &S, jj, 0, 0};
                int n0 = 0, n1 = 0;
                long long in0 = -1, in1 = -1;
                if (k > 0) {
                    mt.a = Wt[k].p + S.ro[jj];
                    mt.ma = bsz[sep[k - 1]];
                    mt.lda = static_cast<int>(S.rows());
                    n0 = mt.ma;
                    in0 = X_ + boff[sep[k - 1]];
                }
                if (k < P - 1) {
                    const double* w = Wb[k].p + S.ro[jj];
                    const int mw = bsz[sep[k]];
                    if (n0 == 0) {
                        mt.a = w;
                        mt.ma = mw;
                        mt.lda = static_cast<int>(S.rows());
                        n0 = mw;
                        in0 = X_ + boff[sep[k]];
                    } else {
                        mt.c = w;
                        mt.mc = mw;
                        mt.ldc = static_cast<int>(S.rows());
                        n1 = mw;
                        in1 = X_ + boff[sep[k]];
                    }
                }
                DenseTask tk = add(mt, bsz[j], n0, in0, -1, n1, in1, -1, boff[j]);
                tk.acc = 1;
                ch[jj <= S.t ? 2 * k : 2 * k + 1].push_back(tk);
            }
        }
    }
    // ---- fill the step matrices (row-major = col-major of the transpose, leading dim ld)
    store.alloc(std::max<long long>(o, 1));
    for (const Mat& mt : mats) {
        double* X = store.p + mt.off;
        const int ld = mt.ld;
        if (mt.kind == MK_GSTEP) {  // [-C(s-1) | -C(s)^T] -> [-C(s-1)^T; -C(s)]
            const int ms = mt.lda;
            PDG_CUBLAS_D(cublasDgeam(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, mt.ma, ms, &mone, mt.a, ms, &zero, mt.a, ms, X, ld));
            PDG_CUBLAS_D(cublasDgeam(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, mt.mc, ms, &mone, mt.c, mt.ldc, &zero, mt.c, mt.ldc,
                                     X + mt.ma, ld));
            continue;
        }
        if (mt.kind == MK_CORR) {  // rows of -[W_top | W_bot] -> [-W_top[rows]^T; -W_bot[rows]^T]
            const int mj = mt.sys->m[mt.j];
            PDG_CUBLAS_D(cublasDgeam(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, mt.ma, mj, &mone, mt.a, mt.lda, &zero, mt.a, mt.lda,
                                     X, ld));
            if (mt.c)
                PDG_CUBLAS_D(cublasDgeam(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, mt.mc, mj, &mone, mt.c, mt.ldc, &zero, mt.c,
                                         mt.ldc, X + mt.ma, ld));
            continue;
        }
        const TriSys& S = *mt.sys;
        const int j = mt.j, mj = S.m[j], nn = S.nb();
        if (S.lu) {  // twisted block LU: LP = L^{-1} P, Ui = U^{-1} (module comment, non-symmetric form)
            auto trT = [&](const double* A_, double* dst) {
                PDG_CUBLAS_D(cublasDgeam(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, mj, mj, &one, A_, mj, &zero, A_, mj, dst, ld));
            };
            switch (mt.kind) {
                case MK_TOPF:
                case MK_PTOP:  // [LP_j | -LP_j Kt_{j-1}] -> [LP_j^T; -Kt_{j-1}^T LP_j^T]
                    trT(S.Li(j), X);
                    if (j > 0)
                        PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_T, S.m[j - 1], mj, mj, &mone, S.Kt(j - 1), mj,
                                                 S.Li(j), mj, &zero, X + mj, ld));
                    break;
                case MK_BOTF:  // [LP'_j | -LP'_j Kb_{j+1}] -> [LP'_j^T; -Kb_{j+1}^T LP'_j^T]
                    trT(S.Li(j), X);
                    if (j < nn - 1)
                        PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_T, S.m[j + 1], mj, mj, &mone, S.Kb(j + 1), mj,
                                                 S.Li(j), mj, &zero, X + mj, ld));
                    break;
                case MK_PBOT:  // -LP_t Kb_{t+1} -> -Kb_{t+1}^T LP_t^T
                    PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_T, S.m[j + 1], mj, mj, &mone, S.Kb(j + 1), mj,
                                             S.Li(j), mj, &zero, X, ld));
                    break;
                case MK_TWIST:  // [Ui_t | Ui_t] -> [Ui_t^T; Ui_t^T]
                    trT(S.Ui(j), X);
                    if (j < nn - 1) trT(S.Ui(j), X + mj);
                    break;
                case MK_TOPB:  // [Ui_j | -Ui_j Ku_j] -> [Ui_j^T; -Ku_j^T Ui_j^T]
                    trT(S.Ui(j), X);
                    PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_T, S.m[j + 1], mj, mj, &mone, S.Ku(j), mj,
                                             S.Ui(j), mj, &zero, X + mj, ld));
                    break;
                default:  // MK_BOTB: [Ui'_j | -Ui'_j Kbu_j] -> [Ui'_j^T; -Kbu_j^T Ui'_j^T]
                    trT(S.Ui(j), X);
                    PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_T, S.m[j - 1], mj, mj, &mone, S.Kbu(j), mj,
                                             S.Ui(j), mj, &zero, X + mj, ld));
                    break;
            }
            continue;
        }
        switch (mt.kind) {
            case MK_TOPF:
            case MK_PTOP:  // [Linv_j | -Linv_j K_{j-1}] -> [Linv_j^T; -K_{j-1}^T Linv_j^T]
                PDG_CUBLAS_D(cublasDgeam(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, mj, mj, &one, S.Li(j), mj, &zero, S.Li(j), mj, X, ld));
                if (j > 0)
                    PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_T, S.m[j - 1], mj, mj, &mone, S.Kt(j - 1), mj,
                                             S.Li(j), mj, &zero, X + mj, ld));
                break;
            case MK_BOTF:  // [Linv'_j | -Linv'_j K'_{j+1}] -> [Linv'_j^T; -K'_{j+1}^T Linv'_j^T]
                PDG_CUBLAS_D(cublasDgeam(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, mj, mj, &one, S.Li(j), mj, &zero, S.Li(j), mj, X, ld));
                if (j < nn - 1)
                    PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_T, S.m[j + 1], mj, mj, &mone, S.Kb(j + 1), mj,
                                             S.Li(j), mj, &zero, X + mj, ld));
                break;
            case MK_PBOT:  // [-Linv_t K'_{t+1}] -> -K'_{t+1}^T Linv_t^T
                PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_T, S.m[j + 1], mj, mj, &mone, S.Kb(j + 1), mj,
                                         S.Li(j), mj, &zero, X, ld));
                break;
            case MK_TWIST:  // [Linv_t^T | Linv_t^T] -> [Linv_t; Linv_t]
                PDG_CUBLAS_D(cublasDgeam(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, mj, mj, &one, S.Li(j), mj, &zero, S.Li(j), mj, X, ld));
                if (j < nn - 1)
                    PDG_CUBLAS_D(cublasDgeam(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, mj, mj, &one, S.Li(j), mj, &zero, S.Li(j), mj,
                                             X + mj, ld));
                break;
            case MK_TOPB:  // [Linv_j^T | -Linv_j^T K_j^T] -> [Linv_j; -K_j Linv_j]
                PDG_CUBLAS_D(cublasDgeam(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, mj, mj, &one, S.Li(j), mj, &zero, S.Li(j), mj, X, ld));
                PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, S.m[j + 1], mj, mj, &mone, S.Kt(j), S.m[j + 1],
                                         S.Li(j), mj, &zero, X + mj, ld));
                break;
            default:  // MK_BOTB: [Linv'_j^T | -Linv'_j^T K'_j^T] -> [Linv'_j; -K'_j Linv'_j]
                PDG_CUBLAS_D(cublasDgeam(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, mj, mj, &one, S.Li(j), mj, &zero, S.Li(j), mj, X, ld));
                PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, S.m[j - 1], mj, mj, &mone, S.Kb(j), S.m[j - 1],
                                         S.Li(j), mj, &zero, X + mj, ld));
                break;
        }
    }
    size_t L = 0;
    for (auto& c : ch) L = std::max(L, c.size());
    dsched.assign(L * nchains, idle);
    for (int c = 0; c < nchains; ++c)
        for (size_t s = 0; s < ch[c].size(); ++s) dsched[s * nchains + c] = ch[c][s];
    d_dsched.upload(dsched, st);
    d_lln = lltop;
    // ---- kernel configuration ------------------------------------------------------
    require(2 * max_b <= 256 * DNI, "block-tridiagonal solver: blocks too large for the dense sweep kernel");
    int dev = 0;
    PDG_CUDA(cudaGetDevice(&dev));
    int optin = 0;
    PDG_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    PDG_CUDA(cudaFuncSetAttribute(k_sweep_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    const int nsteps = static_cast<int>(L);
    d_ldmax = ldmax;
    const size_t fixed = sizeof(double) * 8 * 16 + 8 * 16 + sizeof(DenseTask) * nsteps + 64;
    const size_t unit = sizeof(double) * 8 * ldmax;
    require(fixed + unit <= (size_t)optin - 1024, "block-tridiagonal solver: dense sweep shared memory");
    d_stages = static_cast<int>(std::min<size_t>(((size_t)optin - 1024 - fixed) / unit, 16));
    d_smem = fixed + unit * d_stages;
    int occ = 0;
    PDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sweep_dense, 256, d_smem));
    require(occ >= 1, "block-tridiagonal solver: dense sweep kernel cannot be resident");
    ll.alloc((size_t)max_rhs * d_lln);
    ll.zero(st);
    wb.alloc((size_t)n * max_rhs);
    wx.alloc((size_t)n * max_rhs);
    PDG_CUDA(cudaStreamSynchronize(st));
}

void BlockTriChol::solve_dense(const double* b, double* x, int nrhs, cudaStream_t st) {
    unsigned flag = static_cast<unsigned>(++call);
    if (flag == 0) flag = static_cast<unsigned>(++call);  // 0 = never published
    int nsteps = static_cast<int>(dsched.size() / nchains), nr = nrhs, n_ = n, ldm = d_ldmax, stg = d_stages, g = d_g;
    int nch = nchains;
    int pf = 4;
    if (const char* e = std::getenv("PDG_SWEEP_PF")) pf = std::atoi(e);
    long long lln = d_lln;
    const DenseTask* sched = d_dsched.p;
    const double* sp = store.p;
    uint4* llp = ll.p;
    unsigned long long* dbgp = nullptr;
    dbg_steps = nsteps;
    if (debug_timing) {
        dbg.alloc((size_t)nch * g * nsteps * 4);
        dbg.zero(st);
        dbgp = dbg.p;
    }
    void* args[] = {&nsteps, &sched, &nr, &n_, &sp, &ldm, &b, &x, &llp, &lln, &flag, &stg, &pf, &g, &nch, &dbgp};
    PDG_CUDA(cudaLaunchCooperativeKernel((void*)k_sweep_dense, nch * g, 256, args, d_smem, st));
    count_launch(1);
    PDG_CHECK_LAUNCH();
}

}  // namespace pdg
