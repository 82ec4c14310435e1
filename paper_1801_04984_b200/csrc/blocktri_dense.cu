// General mode of the twisted block-tridiagonal solver (any coupling
// pattern; used for the flow Schur complement in face-row order). With the
// twisted Cholesky factors (top L_j, K_j = L_{j+1,j}; bottom L'_j, K'_j =
// L_{j-1,j}; twist L_t) and Linv = L^{-1}, every step of the solve is
// "outputs = M_s * [seg0; seg1]" with a precomputed row-major M_s, and the whole
// solve (forward, twist, backward of both chains) is one persistent kernel:
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
                  unsigned flag, int stages, int pf, int g, unsigned long long* dbg) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* ring = reinterpret_cast<double*>(smem_raw);  // [stages][8 rows][ldmax]
    double* red = ring + (size_t)stages * 8 * ldmax;      // [8 warps][16]
    unsigned long long* full = reinterpret_cast<unsigned long long*>(red + 8 * 16);
    DenseTask* tsh = reinterpret_cast<DenseTask*>(full + stages);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, lt = threadIdx.x;
    const int chain = static_cast<int>(blockIdx.x) < g ? 0 : 1;
    const int row0 = (chain ? blockIdx.x - g : blockIdx.x) * 8;
    auto stamp = [&](int s, int ph) {
        if (dbg && lt == 0) dbg[((size_t)blockIdx.x * nsteps + s) * 4 + ph] = globaltimer();
    };
    for (int i = lt; i < nsteps; i += blockDim.x) tsh[i] = sched_g[2 * i + chain];
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
    for (int s = 0; s < nsteps; ++s) {
        const DenseTask tk = tsh[s];
        stamp(s, 0);
        if (issuer) prefetch_l2(s + pf);
        const bool active = tk.moff >= 0;
        if (active) {
            const int nin = tk.n0 + tk.n1;
            // this thread's inputs: seg 0 from b (in0 < 0) or LL lines, seg 1 from LL lines
            double y[2][DNI];
            unsigned pending = 0;
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
                if (tk.out_ll >= 0) ll_store(ll + kk * lln + tk.out_ll + r, val, flag);
                if (tk.out_x >= 0) x[(long long)kk * n + tk.out_x + r] = val;
            }
        }
        stamp(s, 2);
    }
}

}  // namespace

void BlockTriChol::dense_finish(LaHandles& h, const double* dense, const double* kp, const std::vector<long long>& oKp,
                                cudaStream_t st) {
    const int t = twist;
    auto Kt = [&](int j) { return dense + dC_[j]; };  // K_j = L_{j+1,j}, m_{j+1} x m_j col-major (top, j < t)
    auto Kb = [&](int j) { return kp + oKp[j]; };     // K'_j = L_{j-1,j}, m_{j-1} x m_j col-major (bottom, j > t)
    // ---- Linv_j (lower triangular, col-major) ------------------------------------------
    std::vector<long long> ol(nb);
    long long tot = 0;
    for (int j = 0; j < nb; ++j) {
        ol[j] = tot;
        tot += (long long)bsz[j] * bsz[j];
    }
    DBuf<double> linv(tot);
    const double one = 1.0, mone = -1.0, zero = 0.0;
    for (int j = 0; j < nb; ++j) {
        const int mj = bsz[j];
        k_identity_cm<<<grid_for((long long)mj * mj, 256), 256, 0, st>>>(mj, linv.p + ol[j]);
        PDG_CHECK_LAUNCH();
        PDG_CUBLAS_D(cublasDtrsm(h.blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, mj,
                                 mj, &one, dense + dD_[j], mj, linv.p + ol[j], mj));
    }
    auto Li = [&](int j) { return linv.p + ol[j]; };
    // ---- per-step matrices (row-major = col-major of the transpose) -------------------
    auto pad = [](int v) { return (v + 1) & ~1; };
    auto al = [](long long v) { return (v + 31) & ~31LL; };
    const long long X_ = n, PT = 2LL * n, PB = 2LL * n + bsz[t];
    d_lln = 2LL * n + 2LL * bsz[t];
    struct Mat {
        int kind, j;  // 0 top fwd, 1 bottom fwd, 2 p_top, 3 p_bot, 4 twist, 5 top bwd, 6 bottom bwd
        long long off;
        int ld;
    };
    std::vector<DenseTask> top, bot;
    std::vector<Mat> mats;
    long long o = 0;
    int ldmax = 2;
    const DenseTask idle{-1, -1, -1, -1, -1, -1, 0, 0, 0, 0};
    factor_bytes = 0.0;
    auto add = [&](int kind, int j, int mout, int n0, long long in0, long long b0, int n1, long long in1,
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
        mats.push_back({kind, j, o, tk.ld});
        o = al(o + (long long)mout * tk.ld);
        factor_bytes += 8.0 * mout * (n0 + n1);
        return tk;
    };
    // forward: y_j of the top blocks, then p_top; bottom blocks, then p_bot
    for (int j = 0; j < t; ++j)
        top.push_back(add(0, j, bsz[j], bsz[j], -1, boff[j], j > 0 ? bsz[j - 1] : 0, j > 0 ? boff[j - 1] : -1, boff[j], -1));
    top.push_back(add(2, t, bsz[t], bsz[t], -1, boff[t], t > 0 ? bsz[t - 1] : 0, t > 0 ? boff[t - 1] : -1, PT, -1));
    for (int j = nb - 1; j > t; --j)
        bot.push_back(add(1, j, bsz[j], bsz[j], -1, boff[j], j < nb - 1 ? bsz[j + 1] : 0, j < nb - 1 ? boff[j + 1] : -1,
                          boff[j], -1));
    if (t < nb - 1) bot.push_back(add(3, t, bsz[t], bsz[t + 1], boff[t + 1], -1, 0, -1, PB, -1));
    const int L = std::max(top.size(), bot.size());
    while ((int)top.size() < L) top.push_back(idle);
    while ((int)bot.size() < L) bot.push_back(idle);
    // twist (top chain)
    top.push_back(add(4, t, bsz[t], bsz[t], PT, -1, t < nb - 1 ? bsz[t] : 0, t < nb - 1 ? PB : -1, X_ + boff[t], boff[t]));
    bot.push_back(idle);
    for (int s = 1; s < nb; ++s) {
        const int jt = t - s, jb = t + s;
        if (jt < 0 && jb > nb - 1) break;
        top.push_back(jt >= 0 ? add(5, jt, bsz[jt], bsz[jt], boff[jt], -1, bsz[jt + 1], X_ + boff[jt + 1],
                                    jt > 0 ? X_ + boff[jt] : -1, boff[jt])
                              : idle);
        bot.push_back(jb <= nb - 1 ? add(6, jb, bsz[jb], bsz[jb], boff[jb], -1, bsz[jb - 1], X_ + boff[jb - 1],
                                         jb < nb - 1 ? X_ + boff[jb] : -1, boff[jb])
                                   : idle);
    }
    store.alloc(std::max<long long>(o, 1));
    for (const Mat& mt : mats) {
        const int j = mt.j, mj = bsz[j], ld = mt.ld;
        double* X = store.p + mt.off;  // col-major (row length) x (output rows), leading dimension ld
        switch (mt.kind) {
            case 0:    // [Linv_j | -Linv_j K_{j-1}]  ->  [Linv_j^T; -K_{j-1}^T Linv_j^T]
            case 2: {  // p_top, the same with j = t
                PDG_CUBLAS_D(cublasDgeam(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, mj, mj, &one, Li(j), mj, &zero, Li(j), mj, X, ld));
                if (j > 0)
                    PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_T, bsz[j - 1], mj, mj, &mone, Kt(j - 1), mj, Li(j),
                                             mj, &zero, X + mj, ld));
                break;
            }
            case 1: {  // [Linv'_j | -Linv'_j K'_{j+1}]  ->  [Linv'_j^T; -K'_{j+1}^T Linv'_j^T]
                PDG_CUBLAS_D(cublasDgeam(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, mj, mj, &one, Li(j), mj, &zero, Li(j), mj, X, ld));
                if (j < nb - 1)
                    PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_T, bsz[j + 1], mj, mj, &mone, Kb(j + 1), mj, Li(j),
                                             mj, &zero, X + mj, ld));
                break;
            }
            case 3:  // [-Linv_t K'_{t+1}]  ->  -K'_{t+1}^T Linv_t^T
                PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_T, bsz[j + 1], mj, mj, &mone, Kb(j + 1), mj, Li(j), mj,
                                         &zero, X, ld));
                break;
            case 4: {  // [Linv_t^T | Linv_t^T]  ->  [Linv_t; Linv_t]
                PDG_CUBLAS_D(cublasDgeam(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, mj, mj, &one, Li(j), mj, &zero, Li(j), mj, X, ld));
                if (t < nb - 1)
                    PDG_CUBLAS_D(
                        cublasDgeam(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, mj, mj, &one, Li(j), mj, &zero, Li(j), mj, X + mj, ld));
                break;
            }
            case 5: {  // [Linv_j^T | -Linv_j^T K_j^T]  ->  [Linv_j; -K_j Linv_j]
                PDG_CUBLAS_D(cublasDgeam(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, mj, mj, &one, Li(j), mj, &zero, Li(j), mj, X, ld));
                PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, bsz[j + 1], mj, mj, &mone, Kt(j), bsz[j + 1],
                                         Li(j), mj, &zero, X + mj, ld));
                break;
            }
            default: {  // [Linv'_j^T | -Linv'_j^T K'_j^T]  ->  [Linv'_j; -K'_j Linv'_j]
                PDG_CUBLAS_D(cublasDgeam(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, mj, mj, &one, Li(j), mj, &zero, Li(j), mj, X, ld));
                PDG_CUBLAS_D(cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, bsz[j - 1], mj, mj, &mone, Kb(j), bsz[j - 1],
                                         Li(j), mj, &zero, X + mj, ld));
                break;
            }
        }
    }
    dsched.clear();
    for (size_t s = 0; s < top.size(); ++s) {
        dsched.push_back(top[s]);
        dsched.push_back(bot[s]);
    }
    d_dsched.upload(dsched, st);
    // ---- kernel configuration ------------------------------------------------------
    require(2 * max_b <= 256 * DNI, "block-tridiagonal solver: blocks too large for the dense sweep kernel");
    int dev = 0;
    PDG_CUDA(cudaGetDevice(&dev));
    int optin = 0;
    PDG_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    PDG_CUDA(cudaFuncSetAttribute(k_sweep_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    const int nsteps = static_cast<int>(dsched.size() / 2);
    d_ldmax = ldmax;
    d_g = (max_b + 7) / 8;
    require(2 * d_g <= num_sms(), "block-tridiagonal solver: blocks too large for the dense sweep kernel");
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
    int nsteps = static_cast<int>(dsched.size() / 2), nr = nrhs, n_ = n, ldm = d_ldmax, stg = d_stages, g = d_g;
    int pf = 4;
    if (const char* e = std::getenv("PDG_SWEEP_PF")) pf = std::atoi(e);
    long long lln = d_lln;
    const DenseTask* sched = d_dsched.p;
    const double* sp = store.p;
    uint4* llp = ll.p;
    unsigned long long* dbgp = nullptr;
    dbg_steps = nsteps;
    if (debug_timing) {
        dbg.alloc((size_t)2 * g * nsteps * 4);
        dbg.zero(st);
        dbgp = dbg.p;
    }
    void* args[] = {&nsteps, &sched, &nr, &n_, &sp, &ldm, &b, &x, &llp, &lln, &flag, &stg, &pf, &g, &dbgp};
    PDG_CUDA(cudaLaunchCooperativeKernel((void*)k_sweep_dense, 2 * g, 256, args, d_smem, st));
    count_launch(1);
    PDG_CHECK_LAUNCH();
}

}  // namespace pdg
