// Twisted block-tridiagonal Cholesky: layout, scatter of the dense blocks and
// the factorisation with cuSOLVER/cuBLAS (setup only). The solve is one
// persistent kernel per call: blocktri_local.cu (chunk-local couplings, the
// displacement block) or blocktri_dense.cu (any coupling, the flow block).
#include <algorithm>

#include "blocktri.cuh"

namespace pdg {

#define PDG_CUBLAS(call)                                                                                          \
    do {                                                                                                          \
        cublasStatus_t s_ = (call);                                                                               \
        if (s_ != CUBLAS_STATUS_SUCCESS)                                                                          \
            throw ::pdg::Error(PDG_CUDA_ERROR, std::string(#call) + ": cublas status " + std::to_string((int)s_)); \
    } while (0)
#define PDG_CUSOLVER(call)                                                                                          \
    do {                                                                                                            \
        cusolverStatus_t s_ = (call);                                                                               \
        if (s_ != CUSOLVER_STATUS_SUCCESS)                                                                          \
            throw ::pdg::Error(PDG_CUDA_ERROR, std::string(#call) + ": cusolver status " + std::to_string((int)s_)); \
    } while (0)

// cuBLAS / cuSOLVER handles are expensive to create (tens of ms each): one pair per host thread
// and device, created on first use and reused by every factorization (handles are not
// thread-safe, hence thread_local; they are released with the thread).
namespace {
struct HandleCache {
    cublasHandle_t blas[64] = {};
    cusolverDnHandle_t solver[64] = {};
    ~HandleCache() {
        for (int d = 0; d < 64; ++d) {
            if (blas[d]) cublasDestroy(blas[d]);
            if (solver[d]) cusolverDnDestroy(solver[d]);
        }
    }
};
thread_local HandleCache g_handles;
}  // namespace

LaHandles::LaHandles(cudaStream_t st) {
    int dev = 0;
    PDG_CUDA(cudaGetDevice(&dev));
    dev %= 64;
    if (!g_handles.blas[dev]) PDG_CUBLAS(cublasCreate(&g_handles.blas[dev]));
    if (!g_handles.solver[dev]) PDG_CUSOLVER(cusolverDnCreate(&g_handles.solver[dev]));
    blas = g_handles.blas[dev];
    solver = g_handles.solver[dev];
    PDG_CUBLAS(cublasSetStream(blas, st));
    PDG_CUSOLVER(cusolverDnSetStream(solver, st));
}
LaHandles::~LaHandles() {}

namespace {

// dense diagonal blocks D_j, sub-diagonal C_j = A_{j+1,j} and (non-symmetric
// matrices, dU != null) super-diagonal U_j = A_{j,j+1}, all col-major
__global__ void k_scatter_blocks(int n, const int* off, const int* idx, const double* val, const int* inv_perm,
                                 const int* blk_of, const int* loc_of, const int* bsz, const long long* dD,
                                 const long long* dC, const long long* dU, double* dense, int* err) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const int nr = inv_perm ? inv_perm[r] : r;
        const int jr = blk_of[nr], lr = loc_of[nr];
        for (int k = off[r]; k < off[r + 1]; ++k) {
            const int nc = inv_perm ? inv_perm[idx[k]] : idx[k];
            const int jc = blk_of[nc], lc = loc_of[nc];
            if (jc == jr)
                dense[dD[jr] + lr + (long long)lc * bsz[jr]] = val[k];
            else if (jr == jc + 1)
                dense[dC[jc] + lr + (long long)lc * bsz[jr]] = val[k];
            else if (jc == jr + 1) {
                if (dU) dense[dU[jr] + lr + (long long)lc * bsz[jr]] = val[k];
            } else
                atomicOr(err, 1);
        }
    }
}

__global__ void k_gather(int n, int nrhs, const int* perm, const double* b, long long ldb, double* out) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)n * nrhs;
         t += (long long)gridDim.x * blockDim.x) {
        const int r = static_cast<int>(t % n), k = static_cast<int>(t / n);
        out[t] = b[(perm ? perm[r] : r) + k * ldb];
    }
}
__global__ void k_scatter(int n, int nrhs, const int* perm, const double* in, double* x, long long ldx) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)n * nrhs;
         t += (long long)gridDim.x * blockDim.x) {
        const int r = static_cast<int>(t % n), k = static_cast<int>(t / n);
        x[(perm ? perm[r] : r) + k * ldx] = in[t];
    }
}

}  // namespace

void BlockTriChol::layout(int n_, const std::vector<int>& perm_host, const std::vector<int>& block_sizes) {
    n = n_;
    bsz = block_sizes;
    nb = static_cast<int>(bsz.size());
    boff.assign(nb + 1, 0);
    for (int j = 0; j < nb; ++j) boff[j + 1] = boff[j] + bsz[j];
    require(nb >= 1 && boff[nb] == n, "block-tridiagonal solver: block sizes do not sum to n");
    max_b = *std::max_element(bsz.begin(), bsz.end());
    std::vector<int> blk(n), loc(n);
    for (int j = 0; j < nb; ++j)
        for (int r = 0; r < bsz[j]; ++r) {
            blk[boff[j] + r] = j;
            loc[boff[j] + r] = r;
        }
    blk_of.upload(blk);
    loc_of.upload(loc);
    if (!perm_host.empty()) {
        require(static_cast<int>(perm_host.size()) == n, "block-tridiagonal solver: bad permutation size");
        std::vector<int> inv(n, -1);
        for (int i = 0; i < n; ++i) inv[perm_host[i]] = i;
        perm.upload(perm_host);
        inv_perm.upload(inv);
    }
    dD_.assign(nb, 0);
    dC_.assign(nb, 0);
    long long o = 0;
    for (int j = 0; j < nb; ++j) {
        dD_[j] = o;
        o += (long long)bsz[j] * bsz[j];
    }
    for (int j = 0; j + 1 < nb; ++j) {
        dC_[j] = o;
        o += (long long)bsz[j + 1] * bsz[j];
    }
    dU_.assign(nb, -1);
    if (!symmetric)
        for (int j = 0; j + 1 < nb; ++j) {
            dU_[j] = o;
            o += (long long)bsz[j] * bsz[j + 1];
        }
    dtot_ = o;
    d_bsz.upload(bsz);
    d_boff.upload(std::vector<int>(boff.begin(), boff.end() - 1));
    twist = (nb - 1) / 2;
}

void BlockTriChol::factor(int n_, const int* off, const int* idx, const double* val, const std::vector<int>& perm_host,
                          const std::vector<int>& block_sizes, int max_rhs_, cudaStream_t st) {
    layout(n_, perm_host, block_sizes);
    max_rhs = max_rhs_;
    DBuf<double> dense(dtot_);
    dense.zero(st);
    DBuf<long long> ddD, ddC, ddU;
    ddD.upload(dD_, st);
    ddC.upload(dC_, st);
    if (!symmetric) ddU.upload(dU_, st);
    DBuf<int> err(1);
    err.zero(st);
    k_scatter_blocks<<<grid_for(n, 256), 256, 0, st>>>(n, off, idx, val, perm.n ? inv_perm.p : nullptr, blk_of.p,
                                                        loc_of.p, d_bsz.p, ddD.p, ddC.p, symmetric ? nullptr : ddU.p,
                                                        dense.p, err.p);
    PDG_CHECK_LAUNCH();
    int herr = 0;
    PDG_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    require(herr == 0, "block-tridiagonal solver: matrix is not block tridiagonal in the given ordering");
    factor_dense(dense.p, st);
}

void BlockTriChol::factor_dense(double* dense, cudaStream_t st) {
    if (!symmetric) {  // twisted block LU, dense-sweep solve
        dense_setup(dense, st);
        return;
    }
    local_prepare(dense, st);  // before the couplings are overwritten by the factorisation
    if (!local) {
        dense_setup(dense, st);
        return;
    }
    LaHandles h(st);
    const int t = twist;
    int lwork = 0;
    PDG_CUSOLVER(cusolverDnDpotrf_bufferSize(h.solver, CUBLAS_FILL_MODE_LOWER, max_b, dense, max_b, &lwork));
    DBuf<double> work(std::max(lwork, 1));
    DBuf<int> info(nb);
    info.zero(st);
    const double one = 1.0, mone = -1.0, zero = 0.0;
    auto D = [&](int j) { return dense + dD_[j]; };
    auto C = [&](int j) { return dense + dC_[j]; };  // A_{j+1,j}, m_{j+1} x m_j, becomes K_j (top)
    // K'_j = A_{j-1,j} L'_j^{-T} (m_{j-1} x m_j) for the bottom part
    std::vector<long long> oKp(nb, -1);
    long long kp_tot = 0;
    for (int j = t + 1; j < nb; ++j) {
        oKp[j] = kp_tot;
        kp_tot += (long long)bsz[j - 1] * bsz[j];
    }
    DBuf<double> kp(std::max<long long>(kp_tot, 1));
    // top: blocks 0..t-1
    for (int j = 0; j < t; ++j) {
        const int mj = bsz[j];
        if (j > 0)
            PDG_CUBLAS(cublasDsyrk(h.blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, mj, bsz[j - 1], &mone, C(j - 1), mj, &one,
                                   D(j), mj));
        PDG_CUSOLVER(cusolverDnDpotrf(h.solver, CUBLAS_FILL_MODE_LOWER, mj, D(j), mj, work.p, lwork, info.p + j));
        PDG_CUBLAS(cublasDtrsm(h.blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT,
                               bsz[j + 1], mj, &one, D(j), mj, C(j), bsz[j + 1]));
    }
    // bottom: blocks nb-1..t+1
    for (int j = nb - 1; j > t; --j) {
        const int mj = bsz[j];
        if (j < nb - 1)
            PDG_CUBLAS(cublasDsyrk(h.blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, mj, bsz[j + 1], &mone, kp.p + oKp[j + 1],
                                   mj, &one, D(j), mj));
        PDG_CUSOLVER(cusolverDnDpotrf(h.solver, CUBLAS_FILL_MODE_LOWER, mj, D(j), mj, work.p, lwork, info.p + j));
        // K'_j = C_{j-1}^T L'_j^{-T}
        const int mp = bsz[j - 1];
        PDG_CUBLAS(cublasDgeam(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, mp, mj, &one, C(j - 1), mj, &zero, kp.p + oKp[j], mp,
                               kp.p + oKp[j], mp));
        PDG_CUBLAS(cublasDtrsm(h.blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, mp,
                               mj, &one, D(j), mj, kp.p + oKp[j], mp));
    }
    // twist block
    {
        const int mt = bsz[t];
        if (t > 0)
            PDG_CUBLAS(cublasDsyrk(h.blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, mt, bsz[t - 1], &mone, C(t - 1), mt, &one,
                                   D(t), mt));
        if (t + 1 < nb)
            PDG_CUBLAS(cublasDsyrk(h.blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, mt, bsz[t + 1], &mone, kp.p + oKp[t + 1],
                                   mt, &one, D(t), mt));
        PDG_CUSOLVER(cusolverDnDpotrf(h.solver, CUBLAS_FILL_MODE_LOWER, mt, D(t), mt, work.p, lwork, info.p + t));
    }
    std::vector<int> hinfo = info.download(st);
    for (int j = 0; j < nb; ++j)
        if (hinfo[j] != 0)
            throw Error(PDG_NOT_CONVERGED, "dense LU: matrix is singular to working precision (block " +
                                               std::to_string(j) + " not positive definite)");
    local_finish(dense, st);
}

void BlockTriChol::solve(const double* b, long long ldb, double* x, long long ldx, int nrhs, cudaStream_t st) {
    ProfScope prof(prof_phase, st, alg_bytes(nrhs));
    require(nrhs >= 1 && nrhs <= max_rhs && nrhs <= 2, "block-tridiagonal solve: bad nrhs");
    if (local) {
        solve_local(b, ldb, x, ldx, nrhs, st);
        return;
    }
    const int* pp = perm.n ? perm.p : nullptr;
    const long long tot = (long long)n * nrhs;
    k_gather<<<grid_for(tot, 256), 256, 0, st>>>(n, nrhs, pp, b, ldb, wb.p);
    solve_dense(wb.p, wx.p, nrhs, st);
    k_scatter<<<grid_for(tot, 256), 256, 0, st>>>(n, nrhs, pp, wx.p, x, ldx);
    count_launch(2);
    PDG_CHECK_LAUNCH();
}

}  // namespace pdg
