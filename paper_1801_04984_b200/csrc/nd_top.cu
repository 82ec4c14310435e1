// Dense top of the nested-dissection solve (nd.cuh, PDG_ND_TOP / PDG_ND_FLOW_TOP).
//
// The fronts of depth <= top_depth (the top separators; pivot positions [top0, n) in the
// elimination order) are not solved front by front. With T their pivots and L the rest,
// block elimination gives
//     x_T = S_TT^{-1} (b_T - L_TL L_LL^{-1} b_L),   S_TT = L_TT L_TT^T,
// and the update vectors the forward pass of the fronts below T already produces (their
// contributions into the contribution slots of the depth-top_depth fronts) sum to
// L_TL L_LL^{-1} b_L. So one solve is: the forward pass of the fronts below T, the top
// right-hand side c_T = b_T - (those contributions, in a fixed order), ONE dense GEMV
// x_T = G c_T with G = S_TT^{-1} = (A^{-1})_TT (setup: L_TT assembled from the top fronts'
// factored frontal matrices, cuSOLVER potri), then the backward pass of the fronts below,
// which reads x_T as the boundary values of the fronts next to T. This replaces
// 2 (top_depth + 1) dependent levels by two launches, for |T|^2 doubles streamed instead of
// the top fronts' M and M^T.
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "blocktri.cuh"
#include "nd.cuh"

namespace pdg {

namespace {

constexpr int kTopThreads = 512;
constexpr int kTopCap = 6144;  // |T| at most (G <= 302 MB; the GEMV holds c_T in shared memory)

// L_TT (col-major ntop x ntop) <- one top front's factored frontal matrix (col-major f x f:
// L_SS in the leading s x s lower triangle, L_BS below it); rows of the boundary dofs at
// their pivot positions
__global__ void k_nd_top_scatter(const double* Fk, int f, int s, int col0, const int* bpos_f, int top0, double* L,
                                 int ntop) {
    const long long tot = (long long)f * s;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
        const int i = static_cast<int>(t % f), j = static_cast<int>(t / f);
        if (i < j) continue;
        const int row = i < s ? col0 + i : bpos_f[i - s] - top0;
        L[row + (long long)(col0 + j) * ntop] = Fk[i + (long long)j * f];
    }
}

// G (row-major ntop x ldg, zero padded) <- the symmetric inverse from potri's lower triangle
__global__ void k_nd_top_sym(const double* Li, int ntop, double* G, int ldg) {
    const long long tot = (long long)ntop * ldg;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
        const int r = static_cast<int>(t / ldg), c = static_cast<int>(t % ldg);
        double v = 0.0;
        if (c < ntop) v = r >= c ? Li[r + (long long)c * ntop] : Li[c + (long long)r * ntop];
        G[t] = v;
    }
}

struct TopArgs {
    const double* G;
    const double* b;
    long long ldb;
    double* x;
    long long ldx;
    double* xpos;
    const double* cb;
    long long cbtot;
    double* c;
    const int* sdofs;
    const int* coff;
    const int* clist;
    const int* stop;
    int n, nrhs, top0, ntop, ldg, rows_per_cta;
    long long pf_bytes;
};

// c_T[k][p] = b[k][dof(p)] - its contributions (fixed order); padding zero
__global__ void k_nd_top_rhs(TopArgs a) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (a.stop && *a.stop) return;  // speculative GMRES step after the cycle ended
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= 2 * a.ldg) return;
    const int k = e / a.ldg, p = e - k * a.ldg;
    double v = 0.0;
    if (k < a.nrhs && p < a.ntop) {
        v = a.b[k * a.ldb + __ldg(a.sdofs + a.top0 + p)];
        const double* cbk = a.cb + k * a.cbtot;
        for (int j = __ldg(a.coff + p), j1 = __ldg(a.coff + p + 1); j < j1; ++j) v = v - __ldcg(cbk + __ldg(a.clist + j));
    }
    a.c[e] = v;
}

// x_T = G c_T: rows_per_cta rows per block, one warp per row (lanes over the columns in
// 512 B coalesced loads, 4 independent chains per right-hand side, then a butterfly: a
// fixed order, bit-identical repeats); c_T in shared memory. The block's rows of G are
// prefetched into L2 (pf_bytes) before the dependency wait: G is static.
__global__ void __launch_bounds__(kTopThreads, 2) k_nd_top_gemv(TopArgs a) {
    extern __shared__ __align__(16) double cs[];  // [2][ldg]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int r0 = blockIdx.x * a.rows_per_cta, r1 = min(a.ntop, r0 + a.rows_per_cta);
    if (a.pf_bytes > 0 && r1 > r0) {
        const long long bytes = min(a.pf_bytes, (long long)(r1 - r0) * a.ldg * 8);
        const char* base = reinterpret_cast<const char*>(a.G + (long long)r0 * a.ldg);
        for (long long off = (long long)tid * 8192; off < bytes; off += (long long)kTopThreads * 8192)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + off),
                         "r"(static_cast<unsigned>(min(8192LL, bytes - off)))
                         : "memory");
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (a.stop && *a.stop) return;
    {
        const double2* src = reinterpret_cast<const double2*>(a.c);
        double2* dst = reinterpret_cast<double2*>(cs);
        for (int i = tid; i < a.ldg; i += kTopThreads) dst[i] = __ldcg(src + i);  // 2 ldg doubles
    }
    __syncthreads();
    const int nit = a.ldg >> 6;  // 64 doubles (512 B) per warp iteration
    const double2* c0 = reinterpret_cast<const double2*>(cs) + lane;
    const double2* c1 = reinterpret_cast<const double2*>(cs + a.ldg) + lane;
    for (int r = r0 + warp; r < r1; r += kTopThreads / 32) {
        const double2* g = reinterpret_cast<const double2*>(a.G + (long long)r * a.ldg) + lane;
        double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0, q0 = 0.0, q1 = 0.0, q2 = 0.0, q3 = 0.0;
        int it = 0;
        for (; it + 3 < nit; it += 4) {
            const double2 m0 = __ldcs(g + it * 32), m1 = __ldcs(g + (it + 1) * 32);
            const double2 m2 = __ldcs(g + (it + 2) * 32), m3 = __ldcs(g + (it + 3) * 32);
            const double2 a0 = c0[it * 32], a1 = c0[(it + 1) * 32], a2 = c0[(it + 2) * 32], a3 = c0[(it + 3) * 32];
            const double2 b0 = c1[it * 32], b1 = c1[(it + 1) * 32], b2 = c1[(it + 2) * 32], b3 = c1[(it + 3) * 32];
            p0 = fma(m0.x, a0.x, p0);
            p1 = fma(m0.y, a0.y, p1);
            q0 = fma(m0.x, b0.x, q0);
            q1 = fma(m0.y, b0.y, q1);
            p2 = fma(m1.x, a1.x, p2);
            p3 = fma(m1.y, a1.y, p3);
            q2 = fma(m1.x, b1.x, q2);
            q3 = fma(m1.y, b1.y, q3);
            p0 = fma(m2.x, a2.x, p0);
            p1 = fma(m2.y, a2.y, p1);
            q0 = fma(m2.x, b2.x, q0);
            q1 = fma(m2.y, b2.y, q1);
            p2 = fma(m3.x, a3.x, p2);
            p3 = fma(m3.y, a3.y, p3);
            q2 = fma(m3.x, b3.x, q2);
            q3 = fma(m3.y, b3.y, q3);
        }
        for (; it < nit; ++it) {
            const double2 m0 = __ldcs(g + it * 32), a0 = c0[it * 32], b0 = c1[it * 32];
            p0 = fma(m0.x, a0.x, p0);
            p1 = fma(m0.y, a0.y, p1);
            q0 = fma(m0.x, b0.x, q0);
            q1 = fma(m0.y, b0.y, q1);
        }
        double s0 = (p0 + p1) + (p2 + p3), s1 = (q0 + q1) + (q2 + q3);
        for (int o = 1; o < 32; o <<= 1) {
            s0 += __shfl_xor_sync(0xffffffffu, s0, o);
            s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        }
        if (lane == 0) {
            const int d = __ldg(a.sdofs + a.top0 + r);
            a.xpos[a.top0 + r] = s0;
            a.x[d] = s0;
            if (a.nrhs > 1) {
                a.xpos[(long long)a.n + a.top0 + r] = s1;
                a.x[a.ldx + d] = s1;
            }
        }
    }
}

}  // namespace

// PDG_ND_TOP (displacement solves) / PDG_ND_FLOW_TOP (flux solves): the deepest front level
// of the dense top (-1: none); the setup lowers it until |T| fits kTopCap
int nd_top_default(int prof_phase) {
    const char* e = std::getenv(prof_phase == PROF_A_SOLVE ? "PDG_ND_TOP" : "PDG_ND_FLOW_TOP");
    if (e) return std::atoi(e);
    return prof_phase == PROF_A_SOLVE ? 2 : 5;
}

void NdChol::build_top(const std::vector<int>& hbp, const std::vector<std::vector<int>>& children,
                       const std::vector<long long>& fo, const double* dense, LaHandles& h, cudaStream_t st) {
    const int nf = static_cast<int>(fronts.size());
    int kt = nf;
    while (kt > 0 && fronts[kt - 1].depth <= top_depth) --kt;
    for (int k = 0; k < kt; ++k) require(fronts[k].depth > top_depth, "nested dissection: top fronts not last");
    require(kt < nf && kt > 0, "nested dissection: empty top");
    top0 = fronts[kt].sdof;
    ntop = n - top0;
    ldg = (ntop + 63) / 64 * 64;
    // L_TT from the top fronts' factors, then G = (L_TT L_TT^T)^{-1}
    DBuf<double> L((size_t)ntop * ntop);
    L.zero(st);
    for (int k = kt; k < nf; ++k) {
        const NdFront& F = fronts[k];
        const int f = F.s + F.b;
        k_nd_top_scatter<<<grid_for((long long)f * F.s, 256), 256, 0, st>>>(dense + fo[k], f, F.s, F.sdof - top0,
                                                                          bpos.p + F.bdof, top0, L.p, ntop);
        PDG_CHECK_LAUNCH();
    }
    {
        int lwork = 0;
        if (cusolverDnDpotri_bufferSize(h.solver, CUBLAS_FILL_MODE_LOWER, ntop, L.p, ntop, &lwork) != CUSOLVER_STATUS_SUCCESS)
            throw Error(PDG_CUDA_ERROR, "nested dissection: potri workspace query failed");
        DBuf<double> work((size_t)std::max(lwork, 1));
        DBuf<int> info(1);
        info.zero(st);
        if (cusolverDnDpotri(h.solver, CUBLAS_FILL_MODE_LOWER, ntop, L.p, ntop, work.p, lwork, info.p) !=
            CUSOLVER_STATUS_SUCCESS)
            throw Error(PDG_CUDA_ERROR, "nested dissection: potri failed");
        const std::vector<int> hi = info.download(st);
        if (hi[0] != 0) throw Error(PDG_NOT_CONVERGED, "nested dissection: top Schur complement singular");
    }
    gtop.alloc((size_t)ntop * ldg);
    k_nd_top_sym<<<grid_for((long long)ntop * ldg, 256), 256, 0, st>>>(L.p, ntop, gtop.p, ldg);
    PDG_CHECK_LAUNCH();
    // contributions: the children's slots of every depth-top_depth front, at the front's
    // local positions (pivots, then boundary dofs), fronts in order, child 0 then 1
    std::vector<std::vector<int>> lists(ntop);
    for (int k = kt; k < nf; ++k) {
        const NdFront& F = fronts[k];
        if (F.depth != top_depth) continue;
        const int f = F.s + F.b, nch = static_cast<int>(children[k].size());
        for (int i = 0; i < f; ++i) {
            const int p = (i < F.s ? F.sdof + i : hbp[F.bdof + i - F.s]) - top0;
            require(p >= 0 && p < ntop, "nested dissection: top boundary outside the top");
            for (int q = 0; q < nch; ++q) lists[p].push_back(F.cboff + q * f + i);
        }
    }
    std::vector<int> coff(ntop + 1, 0), cl;
    for (int p = 0; p < ntop; ++p) {
        cl.insert(cl.end(), lists[p].begin(), lists[p].end());
        coff[p + 1] = static_cast<int>(cl.size());
    }
    if (cl.empty()) cl.push_back(0);
    top_coff.upload(coff, st);
    top_clist.upload(cl, st);
    ctop.alloc((size_t)2 * ldg);
    ctop.zero(st);
    // bytes per solve: the fronts below T (M and M^T once each) and G once
    factor_bytes = 0.0;
    for (int k = 0; k < kt; ++k) factor_bytes += 16.0 * (double)(fronts[k].s + fronts[k].b) * fronts[k].s;
    factor_bytes += 8.0 * (double)ntop * ntop;
    // the attribute is per device and only ever raised: the largest seen on this device
    static size_t attr[64] = {};
    int dev = 0;
    PDG_CUDA(cudaGetDevice(&dev));
    const size_t smem = 2 * (size_t)ldg * sizeof(double);
    if (smem > attr[dev % 64]) {
        PDG_CUDA(cudaFuncSetAttribute(k_nd_top_gemv, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        attr[dev % 64] = smem;
    }
    PDG_CUDA(cudaStreamSynchronize(st));
}

void NdChol::solve_top(const double* b, long long ldb, double* x, long long ldx, int nrhs, cudaStream_t st) {
    int dev = 0, nsm = 0;
    PDG_CUDA(cudaGetDevice(&dev));
    PDG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    static const int bpsm = std::getenv("PDG_ND_TOP_BLOCKS") ? std::max(1, std::atoi(std::getenv("PDG_ND_TOP_BLOCKS"))) : 2;
    static const long long pf = std::getenv("PDG_ND_TOP_PF") ? std::atoll(std::getenv("PDG_ND_TOP_PF")) : 0;
    TopArgs a{};
    a.G = gtop.p;
    a.b = b;
    a.ldb = ldb;
    a.x = x;
    a.ldx = ldx;
    a.xpos = xpos.p;
    a.cb = cbuf.p;
    a.cbtot = cbtot;
    a.c = ctop.p;
    a.sdofs = sdofs.p;
    a.coff = top_coff.p;
    a.clist = top_clist.p;
    a.stop = guard;
    a.n = n;
    a.nrhs = nrhs;
    a.top0 = top0;
    a.ntop = ntop;
    a.ldg = ldg;
    const int grid = bpsm * nsm;
    a.rows_per_cta = (ntop + grid - 1) / grid;
    a.pf_bytes = pf;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>((2 * ldg + 255) / 256));
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    PDG_CUDA(cudaLaunchKernelEx(&cfg, k_nd_top_rhs, a));
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(kTopThreads);
    cfg.dynamicSmemBytes = 2 * (size_t)ldg * sizeof(double);
    PDG_CUDA(cudaLaunchKernelEx(&cfg, k_nd_top_gemv, a));
    count_launch(2);
    PDG_CHECK_LAUNCH();
}

int nd_top_cap() { return kTopCap; }

}  // namespace pdg
