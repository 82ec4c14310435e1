// Level-synchronous solve of the LOCAL subtrees of the hybrid nested-dissection solve
// (NdChol::local_lvl; PDG_ND_LOCAL_LEVELS=1). The chunk kernel (nd.cu) runs a local subtree as
// ~15 tasks per pass on one CTA, each through stage -> gather -> compute -> signal; measured,
// that chain and not bandwidth bounds it. Here a CTA takes ALL fronts of one
// depth of its subtree at once (8 leaves, then 4, 2, 1 fronts): their input vectors are formed in
// shared memory in one round of loads, then the 16 warps stream groups of 8 rows of all those
// fronts straight from the row-major factor store (16-byte loads, the zero triangle of L_SS^{-1}
// skipped), then the CTA moves up (forward) or down (backward) one depth. The math per front is
// that of nd_stream.cu:
//   forward   [y_S; u_F] = M (b_S - w_C1|S - w_C2|S),  w_F = u_F + w_C1|B + w_C2|B  (into the parent's slot)
//   backward  x_S = M^T [y_S; -x_B]
// Sums run in a fixed order: repeats are bit-identical.
#include <algorithm>
#include <cstdlib>

#include "nd.cuh"

namespace pdg {

namespace {

constexpr int kLThreads = 512;
constexpr int kLWarps = kLThreads / 32;
constexpr int kLRows = 8;        // rows per warp item
constexpr int kLMaxFronts = 64;  // fronts of one depth of one subtree

struct LocalArgs {
    const NdLocalFront* fronts;
    const int* cta_off;  // per CTA: its levels [cta_off[c], cta_off[c + 1]) (root level first)
    const int* lev_off;  // per level: its fronts [lev_off[l], lev_off[l + 1])
    const int* sdofs;
    const int* bpos;
    const int* cbdst;
    const double* store;
    const double* b;
    long long ldb;
    double* x;
    long long ldx;
    double* y;
    double* xpos;
    double* cb;
    long long cbtot;
    int n;
    const int* stop;
};

template <int NR, int PASS>
__global__ void __launch_bounds__(kLThreads, 1) k_nd_local(LocalArgs a) {
    if (a.stop && *a.stop) return;  // speculative GMRES step after the cycle ended
    extern __shared__ __align__(16) double vs[];  // per front of the level: NR x stride input vectors
    __shared__ int voff[kLMaxFronts + 1], ioff[kLMaxFronts + 1];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int l0 = a.cta_off[blockIdx.x], l1 = a.cta_off[blockIdx.x + 1];
    for (int li = 0; li < l1 - l0; ++li) {
        const int l = PASS == 1 ? l1 - 1 - li : l0 + li;  // forward: deepest level first
        const int f0 = a.lev_off[l], nf = a.lev_off[l + 1] - f0;
        if (tid < nf) {  // sizes, then an exclusive scan by one thread (at most 64 entries)
            const NdLocalFront& F = a.fronts[f0 + tid];
            voff[tid + 1] = NR * F.ldt;
            ioff[tid + 1] = ((PASS == 1 ? F.s + F.b : F.s) + kLRows - 1) / kLRows;
        }
        // the next depth's matrices into L2 while this depth runs (static data)
        if (li + 1 < l1 - l0 && warp == kLWarps - 1) {
            const int ln = PASS == 1 ? l - 1 : l + 1;
            for (int f = a.lev_off[ln] + lane; f < a.lev_off[ln + 1]; f += 32) {
                const NdLocalFront& F = a.fronts[f];
                const double* base = a.store + (PASS == 1 ? F.moff : F.mtoff);
                const long long bytes = 8LL * (PASS == 1 ? (long long)(F.s + F.b) * F.ldm : (long long)F.s * F.ldt);
                for (long long off = 0; off < bytes; off += 65536)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<const char*>(base) + off),
                                 "r"(static_cast<unsigned>(min(65536LL, bytes - off)))
                                 : "memory");
            }
        }
        __syncthreads();
        if (tid == 0) {
            voff[0] = ioff[0] = 0;
            for (int f = 0; f < nf; ++f) {
                voff[f + 1] += voff[f];
                ioff[f + 1] += ioff[f];
            }
        }
        __syncthreads();
        // ---- phase A: the input vectors of all fronts of this depth, one flat round of loads ----
        {
            int f = 0;
            for (int e = tid; e < voff[nf]; e += kLThreads) {
                while (e >= voff[f + 1]) ++f;
                const NdLocalFront& F = a.fronts[f0 + f];
                const int len = PASS == 1 ? F.s : F.s + F.b;
                const int sb = F.s + F.b;
                const int el = e - voff[f], k = el / F.ldt, c = el - k * F.ldt;
                double val = 0.0;
                if (c < len) {
                    if (PASS == 1) {
                        const double* cbk = a.cb + k * a.cbtot + F.cboff;
                        val = (a.b[k * a.ldb + __ldg(a.sdofs + F.sdof + c)] - __ldcg(cbk + c)) - __ldcg(cbk + sb + c);
                    } else {
                        val = c < F.s ? __ldcg(a.y + (long long)k * a.n + F.sdof + c)
                                      : -__ldcg(a.xpos + (long long)k * a.n + __ldg(a.bpos + F.bdof + c - F.s));
                    }
                }
                vs[e] = val;
            }
        }
        __syncthreads();
        // ---- phase B: groups of 8 rows over the warps ----
        const int nitems = ioff[nf];
        int f = 0;
        for (int it = warp; it < nitems; it += kLWarps) {
            while (it >= ioff[f + 1]) ++f;
            const NdLocalFront F = a.fronts[f0 + f];
            const int rows = PASS == 1 ? F.s + F.b : F.s;
            const int r0 = (it - ioff[f]) * kLRows, nrow = min(kLRows, rows - r0);
            const int ld = PASS == 1 ? F.ldm : F.ldt;
            // columns that can be nonzero: forward rows r < s have entries up to column r; backward
            // row r (of L_SS^{-T} | G^T) from column r on
            int c0 = 0, c1 = ld;
            if (PASS == 1) {
                if (r0 + nrow <= F.s) c1 = min(ld, (r0 + nrow + 1) & ~1);
            } else {
                c0 = r0 & ~1;
            }
            const double* rowp = a.store + (PASS == 1 ? F.moff : F.mtoff) + (long long)r0 * ld;
            const double* v = vs + voff[f];
            double acc[kLRows][NR];
#pragma unroll
            for (int j = 0; j < kLRows; ++j)
#pragma unroll
                for (int k = 0; k < NR; ++k) acc[j][k] = 0.0;
            const int p0 = c0 >> 1, p1 = c1 >> 1;
            if (nrow == kLRows) {
                for (int p = p0 + lane; p < p1; p += 32) {
                    double2 m[kLRows];
#pragma unroll
                    for (int j = 0; j < kLRows; ++j) m[j] = __ldcs(reinterpret_cast<const double2*>(rowp + (long long)j * ld) + p);
#pragma unroll
                    for (int k = 0; k < NR; ++k) {
                        const double2 w = *reinterpret_cast<const double2*>(v + k * F.ldt + 2 * p);
#pragma unroll
                        for (int j = 0; j < kLRows; ++j) acc[j][k] = fma(m[j].y, w.y, fma(m[j].x, w.x, acc[j][k]));
                    }
                }
            } else {
                for (int p = p0 + lane; p < p1; p += 32) {
#pragma unroll
                    for (int j = 0; j < kLRows; ++j)
                        if (j < nrow) {
                            const double2 m = __ldcs(reinterpret_cast<const double2*>(rowp + (long long)j * ld) + p);
#pragma unroll
                            for (int k = 0; k < NR; ++k) {
                                const double2 w = *reinterpret_cast<const double2*>(v + k * F.ldt + 2 * p);
                                acc[j][k] = fma(m.y, w.y, fma(m.x, w.x, acc[j][k]));
                            }
                        }
                }
            }
#pragma unroll
            for (int j = 0; j < kLRows; ++j)
#pragma unroll
                for (int k = 0; k < NR; ++k) {
                    double s = acc[j][k];
                    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                    acc[j][k] = s;
                }
            if (lane < nrow) {
                const int gr = r0 + lane;
#pragma unroll
                for (int k = 0; k < NR; ++k) {
                    double s = 0.0;
#pragma unroll
                    for (int j = 0; j < kLRows; ++j)
                        if (j == lane) s = acc[j][k];
                    if (PASS == 2) {
                        a.xpos[(long long)k * a.n + F.sdof + gr] = s;
                        a.x[k * a.ldx + __ldg(a.sdofs + F.sdof + gr)] = s;
                    } else if (gr < F.s) {
                        a.y[(long long)k * a.n + F.sdof + gr] = s;
                    } else {  // update vector entry plus the children's pass-through, into the parent's slot
                        const double* cbk = a.cb + k * a.cbtot + F.cboff;
                        const double tail = __ldcg(cbk + gr) + __ldcg(cbk + (F.s + F.b) + gr);
                        a.cb[k * a.cbtot + __ldg(a.cbdst + F.bdof + gr - F.s)] = s + tail;
                    }
                }
            }
        }
        __syncthreads();  // this depth's outputs are written before the next depth's gather reads them
    }
}

}  // namespace

// Per subtree root (a front at depth hybrid_top + 1) one CTA; its levels root first.
void NdChol::build_local(const std::vector<std::vector<int>>& children, cudaStream_t st) {
    local_lvl = false;
    const char* e = std::getenv("PDG_ND_LOCAL_LEVELS");
    if (!hybrid || !(e && std::atoi(e) == 1)) return;
    const int ld0 = hybrid_top + 1;
    std::vector<NdLocalFront> lf;
    std::vector<int> cta_off{0}, lev_off{0};
    size_t smem_need = 0;
    for (int k = 0; k < nfront; ++k) {
        if (fronts[k].depth != ld0) continue;
        std::vector<int> level{k};
        while (!level.empty()) {
            if (level.size() > (size_t)kLMaxFronts) return;  // (not with binary dissections below 2^6 levels)
            size_t by = 0;
            std::vector<int> next;
            for (int f : level) {
                const NdFront& F = fronts[f];
                lf.push_back({F.moff, F.mtoff, F.ldm, F.ldt, F.s, F.b, F.sdof, F.bdof, F.cboff, 0});
                by += (size_t)max_rhs * F.ldt * sizeof(double);
                for (int c : children[f]) next.push_back(c);
            }
            smem_need = std::max(smem_need, by);
            lev_off.push_back(static_cast<int>(lf.size()));
            level.swap(next);
        }
        cta_off.push_back(static_cast<int>(lev_off.size()) - 1);
    }
    if (cta_off.size() < 2 || smem_need > 200 * 1024) return;
    d_lfronts.upload(lf, st);
    d_lcta.upload(cta_off, st);
    d_llev.upload(lev_off, st);
    local_ctas = static_cast<int>(cta_off.size()) - 1;
    local_smem = smem_need;
    for (auto* fn : {(const void*)k_nd_local<1, 1>, (const void*)k_nd_local<1, 2>, (const void*)k_nd_local<2, 1>,
                     (const void*)k_nd_local<2, 2>})
        PDG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(200 * 1024)));
    PDG_CUDA(cudaStreamSynchronize(st));
    local_lvl = true;
}

void NdChol::solve_local(int pass, const double* b, long long ldb, double* x, long long ldx, int nrhs, cudaStream_t st) {
    LocalArgs a{d_lfronts.p, d_lcta.p, d_llev.p, sdofs.p, bpos.p, cbdst.p, store.p, b, ldb, x, ldx, y.p, xpos.p, cbuf.p, cbtot, n, guard};
    if (nrhs == 1) {
        if (pass == 1) k_nd_local<1, 1><<<local_ctas, kLThreads, local_smem, st>>>(a);
        else k_nd_local<1, 2><<<local_ctas, kLThreads, local_smem, st>>>(a);
    } else {
        if (pass == 1) k_nd_local<2, 1><<<local_ctas, kLThreads, local_smem, st>>>(a);
        else k_nd_local<2, 2><<<local_ctas, kLThreads, local_smem, st>>>(a);
    }
    count_launch(1);
    PDG_CHECK_LAUNCH();
}

}  // namespace pdg
