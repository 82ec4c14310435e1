// Twisted block-tridiagonal Cholesky: factorisation with cuSOLVER/cuBLAS
// (setup only), solve with hand-written kernels: two bandwidth-bound
// block-diagonal GEMV passes and two persistent cooperative recurrences, each
// running a top and a bottom chain concurrently as a barrier-free dataflow
// with TMA-streamed matrix rows.
#include <algorithm>

#include "blocktri.cuh"
#include "llsync.cuh"

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

LaHandles::LaHandles(cudaStream_t st) {
    PDG_CUBLAS(cublasCreate(&blas));
    PDG_CUBLAS(cublasSetStream(blas, st));
    PDG_CUSOLVER(cusolverDnCreate(&solver));
    PDG_CUSOLVER(cusolverDnSetStream(solver, st));
}
LaHandles::~LaHandles() {
    if (blas) cublasDestroy(blas);
    if (solver) cusolverDnDestroy(solver);
}

namespace {

__global__ void k_scatter_blocks(int n, const int* off, const int* idx, const double* val, const int* inv_perm,
                                 const int* blk_of, const int* loc_of, const int* bsz, const long long* dD,
                                 const long long* dC, double* dense, int* err) {
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
            else if (jc != jr + 1)
                atomicOr(err, 1);
        }
    }
}

__global__ void k_identity(int m, double* a) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * m;
         t += (long long)gridDim.x * blockDim.x)
        a[t] = (t % m == t / m) ? 1.0 : 0.0;
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

// c_j = Linv_j b_j on the row-major copy of Linv: one warp per row, all
// right-hand sides (the factor is read once).
__global__ void __launch_bounds__(256) k_blockdiag_lower_rows(int n, int nrhs, const int* __restrict__ blk_of,
                                                              const int* __restrict__ loc_of, const int* __restrict__ boff,
                                                              const long long* __restrict__ olinvr,
                                                              const int* __restrict__ ldl, const double* __restrict__ L,
                                                              const double* __restrict__ b, double* __restrict__ c) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; w < n; w += warps) {
        const int r = static_cast<int>(w);
        const int j = blk_of[r], lr = loc_of[r];
        const double* row = L + olinvr[j] + (long long)lr * ldl[j];
        const double* b0 = b + boff[j];
        const double* b1 = b0 + n;
        double s0 = 0.0, s1 = 0.0;
#pragma unroll 4
        for (int col = lane; col <= lr; col += 32) {
            const double l = __ldcs(row + col);
            s0 += l * b0[col];
            if (nrhs > 1) s1 += l * b1[col];
        }
        for (int o = 16; o; o >>= 1) {
            s0 += __shfl_xor_sync(0xffffffffu, s0, o);
            s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        }
        if (lane == 0) {
            c[r] = s0;
            if (nrhs > 1) c[n + r] = s1;
        }
    }
}

// e_j = Linv_j^T y_j on the col-major copy: one warp per output (a column of Linv_j).
__global__ void __launch_bounds__(256) k_blockdiag_upper(int n, int nrhs, const int* __restrict__ blk_of,
                                                         const int* __restrict__ loc_of, const int* __restrict__ bsz,
                                                         const int* __restrict__ boff, const long long* __restrict__ olinv,
                                                         const double* __restrict__ L, const double* __restrict__ y,
                                                         double* __restrict__ e) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; w < n; w += warps) {
        const int r = static_cast<int>(w);
        const int j = blk_of[r], lc = loc_of[r], m = bsz[j];
        const double* col = L + olinv[j] + (long long)lc * m;
        const double* y0 = y + boff[j];
        const double* y1 = y0 + n;
        double s0 = 0.0, s1 = 0.0;
#pragma unroll 4
        for (int row = lc + lane; row < m; row += 32) {
            const double l = __ldcs(col + row);
            s0 += l * y0[row];
            if (nrhs > 1) s1 += l * y1[row];
        }
        for (int o = 16; o; o >>= 1) {
            s0 += __shfl_xor_sync(0xffffffffu, s0, o);
            s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        }
        if (lane == 0) {
            e[r] = s0;
            if (nrhs > 1) e[n + r] = s1;
        }
    }
}

using namespace dev;

// Poll-and-gather the nrhs right-hand sides of one source block into shared
// memory: every line load of the thread is issued before any flag is checked.
__device__ __forceinline__ void ll_gather(const uint4* ll, int n, int nrhs, int off, int m, unsigned flag, double* ysh,
                                          int max_b) {
    constexpr int PER = 5;  // rows per thread per right-hand side kept in flight (256 threads: m <= 1280)
    const uint4* src0 = ll + off;
    const uint4* src1 = ll + (long long)n + off;
    uint4 v0[PER], v1[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int r = threadIdx.x + q * 256;
        if (r < m) {
            v0[q] = ll_peek(src0 + r);
            if (nrhs > 1) v1[q] = ll_peek(src1 + r);
        }
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int r = threadIdx.x + q * 256;
        if (r < m) {
            while (v0[q].y != flag || v0[q].w != flag) v0[q] = ll_peek(src0 + r);
            ysh[r] = ll_value(v0[q]);
            if (nrhs > 1) {
                while (v1[q].y != flag || v1[q].w != flag) v1[q] = ll_peek(src1 + r);
                ysh[max_b + r] = ll_value(v1[q]);
            }
        }
    }
    for (int r = threadIdx.x + PER * 256; r < m; r += 256)
        for (int k = 0; k < nrhs; ++k) {
            const uint4* p = (k ? src1 : src0) + r;
            uint4 x = ll_peek(p);
            while (x.y != flag || x.w != flag) x = ll_peek(p);
            ysh[k * max_b + r] = ll_value(x);
        }
}

// The recurrence of one substitution (forward or backward): nsteps steps, two
// concurrent chains (CTAs [0,g0) run chain 0, the rest chain 1), rpc rows per
// CTA (rpc/8 per warp). Task rows whose matrix is streamed (single-source
// tasks) arrive in a shared-memory ring filled by cp.async.bulk ahead of time;
// the twist task (two sources) reads its two matrices from global memory.
// Row values are exchanged as LL lines flagged with the call number.
__global__ void __launch_bounds__(288, 1) k_recurrence(int nsteps, int nb, const RecTask* __restrict__ sched_g, int nrhs,
                                                      int n, const int* __restrict__ bsz_g, const int* __restrict__ boff_g,
                                                      const double* __restrict__ store, const double* __restrict__ rhs,
                                                      double* __restrict__ out, uint4* ll, unsigned flag, int stages,
                                                      int rpc, int maxld, int max_b, int g0,
                                                      unsigned long long* dbg) {
    // dbg (debug only, normally null): per CTA and step, %globaltimer at step
    // start, after the source gather, after the row stores (4 slots per step).
    auto stamp = [&](int s, int ph) {
        if (dbg && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            dbg[((size_t)blockIdx.x * nsteps + s) * 4 + ph] = t;
        }
    };
    // The ring holds `stages` units of 8 rows; step s uses units s*upr .. s*upr+upr-1
    // (upr = rpc/8), unit u lives in slot u % stages with its own mbarrier, so
    // up to stages - upr units of the following steps are in flight.
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* ring = reinterpret_cast<double*>(smem_raw);
    double* ysh = ring + (size_t)stages * 8 * maxld;  // [2 sources][2 rhs][max_b]
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(ysh + 4 * max_b);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int chain = static_cast<int>(blockIdx.x) < g0 ? 0 : 1;
    // this chain's schedule and the block metadata live in shared memory: every
    // per-step lookup is on the critical path and a global load costs ~1 us
    RecTask* tsh = reinterpret_cast<RecTask*>(mbar + 2 * stages);
    int* bsz = reinterpret_cast<int*>(tsh + nsteps);
    int* boff = bsz + nb;
    for (int i = threadIdx.x; i < nsteps; i += blockDim.x) tsh[i] = sched_g[2 * i + chain];
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        bsz[i] = bsz_g[i];
        boff[i] = boff_g[i];
    }
    __syncthreads();
    const int row0 = (chain ? blockIdx.x - g0 : blockIdx.x) * rpc;
    const int rpw = rpc >> 3, upr = rpc >> 3;
    const int nunits = nsteps * upr;
    // warps 0-7 consume (gather, dot products, publish); warp 8 produces: it
    // streams ring units with cp.async.bulk as soon as the consumers release
    // a slot (full/empty mbarrier pair per slot), off the critical path.
    unsigned long long* full = mbar;
    unsigned long long* empty = mbar + stages;
    auto streamed = [&](const RecTask& t) { return t.tgt >= 0 && t.src1 >= 0 && t.src2 < 0; };
    auto consumers_sync = [] { asm volatile("bar.sync 1, 256;" ::: "memory"); };
    if (threadIdx.x == 0) {
        for (int k = 0; k < stages; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 8) {  // ---- producer
        if (lane == 0)
            for (int u = 0; u < nunits; ++u) {
                const int k = u % stages, use = u / stages;
                if (use > 0) mbar_wait(&empty[k], static_cast<unsigned>((use - 1) & 1));
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                const int s = u / upr, part = u % upr;
                const RecTask t = tsh[s];
                const int r0 = row0 + 8 * part;
                int nrows = 0;
                if (streamed(t)) {
                    nrows = bsz[t.tgt] - r0;
                    nrows = nrows < 0 ? 0 : (nrows > 8 ? 8 : nrows);
                }
                mbar_arrive_expect_tx(&full[k], static_cast<unsigned>(nrows * t.ld1 * 8));
                for (int r = 0; r < nrows; ++r)
                    bulk_g2s(ring + ((size_t)k * 8 + r) * maxld, store + t.off1 + (long long)(r0 + r) * t.ld1,
                             static_cast<unsigned>(t.ld1 * 8), &full[k]);
            }
        return;
    }
    for (int s = 0; s < nsteps; ++s) {  // ---- consumers
        const RecTask t = tsh[s];
        stamp(s, 0);
        if (t.tgt >= 0) {
            const int mj = bsz[t.tgt], oj = boff[t.tgt];
            if (t.src1 < 0 && t.src2 < 0) {  // copy task
                if (threadIdx.x < rpc * nrhs) {
                    const int r = row0 + threadIdx.x % rpc, k = threadIdx.x / rpc;
                    if (r < mj) {
                        const long long idx = (long long)k * n + oj + r;
                        const double v = rhs[idx];
                        out[idx] = v;
                        ll_store(&ll[idx], v, flag);
                    }
                }
            } else {
                // this lane's right-hand-side values for its rows, loaded before the
                // (long) wait for the source blocks so they are off the critical path
                double rv[2] = {0.0, 0.0};
                if (lane < nrhs)
                    for (int q = 0; q < rpw && q < 2; ++q) {
                        const int r = row0 + warp * rpw + q;
                        if (r < mj) rv[q] = rhs[(long long)lane * n + oj + r];
                    }
                int m1 = 0, m2 = 0;
                if (t.src1 >= 0) {
                    m1 = bsz[t.src1];
                    ll_gather(ll, n, nrhs, boff[t.src1], m1, flag, ysh, max_b);
                }
                if (t.src2 >= 0) {
                    m2 = bsz[t.src2];
                    ll_gather(ll, n, nrhs, boff[t.src2], m2, flag, ysh + 2 * max_b, max_b);
                }
                consumers_sync();
                stamp(s, 1);
                const bool st_ = t.src2 < 0;
                // two streamed rows per warp: one pass over the columns, y read once
                // from shared memory for both rows (the pass is smem-bandwidth bound)
                const int lr0 = warp * rpw;
                if (st_ && rpw == 2 && row0 + lr0 + 1 < mj) {
                    const int u = s * upr + (lr0 >> 3), k = u % stages;
                    mbar_wait(&full[k], static_cast<unsigned>((u / stages) & 1));
                    const double* ra = ring + ((size_t)k * 8 + (lr0 & 7)) * maxld;
                    const double* rb = ra + maxld;
                    double a0[2] = {0.0, 0.0}, a1[2] = {0.0, 0.0}, b0[2] = {0.0, 0.0}, b1[2] = {0.0, 0.0};
                    int c = lane;
                    for (; c + 32 < m1; c += 64) {
#pragma unroll
                        for (int p = 0; p < 2; ++p) {
                            const double y0 = ysh[c + 32 * p], y1 = ysh[max_b + c + 32 * p];
                            const double va = ra[c + 32 * p], vb = rb[c + 32 * p];
                            a0[p] += va * y0;
                            a1[p] += va * y1;
                            b0[p] += vb * y0;
                            b1[p] += vb * y1;
                        }
                    }
                    for (; c < m1; c += 32) {
                        const double y0 = ysh[c], y1 = ysh[max_b + c];
                        a0[0] += ra[c] * y0;
                        a1[0] += ra[c] * y1;
                        b0[0] += rb[c] * y0;
                        b1[0] += rb[c] * y1;
                    }
                    double acc[4] = {a0[0] + a0[1], a1[0] + a1[1], b0[0] + b0[1], b1[0] + b1[1]};
#pragma unroll
                    for (int o = 16; o; o >>= 1)
#pragma unroll
                        for (int i = 0; i < 4; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
                    // prefetched rhs of (row q, rhs kk) sits in lane kk's rv[q]
                    const double r0v = __shfl_sync(0xffffffffu, rv[0], lane & 1);
                    const double r1v = __shfl_sync(0xffffffffu, rv[1], lane & 1);
                    if (lane < 4) {  // lane = 2 * row + rhs
                        const int q = lane >> 1, kk = lane & 1;
                        if (kk < nrhs) {
                            const long long idx = (long long)kk * n + oj + row0 + lr0 + q;
                            const double sub = q == 0 ? (kk == 0 ? acc[0] : acc[1]) : (kk == 0 ? acc[2] : acc[3]);
                            const double v = (q == 0 ? r0v : r1v) - sub;
                            ll_store(&ll[idx], v, flag);
                            out[idx] = v;
                        }
                    }
                } else
                for (int q = 0; q < rpw; ++q) {
                    const int lr = warp * rpw + q;
                    const int r = row0 + lr;
                    if (r >= mj) break;
                    const int u = s * upr + (lr >> 3), k = u % stages;
                    if (st_) mbar_wait(&full[k], static_cast<unsigned>((u / stages) & 1));
                    // four independent partial sums per right-hand side (breaks the
                    // dependent DFMA chain; fixed order, so still deterministic)
                    double a0[4] = {0.0, 0.0, 0.0, 0.0}, a1[4] = {0.0, 0.0, 0.0, 0.0};
                    const double* row1 =
                        st_ ? ring + ((size_t)k * 8 + (lr & 7)) * maxld : store + t.off1 + (long long)r * t.ld1;
                    if (t.src1 >= 0) {
                        int c = lane;
                        for (; c + 96 < m1; c += 128) {
#pragma unroll
                            for (int p = 0; p < 4; ++p) {
                                const double v = row1[c + 32 * p];
                                a0[p] += v * ysh[c + 32 * p];
                                if (nrhs > 1) a1[p] += v * ysh[max_b + c + 32 * p];
                            }
                        }
                        for (; c < m1; c += 32) {
                            const double v = row1[c];
                            a0[0] += v * ysh[c];
                            if (nrhs > 1) a1[0] += v * ysh[max_b + c];
                        }
                    }
                    if (t.src2 >= 0) {
                        const double* row2 = store + t.off2 + (long long)r * t.ld2;
                        for (int c = lane; c < m2; c += 32) {
                            const double v = __ldcs(row2 + c);
                            a0[1] += v * ysh[2 * max_b + c];
                            if (nrhs > 1) a1[1] += v * ysh[3 * max_b + c];
                        }
                    }
                    double acc0 = (a0[0] + a0[1]) + (a0[2] + a0[3]);
                    double acc1 = (a1[0] + a1[1]) + (a1[2] + a1[3]);
                    for (int o = 16; o; o >>= 1) {
                        acc0 += __shfl_xor_sync(0xffffffffu, acc0, o);
                        acc1 += __shfl_xor_sync(0xffffffffu, acc1, o);
                    }
                    if (lane < nrhs) {
                        const long long idx = (long long)lane * n + oj + r;
                        const double v = (q < 2 ? rv[q] : rhs[idx]) - (lane == 0 ? acc0 : acc1);
                        ll_store(&ll[idx], v, flag);
                        out[idx] = v;
                    }
                }
            }
        }
        // release this step's ring units (every consumer warp arrives once per
        // unit). Each unit's full phase is awaited first -- also for units that
        // carried no rows -- so consumers can never run a phase ahead of the
        // producer on a slot (an mbarrier parity wait cannot tell phase p from p+2).
        __syncwarp();
        for (int p = 0; p < upr; ++p) {
            const int u = s * upr + p;
            mbar_wait(&full[u % stages], static_cast<unsigned>((u / stages) & 1));
        }
        if (lane == 0)
            for (int p = 0; p < upr; ++p) {
                unsigned long long* e = &empty[(s * upr + p) % stages];
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(e)) : "memory");
            }
        consumers_sync();  // ysh free for reuse
        stamp(s, 2);
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
    DBuf<long long> ddD, ddC;
    ddD.upload(dD_, st);
    ddC.upload(dC_, st);
    DBuf<int> err(1);
    err.zero(st);
    k_scatter_blocks<<<grid_for(n, 256), 256, 0, st>>>(n, off, idx, val, perm.n ? inv_perm.p : nullptr, blk_of.p,
                                                        loc_of.p, d_bsz.p, ddD.p, ddC.p, dense.p, err.p);
    PDG_CHECK_LAUNCH();
    int herr = 0;
    PDG_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    require(herr == 0, "block-tridiagonal solver: matrix is not block tridiagonal in the given ordering");
    factor_dense(dense.p, st);
}

void BlockTriChol::factor_dense(double* dense, cudaStream_t st) {
    local_prepare(dense, st);  // before the couplings are overwritten by the factorisation
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
    if (local) {
        local_finish(dense, st);
        return;
    }
    // ---- solve-time storage ---------------------------------------------------
    auto pad = [](int m) { return (m + 1) & ~1; };                    // 16-byte rows (cp.async.bulk)
    auto al = [](long long v) { return (v + 31) & ~31LL; };           // 256-byte aligned matrices
    o_linv.assign(nb, 0);
    o_linvr.assign(nb, 0);
    ld_l.assign(nb, 0);
    std::vector<long long> oF(nb, -1), oG(nb, -1), oN(nb, -1);
    std::vector<int> ldF(nb, 0), ldG(nb, 0), ldN(nb, 0);
    long long o = 0;
    factor_bytes = 0.0;
    for (int j = 0; j < nb; ++j) {
        const int mj = bsz[j];
        o_linv[j] = o;
        o = al(o + (long long)mj * mj);
        ld_l[j] = pad(mj);
        o_linvr[j] = o;
        o = al(o + (long long)mj * ld_l[j]);
        factor_bytes += 8.0 * mj * (mj + 1);  // lower triangle, read by both passes
        if (j >= 1 && j <= t) {
            ldF[j] = pad(bsz[j - 1]);
            oF[j] = o;
            o = al(o + (long long)mj * ldF[j]);
            factor_bytes += 8.0 * mj * bsz[j - 1];
        }
        if (j >= t && j + 1 < nb) {
            ldG[j] = pad(bsz[j + 1]);
            oG[j] = o;
            o = al(o + (long long)mj * ldG[j]);
            factor_bytes += 8.0 * mj * bsz[j + 1];
        }
        if (j != t) {
            const int src = j < t ? j + 1 : j - 1;
            ldN[j] = pad(bsz[src]);
            oN[j] = o;
            o = al(o + (long long)mj * ldN[j]);
            factor_bytes += 8.0 * mj * bsz[src];
        }
    }
    store.alloc(o);
    store.zero(st);
    for (int j = 0; j < nb; ++j) {
        const int mj = bsz[j];
        double* Lj = store.p + o_linv[j];
        k_identity<<<grid_for((long long)mj * mj, 256), 256, 0, st>>>(mj, Lj);
        PDG_CHECK_LAUNCH();
        PDG_CUBLAS(cublasDtrsm(h.blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, mj, mj,
                               &one, D(j), mj, Lj, mj));
        PDG_CUBLAS(cublasDgeam(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, mj, mj, &one, Lj, mj, &zero, Lj, mj,
                               store.p + o_linvr[j], ld_l[j]));
        if (oF[j] >= 0)  // F_j row-major = (K_{j-1}^T Linv_j^T) col-major, K_{j-1}: m_j x m_{j-1}
            PDG_CUBLAS(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_T, bsz[j - 1], mj, mj, &one, C(j - 1), mj, Lj, mj, &zero,
                                   store.p + oF[j], ldF[j]));
        if (oG[j] >= 0)  // G_j row-major = (K'_{j+1}^T Linv_j^T) col-major, K'_{j+1}: m_j x m_{j+1}
            PDG_CUBLAS(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_T, bsz[j + 1], mj, mj, &one, kp.p + oKp[j + 1], mj, Lj, mj,
                                   &zero, store.p + oG[j], ldG[j]));
        if (oN[j] >= 0 && j < t)  // N_j row-major = (K_j Linv_j) col-major, K_j: m_{j+1} x m_j
            PDG_CUBLAS(cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, bsz[j + 1], mj, mj, &one, C(j), bsz[j + 1], Lj, mj,
                                   &zero, store.p + oN[j], ldN[j]));
        if (oN[j] >= 0 && j > t)  // N'_j row-major = (K'_j Linv_j) col-major, K'_j: m_{j-1} x m_j
            PDG_CUBLAS(cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, bsz[j - 1], mj, mj, &one, kp.p + oKp[j], bsz[j - 1],
                                   Lj, mj, &zero, store.p + oN[j], ldN[j]));
    }
    d_olinv.upload(o_linv, st);
    d_olinvr.upload(o_linvr, st);
    d_ldl.upload(ld_l, st);
    // ---- schedules ------------------------------------------------------------------
    const RecTask idle{-1, -1, -1, 0, 0, 0, 0};
    auto copy_task = [&](int j) { return RecTask{j, -1, -1, 0, 0, 0, 0}; };
    fwd.clear();
    bwd.clear();
    {  // forward: chains start at 0 and nb-1, meet at the twist
        fwd.push_back(t >= 1 ? copy_task(0) : idle);
        fwd.push_back(nb - 1 > t ? copy_task(nb - 1) : idle);
        const int L = std::max({t - 1, nb - 2 - t, 0});
        for (int s = 1; s <= L; ++s) {
            const int jt = s, jb = nb - 1 - s;
            fwd.push_back(jt <= t - 1 ? RecTask{jt, jt - 1, -1, ldF[jt], 0, oF[jt], 0} : idle);
            fwd.push_back(jb >= t + 1 ? RecTask{jb, jb + 1, -1, ldG[jb], 0, oG[jb], 0} : idle);
        }
        RecTask tw{t, -1, -1, 0, 0, 0, 0};
        if (t >= 1) {
            tw.src1 = t - 1;
            tw.ld1 = ldF[t];
            tw.off1 = oF[t];
        }
        if (t + 1 < nb) {
            if (tw.src1 < 0) {
                tw.src1 = t + 1;
                tw.ld1 = ldG[t];
                tw.off1 = oG[t];
            } else {
                tw.src2 = t + 1;
                tw.ld2 = ldG[t];
                tw.off2 = oG[t];
            }
        }
        fwd.push_back(tw);
        fwd.push_back(idle);
    }
    {  // backward: from the twist outwards
        bwd.push_back(copy_task(t));
        bwd.push_back(idle);
        const int L = std::max(t, nb - 1 - t);
        for (int s = 1; s <= L; ++s) {
            const int jt = t - s, jb = t + s;
            bwd.push_back(jt >= 0 ? RecTask{jt, jt + 1, -1, ldN[jt], 0, oN[jt], 0} : idle);
            bwd.push_back(jb <= nb - 1 ? RecTask{jb, jb - 1, -1, ldN[jb], 0, oN[jb], 0} : idle);
        }
    }
    d_fwd.upload(fwd, st);
    d_bwd.upload(bwd, st);
    // ---- recurrence kernel configuration -------------------------------------------
    int dev = 0;
    PDG_CUDA(cudaGetDevice(&dev));
    int optin = 0;
    PDG_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    PDG_CUDA(cudaFuncSetAttribute(k_recurrence, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    maxld = pad(max_b);
    int top_rows = 0, bot_rows = 0;
    for (int j = 0; j <= t; ++j) top_rows = std::max(top_rows, bsz[j]);
    for (int j = t + 1; j < nb; ++j) bot_rows = std::max(bot_rows, bsz[j]);
    const size_t meta = sizeof(RecTask) * std::max(fwd.size(), bwd.size()) / 2 + sizeof(int) * 2 * nb + 64;
    const size_t fixed = sizeof(double) * 4 * max_b + 8 * 2 * 32 + meta;  // ysh + full/empty mbarriers + metadata
    const size_t unit = sizeof(double) * 8 * maxld;  // one ring unit = 8 rows
    bool ok = false;
    for (rpc = 8; rpc <= 64; rpc += 8) {
        g0 = (top_rows + rpc - 1) / rpc;
        g1 = (bot_rows + rpc - 1) / rpc;
        if (fixed + unit * (rpc / 8) > (size_t)optin - 1024) continue;
        stages = static_cast<int>(std::min<size_t>(((size_t)optin - 1024 - fixed) / unit, 32));
        if (g0 + g1 <= num_sms()) {
            ok = true;
            break;
        }
    }
    require(ok, "block-tridiagonal solver: blocks too large for the recurrence kernel");
    smem = unit * stages + fixed;
    int occ = 0;
    PDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_recurrence, 288, smem));
    require(occ >= 1, "block-tridiagonal solver: recurrence kernel cannot be resident");
    ll.alloc((size_t)n * max_rhs);
    ll.zero(st);
    wb.alloc((size_t)n * max_rhs);
    wc.alloc((size_t)n * max_rhs);
    wy.alloc((size_t)n * max_rhs);
    we.alloc((size_t)n * max_rhs);
    wx.alloc((size_t)n * max_rhs);
    PDG_CUDA(cudaStreamSynchronize(st));
}

void BlockTriChol::recurrence(const DBuf<RecTask>& sched, int nsteps, const double* in, double* out, int nrhs,
                              cudaStream_t st) {
    unsigned flag = static_cast<unsigned>(++call);
    if (flag == 0) flag = static_cast<unsigned>(++call);  // 0 = never published
    int ns = nsteps, nr = nrhs, n_ = n, stg = stages, rp = rpc, mld = maxld, mb = max_b, gg0 = g0;
    const RecTask* a1 = sched.p;
    const int* a2 = d_bsz.p;
    const int* a3 = d_boff.p;
    const double* a4 = store.p;
    const double* a5 = in;
    double* a6 = out;
    uint4* a7 = ll.p;
    unsigned long long* dbgp = nullptr;
    dbg_steps = nsteps;
    if (debug_timing) {
        dbg.alloc((size_t)(g0 + g1) * nsteps * 4);
        dbg.zero(st);
        dbgp = dbg.p;
    }
    int nb_ = nb;
    void* args[] = {&ns, &nb_, &a1, &nr, &n_, &a2, &a3, &a4, &a5, &a6, &a7, &flag, &stg, &rp, &mld, &mb, &gg0, &dbgp};
    PDG_CUDA(cudaLaunchCooperativeKernel((void*)k_recurrence, g0 + g1, 288, args, smem, st));
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
    k_blockdiag_lower_rows<<<grid_for((long long)n * 32, 256), 256, 0, st>>>(n, nrhs, blk_of.p, loc_of.p, d_boff.p,
                                                                              d_olinvr.p, d_ldl.p, store.p, wb.p, wc.p);
    recurrence(d_fwd, static_cast<int>(fwd.size() / 2), wc.p, wy.p, nrhs, st);
    k_blockdiag_upper<<<grid_for((long long)n * 32, 256), 256, 0, st>>>(n, nrhs, blk_of.p, loc_of.p, d_bsz.p, d_boff.p,
                                                                         d_olinv.p, store.p, wy.p, we.p);
    recurrence(d_bwd, static_cast<int>(bwd.size() / 2), we.p, wx.p, nrhs, st);
    k_scatter<<<grid_for(tot, 256), 256, 0, st>>>(n, nrhs, pp, wx.p, x, ldx);
    count_launch(6);
    PDG_CHECK_LAUNCH();
}

}  // namespace pdg
