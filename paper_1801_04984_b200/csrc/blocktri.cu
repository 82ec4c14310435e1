// Block-tridiagonal Cholesky: factorisation with cuSOLVER/cuBLAS (setup
// only), solve with hand-written kernels (two bandwidth-bound block-diagonal
// GEMV passes and two persistent cooperative recurrences).
#include <cooperative_groups.h>

#include <algorithm>

#include "blocktri.cuh"

namespace pdg {

#define PDG_CUBLAS(call)                                                                        \
    do {                                                                                        \
        cublasStatus_t s_ = (call);                                                             \
        if (s_ != CUBLAS_STATUS_SUCCESS)                                                        \
            throw ::pdg::Error(PDG_CUDA_ERROR, std::string(#call) + ": cublas status " + std::to_string((int)s_)); \
    } while (0)
#define PDG_CUSOLVER(call)                                                                      \
    do {                                                                                        \
        cusolverStatus_t s_ = (call);                                                           \
        if (s_ != CUSOLVER_STATUS_SUCCESS)                                                      \
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
                                 const long long* dC, double* D, double* C, int* err) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const int nr = inv_perm ? inv_perm[r] : r;
        const int jr = blk_of[nr], lr = loc_of[nr];
        for (int k = off[r]; k < off[r + 1]; ++k) {
            const int nc = inv_perm ? inv_perm[idx[k]] : idx[k];
            const int jc = blk_of[nc], lc = loc_of[nc];
            if (jc == jr)
                D[dD[jr] + lr + (long long)lc * bsz[jr]] = val[k];
            else if (jr == jc + 1)
                C[dC[jc] + lr + (long long)lc * bsz[jr]] = val[k];
            else if (jc != jr + 1)
                atomicOr(err, 1);
        }
    }
}

__global__ void k_identity(int m, double* a) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * m; t += (long long)gridDim.x * blockDim.x)
        a[t] = (t % m == t / m) ? 1.0 : 0.0;
}

// ---- solve kernels -------------------------------------------------------------
__global__ void k_gather(int n, int nrhs, const int* perm, const double* b, long long ldb, double* out) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)n * nrhs; t += (long long)gridDim.x * blockDim.x) {
        const int r = static_cast<int>(t % n), k = static_cast<int>(t / n);
        out[t] = b[(perm ? perm[r] : r) + k * ldb];
    }
}
__global__ void k_scatter(int n, int nrhs, const int* perm, const double* in, double* x, long long ldx) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)n * nrhs; t += (long long)gridDim.x * blockDim.x) {
        const int r = static_cast<int>(t % n), k = static_cast<int>(t / n);
        x[(perm ? perm[r] : r) + k * ldx] = in[t];
    }
}

// c_j = Linv_j b_j : one thread per row (all right-hand sides, so L is read
// once); Linv col-major lower, row r uses cols 0..r; loads unrolled x8.
__global__ void __launch_bounds__(256) k_blockdiag_lower(int n, int nrhs, const int* __restrict__ blk_of,
                                                         const int* __restrict__ loc_of, const int* __restrict__ bsz,
                                                         const int* __restrict__ boff, const long long* __restrict__ olinv,
                                                         const double* __restrict__ L, const double* __restrict__ b,
                                                         double* __restrict__ c) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const int j = blk_of[r], lr = loc_of[r], m = bsz[j];
        const double* Lr = L + olinv[j] + lr;
        const double* b0 = b + boff[j];
        const double* b1 = b0 + n;
        double s0 = 0.0, s1 = 0.0;
        if (nrhs > 1) {
#pragma unroll 8
            for (int col = 0; col <= lr; ++col) {
                const double l = __ldcs(Lr + (long long)col * m);
                s0 += l * b0[col];
                s1 += l * b1[col];
            }
            c[n + r] = s1;
        } else {
#pragma unroll 8
            for (int col = 0; col <= lr; ++col) s0 += __ldcs(Lr + (long long)col * m) * b0[col];
        }
        c[r] = s0;
    }
}

// e_j = Linv_j^T y_j : one warp per output (all right-hand sides); column lc
// of Linv_j, rows lc..m-1 contiguous.
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

__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned int* gen = bar + 1;
        const unsigned int g = *gen;
        __threadfence();
        const unsigned int arrived = atomicAdd(bar, 1u);
        if (arrived == nblocks - 1) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) __nanosleep(16);
        }
        __threadfence();
    }
    __syncthreads();
}

// Forward (dir = +1): y_0 = c_0, y_j = c_j - M_j y_{j-1} (M_j: bsz_j x bsz_{j-1} row-major).
// Backward (dir = -1): x_{nb-1} = e_{nb-1}, x_j = e_j - N_j x_{j+1} (N_j: bsz_j x bsz_{j+1}).
// One warp per matrix row. The row a warp needs at step s+1 does not depend on
// the recurrence, so it is loaded into registers (R doubles per lane) before
// the grid barrier of step s+1: HBM latency overlaps the barrier.
template <int R>
__global__ void __launch_bounds__(256) k_recurrence(int nb, int nrhs, int n, int dir, const int* __restrict__ bsz,
                                                    const int* __restrict__ boff, const long long* __restrict__ omat,
                                                    const int* __restrict__ ldm, const double* __restrict__ store,
                                                    const double* __restrict__ rhs, double* __restrict__ out,
                                                    unsigned int* bar) {
    extern __shared__ double sh[];  // previous block's solution, nrhs * max_b
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const int gwarp = blockIdx.x * wpb + warp;
    const int nwarps = gridDim.x * wpb;
    {
        const int j0 = dir > 0 ? 0 : nb - 1;
        const int m0 = bsz[j0], o0 = boff[j0];
        for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < m0 * nrhs; t += gridDim.x * blockDim.x) {
            const int r = t % m0, k = t / m0;
            out[(long long)k * n + o0 + r] = rhs[(long long)k * n + o0 + r];
        }
    }
    double v[R];
    auto prefetch = [&](int s) {
        const int j = dir > 0 ? s : nb - 1 - s;
        const int jp = dir > 0 ? j - 1 : j + 1;
        const int mj = bsz[j], mp = bsz[jp];
        if (gwarp < mj) {
            const double* row = store + omat[j] + (long long)gwarp * ldm[j];
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const int c = lane + 32 * k;
                v[k] = c < mp ? __ldcs(row + c) : 0.0;
            }
        }
    };
    if (nb > 1) prefetch(1);
    for (int s = 1; s < nb; ++s) {
        const int j = dir > 0 ? s : nb - 1 - s;
        const int jp = dir > 0 ? j - 1 : j + 1;
        const int mj = bsz[j], mp = bsz[jp], oj = boff[j], op = boff[jp];
        grid_barrier(bar, gridDim.x);
        for (int t = threadIdx.x; t < mp * nrhs; t += blockDim.x) {
            const int r = t % mp, k = t / mp;
            sh[k * mp + r] = __ldcg(&out[(long long)k * n + op + r]);
        }
        __syncthreads();
        if (gwarp < mj) {
            double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const int c = lane + 32 * k;
                if (c < mp) {
                    acc0 += v[k] * sh[c];
                    if (nrhs > 1) acc1 += v[k] * sh[mp + c];
                }
            }
            for (int o = 16; o; o >>= 1) {
                acc0 += __shfl_xor_sync(0xffffffffu, acc0, o);
                acc1 += __shfl_xor_sync(0xffffffffu, acc1, o);
            }
            if (lane == 0) {
                out[oj + gwarp] = rhs[oj + gwarp] - acc0;
                if (nrhs > 1) out[(long long)n + oj + gwarp] = rhs[(long long)n + oj + gwarp] - acc1;
            }
        }
        // rows beyond one per warp (only when the grid has fewer warps than rows)
        const double* Mj = store + omat[j];
        for (int w = gwarp + nwarps; w < mj; w += nwarps) {
            const double* row = Mj + (long long)w * ldm[j];
            double acc0 = 0.0, acc1 = 0.0;
            for (int c = lane; c < mp; c += 32) {
                const double x = __ldcs(&row[c]);
                acc0 += x * sh[c];
                if (nrhs > 1) acc1 += x * sh[mp + c];
            }
            for (int o = 16; o; o >>= 1) {
                acc0 += __shfl_xor_sync(0xffffffffu, acc0, o);
                acc1 += __shfl_xor_sync(0xffffffffu, acc1, o);
            }
            if (lane == 0) {
                out[oj + w] = rhs[oj + w] - acc0;
                if (nrhs > 1) out[(long long)n + oj + w] = rhs[(long long)n + oj + w] - acc1;
            }
        }
        if (s + 1 < nb) prefetch(s + 1);
    }
}

// ---- TMA-pipelined recurrence ---------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1D bulk copy global -> shared (TMA engine), completion counted on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// LL line (the NCCL "LL" idea): a double travels as two 32-bit halves, each
// paired with a 32-bit flag in one 8-byte-atomic unit, 16 bytes per value.
// One volatile 16-byte store publishes value+flag; a reader polls the line
// and accepts it when both flags match -- no release/acquire fences.
__device__ __forceinline__ void ll_store(uint4* p, double v, unsigned flag) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(static_cast<unsigned>(b)), "r"(flag),
                 "r"(static_cast<unsigned>(b >> 32)), "r"(flag)
                 : "memory");
}
__device__ __forceinline__ uint4 ll_peek(const uint4* p) {
    uint4 v;
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
__device__ __forceinline__ double ll_load(const uint4* p, unsigned flag) {
    unsigned a, f0, c, f1;
    do {
        asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(a), "=r"(f0), "=r"(c), "=r"(f1)
                     : "l"(p)
                     : "memory");
    } while (f0 != flag || f1 != flag);
    return __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(c) << 32) | a));
}

// Same recurrence as k_recurrence, one CTA per 8 consecutive rows of every
// block (one warp per row), as a dataflow without grid barriers: the writer of
// row r publishes it as an LL line flagged with the call number; a consumer
// polls exactly the lines it reads. The rows of the matrices a CTA needs in
// the next `stages` steps do not depend on the recurrence, so thread 0
// streams them into a shared-memory ring with cp.async.bulk (TMA) + mbarriers
// ahead of time: the per-step critical path is one L2 round trip.
__global__ void __launch_bounds__(256, 1) k_recurrence_tma(int nb, int nrhs, int n, int dir, const int* __restrict__ bsz,
                                                          const int* __restrict__ boff, const long long* __restrict__ omat,
                                                          const int* __restrict__ ldm, const double* __restrict__ store,
                                                          const double* __restrict__ rhs, double* __restrict__ out,
                                                          uint4* ll, unsigned flag, int stages, int maxld, int max_b) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* buf = reinterpret_cast<double*>(smem_raw);
    double* ysh = buf + (size_t)stages * 8 * maxld;
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(ysh + 2 * max_b);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int row0 = blockIdx.x * 8;
    auto blk = [&](int s) { return dir > 0 ? s : nb - 1 - s; };
    auto issue = [&](int s) {  // thread 0
        const int k = (s - 1) % stages;
        const int j = blk(s), mj = bsz[j], ld = ldm[j];
        int nrows = mj - row0;
        nrows = nrows < 0 ? 0 : (nrows > 8 ? 8 : nrows);
        mbar_arrive_expect_tx(&mbar[k], static_cast<unsigned>(nrows * ld * 8));
        for (int r = 0; r < nrows; ++r)
            bulk_g2s(buf + ((size_t)k * 8 + r) * maxld, store + omat[j] + (long long)(row0 + r) * ld,
                     static_cast<unsigned>(ld * 8), &mbar[k]);
    };
    if (threadIdx.x == 0) {
        for (int k = 0; k < stages; ++k) mbar_init(&mbar[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int s = 1; s <= stages && s < nb; ++s) issue(s);
    {  // step 0: this CTA's rows of the first block are the right-hand side itself
        const int j0 = blk(0), m0 = bsz[j0], o0 = boff[j0];
        if (threadIdx.x < 8 * nrhs) {
            const int r = row0 + (threadIdx.x & 7), k = threadIdx.x >> 3;
            if (r < m0) {
                const double v = rhs[(long long)k * n + o0 + r];
                out[(long long)k * n + o0 + r] = v;
                ll_store(&ll[(long long)k * n + o0 + r], v, flag);
            }
        }
    }
    for (int s = 1; s < nb; ++s) {
        const int j = blk(s), jp = dir > 0 ? j - 1 : j + 1;
        const int mj = bsz[j], mp = bsz[jp], oj = boff[j], op = boff[jp];
        {
            // issue every line load of this thread first (independent, all in
            // flight together), then re-poll only the lines not yet published
            constexpr int PER = 9;
            const int total = mp * nrhs;
            uint4 v[PER];
#pragma unroll
            for (int q = 0; q < PER; ++q) {
                const int t = threadIdx.x + q * blockDim.x;
                if (t < total) v[q] = ll_peek(&ll[(long long)(t / mp) * n + op + (t % mp)]);
            }
#pragma unroll
            for (int q = 0; q < PER; ++q) {
                const int t = threadIdx.x + q * blockDim.x;
                if (t < total) {
                    const uint4* p = &ll[(long long)(t / mp) * n + op + (t % mp)];
                    while (v[q].y != flag || v[q].w != flag) v[q] = ll_peek(p);
                    ysh[(t / mp) * max_b + (t % mp)] = __longlong_as_double(
                        static_cast<long long>((static_cast<unsigned long long>(v[q].z) << 32) | v[q].x));
                }
            }
            for (int t = threadIdx.x + PER * blockDim.x; t < total; t += blockDim.x)
                ysh[(t / mp) * max_b + (t % mp)] = ll_load(&ll[(long long)(t / mp) * n + op + (t % mp)], flag);
        }
        __syncthreads();
        const int k = (s - 1) % stages;
        mbar_wait(&mbar[k], static_cast<unsigned>(((s - 1) / stages) & 1));
        const int r = row0 + warp;
        if (r < mj) {
            const double* row = buf + ((size_t)k * 8 + warp) * maxld;
            double acc0 = 0.0, acc1 = 0.0;
            for (int c = lane; c < mp; c += 32) {
                const double v = row[c];
                acc0 += v * ysh[c];
                if (nrhs > 1) acc1 += v * ysh[max_b + c];
            }
            for (int o = 16; o; o >>= 1) {
                acc0 += __shfl_xor_sync(0xffffffffu, acc0, o);
                acc1 += __shfl_xor_sync(0xffffffffu, acc1, o);
            }
            if (lane < nrhs) {
                const long long idx = (long long)lane * n + oj + r;
                const double v = rhs[idx] - (lane == 0 ? acc0 : acc1);
                ll_store(&ll[idx], v, flag);
                out[idx] = v;
            }
        }
        __syncthreads();  // stage buffer and ysh free for reuse
        if (threadIdx.x == 0 && s + stages < nb) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(s + stages);
        }
    }
}

// c_j = Linv_j b_j on the row-major copy of Linv: one warp per row (balanced
// across the triangle), all right-hand sides.
__global__ void __launch_bounds__(256) k_blockdiag_lower_rows(int n, int nrhs, const int* __restrict__ blk_of,
                                                              const int* __restrict__ loc_of, const int* __restrict__ boff,
                                                              const long long* __restrict__ olinvr, const int* __restrict__ ldl,
                                                              const double* __restrict__ L, const double* __restrict__ b,
                                                              double* __restrict__ c) {
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

using RecFn = void (*)(int, int, int, int, const int*, const int*, const long long*, const int*, const double*,
                       const double*, double*, unsigned int*);
RecFn pick_recurrence(int max_b) {
    const int r = (max_b + 31) / 32;
    if (r <= 4) return k_recurrence<4>;
    if (r <= 9) return k_recurrence<9>;
    if (r <= 17) return k_recurrence<17>;
    if (r <= 33) return k_recurrence<33>;
    return k_recurrence<64>;
}

}  // namespace

void BlockTriChol::layout(int n_, const std::vector<int>& perm_host, const std::vector<int>& block_sizes) {
    n = n_;
    bsz = block_sizes;
    nb = static_cast<int>(bsz.size());
    boff.assign(nb + 1, 0);
    for (int j = 0; j < nb; ++j) boff[j + 1] = boff[j] + bsz[j];
    require(boff[nb] == n, "block-tridiagonal solver: block sizes do not sum to n");
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
}

void BlockTriChol::factor(int n_, const int* off, const int* idx, const double* val, const std::vector<int>& perm_host,
                          const std::vector<int>& block_sizes, int max_rhs_, cudaStream_t st) {
    layout(n_, perm_host, block_sizes);
    max_rhs = max_rhs_;
    DBuf<double> dense(dtot_);
    dense.zero(st);
    DBuf<long long> ddD(nb), ddC(nb);
    ddD.upload(dD_, st);
    ddC.upload(dC_, st);
    DBuf<int> err(1);
    err.zero(st);
    k_scatter_blocks<<<grid_for(n, 256), 256, 0, st>>>(n, off, idx, val, perm.n ? inv_perm.p : nullptr, blk_of.p,
                                                        loc_of.p, d_bsz.p, ddD.p, ddC.p, dense.p, dense.p, err.p);
    PDG_CHECK_LAUNCH();
    int herr = 0;
    PDG_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    require(herr == 0, "block-tridiagonal solver: matrix is not block tridiagonal in the given ordering");
    factor_dense(dense.p, dense.p, st);
}

void BlockTriChol::factor_dense(double* Dbase, double* Cbase, cudaStream_t st) {
    LaHandles h(st);
    int lwork = 0;
    PDG_CUSOLVER(cusolverDnDpotrf_bufferSize(h.solver, CUBLAS_FILL_MODE_LOWER, max_b, Dbase, max_b, &lwork));
    DBuf<double> work(std::max(lwork, 1));
    DBuf<int> info(nb);
    info.zero(st);
    const double one = 1.0, mone = -1.0, zero = 0.0;
    for (int j = 0; j < nb; ++j) {
        const int mj = bsz[j];
        double* Dj = Dbase + dD_[j];
        if (j > 0) {
            const int mp = bsz[j - 1];
            PDG_CUBLAS(cublasDsyrk(h.blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, mj, mp, &mone, Cbase + dC_[j - 1], mj, &one,
                                   Dj, mj));
        }
        PDG_CUSOLVER(cusolverDnDpotrf(h.solver, CUBLAS_FILL_MODE_LOWER, mj, Dj, mj, work.p, lwork, info.p + j));
        if (j + 1 < nb)
            PDG_CUBLAS(cublasDtrsm(h.blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT,
                                   bsz[j + 1], mj, &one, Dj, mj, Cbase + dC_[j], bsz[j + 1]));
    }
    std::vector<int> hinfo = info.download(st);
    for (int j = 0; j < nb; ++j)
        if (hinfo[j] != 0)
            throw Error(PDG_NOT_CONVERGED, "dense LU: matrix is singular to working precision (block " +
                                               std::to_string(j) + " not positive definite)");
    // solve-time storage
    // Row strides are padded to an even number of doubles so every row is a
    // 16-byte aligned, 16-byte multiple span (cp.async.bulk requirement).
    auto pad = [](int m) { return (m + 1) & ~1; };
    o_linv.assign(nb, 0);
    o_linvr.assign(nb, 0);
    o_m.assign(nb, -1);
    o_n.assign(nb, -1);
    ld_m.assign(nb, 0);
    ld_n.assign(nb, 0);
    ld_l.assign(nb, 0);
    long long o = 0;
    auto al = [](long long v) { return (v + 31) & ~31LL; };  // 256-byte aligned matrices
    for (int j = 0; j < nb; ++j) {
        o_linv[j] = o;
        o = al(o + (long long)bsz[j] * bsz[j]);
        ld_l[j] = pad(bsz[j]);
        o_linvr[j] = o;
        o = al(o + (long long)bsz[j] * ld_l[j]);
        if (j > 0) {
            ld_m[j] = pad(bsz[j - 1]);
            o_m[j] = o;
            o = al(o + (long long)bsz[j] * ld_m[j]);
        }
        if (j + 1 < nb) {
            ld_n[j] = pad(bsz[j + 1]);
            o_n[j] = o;
            o = al(o + (long long)bsz[j] * ld_n[j]);
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
                               &one, Dbase + dD_[j], mj, Lj, mj));
        // row-major Linv (col-major Linv^T) for the forward block-diagonal pass
        PDG_CUBLAS(cublasDgeam(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, mj, mj, &one, Lj, mj, &zero, Lj, mj,
                               store.p + o_linvr[j], ld_l[j]));
        if (j > 0) {  // M_j row-major = M_j^T col-major (m_{j-1} x m_j) = K_{j-1}^T Linv_j^T
            const int mp = bsz[j - 1];
            PDG_CUBLAS(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_T, mp, mj, mj, &one, Cbase + dC_[j - 1], mj, Lj, mj, &zero,
                                   store.p + o_m[j], ld_m[j]));
        }
        if (j + 1 < nb) {  // N_j row-major = N_j^T col-major (m_{j+1} x m_j) = K_j Linv_j
            const int mn = bsz[j + 1];
            PDG_CUBLAS(cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, mn, mj, mj, &one, Cbase + dC_[j], mn, Lj, mj, &zero,
                                   store.p + o_n[j], ld_n[j]));
        }
    }
    d_olinv.upload(o_linv, st);
    d_olinvr.upload(o_linvr, st);
    d_om.upload(o_m, st);
    d_on.upload(o_n, st);
    d_ldm.upload(ld_m, st);
    d_ldn.upload(ld_n, st);
    d_ldl.upload(ld_l, st);
    counter.alloc(2);
    ll.alloc((size_t)n * max_rhs);
    ll.zero(st);
    bar.alloc(2);
    bar.zero(st);
    wb.alloc((size_t)n * max_rhs);
    wc.alloc((size_t)n * max_rhs);
    wy.alloc((size_t)n * max_rhs);
    we.alloc((size_t)n * max_rhs);
    wx.alloc((size_t)n * max_rhs);
    int dev = 0, occ = 0;
    PDG_CUDA(cudaGetDevice(&dev));
    // TMA pipeline: one CTA per 8 rows, smem ring of `stages` x 8 rows
    maxld = (max_b + 1) & ~1;
    tma_blocks = (max_b + 7) / 8;
    {
        const size_t stage_bytes = sizeof(double) * 8 * maxld;
        const size_t fixed = sizeof(double) * 2 * max_b + 64 * 8;
        const size_t cap = 220 * 1024;
        tma_stages = cap > fixed ? static_cast<int>(std::min<size_t>((cap - fixed) / stage_bytes, 8)) : 0;
        tma_smem = stage_bytes * tma_stages + sizeof(double) * 2 * max_b + sizeof(unsigned long long) * tma_stages;
        if (tma_stages >= 2 && tma_blocks <= num_sms()) {
            // the attribute is per function (shared by every solver instance): set the device maximum
            int optin = 0;
            PDG_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
            PDG_CUDA(cudaFuncSetAttribute(k_recurrence_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
            int occ_t = 0;
            PDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_t, k_recurrence_tma, 256, tma_smem));
            use_tma = occ_t >= 1;
        }
    }
    const size_t shmem = sizeof(double) * max_b * max_rhs;
    rec_fn = (void*)pick_recurrence(max_b);
    if (shmem > 48 * 1024)
        PDG_CUDA(cudaFuncSetAttribute(rec_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem));
    PDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rec_fn, 256, shmem));
    require(occ >= 1, "block-tridiagonal solver: recurrence kernel cannot be resident");
    // one warp per row of the largest block (8 warps per CTA), capped by co-residency:
    // a smaller grid makes the per-step grid barrier cheaper.
    const int want = (max_b + 7) / 8;
    coop_blocks = std::max(1, std::min(want, num_sms() * occ));
    PDG_CUDA(cudaStreamSynchronize(st));
}

double BlockTriChol::alg_bytes(int nrhs) const {
    double e = 0.0;
    for (int j = 0; j < nb; ++j) {
        e += (double)bsz[j] * (bsz[j] + 1);  // Linv lower triangle, read twice
        if (j > 0) e += (double)bsz[j] * bsz[j - 1];
        if (j + 1 < nb) e += (double)bsz[j] * bsz[j + 1];
    }
    return 8.0 * e + 16.0 * n * nrhs;
}

void BlockTriChol::recurrence(int dir, const double* in, double* out, int nrhs, cudaStream_t st) {
    int nb_ = nb, nrhs_ = nrhs, n_ = n, dir_ = dir;
    const int* a1 = d_bsz.p;
    const int* a2 = d_boff.p;
    const long long* a3 = dir > 0 ? d_om.p : d_on.p;
    const int* a4 = dir > 0 ? d_ldm.p : d_ldn.p;
    const double* a5 = store.p;
    const double* a6 = in;
    double* a7 = out;
    if (use_tma) {
        uint4* a8 = ll.p;
        unsigned call = static_cast<unsigned>(++tag_call);
        if (call == 0) call = static_cast<unsigned>(++tag_call);  // 0 is the initial (never-published) flag
        int st_ = tma_stages, mld = maxld, mb = max_b;
        void* args[] = {&nb_, &nrhs_, &n_, &dir_, &a1, &a2, &a3, &a4, &a5, &a6, &a7, &a8, &call, &st_, &mld, &mb};
        PDG_CUDA(cudaLaunchCooperativeKernel((void*)k_recurrence_tma, tma_blocks, 256, args, tma_smem, st));
    } else {
        unsigned int* a8 = bar.p;
        void* args[] = {&nb_, &nrhs_, &n_, &dir_, &a1, &a2, &a3, &a4, &a5, &a6, &a7, &a8};
        PDG_CUDA(cudaLaunchCooperativeKernel(rec_fn, coop_blocks, 256, args, sizeof(double) * max_b * nrhs, st));
    }
}

void BlockTriChol::solve(const double* b, long long ldb, double* x, long long ldx, int nrhs, cudaStream_t st) {
    ProfScope prof(prof_phase, st, alg_bytes(nrhs));
    require(nrhs >= 1 && nrhs <= max_rhs && nrhs <= 2, "block-tridiagonal solve: bad nrhs");
    const int* pp = perm.n ? perm.p : nullptr;
    const long long tot = (long long)n * nrhs;
    k_gather<<<grid_for(tot, 256), 256, 0, st>>>(n, nrhs, pp, b, ldb, wb.p);
    k_blockdiag_lower_rows<<<grid_for((long long)n * 32, 256), 256, 0, st>>>(n, nrhs, blk_of.p, loc_of.p, d_boff.p,
                                                                              d_olinvr.p, d_ldl.p, store.p, wb.p, wc.p);
    recurrence(+1, wc.p, wy.p, nrhs, st);
    k_blockdiag_upper<<<grid_for((long long)n * 32, 256), 256, 0, st>>>(n, nrhs, blk_of.p, loc_of.p, d_bsz.p, d_boff.p,
                                                                         d_olinv.p, store.p, wy.p, we.p);
    recurrence(-1, we.p, wx.p, nrhs, st);
    k_scatter<<<grid_for(tot, 256), 256, 0, st>>>(n, nrhs, pp, wx.p, x, ldx);
    count_launch(6);
    PDG_CHECK_LAUNCH();
}

}  // namespace pdg
