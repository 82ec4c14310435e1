// Local-coupling mode of the twisted block-tridiagonal solver: inverse twisted
// Schur complements + chunk-local couplings, one persistent sweep kernel per
// solve (forward, twist and backward of both chains). Used for the
// displacement block A in cell-row order: the SIPG coupling between two cell
// rows only joins vertically adjacent cells, so C_j = A_{j+1,j} is block
// diagonal in 8x8 cell chunks (assembly.hpp:177-395, interior faces).
#include <algorithm>
#include <cstdlib>

#include "blocktri.cuh"
#include "llsync.cuh"

namespace pdg {

using namespace dev;

namespace {

// flag couplings outside the 8x8 diagonal chunks of every C_j (m x m, col-major)
__global__ void k_check_local(long long total, int m, const double* __restrict__ c, int* err) {
    const long long mm = (long long)m * m;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long e = t % mm;
        const int row = static_cast<int>(e % m), col = static_cast<int>(e / m);
        if ((row >> 3) != (col >> 3) && c[t] != 0.0) atomicOr(err, 1);
    }
}

// cloc[j][cell][r][q] = C_j(8 cell + r, 8 cell + q)
__global__ void k_extract_cloc(int nc, int m, const double* __restrict__ c, double* __restrict__ cloc) {
    const long long total = (long long)nc * m * 8;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int q = static_cast<int>(t & 7);
        const long long jr = t >> 3;
        const int r = static_cast<int>(jr % m);
        const long long j = jr / m;
        const int cell = r >> 3;
        cloc[((j * (m >> 3) + cell) * 8 + (r & 7)) * 8 + q] = c[j * m * m + r + (long long)(cell * 8 + q) * m];
    }
}

// full symmetric matrix (row-major, stride ld) from the lower triangle of a col-major m x m
__global__ void k_symm_store(int m, const double* __restrict__ lo, int ld, double* __restrict__ out) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * m;
         t += (long long)gridDim.x * blockDim.x) {
        const int r = static_cast<int>(t / m), c = static_cast<int>(t % m);
        out[(long long)r * ld + c] = r >= c ? lo[r + (long long)c * m] : lo[c + (long long)r * m];
    }
}

// This thread's input values: columns c0, c0+1, c0+512, c0+513 (pairs valid
// when c0 + 512 i < m) of every right-hand side, polled from LL lines at src
// (stride lln per right-hand side). Every round re-issues the loads of all
// lines still pending before checking any, so a round costs one L2 round trip
// however many lines are late. Returns (or adds into) y[k][i][e].
__device__ __forceinline__ void poll_pairs(const uint4* src, long long lln, int nrhs, int m, int c0, unsigned flag,
                                           double (&y)[2][2][2], bool accumulate) {
    unsigned pending = 0;
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int i = 0; i < 2; ++i)
            if (k < nrhs && c0 + 512 * i < m) pending |= 3u << (4 * k + 2 * i);
    uint4 v[8];
    // warp-uniform rounds (lanes stay converged: a lane spinning alone on a
    // divergent path would stall its whole warp)
    while (__any_sync(0xffffffffu, pending != 0)) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (pending & (1u << q)) v[q] = ll_peek(src + (q >> 2) * lln + c0 + 512 * ((q >> 1) & 1) + (q & 1));
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if ((pending & (1u << q)) && ll_ready(v[q], flag)) {
                const double val = ll_value(v[q]);
                double& d = y[q >> 2][(q >> 1) & 1][q & 1];
                d = accumulate ? d + val : val;
                pending &= ~(1u << q);
            }
    }
}

// Sum of 32 per-lane values across the warp, reduce-scatter style: on return
// lane l holds the warp total of index l (31 shuffles, fixed order).
__device__ __forceinline__ double warp_reduce_scatter32(double (&v)[32], int lane) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const bool up = lane & o;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const double send = up ? v[i] : v[i + o];
            const double keep = up ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0];
}

// The whole solve of one right-hand-side pair. CTAs [0, g) run the top chain,
// [g, 2g) the bottom chain; CTA i of a chain owns rows [i RPC, (i+1) RPC) of
// every block. Each thread owns the column pairs c0 = 2 tid + 512 i (m <= 1024)
// of all owned rows: it polls exactly the LL lines of its columns and
// multiplies them into its partial sums as soon as they arrive, so the
// matrix-vector product overlaps the dataflow wait (no CTA-wide gather). The
// Sinv rows stream into a shared-memory ring of 8-row units (cp.async.bulk,
// one full mbarrier per slot, refilled by one elected thread after each step)
// behind an L2 prefetch `pf` steps ahead. Per step: poll + partial products ->
// warp reduce-scatter -> warp 0 sums the 8 warp partials in order, forms the
// owned rows of the next step's input with the 8x8 coupling chunk and
// publishes them as LL lines. LL regions (per right-hand side, stride lln):
// [0, n) forward w, [n, 2n) backward inputs, [2n, 2n+m) top part of the twist
// input, [2n+m, 2n+2m) bottom part.
template <int RPC>
__global__ void __launch_bounds__(256, 1)
    k_sweep(int nsteps, int nb, int t, int m, const SweepTask* __restrict__ sched_g, int nrhs, int n,
            const double* __restrict__ sinv, long long sstride, int ld, const double* __restrict__ cloc,
            const double* __restrict__ b, long long ldb, double* __restrict__ x, long long ldx,
            double* __restrict__ wsave, uint4* ll, long long lln, unsigned flag, int stages, int pf, int g,
            unsigned long long* dbg) {
    static_assert(RPC == 8 || RPC == 16, "rows per CTA");
    constexpr int UPR = RPC / 8;  // ring units per step
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* ring = reinterpret_cast<double*>(smem_raw);  // [stages][8 rows][ld]
    double* red = ring + (size_t)stages * 8 * ld;         // [8 warps][32] partial sums
    double* csh = red + 8 * 32;                           // [32 lanes of warp 0][8] coupling row, then base
    unsigned long long* full = reinterpret_cast<unsigned long long*>(csh + 32 * 9);
    unsigned long long* wst = full + stages;  // debug: [3] per-step maxima
    SweepTask* tsh = reinterpret_cast<SweepTask*>(wst + 4);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lt = threadIdx.x;
    const int c0 = 2 * lt;
    if (lt < 3) wst[lt] = 0;
    const int chain = static_cast<int>(blockIdx.x) < g ? 0 : 1;
    const int row0 = (chain ? blockIdx.x - g : blockIdx.x) * RPC;
    const int nrow = min(RPC, m - row0);
    auto stamp = [&](int s, int ph) {
        if (dbg && threadIdx.x == 0) dbg[((size_t)blockIdx.x * nsteps + s) * 4 + ph] = globaltimer();
    };
    for (int i = threadIdx.x; i < nsteps; i += blockDim.x) tsh[i] = sched_g[2 * i + chain];
    const int nunits = nsteps * UPR;
    // unit u = rows [r0, r0 + 8) of Sinv_blk: contiguous (ld == m)
    auto unit_src = [&](int u, int& nrows) -> const double* {
        const SweepTask tk = tsh[u / UPR];
        const int r0 = 8 * (u % UPR);
        nrows = tk.kind != SW_IDLE ? max(0, min(8, nrow - r0)) : 0;
        return sinv + tk.blk * sstride + (long long)(row0 + r0) * ld;
    };
    auto prefetch_l2 = [&](int u) {
        if (u >= nunits) return;
        int nr;
        const double* src = unit_src(u, nr);
        if (nr) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(nr * ld * 8) : "memory");
    };
    auto issue = [&](int u) {
        if (u >= nunits) return;
        const int k = u % stages;
        int nr;
        const double* src = unit_src(u, nr);
        mbar_arrive_expect_tx(&full[k], static_cast<unsigned>(nr * ld * 8));
        if (nr) bulk_g2s(ring + (size_t)k * 8 * ld, src, static_cast<unsigned>(nr * ld * 8), &full[k]);
    };
    const bool issuer = lt == 7 * 32;  // off the publishing warp
    if (issuer) {
        for (int k = 0; k < stages; ++k) mbar_init(&full[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (issuer) {
        for (int u = 0; u < min(pf * UPR, nunits); ++u) prefetch_l2(u);
        for (int u = 0; u < stages; ++u) issue(u);
    }
    // warp 0 lane = kk * RPC + lr owns row lr, right-hand side kk of the step's result
    const int kk = lane / RPC, lr = lane % RPC;
    const int r_own = row0 + lr;
    const bool owner = warp == 0 && kk < nrhs && r_own < m;
    for (int s = 0; s < nsteps; ++s) {
        const SweepTask tk = tsh[s];
        stamp(s, 0);
        if (issuer)
            for (int p = 0; p < UPR; ++p) prefetch_l2((s + pf) * UPR + p);
        // the owned rows of the next step's input vector: target block tb at LL
        // offset reg, coupling chunk of C_cj (transposed or not), base 0 / rhs / saved w
        int tb = -1, cj = 0, basek = 0;
        bool tr = false, save = false;
        long long reg = 0;
        const int j = tk.blk;
        if (tk.kind == SW_FIRST || tk.kind == SW_FWD) {
            if (chain == 0) {
                if (j + 1 < t) { tb = j + 1; reg = (long long)tb * m; cj = j; basek = 1; save = true; }
                else if (j + 1 == t) { tb = t; reg = 2LL * n; cj = j; basek = 1; }
            } else {
                if (j - 1 > t) { tb = j - 1; reg = (long long)tb * m; cj = j - 1; tr = true; basek = 1; save = true; }
                else if (j - 1 == t) { tb = t; reg = 2LL * n + m; cj = j - 1; tr = true; }
            }
        } else if (tk.kind != SW_IDLE) {  // twist or backward
            if (chain == 0) {
                if (j - 1 >= 0) { tb = j - 1; reg = (long long)n + (long long)tb * m; cj = j - 1; tr = true; basek = 2; }
            } else if (j + 1 <= nb - 1) {
                tb = j + 1; reg = (long long)n + (long long)tb * m; cj = j; basek = 2;
            }
        }
        // its operands, loaded before the wait (off the critical path) into this
        // lane's own shared-memory slot
        const bool pub = owner && tb >= 0;
        if (pub) {
            double* cs = csh + lane * 9;
            cs[8] = basek == 1 ? b[kk * ldb + (long long)tb * m + r_own]
                               : basek == 2 ? wsave[kk * (long long)n + (long long)tb * m + r_own] : 0.0;
            const double* cp = cloc + ((long long)cj * (m >> 3) + (r_own >> 3)) * 64;
#pragma unroll
            for (int q = 0; q < 8; ++q) cs[q] = tr ? cp[q * 8 + (r_own & 7)] : cp[(r_own & 7) * 8 + q];
        }
        const bool active = tk.kind != SW_IDLE;
        if (active) {
            if (tk.kind == SW_FIRST && owner)
                wsave[kk * (long long)n + (long long)j * m + r_own] = b[kk * ldb + (long long)j * m + r_own];
            // this thread's input values
            double y[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};
            if (tk.kind == SW_FIRST || (tk.kind == SW_TWIST && t == 0)) {
                const int jb = tk.kind == SW_FIRST ? j : t;
#pragma unroll
                for (int k = 0; k < 2; ++k)
#pragma unroll
                    for (int i = 0; i < 2; ++i)
                        if (k < nrhs && c0 + 512 * i < m) {
                            const double2 v2 =
                                *reinterpret_cast<const double2*>(b + k * ldb + (long long)jb * m + c0 + 512 * i);
                            y[k][i][0] = v2.x;
                            y[k][i][1] = v2.y;
                        }
            }
            if (tk.kind == SW_TWIST) {
                if (t > 0) poll_pairs(ll + 2LL * n, lln, nrhs, m, c0, flag, y, false);
                if (t < nb - 1) poll_pairs(ll + 2LL * n + m, lln, nrhs, m, c0, flag, y, true);
            } else if (tk.kind != SW_FIRST) {
                poll_pairs(ll + (tk.kind == SW_BWD ? (long long)n : 0LL) + (long long)j * m, lln, nrhs, m, c0, flag, y,
                           false);
            }
            if (dbg && lane == 0) atomicMax(&wst[0], globaltimer());  // last warp's inputs polled
#pragma unroll
            for (int p = 0; p < UPR; ++p) {
                const int u = s * UPR + p;
                mbar_wait(&full[u % stages], static_cast<unsigned>((u / stages) & 1));
            }
            if (dbg && lane == 0) atomicMax(&wst[2], globaltimer());  // last warp's rows ready
            // owned rows of Sinv_j times this thread's inputs
            double v[32];  // [rhs][row]
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.0;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int c = c0 + 512 * i;
                if (c < m)
#pragma unroll
                    for (int r = 0; r < RPC; ++r) {
                        const int u = s * UPR + (r >> 3);
                        const double2 a =
                            r < nrow ? *reinterpret_cast<const double2*>(ring + ((size_t)(u % stages) * 8 + (r & 7)) * ld + c)
                                     : make_double2(0.0, 0.0);
                        v[r] += a.x * y[0][i][0];
                        v[r] += a.y * y[0][i][1];
                        v[RPC + r] += a.x * y[1][i][0];
                        v[RPC + r] += a.y * y[1][i][1];
                    }
            }
            red[warp * 32 + lane] = warp_reduce_scatter32(v, lane);
            if (dbg && lane == 0) atomicMax(&wst[1], globaltimer());  // last warp's partials done
        }
        __syncthreads();  // partials complete, this step's ring slots free
        if (dbg && lt == 0) {
            dbg[((size_t)blockIdx.x * nsteps + s) * 4 + 1] = wst[0];
            dbg[((size_t)blockIdx.x * nsteps + s) * 4 + 3] = wst[1];
            dbg[((size_t)blockIdx.x * nsteps + s) * 4 + 2] = wst[2];
            wst[0] = wst[1] = wst[2] = 0;
        }
        if (issuer) {
            // refill the freed slots with the units `stages` ahead (a unit is issued only
            // after every thread finished the step that used its slot, so a parity wait
            // never sees a slot two phases ahead)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
            for (int p = 0; p < UPR; ++p) issue(s * UPR + p + stages);
        }
        if (active && warp == 0) {
            double val = 0.0;
#pragma unroll
            for (int w = 0; w < 8; ++w) val += red[w * 32 + lane];
            const bool store_x = tk.kind == SW_BWD || (tk.kind == SW_TWIST && chain == 0);
            if (owner && store_x) x[kk * ldx + (long long)j * m + r_own] = val;
            // publish the owned rows of the next input: base - C v (fixed order); the
            // 8 values of this row's cell sit in lanes (lane & ~7) .. + 7
            const double* cs = csh + lane * 9;
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const double vq = __shfl_sync(0xffffffffu, val, (lane & ~7) + q);
                acc += (pub ? cs[q] : 0.0) * vq;
            }
            if (pub) {
                const double nv = cs[8] - acc;
                ll_store(ll + kk * lln + reg + r_own, nv, flag);
                if (save) wsave[kk * (long long)n + (long long)tb * m + r_own] = nv;
            }
        }
        if (!dbg) stamp(s, 2);
    }
}

}  // namespace

bool BlockTriChol::local_prepare(double* dense, cudaStream_t st) {
    local = false;
    if (!allow_local || perm.n || nb < 1) return false;
    const int m = bsz[0];
    if (m % 8 != 0 || m > 1024) return false;  // k_sweep: two column pairs per thread
    for (int j = 0; j < nb; ++j)
        if (bsz[j] != m) return false;
    const int nc = nb - 1;
    if (nc > 0) {
        DBuf<int> err(1);
        err.zero(st);
        const long long total = (long long)nc * m * m;
        k_check_local<<<grid_for(total, 256), 256, 0, st>>>(total, m, dense + dC_[0], err.p);
        PDG_CHECK_LAUNCH();
        if (err.download(st)[0] != 0) return false;
        cloc.alloc((size_t)nc * m * 8);
        k_extract_cloc<<<grid_for((long long)nc * m * 8, 256), 256, 0, st>>>(nc, m, dense + dC_[0], cloc.p);
        PDG_CHECK_LAUNCH();
    } else {
        cloc.alloc(8);
    }
    local = true;
    return true;
}

void BlockTriChol::local_finish(double* dense, cudaStream_t st) {
    const int m = bsz[0], t = twist;
    {
        cusolverDnHandle_t h = nullptr;
        if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS) throw Error(PDG_CUDA_ERROR, "cusolverDnCreate failed");
        struct Guard {
            cusolverDnHandle_t h;
            ~Guard() { cusolverDnDestroy(h); }
        } guard{h};
        if (cusolverDnSetStream(h, st) != CUSOLVER_STATUS_SUCCESS) throw Error(PDG_CUDA_ERROR, "cusolverDnSetStream failed");
        int lwork = 0;
        if (cusolverDnDpotri_bufferSize(h, CUBLAS_FILL_MODE_LOWER, m, dense + dD_[0], m, &lwork) != CUSOLVER_STATUS_SUCCESS)
            throw Error(PDG_CUDA_ERROR, "cusolverDnDpotri_bufferSize failed");
        DBuf<double> work(std::max(lwork, 1));
        DBuf<int> info(nb);
        info.zero(st);
        ld_s = (m + 1) & ~1;
        sinv_stride = ((long long)m * ld_s + 31) & ~31LL;
        store.alloc((size_t)nb * sinv_stride);
        for (int j = 0; j < nb; ++j) {
            // Sinv_j = (L_j L_j^T)^{-1} from the Cholesky factor of the twisted Schur complement
            if (cusolverDnDpotri(h, CUBLAS_FILL_MODE_LOWER, m, dense + dD_[j], m, work.p, lwork, info.p + j) !=
                CUSOLVER_STATUS_SUCCESS)
                throw Error(PDG_CUDA_ERROR, "cusolverDnDpotri failed");
            k_symm_store<<<grid_for((long long)m * m, 256), 256, 0, st>>>(m, dense + dD_[j], ld_s,
                                                                           store.p + j * sinv_stride);
            PDG_CHECK_LAUNCH();
        }
        std::vector<int> hinfo = info.download(st);
        for (int j = 0; j < nb; ++j)
            if (hinfo[j] != 0)
                throw Error(PDG_NOT_CONVERGED, "dense LU: matrix is singular to working precision (block " +
                                                   std::to_string(j) + " not invertible)");
    }
    factor_bytes = 16.0 * m * (double)m * nb + 16.0 * 8.0 * m * (nb - 1);
    // ---- schedule: forward (top 0..t-1, bottom nb-1..t+1), twist, backward --------
    sweep.clear();
    const SweepTask idle{-1, SW_IDLE};
    const int L = std::max(t, nb - 1 - t);
    for (int s = 0; s < L; ++s) {
        sweep.push_back(s < t ? SweepTask{s, s == 0 ? SW_FIRST : SW_FWD} : idle);
        const int jb = nb - 1 - s;
        sweep.push_back(jb > t ? SweepTask{jb, s == 0 ? SW_FIRST : SW_FWD} : idle);
    }
    sweep.push_back(SweepTask{t, SW_TWIST});
    sweep.push_back(SweepTask{t, SW_TWIST});
    for (int s = 1; s <= L; ++s) {
        sweep.push_back(t - s >= 0 ? SweepTask{t - s, SW_BWD} : idle);
        sweep.push_back(t + s <= nb - 1 ? SweepTask{t + s, SW_BWD} : idle);
    }
    d_sweep.upload(sweep, st);
    // ---- kernel configuration: rows per CTA (8 or 16, one CTA per SM), ring stages --
    int dev = 0;
    PDG_CUDA(cudaGetDevice(&dev));
    int optin = 0;
    PDG_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    // (the attribute is per function, shared by every solver instance: set the device maximum)
    PDG_CUDA(cudaFuncSetAttribute(k_sweep<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    PDG_CUDA(cudaFuncSetAttribute(k_sweep<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    const int nsteps = static_cast<int>(sweep.size() / 2);
    sw_rpc = 2 * ((m + 7) / 8) <= num_sms() ? 8 : 16;
    sw_g = (m + sw_rpc - 1) / sw_rpc;
    require(2 * sw_g <= num_sms(), "block-tridiagonal solver: blocks too large for the sweep kernel");
    const size_t fixed = sizeof(double) * (8 * 32 + 32 * 9) + 8 * 16 + sizeof(SweepTask) * nsteps + 64;
    const size_t unit = sizeof(double) * 8 * ld_s;
    require(fixed + unit * (sw_rpc / 8) <= (size_t)optin - 1024, "block-tridiagonal solver: sweep kernel shared memory");
    sw_stages = static_cast<int>(std::min<size_t>(((size_t)optin - 1024 - fixed) / unit, 16));
    sw_smem = fixed + unit * sw_stages;
    int occ = 0;
    PDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sw_rpc == 8 ? k_sweep<8> : k_sweep<16>, 256, sw_smem));
    require(occ >= 1, "block-tridiagonal solver: sweep kernel cannot be resident");
    ll.alloc((size_t)max_rhs * (2 * (size_t)n + 2 * (size_t)m));
    ll.zero(st);
    wsave.alloc((size_t)n * max_rhs);
    PDG_CUDA(cudaStreamSynchronize(st));
}

void BlockTriChol::solve_local(const double* b, long long ldb, double* x, long long ldx, int nrhs, cudaStream_t st) {
    unsigned flag = static_cast<unsigned>(++call);
    if (flag == 0) flag = static_cast<unsigned>(++call);  // 0 = never published
    int nsteps = static_cast<int>(sweep.size() / 2), nb_ = nb, t = twist, m = bsz[0], nr = nrhs, n_ = n;
    int ld = ld_s, g = sw_g, stg = sw_stages;
    int pf = 2;  // L2 prefetch distance (steps)
    if (const char* e = std::getenv("PDG_SWEEP_PF")) pf = std::atoi(e);
    long long ss = sinv_stride, lb = ldb, lx = ldx, lln = 2LL * n + 2LL * m;
    const SweepTask* sched = d_sweep.p;
    const double* sv = store.p;
    const double* cl = cloc.p;
    double* ws = wsave.p;
    uint4* llp = ll.p;
    unsigned long long* dbgp = nullptr;
    dbg_steps = nsteps;
    if (debug_timing) {
        dbg.alloc((size_t)2 * g * nsteps * 4);
        dbg.zero(st);
        dbgp = dbg.p;
    }
    void* args[] = {&nsteps, &nb_, &t, &m, &sched, &nr, &n_, &sv, &ss, &ld, &cl, &b, &lb,
                    &x, &lx, &ws, &llp, &lln, &flag, &stg, &pf, &g, &dbgp};
    PDG_CUDA(cudaLaunchCooperativeKernel(sw_rpc == 8 ? (void*)k_sweep<8> : (void*)k_sweep<16>, 2 * g, 256, args, sw_smem, st));
    count_launch(1);
    PDG_CHECK_LAUNCH();
}

}  // namespace pdg
