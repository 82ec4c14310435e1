// Nested-dissection multifrontal Cholesky (see nd.cuh).
#include <cooperative_groups.h>
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <numeric>
#include <queue>
#include <string>

#include "blocktri.cuh"
#include "llsync.cuh"
#include "nd.cuh"

namespace cg = cooperative_groups;

#define PDG_ND_CUSOLVER(call)                                                                                       \
    do {                                                                                                            \
        cusolverStatus_t s_ = (call);                                                                               \
        if (s_ != CUSOLVER_STATUS_SUCCESS)                                                                          \
            throw ::pdg::Error(PDG_CUDA_ERROR, std::string(#call) + ": cusolver status " + std::to_string((int)s_)); \
    } while (0)
#define PDG_ND_CUBLAS(call)                                                                                       \
    do {                                                                                                          \
        cublasStatus_t s_ = (call);                                                                               \
        if (s_ != CUBLAS_STATUS_SUCCESS)                                                                          \
            throw ::pdg::Error(PDG_CUDA_ERROR, std::string(#call) + ": cublas status " + std::to_string((int)s_)); \
    } while (0)

namespace pdg {

namespace {

#ifndef PDG_ND_THREADS
#define PDG_ND_THREADS 256
#endif
#ifndef PDG_ND_BUFS
#define PDG_ND_BUFS 8
#endif
constexpr int kNdThreads = PDG_ND_THREADS;  // compute threads (tuning: tools/nd_variant_sweep.sh)
constexpr int kNdMaxRhs = 2;
constexpr int kNdMaxTaskRows = 1024;  // rows of one task (the update-vector staging in shared memory)
constexpr int kNdComputeWarps = kNdThreads / 32;
#ifndef PDG_ND_PREP
#define PDG_ND_PREP 2
#endif
#ifndef PDG_ND_GATHER
#define PDG_ND_GATHER 4
#endif
#ifndef PDG_ND_MINB
#define PDG_ND_MINB 1
#endif
constexpr int kNdPrepWarps = PDG_ND_PREP;  // input warps
constexpr int kNdBufs = PDG_ND_BUFS;     // pipeline slots (barrier sets); task buffers live in a FIFO arena
constexpr int kNdGatherWarps = PDG_ND_GATHER;  // dependency wait + dependent gather, tasks in order
constexpr int kNdGatherThreads = 32 * kNdGatherWarps;
constexpr int kNdWarpProducer = kNdComputeWarps;
constexpr int kNdWarpStage = kNdWarpProducer + 1;
constexpr int kNdWarpGather = kNdWarpStage + kNdPrepWarps;
constexpr int kNdWarpSignal = kNdWarpGather + kNdGatherWarps;
constexpr int kNdBlock = 32 * (kNdWarpSignal + 1);

// ---------------------------------------------------------------------------
// host: nested dissection
// ---------------------------------------------------------------------------
struct HostFront {
    std::vector<int> snodes, bnodes;
    int parent = -1, depth = 0;
    std::vector<int> children;
};

struct Dissector {
    const std::vector<int>& aoff;  // node adjacency CSR
    const std::vector<int>& adj;
    const std::vector<int>& ndofs;
    std::vector<const std::vector<double>*> cs;  // node coordinates per axis (2 or 3 axes)
    int leaf;
    std::vector<HostFront> fr;
    std::vector<int> node_front, mark, seen;
    int stamp = 0;

    Dissector(const std::vector<int>& o, const std::vector<int>& a, const std::vector<int>& nd,
              const std::vector<double>& x, const std::vector<double>& y, const std::vector<double>* z, int lf)
        : aoff(o), adj(a), ndofs(nd), leaf(lf) {
        cs = {&x, &y};
        if (z) cs.push_back(z);
        const int nn = static_cast<int>(nd.size());
        node_front.assign(nn, -1);
        mark.assign(nn, 0);
        seen.assign(nn, 0);
    }

    // try to cut `nodes` at the line / plane coord == v (axis 0: x, 1: y, 2: z)
    bool try_cut(const std::vector<int>& nodes, int axis, double v, int st, std::vector<int>& sep,
                 std::vector<int>& lo, std::vector<int>& hi) {
        const std::vector<double>& c = *cs[axis];
        sep.clear();
        lo.clear();
        hi.clear();
        for (int u : nodes) {
            if (c[u] < v)
                lo.push_back(u);
            else if (c[u] > v)
                hi.push_back(u);
            else
                sep.push_back(u);
        }
        if (lo.empty() || hi.empty() || sep.empty()) return false;
        for (int u : lo)
            for (int k = aoff[u]; k < aoff[u + 1]; ++k) {
                const int w = adj[k];
                if (mark[w] == st && c[w] > v) return false;
            }
        return true;
    }

    int build(std::vector<int> nodes, int parent, int depth) {
        const int st = ++stamp;
        for (int u : nodes) mark[u] = st;
        std::vector<int> bnd;
        for (int u : nodes)
            for (int k = aoff[u]; k < aoff[u + 1]; ++k) {
                const int w = adj[k];
                if (mark[w] != st && seen[w] != st) {
                    seen[w] = st;
                    if (node_front[w] < 0) throw Error(PDG_INVALID_ARGUMENT, "nested dissection: region boundary outside the ancestor separators");
                    bnd.push_back(w);
                }
            }
        long long dofs = 0;
        for (int u : nodes) dofs += ndofs[u];
        std::vector<int> sep, lo, hi;
        bool cut = false;
        if (dofs > leaf && nodes.size() >= 3) {
            const int nax = static_cast<int>(cs.size());
            double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
            for (int u : nodes)
                for (int a = 0; a < nax; ++a) {
                    mn[a] = std::min(mn[a], (*cs[a])[u]);
                    mx[a] = std::max(mx[a], (*cs[a])[u]);
                }
            // axes by decreasing extent (ties: the lower axis first)
            int order[3] = {0, 1, 2};
            std::stable_sort(order, order + nax, [&](int a, int b) { return mx[a] - mn[a] > mx[b] - mn[b]; });
            for (int t = 0; t < nax && !cut; ++t) {
                const int axis = order[t];
                const std::vector<double>& c = *cs[axis];
                std::vector<double> vals;
                vals.reserve(nodes.size());
                for (int u : nodes) vals.push_back(c[u]);
                std::sort(vals.begin(), vals.end());
                const double med = vals[vals.size() / 2];
                vals.erase(std::unique(vals.begin(), vals.end()), vals.end());
                std::vector<double> cand(vals);
                std::stable_sort(cand.begin(), cand.end(),
                                 [&](double a, double b) { return std::fabs(a - med) < std::fabs(b - med); });
                const int tries = std::min<int>(static_cast<int>(cand.size()), 8);
                for (int k = 0; k < tries && !cut; ++k) cut = try_cut(nodes, axis, cand[k], st, sep, lo, hi);
            }
        }
        const int id = static_cast<int>(fr.size());
        fr.emplace_back();
        fr[id].parent = parent;
        fr[id].depth = depth;
        fr[id].bnodes = std::move(bnd);
        fr[id].snodes = cut ? sep : nodes;
        for (int u : fr[id].snodes) node_front[u] = id;
        if (cut) {
            const int a = build(std::move(lo), id, depth + 1);
            const int b = build(std::move(hi), id, depth + 1);
            fr[id].children = {a, b};
        }
        return id;
    }
};

// ---------------------------------------------------------------------------
// device: numeric factorization helpers (setup)
// ---------------------------------------------------------------------------
__global__ void k_nd_scatter(long long nt, const long long* pos, const double* val, double* F) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nt; t += (long long)gridDim.x * blockDim.x)
        F[pos[t]] = val[t];
}
// parent(lower) += child update matrix (lower), both column-major
__global__ void k_nd_extend_add(double* P, int fp, const double* U, int fc, int bc, const int* map) {
    const long long tot = (long long)bc * bc;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
        const int r = static_cast<int>(t % bc), c = static_cast<int>(t / bc);
        if (r < c) continue;
        const int pr = map[r], pc = map[c];
        const int hi = max(pr, pc), lo = min(pr, pc);
        P[hi + (long long)lo * fp] += U[r + (long long)c * fc];
    }
}
__global__ void k_nd_identity(int s, double* T) {
    const long long tot = (long long)s * s;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x)
        T[t] = (t % s == t / s) ? 1.0 : 0.0;
}
// M (row-major (s+b) x ldm) and M^T (row-major s x ldt) from Linv (s x s, col-major, ld s)
// and G = L_BS Linv (b x s, col-major, ld b); padding zero.
template <typename OutT>
__global__ void k_nd_pack(int s, int b, const double* T, const double* G, OutT* M, int ldm, OutT* MT, int ldt) {
    const long long tot = (long long)(s + b) * ldm;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
        const int r = static_cast<int>(t / ldm), c = static_cast<int>(t % ldm);
        double v = 0.0;
        if (c < s) v = r < s ? T[r + (long long)c * s] : G[(r - s) + (long long)c * b];
        M[t] = static_cast<OutT>(v);
    }
    const long long tt = (long long)s * ldt;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tt; t += (long long)gridDim.x * blockDim.x) {
        const int r = static_cast<int>(t / ldt), c = static_cast<int>(t % ldt);
        double v = 0.0;
        if (c < s)
            v = T[c + (long long)r * s];
        else if (c < s + b)
            v = G[(c - s) + (long long)r * b];
        MT[t] = static_cast<OutT>(v);
    }
}

// Batched factorization of one tree level (setup): one CTA per front does what the cuSOLVER /
// cuBLAS sequence does per front (extend-add of the children's update matrices, partial
// Cholesky of the s pivots with the Schur complement left in F_BB for the parent,
// T = L_SS^{-1}, G = L_BS T, M / M^T packed into the store), so a level of hundreds of small
// fronts is ONE launch instead of ~10 library calls per front (the setup was launch-bound:
// config 1, 2047 + 1023 fronts). Fronts are dense column-major (ld = f), lower triangle.
struct NdFactorDesc {
    long long fo, moff, mtoff;
    long long cfo[2], cmap[2];
    int s, b, ldm, ldt, nchild, front;
    int cs[2], cb[2];
};
constexpr int kFactorThreads = 256;
__global__ void __launch_bounds__(kFactorThreads) k_nd_factor_batch(const NdFactorDesc* descs, double* dense, const int* maps,
                                                                   double* store, int* info) {
    const NdFactorDesc D = descs[blockIdx.x];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = kFactorThreads / 32;
    const int s = D.s, b = D.b, f = s + b;
    double* F = dense + D.fo;
    // 1. extend-add, children in order (their maps are injective: no two entries collide)
    for (int q = 0; q < D.nchild; ++q) {
        const int bc = D.cb[q], fc = D.cs[q] + bc;
        const double* U = dense + D.cfo[q] + D.cs[q] + (long long)D.cs[q] * fc;
        const int* map = maps + D.cmap[q];
        for (long long t = tid; t < (long long)bc * bc; t += kFactorThreads) {
            const int r = static_cast<int>(t % bc), c = static_cast<int>(t / bc);
            if (r < c) continue;
            const int pr = map[r], pc = map[c];
            const int hi = max(pr, pc), lo = min(pr, pc);
            F[hi + (long long)lo * f] += U[r + (long long)c * fc];
        }
        __syncthreads();
    }
    // 2. right-looking partial Cholesky: pivots 0..s-1, updates reach the whole lower triangle
    for (int k = 0; k < s; ++k) {
        if (tid == 0) {
            double d = F[k + (long long)k * f];
            if (!(d > 0.0)) {
                if (info[D.front] == 0) info[D.front] = k + 1;
                d = 1.0;
            }
            F[k + (long long)k * f] = sqrt(d);
        }
        __syncthreads();
        const double dk = F[k + (long long)k * f];
        for (int i = k + 1 + tid; i < f; i += kFactorThreads) F[i + (long long)k * f] /= dk;
        __syncthreads();
        for (int j = k + 1 + warp; j < f; j += nw) {
            const double ljk = F[j + (long long)k * f];
            for (int i = j + lane; i < f; i += 32) F[i + (long long)j * f] -= F[i + (long long)k * f] * ljk;
        }
        __syncthreads();
    }
    // 3. T = L_SS^{-1} straight into M (row-major, ld = ldm): thread j owns column j
    double* M = store + D.moff;
    double* MT = store + D.mtoff;
    for (int j = tid; j < D.ldm; j += kFactorThreads) {
        for (int i = 0; i < s; ++i) {
            double acc = 0.0;
            if (j < s && i >= j) {
                acc = i == j ? 1.0 : 0.0;
                for (int k = j; k < i; ++k) acc -= F[i + (long long)k * f] * M[(long long)k * D.ldm + j];
                acc /= F[i + (long long)i * f];
            }
            M[(long long)i * D.ldm + j] = acc;
        }
    }
    __syncthreads();
    // 4. G = L_BS T into the rows s.. of M
    for (long long t = tid; t < (long long)b * D.ldm; t += kFactorThreads) {
        const int r = static_cast<int>(t / D.ldm), c = static_cast<int>(t % D.ldm);
        double acc = 0.0;
        if (c < s)
            for (int k = c; k < s; ++k) acc += F[(s + r) + (long long)k * f] * M[(long long)k * D.ldm + c];
        M[(long long)(s + r) * D.ldm + c] = acc;
    }
    __syncthreads();
    // 5. M^T (s x ldt)
    for (long long t = tid; t < (long long)s * D.ldt; t += kFactorThreads) {
        const int r = static_cast<int>(t / D.ldt), c = static_cast<int>(t % D.ldt);
        MT[t] = c < f ? M[(long long)c * D.ldm + r] : 0.0;
    }
}

// ---------------------------------------------------------------------------
// device: the solve
// ---------------------------------------------------------------------------
struct NdArgs {
    const NdTask* tasks;
    const int* ctoff;
    const int* sdofs;
    const int* bpos;
    const int* cbdst;  // per boundary entry: its slot in the parent's contribution buffer
    const double* store;
    const double* b;
    long long ldb;
    double* x;
    long long ldx;
    double* y;
    double* xpos;
    double* cb;
    unsigned long long* cnt;
    unsigned long long call;
    long long cbtot;
    int n, nrhs, stages, vmax, max_tasks, pf;
    unsigned stage_bytes;
    unsigned long long* dbg;  // optional: per task, %globaltimer at [inputs ready, signalled, prep done, compute done]
    int nodep;                // debug timing only (PDG_ND_NODEP): skip the dependency waits (wrong results)
    int nomath;               // debug timing only (PDG_ND_NOMATH): consume the matrix chunks without the products
    int fence;                // PDG_ND_FENCE: explicit fence.acq_rel.gpu before each completion release
    const int* stop;          // skip the solve once *stop != 0 (speculative GMRES steps)
    int tile8;                // PDG_ND_TILE8: the 8-row / 32-lane narrow-chunk GEMV instead of the 8-lane groups
    int pairs;                // PDG_ND_PAIRS=1: two warps per chunk (measured slower: 298 vs 287 us at config 1)
};

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add(unsigned long long* p, unsigned long long v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// 16 per-lane values summed across the warp: on return lane l (< 16) holds the
// total of index l (reduce-scatter over each half-warp, then the two halves; fixed order)
__device__ __forceinline__ double warp_reduce_scatter16(double (&v)[16], int lane) {
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) {
        const bool up = lane & o;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const double send = up ? v[i] : v[i + o];
            const double keep = up ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}

// Narrow-row chunk GEMV: the warp as 4 groups of 8 lanes, group q owns R rows of each
// pass (4 R rows per pass), a lane sums its row segment over the columns c2 = lane % 8
// (mod 8) for both right-hand sides (4 independent FMA chains per row), then an 8-lane
// reduce-scatter of the 2 R (row, rhs) sums leaves lane l of the group with sum l.
// Fewer shuffles and more independent chains than the 8-row / 32-lane tile
// (tools/ubench/chunk_gemv.cu: "G8 R4").
template <int R, typename Out>
__device__ __forceinline__ void chunk_g8(const double2* __restrict__ rows2, int nrow, int ld2, const double2* va,
                                         const double2* vb, int lane, Out out, int nr, int start = 0, int step = 1) {
    static_assert(R == 1 || R == 2 || R == 4, "rows per lane group");
    const int lg = lane & 7, grp = lane >> 3;
    for (int rb = start * 4 * R; rb < nrow; rb += step * 4 * R) {
        const int row0 = rb + grp * R;
        double acc[R][4];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r][0] = acc[r][1] = acc[r][2] = acc[r][3] = 0.0;
        for (int c2 = lg; c2 < ld2; c2 += 8) {
            const double2 p = va[c2], q = vb[c2];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double2 m = row0 + r < nrow ? rows2[(size_t)(row0 + r) * ld2 + c2] : make_double2(0.0, 0.0);
                acc[r][0] = fma(m.x, p.x, acc[r][0]);
                acc[r][1] = fma(m.y, p.y, acc[r][1]);
                acc[r][2] = fma(m.x, q.x, acc[r][2]);
                acc[r][3] = fma(m.y, q.y, acc[r][3]);
            }
        }
        double v[2 * R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            v[2 * r] = acc[r][0] + acc[r][1];
            v[2 * r + 1] = acc[r][2] + acc[r][3];
        }
        // reduce-scatter over the 8 lanes of the group (xor offsets stay inside it)
#pragma unroll
        for (int o = R; o >= 1; o >>= 1) {
            const bool up = lg & o;
#pragma unroll
            for (int i = 0; i < o; ++i) {
                const double send = up ? v[i] : v[i + o];
                const double keep = up ? v[i + o] : v[i];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
        double t = v[0];
#pragma unroll
        for (int o = 2 * R; o < 8; o <<= 1) t += __shfl_xor_sync(0xffffffffu, t, o);  // 2 R values over 8 lanes
        const int idx = lg & (2 * R - 1);  // lane's (row, rhs) index: row idx / 2, rhs idx % 2
        const int r = idx >> 1, k = idx & 1;
        if (lg < 2 * R && row0 + r < nrow && k < nr) out(k, row0 + r, t);
    }
}

// Wide-row chunk GEMV: R rows at a time, all 32 lanes over the columns (stride 32),
// 4 independent FMA chains per row; reduce-scatter of the 2 R (row, rhs) sums over the
// low lane bits, then a butterfly over the rest: lane l < 2 R ends with sum l.
template <int R, typename Out>
__device__ __forceinline__ void chunk_wide(const double2* __restrict__ rows2, int nrow, int ld2, const double2* va,
                                           const double2* vb, int lane, Out out, int nr, int start = 0, int step = 1) {
    for (int rb = start * R; rb < nrow; rb += step * R) {
        double acc[R][4];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r][0] = acc[r][1] = acc[r][2] = acc[r][3] = 0.0;
        for (int c2 = lane; c2 < ld2; c2 += 32) {
            const double2 p = va[c2], q = vb[c2];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double2 m = rb + r < nrow ? rows2[(size_t)(rb + r) * ld2 + c2] : make_double2(0.0, 0.0);
                acc[r][0] = fma(m.x, p.x, acc[r][0]);
                acc[r][1] = fma(m.y, p.y, acc[r][1]);
                acc[r][2] = fma(m.x, q.x, acc[r][2]);
                acc[r][3] = fma(m.y, q.y, acc[r][3]);
            }
        }
        double v[2 * R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            v[2 * r] = acc[r][0] + acc[r][1];
            v[2 * r + 1] = acc[r][2] + acc[r][3];
        }
#pragma unroll
        for (int o = R; o >= 1; o >>= 1) {
            const bool up = lane & o;
#pragma unroll
            for (int i = 0; i < o; ++i) {
                const double send = up ? v[i] : v[i + o];
                const double keep = up ? v[i + o] : v[i];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
        double t = v[0];
#pragma unroll
        for (int o = 2 * R; o < 32; o <<= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        const int r = lane >> 1, k = lane & 1;
        if (lane < 2 * R && rb + r < nrow && k < nr) out(k, rb + r, t);
    }
}

// Shared-memory layout of the solve kernel: mbarriers + task descriptors, the TMA
// ring, then the buffer arena: per task (FIFO, offsets placed on the host so small
// tasks pack densely and up to kNdBufs tasks are in flight) [v: rhs x vmt doubles]
// [oix: nrows ints][bix: b ints (backward)]. v holds the task's input vector; for a
// forward task the tail v[k][s ..] also carries the children's updates passing
// through the task's boundary rows.
constexpr unsigned kNdHeader = 2048;
long long round2(long long v) { return (v + 1) & ~1LL; }
// v stride of a task: the row length, and for a non-leaf forward task at least s + b (pass-through tail)
inline int nd_task_vmt(const NdTask& t) { return static_cast<int>(round2((t.type == 1 && !t.leaf) ? std::max(t.ld, t.s + t.b) : t.ld)); }
inline size_t nd_task_buf_bytes(const NdTask& t) {
    const size_t by = (size_t)t.vmt * kNdMaxRhs * sizeof(double) + (size_t)(t.nrows + (t.type == 2 ? t.b : 0)) * sizeof(int);
    return (by + 127) / 128 * 128;
}
__host__ __device__ inline size_t nd_task_bytes(int max_tasks) { return ((size_t)max_tasks * sizeof(NdTask) + 127) / 128 * 128; }

// Warp roles (one CTA per SM, a static task list per CTA in topological order):
//   warps 0-7   compute: chunk j of the CTA's matrix stream is consumed by warp j % 8
//               against the task's gathered input; outputs to y / cb / x. No CTA-wide
//               barrier: a warp moves on to the next task as soon as its chunks are
//               done and that task's input is gathered (no waiting for stragglers);
//   warp 8      TMA producer (lane 0): matrix chunks into the ring, L2 prefetch ahead;
//   warps 9-10  staging (even / odd tasks, independently): for the tasks ahead (up to
//               kNdBufs - 1), the output indices, the boundary pivot positions and the
//               right-hand side b_S - everything that does not depend on other tasks -
//               plus a non-blocking look at the dependency counters;
//   warps 11-14 gather (tasks in order): the dependency wait and the dependent gather
//               (children's update vectors, or y / x of the parent) into the task
//               buffer, while the compute warps still stream the previous tasks;
//   warp 15     signaller (lane 0): once the compute warps are done with a task,
//               publishes its completion counter (release).
// Buffer q cycles staged (staging -> gather), gathered (gather -> compute), done
// (compute -> signaller) and free (gather, once the next task's input is built, +
// signaller -> staging).
__device__ __forceinline__ void gather_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kNdGatherThreads) : "memory"); }

__global__ void __launch_bounds__(kNdBlock, PDG_ND_MINB) k_nd_solve(NdArgs a) {
    using namespace dev;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem);  // [32]
    unsigned long long* empty = full + 32;                                   // [32]
    unsigned long long* staged = empty + 32;                                 // [kNdBufs]
    unsigned long long* done = staged + kNdBufs;                             // [kNdBufs]
    unsigned long long* freeb = done + kNdBufs;                              // [kNdBufs]
    unsigned long long* gathered = freeb + kNdBufs;                          // [kNdBufs]
    NdTask* tbT = reinterpret_cast<NdTask*>(smem + 1024);                    // [kNdBufs]
    int* tbOk = reinterpret_cast<int*>(smem + 1024 + kNdBufs * sizeof(NdTask));  // [kNdBufs] dependencies seen met
    // this CTA's task descriptors: copied into shared memory when they fit the budget the
    // host planned (a.max_tasks > 0), read from global memory (L1-cached) otherwise, so the
    // shared-memory plan does not grow with the mesh
    const bool tsk_smem = a.max_tasks > 0;
    NdTask* tsk_s = reinterpret_cast<NdTask*>(smem + kNdHeader);
    const int t0_ = a.ctoff[blockIdx.x];
    const NdTask* tsk = tsk_smem ? tsk_s : a.tasks + t0_;
    unsigned char* ring = smem + kNdHeader + nd_task_bytes(a.max_tasks);
    unsigned char* arena = ring + (size_t)a.stages * a.stage_bytes;
    auto vbuf = [&](const NdTask& t) { return reinterpret_cast<double*>(arena + t.boff); };
    auto oixbuf = [&](const NdTask& t) { return reinterpret_cast<int*>(vbuf(t) + (size_t)t.vmt * kNdMaxRhs); };
    auto bixbuf = [&](const NdTask& t) { return oixbuf(t) + t.nrows; };
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int t0 = a.ctoff[blockIdx.x], nt = a.ctoff[blockIdx.x + 1] - t0;
    const int nr = a.nrhs;
    if (tid == 0) {
        for (int k = 0; k < a.stages; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], a.pairs ? 2 : 1);
        }
        for (int k = 0; k < kNdBufs; ++k) {
            mbar_init(&staged[k], 1);
            mbar_init(&done[k], kNdComputeWarps);
            mbar_init(&freeb[k], 2);
            mbar_init(&gathered[k], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tsk_smem) {
        static_assert(sizeof(NdTask) % 4 == 0, "NdTask is copied as ints");
        const int* src = reinterpret_cast<const int*>(a.tasks + t0);
        int* dst = reinterpret_cast<int*>(tsk_s);
        const int words = nt * static_cast<int>(sizeof(NdTask) / 4);
        for (int w = tid; w < words; w += kNdBlock) dst[w] = src[w];
    }
    __syncthreads();
    if (a.stop && *a.stop) {  // skipped call: completion counters advance as if every task ran
        for (int i = tid; i < nt; i += kNdBlock) atomicAdd(a.cnt + tsk[i].signal, 1ull);
        return;
    }
    if (warp == kNdWarpProducer) {  // TMA producer
        if (lane == 0) {
            // two cursors over this CTA's matrix chunks: the ring fill, and an L2
            // prefetch running pf chunks ahead of it (keeps HBM busy through dependency waits)
            int ti = 0, tr = 0, pi = 0, pr = 0, seq = 0, pseq = 0;
            NdTask Ti{}, Tp{};
            int ti_loaded = -1, pi_loaded = -1;
            auto next = [&](int& i, int& r, NdTask& T, int& loaded) -> bool {
                while (i < nt) {
                    if (loaded != i) {
                        T = tsk[i];
                        loaded = i;
                    }
                    if (r < T.nrows) return true;
                    ++i;
                    r = 0;
                }
                return false;
            };
            while (true) {
                while (pseq < seq + a.pf && next(pi, pr, Tp, pi_loaded)) {
                    const int rpc = static_cast<int>(a.stage_bytes / (8u * Tp.ld));
                    const unsigned bytes = static_cast<unsigned>(min(rpc, Tp.nrows - pr)) * Tp.ld * 8u;
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.store + Tp.src + (long long)pr * Tp.ld),
                                 "r"(bytes)
                                 : "memory");
                    pr += rpc;
                    ++pseq;
                }
                if (!next(ti, tr, Ti, ti_loaded)) break;
                const int rpc = static_cast<int>(a.stage_bytes / (8u * Ti.ld));
                const int k = seq % a.stages;
                if (seq >= a.stages) mbar_wait(&empty[k], static_cast<unsigned>(((seq / a.stages) - 1) & 1));
                const unsigned bytes = static_cast<unsigned>(min(rpc, Ti.nrows - tr)) * Ti.ld * 8u;
                mbar_arrive_expect_tx(&full[k], bytes);
                bulk_g2s(ring + (size_t)k * a.stage_bytes, a.store + Ti.src + (long long)tr * Ti.ld, bytes, &full[k]);
                tr += rpc;
                ++seq;
                if (pseq < seq) {  // prefetch cursor never behind the fill
                    pi = ti;
                    pr = tr;
                    pseq = seq;
                }
            }
        }
        return;
    }
    if (warp == kNdWarpSignal) {  // signaller
        if (lane == 0)
            for (int i = 0; i < nt; ++i) {
                const int q = i % kNdBufs;
                mbar_wait(&done[q], static_cast<unsigned>((i / kNdBufs) & 1));
                if (a.dbg) a.dbg[((size_t)(t0 + i)) * 4 + 3] = globaltimer();
                const int sig = tbT[q].signal;
                // the compute warps' outputs reach this thread through the done barrier (release /
                // acquire at CTA scope); the gpu-scope release below is cumulative over them.
                // PDG_ND_FENCE (debug): an explicit fence.acq_rel.gpu first
                if (a.fence) asm volatile("fence.acq_rel.gpu;" ::: "memory");
                red_release_add(a.cnt + sig, 1ull);
                if (a.dbg) a.dbg[((size_t)(t0 + i)) * 4 + 1] = globaltimer();
                mbar_arrive(&freeb[q]);
            }
        return;
    }
    constexpr int kB = 8;  // loads in flight per thread
    if (warp >= kNdWarpStage && warp < kNdWarpStage + kNdPrepWarps) {  // staging warps: task j = w mod kNdPrepWarps
        const int w = warp - kNdWarpStage;
        for (int j = w; j < nt; j += kNdPrepWarps) {
            const int q = j % kNdBufs;
            const NdTask& T = tsk[j];
            // the slot's previous task and the arena space (both released in task order;
            // fdep is monotone and <= j - 2, so this warp's waits never alias a barrier phase)
            const int wt = max(j - kNdBufs, T.fdep);
            if (wt >= 0) mbar_wait(&freeb[wt % kNdBufs], static_cast<unsigned>((wt / kNdBufs) & 1));
            const bool fresh = j == 0 || T.front != tsk[j - 1].front || T.type != tsk[j - 1].type;
            double* v = vbuf(T);
            int* oix = oixbuf(T);
            int* bix = bixbuf(T);
            const int vm = T.vmt;
            const int len = T.ncols, lp = T.ld;
            // output indices of the task's rows
            for (int r0 = lane; r0 < T.nrows; r0 += 32 * kB) {
                int o[kB];
#pragma unroll
                for (int u = 0; u < kB; ++u) {
                    const int r = r0 + u * 32, gr = T.r0 + r;
                    o[u] = r >= T.nrows ? 0
                                        : T.type == 2 ? a.sdofs[T.sdof + gr] : (gr >= T.s ? a.cbdst[T.bdof + gr - T.s] : 0);
                }
#pragma unroll
                for (int u = 0; u < kB; ++u)
                    if (r0 + u * 32 < T.nrows) oix[r0 + u * 32] = o[u];
            }
            if (fresh && T.type == 1) {  // b_S (and the padding)
                const int tot = lp * nr;
                for (int c0 = lane; c0 < tot; c0 += 32 * kB) {
                    int d[kB];
#pragma unroll
                    for (int u = 0; u < kB; ++u) {
                        const int c = c0 + u * 32, cc = c % lp;
                        d[u] = (c < tot && cc < len) ? a.sdofs[T.sdof + cc] : -1;
                    }
                    double x[kB];
#pragma unroll
                    for (int u = 0; u < kB; ++u) {
                        const int c = c0 + u * 32, k = c / lp;
                        x[u] = d[u] >= 0 ? a.b[k * a.ldb + d[u]] : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < kB; ++u) {
                        const int c = c0 + u * 32;
                        if (c < tot) v[(c / lp) * vm + c % lp] = x[u];
                    }
                }
            } else if (fresh) {  // backward: the boundary's pivot positions
                for (int c = lane; c < T.b; c += 32) bix[c] = a.bpos[T.bdof + c];
            }
            // a look at the dependency counters, after the other loads are issued
            // (monotone: once met, met for this call)
            int ok = 1;
            if (lane == 0) {
                if (!a.nodep) {
                    if (T.wait0 >= 0 && ld_acquire(a.cnt + T.wait0) < a.call * (unsigned long long)T.need0) ok = 0;
                    if (T.wait1 >= 0 && ld_acquire(a.cnt + T.wait1) < a.call * (unsigned long long)T.need1) ok = 0;
                }
                tbT[q] = T;
                tbOk[q] = ok | (fresh ? 2 : 0);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&staged[q]);
        }
        return;
    }
    if (warp >= kNdWarpGather && warp < kNdWarpGather + kNdGatherWarps) {  // gather warps, tasks in order
        const int gt = tid - kNdWarpGather * 32;
        for (int i = 0; i < nt; ++i) {
            const int q = i % kNdBufs, qp = (i + kNdBufs - 1) % kNdBufs;
            mbar_wait(&staged[q], static_cast<unsigned>((i / kNdBufs) & 1));
            const NdTask T = tbT[q];
            const int flags = tbOk[q];
            const bool fresh = flags & 2;
            double* v = vbuf(T);
            const int* bix = bixbuf(T);
            const int len = T.ncols, lp = T.ld, tot = lp * nr, vm = T.vmt;
            if (!fresh) {  // continuation of the previous task's front: the same input (same stride)
                const double* vprev = vbuf(tsk[i - 1]);
                for (int c = gt; c < vm * nr; c += kNdGatherThreads) v[c] = vprev[c];
            }
            // ---- the dependency wait ----
            if (gt == 0 && !a.nodep && !(flags & 1)) {
                if (T.wait0 >= 0) {
                    const unsigned long long tgt = a.call * (unsigned long long)T.need0;
                    while (ld_acquire(a.cnt + T.wait0) < tgt) {
                    }
                }
                if (T.wait1 >= 0) {
                    const unsigned long long tgt = a.call * (unsigned long long)T.need1;
                    while (ld_acquire(a.cnt + T.wait1) < tgt) {
                    }
                }
            }
            gather_sync();
            if (a.dbg && gt == 0) a.dbg[((size_t)(t0 + i)) * 4] = globaltimer();
            // ---- dependent inputs, one batch of loads ----
            if (T.type == 1 && !T.leaf) {
                const double* c0p = a.cb + T.cboff;
                const double* c1p = c0p + (T.s + T.b);
                // fresh: v[k][cc] -= c0 + c1 for cc < len; every task: the pass-through updates
                // c0 + c1 of its own boundary rows into the tail v[k][gr], gr in [max(r0, s), r0 + nrows)
                const int nf = fresh ? len * nr : 0;
                const int r_lo = max(T.r0, T.s), cnt = max(0, T.r0 + T.nrows - r_lo), tw = cnt * nr;
                for (int cb0 = gt; cb0 < nf + tw; cb0 += kNdGatherThreads * kB) {
                    double w1[kB], w2[kB];
                    int dst[kB];
#pragma unroll
                    for (int u = 0; u < kB; ++u) {
                        const int c = cb0 + u * kNdGatherThreads;
                        int k = 0, col = 0;
                        dst[u] = -1;
                        if (c < nf) {
                            k = c / len;
                            col = c % len;
                            dst[u] = k * vm + col;
                        } else if (c < nf + tw) {
                            const int e = c - nf;
                            k = e / cnt;
                            col = r_lo + e % cnt;
                            dst[u] = k * vm + col;
                        }
                        w1[u] = dst[u] >= 0 ? __ldcg(c0p + k * a.cbtot + col) : 0.0;
                        w2[u] = dst[u] >= 0 ? __ldcg(c1p + k * a.cbtot + col) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < kB; ++u) {
                        const int c = cb0 + u * kNdGatherThreads;
                        if (c < nf)
                            v[dst[u]] = v[dst[u]] - w1[u] - w2[u];
                        else if (c < nf + tw)
                            v[dst[u]] = w1[u] + w2[u];
                    }
                }
            } else if (T.type == 2 && fresh) {  // [y_S; -x_B]
                for (int cb0 = gt; cb0 < tot; cb0 += kNdGatherThreads * kB) {
                    double w[kB];
#pragma unroll
                    for (int u = 0; u < kB; ++u) {
                        const int c = cb0 + u * kNdGatherThreads, k = c / lp, cc = c % lp;
                        w[u] = 0.0;
                        if (c < tot && cc < len)
                            w[u] = cc < T.s ? __ldcg(a.y + (long long)k * a.n + T.sdof + cc)
                                            : -__ldcg(a.xpos + (long long)k * a.n + bix[cc - T.s]);
                    }
#pragma unroll
                    for (int u = 0; u < kB; ++u) {
                        const int c = cb0 + u * kNdGatherThreads;
                        if (c < tot) v[(c / lp) * vm + c % lp] = w[u];
                    }
                }
            }
            gather_sync();
            if (gt == 0) {
                if (a.dbg) a.dbg[((size_t)(t0 + i)) * 4 + 2] = globaltimer();
                mbar_arrive(&gathered[q]);
                if (i > 0) mbar_arrive(&freeb[qp]);  // the previous task's buffer is no longer read by the gather
            }
        }
        return;
    }
    // ---- compute warps: the matrix stream ----
    int seq = 0;  // chunks of this CTA's stream consumed so far (by all compute warps)
    for (int i = 0; i < nt; ++i) {
        const int q = i % kNdBufs;
        const NdTask& Ts = tsk[i];
        const int type = Ts.type, r0t = Ts.r0, nrows = Ts.nrows, ld = Ts.ld, s = Ts.s, sdof = Ts.sdof, leaf = Ts.leaf;
        const int rpc = static_cast<int>(a.stage_bytes / (8u * ld));
        const int nch = (nrows + rpc - 1) / rpc;
        // chunks of this task owned by this warp: seq + c with (seq + c) % 8 == warp
        // chunk owners: warp c % 8, or (pairs) the warp pair c % 4 with the chunk's row passes
        // alternating between the two warps (a consumer then has two ring slots in flight)
        const int ncons = a.pairs ? kNdComputeWarps / 2 : kNdComputeWarps;
        const int me = a.pairs ? warp >> 1 : warp, half = a.pairs ? (warp & 1) : 0, npart = a.pairs ? 2 : 1;
        const int first = (me - seq % ncons + ncons) % ncons;
        // every warp waits for every task's input, chunks or not: keeps the warps within one
        // phase of the gathered / done barriers (a warp skipping tasks could otherwise run a
        // full buffer cycle ahead and alias a barrier phase)
        mbar_wait(&gathered[q], static_cast<unsigned>((i / kNdBufs) & 1));
        if (first < nch) {
            const double* v = vbuf(Ts);
            const int* oix = oixbuf(Ts);
            const int vm = Ts.vmt;
            const double2* va = reinterpret_cast<const double2*>(v);
            const double2* vb = va + (vm >> 1);
            const int ld2 = ld >> 1;
            auto write_out = [&](int k, int lr, double t) {  // row lr of the task, rhs k
                const int gr = r0t + lr;
                if (type == 2) {
                    a.xpos[(long long)k * a.n + sdof + gr] = t;
                    a.x[k * a.ldx + oix[lr]] = t;
                } else if (gr < s) {
                    a.y[(long long)k * a.n + sdof + gr] = t;
                } else {  // update vector entry (+ the pass-through), into the parent's contribution slot
                    const double w = leaf ? 0.0 : v[k * vm + gr];
                    a.cb[k * a.cbtot + oix[lr]] = t + w;
                }
            };
            for (int c = first; c < nch; c += ncons) {
                const int sq = seq + c, rc = c * rpc;
                const int slot = sq % a.stages;
                // warps drift apart (no per-task barrier): before waiting for chunk sq to land, wait
                // until the slot's previous chunk (sq - stages) has been consumed, so a parity wait
                // can never see an older phase of the slot as this chunk's (needs stages >= 8: this
                // warp's previous chunk landed, so sq - stages was issued, so sq - 2 stages was consumed)
                if (sq >= a.stages) mbar_wait(&empty[slot], static_cast<unsigned>(((sq / a.stages) - 1) & 1));
                mbar_wait(&full[slot], static_cast<unsigned>((sq / a.stages) & 1));
                const double2* rows2 = reinterpret_cast<const double2*>(ring + (size_t)slot * a.stage_bytes);
                const int nrow = min(rpc, nrows - rc);
                if (a.nomath) {
                } else if (rpc >= 8 && !a.tile8) {
                    // rows per pass 4 R, with at least npart passes per chunk
                    auto o = [&](int k, int lr, double t) { write_out(k, rc + lr, t); };
                    if (rpc >= 16 * npart)
                        chunk_g8<4>(rows2, nrow, ld2, va, vb, lane, o, nr, half, npart);
                    else if (rpc >= 8 * npart)
                        chunk_g8<2>(rows2, nrow, ld2, va, vb, lane, o, nr, half, npart);
                    else
                        chunk_g8<1>(rows2, nrow, ld2, va, vb, lane, o, nr, half, npart);
                } else if (rpc >= 8) {
                    // narrow rows: groups of 8 rows share each input load, lanes over the
                    // columns, warp reduce-scatter of the 16 (row, rhs) sums (PDG_ND_TILE8)
                    for (int rb = 0; rb < nrow; rb += 8) {
                        const int rn = min(8, nrow - rb);
                        double acc[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) acc[j] = 0.0;
                        for (int c2 = lane; c2 < ld2; c2 += 32) {
                            const double2 pv = va[c2], qv = vb[c2];
#pragma unroll
                            for (int r = 0; r < 8; ++r) {
                                const double2 m = r < rn ? rows2[(size_t)(rb + r) * ld2 + c2] : make_double2(0.0, 0.0);
                                acc[2 * r] = fma(m.y, pv.y, fma(m.x, pv.x, acc[2 * r]));
                                acc[2 * r + 1] = fma(m.y, qv.y, fma(m.x, qv.x, acc[2 * r + 1]));
                            }
                        }
                        const double t = warp_reduce_scatter16(acc, lane);  // lane l < 16: row l/2, rhs l%2
                        const int r = lane >> 1, k = lane & 1;
                        if (lane < 16 && r < rn && k < nr) write_out(k, rc + rb + r, t);
                    }
                } else if (!a.tile8) {
                    // wide rows (fewer than 8 per chunk): R rows at a time over all 32 lanes
                    auto o = [&](int k, int lr, double t) { write_out(k, rc + lr, t); };
                    if (rpc >= 4 * npart)
                        chunk_wide<4>(rows2, nrow, ld2, va, vb, lane, o, nr, half, npart);
                    else if (rpc >= 2 * npart)
                        chunk_wide<2>(rows2, nrow, ld2, va, vb, lane, o, nr, half, npart);
                    else
                        chunk_wide<1>(rows2, nrow, ld2, va, vb, lane, o, nr, half, npart);
                } else {
                    // wide rows (fewer than 8 per chunk): two rows at a time, lanes over the
                    // columns, butterfly over the warp
                    for (int rb = 0; rb < nrow; rb += 2) {
                        const bool two = rb + 1 < nrow;
                        const double2* r0p = rows2 + (size_t)rb * ld2;
                        const double2* r1p = two ? r0p + ld2 : r0p;
                        double acc[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
                        for (int c2 = lane; c2 < ld2; c2 += 32) {
                            const double2 pv = va[c2], qv = vb[c2], m0 = r0p[c2], m1 = r1p[c2];
                            acc[0][0] = fma(m0.x, pv.x, acc[0][0]);
                            acc[0][1] = fma(m0.y, pv.y, acc[0][1]);
                            acc[0][2] = fma(m0.x, qv.x, acc[0][2]);
                            acc[0][3] = fma(m0.y, qv.y, acc[0][3]);
                            acc[1][0] = fma(m1.x, pv.x, acc[1][0]);
                            acc[1][1] = fma(m1.y, pv.y, acc[1][1]);
                            acc[1][2] = fma(m1.x, qv.x, acc[1][2]);
                            acc[1][3] = fma(m1.y, qv.y, acc[1][3]);
                        }
                        double t4[4] = {acc[0][0] + acc[0][1], acc[0][2] + acc[0][3], acc[1][0] + acc[1][1],
                                        acc[1][2] + acc[1][3]};
#pragma unroll
                        for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
                            for (int u = 0; u < 4; ++u) t4[u] += __shfl_xor_sync(0xffffffffu, t4[u], o);
                        // lane 2 r + k writes row rb + r, rhs k
                        const int r = lane >> 1, k = lane & 1;
                        if (lane < 4 && (r == 0 || two) && k < nr)
                            write_out(k, rc + rb + r, lane == 0 ? t4[0] : lane == 1 ? t4[1] : lane == 2 ? t4[2] : t4[3]);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[slot]);
            }
        }
        seq += nch;
        __syncwarp();
        if (lane == 0) mbar_arrive(&done[q]);  // this warp's outputs of task i written (or it had no chunk)
    }
}

}  // namespace

void NdChol::factor(int n_, const std::vector<int>& off, const std::vector<int>& idx, const std::vector<double>& val,
                    const std::vector<int>& node_of, const std::vector<double>& cx, const std::vector<double>& cy,
                    int leaf_dofs, int max_rhs_, cudaStream_t st, const std::vector<double>* cz) {
    n = n_;
    max_rhs = max_rhs_;
    const int stage0 = prof_phase == PROF_A_SOLVE ? SETUP_A_ANALYSIS : SETUP_F_ANALYSIS;
    SetupTimer timer(stage0, st);
    require(max_rhs >= 1 && max_rhs <= kNdMaxRhs, "nested dissection: at most 2 right-hand sides");
    require(static_cast<int>(off.size()) == n + 1 && static_cast<int>(node_of.size()) == n, "nested dissection: bad CSR");
    const int nn = static_cast<int>(cx.size());
    // ---- node graph ----
    std::vector<int> ndofs(nn, 0);
    for (int d = 0; d < n; ++d) {
        require(node_of[d] >= 0 && node_of[d] < nn, "nested dissection: bad node index");
        ++ndofs[node_of[d]];
    }
    std::vector<int> noff(nn + 1, 0), nlist(n);
    for (int u = 0; u < nn; ++u) noff[u + 1] = noff[u] + ndofs[u];
    {
        std::vector<int> fill(noff.begin(), noff.end() - 1);
        for (int d = 0; d < n; ++d) nlist[fill[node_of[d]]++] = d;
    }
    std::vector<int> aoff(nn + 1, 0), adj;
    {
        // one pass over the nonzeros, a neighbour recorded the first time a node's rows meet it
        std::vector<int> mark(nn, -1);
        for (int u = 0; u < nn; ++u) {
            const size_t start = adj.size();
            for (int q = noff[u]; q < noff[u + 1]; ++q) {
                const int d = nlist[q];
                for (int k = off[d]; k < off[d + 1]; ++k) {
                    const int e = node_of[idx[k]];
                    if (e != u && mark[e] != u) {
                        mark[e] = u;
                        adj.push_back(e);
                    }
                }
            }
            std::sort(adj.begin() + start, adj.end());
            aoff[u + 1] = static_cast<int>(adj.size());
        }
    }
    // ---- dissection ----
    Dissector ds(aoff, adj, ndofs, cx, cy, cz, leaf_dofs);
    {
        std::vector<int> all(nn);
        std::iota(all.begin(), all.end(), 0);
        ds.build(std::move(all), -1, 0);
    }
    for (int u = 0; u < nn; ++u) require(ds.node_front[u] >= 0, "nested dissection: unassigned node");
    const int nf = static_cast<int>(ds.fr.size());
    nfront = nf;
    maxdepth = 0;
    for (auto& f : ds.fr) maxdepth = std::max(maxdepth, f.depth);
    // final order: deepest first (children before parents), stable in build order
    std::vector<int> order(nf);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return ds.fr[a].depth > ds.fr[b].depth; });
    std::vector<int> newid(nf);
    for (int k = 0; k < nf; ++k) newid[order[k]] = k;
    // dof lists
    std::vector<int> hs, hb;
    std::vector<int> front_of(n, -1), spos(n, -1);
    fronts.assign(nf, NdFront{});
    std::vector<std::vector<int>> children(nf);
    std::vector<int> parent(nf, -1);
    for (int k = 0; k < nf; ++k) {
        const HostFront& h = ds.fr[order[k]];
        NdFront& F = fronts[k];
        std::vector<int> sd, bd;
        for (int u : h.snodes) sd.insert(sd.end(), nlist.begin() + noff[u], nlist.begin() + noff[u + 1]);
        for (int u : h.bnodes) bd.insert(bd.end(), nlist.begin() + noff[u], nlist.begin() + noff[u + 1]);
        std::sort(sd.begin(), sd.end());
        std::sort(bd.begin(), bd.end());
        F.s = static_cast<int>(sd.size());
        F.b = static_cast<int>(bd.size());
        F.sdof = static_cast<int>(hs.size());
        F.bdof = static_cast<int>(hb.size());
        F.depth = h.depth;
        for (int i = 0; i < F.s; ++i) {
            front_of[sd[i]] = k;
            spos[sd[i]] = F.sdof + i;
        }
        hs.insert(hs.end(), sd.begin(), sd.end());
        hb.insert(hb.end(), bd.begin(), bd.end());
        parent[k] = h.parent < 0 ? -1 : newid[h.parent];
        for (int c : h.children) children[k].push_back(newid[c]);
    }
    require(static_cast<int>(hs.size()) == n, "nested dissection: pivots do not cover the matrix");
    // dense top (nd_top.cu): the deepest front level it covers, lowered until |T| fits
    top_depth = std::min(nd_top_default(prof_phase), maxdepth - 1);
    while (top_depth >= 0) {
        long long nt = 0;
        for (const auto& F : fronts)
            if (F.depth <= top_depth) nt += F.s;
        if (nt <= nd_top_cap()) break;
        --top_depth;
    }
    // contribution buffers: front F holds [child q][s + b] (per right-hand side); the
    // update vector w_C of child q of F (its boundary rows: u_C plus the pass-through
    // of C's own children) is written by C's forward tasks straight into F's slot q at
    // F's local positions, so F's forward reads contiguous inputs after its wait
    cbtot = 0;
    for (auto& F : fronts) {
        F.cboff = static_cast<int>(cbtot);
        cbtot += 2LL * (F.s + F.b);
    }
    require(cbtot < (1LL << 31), "nested dissection: contribution buffer too large");
    const long long nbt = static_cast<long long>(hb.size());
    std::vector<int> hcbdst(std::max<long long>(nbt, 1), -1);
    {
        std::vector<int> lc(n, -1);
        for (int k = 0; k < nf; ++k) {
            const NdFront& F = fronts[k];
            for (int i = 0; i < F.s; ++i) lc[hs[F.sdof + i]] = i;
            for (int i = 0; i < F.b; ++i) lc[hb[F.bdof + i]] = F.s + i;
            require(children[k].size() <= 2, "nested dissection: more than two children");
            for (size_t q = 0; q < children[k].size(); ++q) {
                const NdFront& C = fronts[children[k][q]];
                for (int i = 0; i < C.b; ++i) {
                    const int l = lc[hb[C.bdof + i]];
                    require(l >= 0, "nested dissection: child boundary outside the parent front");
                    hcbdst[C.bdof + i] = F.cboff + static_cast<int>(q) * (F.s + F.b) + l;
                }
            }
            for (int i = 0; i < F.s; ++i) lc[hs[F.sdof + i]] = -1;
            for (int i = 0; i < F.b; ++i) lc[hb[F.bdof + i]] = -1;
        }
        for (long long i = 0; i < nbt; ++i) require(hcbdst[i] >= 0, "nested dissection: boundary entry without a parent slot");
    }
    // ---- storage layout ----
    long long so = 0;
    factor_bytes = 0.0;
    vmax = 0;
    for (auto& F : fronts) {
        // rows start on 16-byte boundaries: even lengths in fp64, multiples of 4 for an fp32 store
        F.ldm = static_cast<int>(fp32_req ? (F.s + 3LL) & ~3LL : round2(F.s));
        F.ldt = static_cast<int>(fp32_req ? (F.s + F.b + 3LL) & ~3LL : round2(F.s + F.b));
        F.moff = so;
        so += (long long)(F.s + F.b) * F.ldm;
        F.mtoff = so;
        so += (long long)F.s * F.ldt;
        factor_bytes += 8.0 * ((double)(F.s + F.b) * F.s * 2.0);
        vmax = std::max(vmax, F.ldt);
    }
    // ---- numeric factorization (multifrontal, stream-serial, children first) ----
    std::vector<long long> fo(nf);
    long long ftot = 0, sbmax = 1;
    int smax = 1, bmax = 1;
    for (int k = 0; k < nf; ++k) {
        const long long f = fronts[k].s + fronts[k].b;
        fo[k] = ftot;
        ftot += f * f;
        smax = std::max(smax, fronts[k].s);
        bmax = std::max(bmax, fronts[k].b);
        sbmax = std::max(sbmax, (long long)fronts[k].s * fronts[k].b);
    }
    // streaming mode (nd_stream.cu): wide fronts (the level kernels hold a front's input vector,
    // s + b doubles per right-hand side plus index lists, in shared memory) or more than 8 GB of
    // dense fronts (3D meshes)
    stream = vmax > 10000 || 8.0 * (double)ftot > 8e9;
    if (const char* e = std::getenv("PDG_ND_STREAM")) stream = std::atoi(e) != 0;
    if (stream) {
        top_depth = -1;
        for (auto& o : fo) o = 0;  // front-relative positions: every front has its own allocation
    }
    fp32 = fp32_req && stream;
    if (fp32)
        store32.alloc((size_t)so);
    else
        store.alloc((size_t)so);
    DBuf<double> dense(stream ? 1 : ftot);
    dense.zero(st);
    std::vector<long long> tstart(nf + 1, 0);  // streaming: the scatter entries of front k
    std::vector<int> loc(n, -1);
    DBuf<long long> dpos;
    DBuf<double> dval;
    {
        std::vector<long long> tpos;
        std::vector<double> tval;
        tpos.reserve(idx.size() / 2 + n);  // the lower triangle
        tval.reserve(idx.size() / 2 + n);
        for (int k = 0; k < nf; ++k) {
            const NdFront& F = fronts[k];
            const long long f = F.s + F.b;
            for (int i = 0; i < F.s; ++i) loc[hs[F.sdof + i]] = i;
            for (int i = 0; i < F.b; ++i) loc[hb[F.bdof + i]] = F.s + i;
            for (int i = 0; i < F.s; ++i) {
                const int d = hs[F.sdof + i];
                for (int q = off[d]; q < off[d + 1]; ++q) {
                    const int lj = loc[idx[q]];
                    if (lj >= i) {
                        tpos.push_back(fo[k] + lj + (long long)i * f);
                        tval.push_back(val[q]);
                    }
                }
            }
            for (int i = 0; i < F.s; ++i) loc[hs[F.sdof + i]] = -1;
            for (int i = 0; i < F.b; ++i) loc[hb[F.bdof + i]] = -1;
            tstart[k + 1] = static_cast<long long>(tpos.size());
        }
        dpos.upload(tpos, st);
        dval.upload(tval, st);
        if (!stream) {
            k_nd_scatter<<<grid_for((long long)tpos.size(), 256), 256, 0, st>>>((long long)tpos.size(), dpos.p, dval.p,
                                                                               dense.p);
            PDG_CHECK_LAUNCH();
        }
        PDG_CUDA(cudaStreamSynchronize(st));
    }
    // extend-add maps
    std::vector<int> hmap;
    std::vector<long long> mapoff(nf, 0);
    for (int k = 0; k < nf; ++k) {
        const NdFront& P = fronts[k];
        for (int i = 0; i < P.s; ++i) loc[hs[P.sdof + i]] = i;
        for (int i = 0; i < P.b; ++i) loc[hb[P.bdof + i]] = P.s + i;
        for (int c : children[k]) {
            mapoff[c] = static_cast<long long>(hmap.size());
            for (int i = 0; i < fronts[c].b; ++i) {
                const int l = loc[hb[fronts[c].bdof + i]];
                require(l >= 0, "nested dissection: child boundary outside the parent front");
                hmap.push_back(l);
            }
        }
        for (int i = 0; i < P.s; ++i) loc[hs[P.sdof + i]] = -1;
        for (int i = 0; i < P.b; ++i) loc[hb[P.bdof + i]] = -1;
    }
    DBuf<int> dmap;
    dmap.upload(hmap, st);
    timer.next(stage0 + 1);  // numeric factorization
    LaHandles h(st);
    int lwork = 0;
    PDG_ND_CUSOLVER(cusolverDnDpotrf_bufferSize(h.solver, CUBLAS_FILL_MODE_LOWER, smax, dense.p, smax, &lwork));
    DBuf<double> work(std::max(lwork, 1)), T((size_t)smax * smax), G(stream ? (size_t)sbmax : (size_t)smax * bmax);
    DBuf<int> info(nf);
    info.zero(st);
    const double one = 1.0, mone = -1.0, zero = 0.0;
    // processing order: by index (deepest level first), or in streaming mode the postorder of the
    // tree, so that only the update matrices on the current root path are alive
    std::vector<int> porder;
    std::vector<double*> fptr(nf, nullptr);
    if (stream) {
        std::vector<std::pair<int, size_t>> stk;
        for (int k = 0; k < nf; ++k)
            if (parent[k] < 0) stk.push_back({k, 0});
        while (!stk.empty()) {
            auto& [k, ci] = stk.back();
            if (ci < children[k].size()) {
                const int c = children[k][ci++];
                stk.push_back({c, 0});
            } else {
                porder.push_back(k);
                stk.pop_back();
            }
        }
        cudaMemPool_t pool;
        int dev = 0;
        PDG_CUDA(cudaGetDevice(&dev));
        PDG_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
        unsigned long long keep = ~0ULL;  // reuse freed front matrices instead of returning them to the driver
        PDG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    } else {
        porder.resize(nf);
        std::iota(porder.begin(), porder.end(), 0);
    }
    // levels of many small fronts: one batched launch per level (k_nd_factor_batch); the few
    // large fronts near the root (and everything in streaming mode) go through cuSOLVER / cuBLAS
    std::vector<char> batched(nf, 0);
    std::vector<int> level_first(maxdepth + 2, -1), level_count(maxdepth + 2, 0);
    bool batch_on = !stream;
    if (const char* e = std::getenv("PDG_ND_FACTOR_BATCH")) batch_on = batch_on && std::atoi(e) != 0;
    for (int k = 0; k < nf; ++k) {
        const int d = fronts[k].depth;
        if (level_first[d] < 0) level_first[d] = k;
        ++level_count[d];
    }
    DBuf<NdFactorDesc> d_descs;
    if (batch_on) {
        std::vector<NdFactorDesc> descs;
        std::vector<int> level_desc0(maxdepth + 2, 0);
        for (int d = maxdepth; d >= 0; --d) {
            level_desc0[d] = static_cast<int>(descs.size());
            int fmax = 0;
            for (int k = level_first[d]; k >= 0 && k < level_first[d] + level_count[d]; ++k)
                fmax = std::max(fmax, fronts[k].s + fronts[k].b);
            if (level_count[d] < 32 || fmax > 1536) continue;
            // one CTA per front pays while its rank-1 updates (~1.45 ns per 1000 s f^2, measured at
            // config 1: 6 / 26 / 50 ms for the levels of 128 / 64 / 32 fronts) stay below the
            // library path's ~0.25 ms of launches per front (PDG_ND_FACTOR_BATCH_COST=0: always batch)
            {
                double sf2 = 0.0;
                for (int k = level_first[d]; k < level_first[d] + level_count[d]; ++k) {
                    const double f = fronts[k].s + fronts[k].b;
                    sf2 = std::max(sf2, fronts[k].s * f * f);
                }
                const bool cost_rule = !(std::getenv("PDG_ND_FACTOR_BATCH_COST") && std::atoi(std::getenv("PDG_ND_FACTOR_BATCH_COST")) == 0);
                const double waves = std::ceil(level_count[d] / 148.0);
                if (cost_rule && 1.45e-9 * sf2 * waves > 0.25e-3 * level_count[d]) continue;
            }
            for (int k = level_first[d]; k < level_first[d] + level_count[d]; ++k) {
                require(fronts[k].depth == d, "nested dissection: fronts of a level are not contiguous");
                NdFactorDesc D{};
                D.fo = fo[k];
                D.moff = fronts[k].moff;
                D.mtoff = fronts[k].mtoff;
                D.s = fronts[k].s;
                D.b = fronts[k].b;
                D.ldm = fronts[k].ldm;
                D.ldt = fronts[k].ldt;
                D.front = k;
                D.nchild = 0;
                for (int c : children[k]) {
                    if (fronts[c].b == 0) continue;
                    D.cfo[D.nchild] = fo[c];
                    D.cmap[D.nchild] = mapoff[c];
                    D.cs[D.nchild] = fronts[c].s;
                    D.cb[D.nchild] = fronts[c].b;
                    ++D.nchild;
                }
                descs.push_back(D);
                batched[k] = 1;
            }
        }
        d_descs.upload(descs, st);
        // launches happen in the loop below, when the level's first front comes up
        for (int d = 0; d <= maxdepth; ++d)
            if (level_first[d] >= 0 && batched[level_first[d]]) level_first[d] = -2 - level_desc0[d];
    }
    // PDG_ND_FACTOR_TIMING: host-synchronised time and flops per library call type (diagnostic)
    const bool ftime = std::getenv("PDG_ND_FACTOR_TIMING") != nullptr;
    double fsec[6] = {0, 0, 0, 0, 0, 0}, fflop[6] = {0, 0, 0, 0, 0, 0};
    std::chrono::steady_clock::time_point ft0;
    auto tick = [&](int which, double flops = 0.0) {
        if (!ftime) return;
        cudaStreamSynchronize(st);
        const auto now = std::chrono::steady_clock::now();
        if (which >= 0) {
            fsec[which] += std::chrono::duration<double>(now - ft0).count();
            fflop[which] += flops;
        }
        ft0 = now;
    };
    for (int k : porder) {
        const NdFront& F = fronts[k];
        const int s = F.s, b = F.b, f = s + b;
        if (batched[k]) {
            const int d = F.depth;
            if (level_first[d] <= -2) {  // first front of a batched level: the whole level in one launch
                const int d0 = -2 - level_first[d];
                tick(-1);
                k_nd_factor_batch<<<level_count[d], kFactorThreads, 0, st>>>(d_descs.p + d0, dense.p, dmap.p, store.p, info.p);
                PDG_CHECK_LAUNCH();
                if (ftime) {
                    tick(5);
                    std::fprintf(stderr, "nd factor batched level depth %d: %d fronts (s %d b %d), cumulative %.4f s\n", d, level_count[d],
                                 F.s, F.b, fsec[5]);
                }
                level_first[d] = -1;
            }
            continue;
        }
        double* Fk = dense.p + fo[k];
        if (stream) {
            PDG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&Fk), sizeof(double) * (size_t)f * f, st));
            fptr[k] = Fk;
            PDG_CUDA(cudaMemsetAsync(Fk, 0, sizeof(double) * (size_t)f * f, st));
            const long long cnt = tstart[k + 1] - tstart[k];
            if (cnt > 0) {
                k_nd_scatter<<<grid_for(cnt, 256), 256, 0, st>>>(cnt, dpos.p + tstart[k], dval.p + tstart[k], Fk);
                PDG_CHECK_LAUNCH();
            }
        }
        for (int c : children[k]) {
            const NdFront& C = fronts[c];
            const int fc = C.s + C.b;
            const double* Fc = stream ? fptr[c] : dense.p + fo[c];
            if (C.b > 0) {
                k_nd_extend_add<<<grid_for((long long)C.b * C.b, 256), 256, 0, st>>>(
                    Fk, f, Fc + C.s + (long long)C.s * fc, fc, C.b, dmap.p + mapoff[c]);
                PDG_CHECK_LAUNCH();
            }
            if (stream) {
                PDG_CUDA(cudaFreeAsync(fptr[c], st));
                fptr[c] = nullptr;
            }
        }
        tick(-1);
        PDG_ND_CUSOLVER(cusolverDnDpotrf(h.solver, CUBLAS_FILL_MODE_LOWER, s, Fk, f, work.p, lwork, info.p + k));
        tick(0, (double)s * s * s / 3.0);
        if (b > 0) {
            PDG_ND_CUBLAS(cublasDtrsm(h.blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T,
                                      CUBLAS_DIAG_NON_UNIT, b, s, &one, Fk, f, Fk + s, f));
            tick(1, (double)b * s * s);
            PDG_ND_CUBLAS(cublasDsyrk(h.blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, b, s, &mone, Fk + s, f, &one,
                                      Fk + s + (long long)s * f, f));
            tick(2, (double)b * b * s);
        }
        k_nd_identity<<<grid_for((long long)s * s, 256), 256, 0, st>>>(s, T.p);
        PDG_CHECK_LAUNCH();
        PDG_ND_CUBLAS(cublasDtrsm(h.blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT,
                                  s, s, &one, Fk, f, T.p, s));
        tick(3, (double)s * s * s);
        if (b > 0)
            PDG_ND_CUBLAS(cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, b, s, s, &one, Fk + s, f, T.p, s, &zero, G.p, b));
        tick(4, 2.0 * b * s * s);
        if (fp32)
            k_nd_pack<float><<<grid_for((long long)f * F.ldm, 256), 256, 0, st>>>(s, b, T.p, G.p, store32.p + F.moff, F.ldm,
                                                                                 store32.p + F.mtoff, F.ldt);
        else
            k_nd_pack<double><<<grid_for((long long)f * F.ldm, 256), 256, 0, st>>>(s, b, T.p, G.p, store.p + F.moff, F.ldm,
                                                                                  store.p + F.mtoff, F.ldt);
        PDG_CHECK_LAUNCH();
        tick(5);
    }
    if (ftime) {
        const char* nm[6] = {"potrf", "trsm L_BS", "syrk", "trsm L^-1", "gemm G", "alloc/scatter/extend-add/pack"};
        for (int i = 0; i < 6; ++i)
            std::fprintf(stderr, "nd factor %-30s %8.3f s %9.2f TFLOP %7.2f TFLOP/s\n", nm[i], fsec[i], fflop[i] / 1e12,
                         fsec[i] > 0 ? fflop[i] / fsec[i] / 1e12 : 0.0);
    }
    if (stream) {  // the roots' front matrices, then the pool's cached blocks back to the driver
        for (int k = 0; k < nf; ++k)
            if (fptr[k]) PDG_CUDA(cudaFreeAsync(fptr[k], st));
        PDG_CUDA(cudaStreamSynchronize(st));
        cudaMemPool_t pool;
        int dev = 0;
        PDG_CUDA(cudaGetDevice(&dev));
        PDG_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
        PDG_CUDA(cudaMemPoolTrimTo(pool, 0));
    }
    std::vector<int> hinfo(nf);
    PDG_CUDA(cudaMemcpyAsync(hinfo.data(), info.p, sizeof(int) * nf, cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    for (int k = 0; k < nf; ++k)
        if (hinfo[k] != 0) throw Error(PDG_NOT_CONVERGED, "nested dissection: front " + std::to_string(k) + " not positive definite");
    timer.next(stage0 + 2);  // solve schedule
    // boundary dofs as pivot positions; buffers shared by both solve kernels
    std::vector<int> hbp(hb.size());
    for (size_t i = 0; i < hb.size(); ++i) hbp[i] = spos[hb[i]];
    sdofs.upload(hs, st);
    bpos.upload(hbp, st);
    cbdst.upload(hcbdst, st);
    counters.alloc((size_t)3 * nf);
    counters.zero(st);
    call = 0;
    y.alloc((size_t)n * max_rhs);
    xpos.alloc((size_t)n * max_rhs);
    cbuf.alloc((size_t)std::max<long long>(cbtot, 1) * max_rhs);
    cbuf.zero(st);  // slots no child writes stay zero
    if (stream) {
        tiles = levels = hybrid = split = false;
        build_stream(st);
        return;
    }
    tiles = nd_tile_default();
    levels = nd_levels_default();
    if (tiles && !levels) top_depth = -1;  // the opt-in dataflow tile kernel solves every front
    if (top_depth >= 0) build_top(hbp, children, fo, dense.p, h, st);
    lvl_min_depth = top_depth + 1;
    if (tiles) {
        build_tiles(children, parent, hs, hbp, hcbdst, st);
        store.release();  // the tile store replaces the row-major one
        return;
    }
    // ---- solve schedule: tasks in topological order, contiguous per phase on the CTAs ----
    // (wide fronts of large meshes do not fit the ring / arena of this kernel: the
    // level-synchronous tile kernels, which stream tiles from global memory, take over)
    auto schedule_chunks = [&]() {
        int dev = 0, nsm = 0;
        PDG_CUDA(cudaGetDevice(&dev));
        PDG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        int task_chunks = 16;
        // no L2 prefetch cursor by default: measured 278 vs 291 us (pf 16) for the config-1
        // displacement solve (tools/nd_sweep.sh, profiles/round2_nd_sweeps.txt)
        pf = 0;
        if (const char* e = std::getenv("PDG_ND_PF")) pf = std::max(0, std::atoi(e));
        if (const char* e = std::getenv("PDG_ND_CHUNKS")) task_chunks = std::max(1, std::atoi(e));
        stages = 16;
        // 16 KB stages for wide fronts (rows of up to 8 KB: more rows per chunk), 12 KB otherwise
        stage_bytes = static_cast<unsigned>(std::max<long long>(vmax >= 1024 ? 16384 : 12288, ((long long)vmax * 8 + 1023) / 1024 * 1024));
        if (const char* e = std::getenv("PDG_ND_STAGES")) stages = std::min(32, std::max(2, std::atoi(e)));
        if (const char* e = std::getenv("PDG_ND_STAGE_KB")) stage_bytes = 1024u * std::max(8, std::atoi(e));
        int ctas_per_sm = PDG_ND_MINB;
        if (const char* e = std::getenv("PDG_ND_CTAS")) ctas_per_sm = std::max(1, std::atoi(e));
        grid = nsm * ctas_per_sm;
        std::vector<int> fwd_tasks(nf, 0), bwd_tasks(nf, 0);
        std::vector<bool> leaf(nf);
        for (int k = 0; k < nf; ++k) leaf[k] = children[k].empty();
        std::vector<std::vector<NdTask>> per_cta(grid);
        auto place = [&](std::vector<NdTask>& ts) {
            double wsum = 0.0;
            for (const auto& t : ts) wsum += 8.0 * t.nrows * t.ld + 64.0 * t.ld;
            double acc = 0.0;
            for (const auto& t : ts) {
                const double w = 8.0 * t.nrows * t.ld + 64.0 * t.ld;
                int q = static_cast<int>((acc + 0.5 * w) / wsum * grid);
                q = std::min(std::max(q, 0), grid - 1);
                per_cta[q].push_back(t);
                acc += w;
            }
        };
        auto base_task = [&](int k, int type) {
            const NdFront& F = fronts[k];
            NdTask t{};
            t.type = type;
            t.front = k;
            t.s = F.s;
            t.b = F.b;
            t.sdof = F.sdof;
            t.bdof = F.bdof;
            t.cboff = F.cboff;
            t.wait0 = t.wait1 = -1;
            t.need0 = t.need1 = 0;
            t.leaf = leaf[k] ? 1 : 0;
            return t;
        };
        auto level_bytes = [&](int type, int depth) {
            double by = 0.0;
            for (const auto& F : fronts)
                if (F.depth == depth) by += 8.0 * (type == 1 ? (double)(F.s + F.b) * F.ldm : (double)F.s * F.ldt);
            return by;
        };
        // subtree mapping: the fronts at depth >= local_depth form subtrees that run entirely on one
        // CTA each (their dependencies stay inside the CTA, in task order); the levels above are
        // spread over all CTAs. Default: the deepest level with no more fronts than CTAs.
        int local_depth = maxdepth + 1;
        {
            std::vector<int> per_depth(maxdepth + 1, 0);
            for (const auto& F : fronts) per_depth[F.depth]++;
            for (int d = maxdepth; d >= 0; --d)
                if (per_depth[d] <= grid) {
                    local_depth = d;
                    break;
                }
            if (const char* e = std::getenv("PDG_ND_LOCAL_DEPTH")) {
                const int v = std::atoi(e);
                local_depth = v < 0 ? maxdepth + 1 : std::min(v, maxdepth + 1);
            }
        }
        std::vector<int> cta_of(nf, -1);  // CTA of a local front
        {
            std::vector<int> roots;
            for (int k = 0; k < nf; ++k)
                if (fronts[k].depth == local_depth) roots.push_back(k);
            const int nr = static_cast<int>(roots.size());
            // PDG_ND_SPLIT_LOCAL: a local subtree on two CTAs (the root and its first child's subtree
            // on one, the second child's subtree on the other) when the grid has room for it
            const bool split_local = std::getenv("PDG_ND_SPLIT_LOCAL") && std::atoi(std::getenv("PDG_ND_SPLIT_LOCAL")) && 2 * nr <= grid;
            const int slots = split_local ? grid / 2 : grid;
            for (int j = 0; j < nr; ++j)
                cta_of[roots[j]] = (split_local ? 2 : 1) * static_cast<int>((long long)j * slots / std::max(nr, 1));
            for (int d = local_depth + 1; d <= maxdepth; ++d)
                for (int k = 0; k < nf; ++k)
                    if (fronts[k].depth == d && parent[k] >= 0) {
                        const int pk = parent[k];
                        const bool second = split_local && d == local_depth + 1 && children[pk].size() > 1 && children[pk][1] == k;
                        cta_of[k] = cta_of[pk] + (second ? 1 : 0);
                    }
        }
        auto matrix_tasks = [&](int type, int depth) {
            std::vector<NdTask> ts;
            for (int k = 0; k < nf; ++k) {
                const NdFront& F = fronts[k];
                if (F.depth != depth) continue;
                const int rows = type == 1 ? F.s + F.b : F.s;
                const int ld = type == 1 ? F.ldm : F.ldt;
                const long long base = type == 1 ? F.moff : F.mtoff;
                const int rpc = std::max(1, static_cast<int>(stage_bytes / (8u * ld)));  // (fronts outside this kernel may be wider)
                // balanced over the CTAs: about level bytes / grid per task, 1..task_chunks chunks;
                // a local front (one CTA runs its whole subtree) in as few tasks as the buffers allow
                const int want = static_cast<int>(std::ceil(level_bytes(type, depth) / grid / stage_bytes));
                const int cap = depth >= local_depth ? kNdMaxTaskRows
                                                     : std::min(kNdMaxTaskRows, rpc * std::max(1, std::min(task_chunks, want)));
                for (int r0 = 0; r0 < rows; r0 += cap) {
                    NdTask t = base_task(k, type);
                    t.src = base + (long long)r0 * ld;
                    t.r0 = r0;
                    t.nrows = std::min(cap, rows - r0);
                    t.ld = ld;
                    t.ncols = type == 1 ? F.s : F.s + F.b;
                    t.signal = 3 * k + type;
                    ts.push_back(t);
                    (type == 1 ? fwd_tasks : bwd_tasks)[k]++;
                }
            }
            return ts;
        };
        std::vector<std::vector<NdTask>> fwd_by_depth(maxdepth + 1), bwd_by_depth(maxdepth + 1);
        for (int d = maxdepth; d >= 0; --d) fwd_by_depth[d] = matrix_tasks(1, d);
        for (int d = 0; d <= maxdepth; ++d) bwd_by_depth[d] = matrix_tasks(2, d);
        // dependencies: forward after both children's forward, backward after the parent's backward
        for (auto& v : fwd_by_depth)
            for (auto& t : v) {
                const auto& ch = children[t.front];
                if (ch.size() > 0) {
                    t.wait0 = 3 * ch[0] + 1;
                    t.need0 = fwd_tasks[ch[0]];
                }
                if (ch.size() > 1) {
                    t.wait1 = 3 * ch[1] + 1;
                    t.need1 = fwd_tasks[ch[1]];
                }
            }
        for (auto& v : bwd_by_depth)
            for (auto& t : v) {
                const int p = parent[t.front];
                if (p >= 0) {
                    t.wait0 = 3 * p + 2;
                    t.need0 = bwd_tasks[p];
                } else {
                    t.wait0 = 3 * t.front + 1;
                    t.need0 = fwd_tasks[t.front];
                }
            }
        auto place_local = [&](std::vector<NdTask>& ts) {
            for (const auto& t : ts) per_cta[cta_of[t.front]].push_back(t);
        };
        // hybrid (PDG_ND_HYBRID): this kernel runs the local subtrees only, as two launches
        // (forward, backward); the levels above run as level kernels in between (nd_tile.cu)
        // with a dense top (top_depth >= 0) the fronts of depth <= top_depth get no tasks
        hybrid = local_depth > 0 && local_depth <= maxdepth && nd_hybrid_default(prof_phase) &&
                 local_depth - 1 > top_depth;
        hybrid_top = local_depth - 1;
        split = hybrid || top_depth >= 0;
        auto in_chunks = [&](int d) { return d > top_depth && (d >= local_depth || !hybrid); };
        for (const auto& F : fronts)
            if (in_chunks(F.depth)) require((long long)F.ldt * 8 <= stage_bytes, "nested dissection: front wider than a ring stage");
        std::vector<std::vector<NdTask>> per_cta_b(split ? grid : 0);
        for (int d = maxdepth; d >= 0; --d) {
            if (!in_chunks(d)) continue;
            if (d >= local_depth)
                place_local(fwd_by_depth[d]);
            else
                place(fwd_by_depth[d]);
        }
        if (split) per_cta.swap(per_cta_b);  // per_cta_b: forward schedule, per_cta: backward
        if (split) per_cta.assign(grid, {});
        for (int d = 0; d <= maxdepth; ++d) {
            if (!in_chunks(d)) continue;
            if (d >= local_depth)
                place_local(bwd_by_depth[d]);
            else
                place(bwd_by_depth[d]);
        }
        if (split) {
            per_cta.swap(per_cta_b);  // per_cta: forward, per_cta_b: backward
            // backward tasks whose parent is solved outside this launch (level kernels, dense
            // top, or none): their inputs are complete in stream order
            for (auto& v : per_cta_b)
                for (auto& t : v) {
                    const int p = parent[t.front];
                    if (p < 0 || !in_chunks(fronts[p].depth)) t.wait0 = -1;
                }
        }
        max_tasks = 0;
        size_t max_buf = 0;
        for (auto* lists : {&per_cta, &per_cta_b})
            for (auto& v : *lists) {
                max_tasks = std::max(max_tasks, static_cast<int>(v.size()));
                for (auto& t : v) {
                    t.vmt = nd_task_vmt(t);
                    max_buf = std::max(max_buf, nd_task_buf_bytes(t));
                }
            }
        static_assert((sizeof(NdTask) + sizeof(int)) * kNdBufs <= kNdHeader - 1024, "task descriptors do not fit the header");
        // shared memory: header, task list, TMA ring, and the buffer arena (at least three of the
        // largest task buffers, so a task's buffer never waits on the previous task's)
        // descriptors in shared memory only up to 12 KB (config 1: 49 tasks = 4.7 KB); beyond it
        // (large meshes) the kernel reads them from global memory
        if (nd_task_bytes(max_tasks) > 12 * 1024 || std::getenv("PDG_ND_TASKS_GLOBAL")) smem_tasks = 0;
        else smem_tasks = max_tasks;
        const size_t fixed = kNdHeader + nd_task_bytes(smem_tasks);
        size_t arena_min = std::max<size_t>(3 * max_buf, 48 * 1024);
        if (const char* e = std::getenv("PDG_ND_ARENA_KB")) arena_min = 1024 * (size_t)std::max(16, std::atoi(e));
        const size_t smem_cap = ctas_per_sm == 1 ? 227 * 1024 : (228 * 1024 / ctas_per_sm - 1024) / 128 * 128;
        require(fixed + arena_min + 2 * (size_t)stage_bytes <= smem_cap, "nested dissection: ring does not fit in shared memory");
        stages = std::min<int>(stages, static_cast<int>((smem_cap - fixed - arena_min) / stage_bytes));
        require(stages >= kNdComputeWarps, "nested dissection: ring shallower than the compute warps (stage size too large)");
        const size_t arena = (smem_cap - fixed - (size_t)stages * stage_bytes) / 128 * 128;
        arena_bytes = arena;
        max_task_buf = max_buf;
        smem = fixed + (size_t)stages * stage_bytes + arena;
        // FIFO placement of the task buffers in the arena (tasks run and release in order)
        for (auto& v : per_cta_b) per_cta.push_back(std::move(v));  // placed like the others, split below
        for (auto& v : per_cta) {
            size_t head = 0;
            int prev_dep = -1;
            for (int j = 0; j < static_cast<int>(v.size()); ++j) {
                const size_t sz = nd_task_buf_bytes(v[j]);
                if (head + sz > arena) head = 0;
                v[j].boff = static_cast<int>(head);
                int dep = -1;
                for (int i = j - 1; i >= 0; --i)
                    if ((size_t)v[i].boff < head + sz && head < (size_t)v[i].boff + nd_task_buf_bytes(v[i])) {
                        dep = i;
                        break;
                    }
                dep = std::max(dep, prev_dep);
                require(dep < 0 || dep <= j - 2, "nested dissection: buffer arena too small (task " + std::to_string(j) + " dep " +
                                          std::to_string(dep) + " head " + std::to_string(head) + " size " + std::to_string(sz) +
                                          " arena " + std::to_string(arena) + " prev " + std::to_string(v[j - 1].boff) + "+" +
                                          std::to_string(nd_task_buf_bytes(v[j - 1])) + ")");
                v[j].fdep = prev_dep = dep;
                head += sz;
            }
        }
        std::vector<NdTask> all, all_b;
        std::vector<int> hct(grid + 1, 0), hct_b(grid + 1, 0);
        for (int q = 0; q < grid; ++q) {
            all.insert(all.end(), per_cta[q].begin(), per_cta[q].end());
            hct[q + 1] = static_cast<int>(all.size());
        }
        if (split) {
            for (int q = 0; q < grid; ++q) {
                all_b.insert(all_b.end(), per_cta[grid + q].begin(), per_cta[grid + q].end());
                hct_b[q + 1] = static_cast<int>(all_b.size());
            }
            d_tasks_b.upload(all_b, st);
            ctoff_b.upload(hct_b, st);
        }
        // the attribute is per device and only ever raised: set the largest seen on this device
        static size_t attr_smem[64] = {};
        if (smem > attr_smem[dev % 64]) {
            PDG_CUDA(cudaFuncSetAttribute(k_nd_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            attr_smem[dev % 64] = smem;
        }
        int per_sm = 0;
        PDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_nd_solve, kNdBlock, smem));
        require(per_sm >= 1 && grid <= per_sm * nsm, "nested dissection: solve grid not co-resident");
    d_tasks.upload(all, st);
        ctoff.upload(hct, st);
        PDG_CUDA(cudaStreamSynchronize(st));
    };
    try {
        schedule_chunks();
        if (hybrid) {  // the top levels as level kernels (tiles for those fronts only)
            lvl_max_depth = hybrid_top;
            build_tiles(children, parent, hs, hbp, hcbdst, st);
        }
    } catch (const Error& e) {
        if (e.status != PDG_INVALID_ARGUMENT || std::getenv("PDG_ND_STRICT")) throw;
        fallback_reason = e.what();
        hybrid = split = false;
        lvl_max_depth = -1;
        tiles = levels = true;
        build_tiles(children, parent, hs, hbp, hcbdst, st);
        store.release();
    }
}

// one launch of the chunk kernel on a task schedule (the hybrid's local forward / backward)
void NdChol::launch_chunks(const NdTask* tasks, const int* cto, const double* b, long long ldb, double* x, long long ldx,
                           int nrhs, cudaStream_t st) {
    NdArgs a{tasks, cto, sdofs.p, bpos.p, cbdst.p, store.p, b, ldb, x, ldx, y.p, xpos.p, cbuf.p, counters.p, call, cbtot, n,
             nrhs, stages, vmax, smem_tasks, pf, stage_bytes, nullptr, 0, 0, std::getenv("PDG_ND_FENCE") != nullptr, guard,
             0, 0};
    void* args[] = {&a};
    PDG_CUDA(cudaLaunchCooperativeKernel((void*)k_nd_solve, grid, kNdBlock, args, smem, st));
    count_launch(1);
    PDG_CHECK_LAUNCH();
}

// PDG_ND_HYBRID: unset -> the displacement solve only (config 1: 275 -> 246 us; the flux
// solve's small top levels are faster in the chunk kernel, 92 vs 106 us); 0 none; 1 both
bool nd_hybrid_default(int prof_phase) {
    const char* e = std::getenv("PDG_ND_HYBRID");
    if (!e) return prof_phase == PROF_A_SOLVE;
    return std::atoi(e) == 1 || (std::atoi(e) == 2 && prof_phase == PROF_A_SOLVE);
}

void NdChol::solve(const double* b, long long ldb, double* x, long long ldx, int nrhs, cudaStream_t st) {
    ProfScope prof(prof_phase, st, alg_bytes(nrhs));
    require(nrhs >= 1 && nrhs <= max_rhs, "nested dissection solve: bad nrhs");
    ++call;
    if (stream) {
        solve_stream(b, ldb, x, ldx, nrhs, st);
        return;
    }
    const int nl = static_cast<int>(lvl_smem.size());
    if (levels) {  // forward levels, the dense top, backward levels
        solve_levels_range(b, ldb, x, ldx, nrhs, 0, top_depth >= 0 ? nl / 2 : nl, st);
        if (top_depth >= 0) {
            solve_top(b, ldb, x, ldx, nrhs, st);
            solve_levels_range(b, ldb, x, ldx, nrhs, nl / 2, nl, st);
        }
        return;
    }
    if (split) {  // local forward (chunk kernel), level kernels, dense top, level kernels, local backward
        launch_chunks(d_tasks.p, ctoff.p, b, ldb, x, ldx, nrhs, st);
        if (hybrid) solve_levels_range(b, ldb, x, ldx, nrhs, 0, nl / 2, st);
        if (top_depth >= 0) solve_top(b, ldb, x, ldx, nrhs, st);
        if (hybrid) solve_levels_range(b, ldb, x, ldx, nrhs, nl / 2, nl, st);
        launch_chunks(d_tasks_b.p, ctoff_b.p, b, ldb, x, ldx, nrhs, st);
        return;
    }
    if (tiles) {
        solve_tiles(b, ldb, x, ldx, nrhs, st);
        return;
    }
    NdArgs a{d_tasks.p, ctoff.p, sdofs.p,    bpos.p, cbdst.p, store.p, b,         ldb,        x,       ldx,
             y.p,       xpos.p,  cbuf.p,     counters.p, call, cbtot,   n,         nrhs,       stages,  vmax,
             smem_tasks, pf,     stage_bytes, nullptr, std::getenv("PDG_ND_NODEP") != nullptr,
             std::getenv("PDG_ND_NOMATH") != nullptr, std::getenv("PDG_ND_FENCE") != nullptr, guard,
             std::getenv("PDG_ND_TILE8") != nullptr,
             std::getenv("PDG_ND_TILE8") == nullptr && std::getenv("PDG_ND_PAIRS") && std::atoi(std::getenv("PDG_ND_PAIRS")) > 0};
    const bool debug = std::getenv("PDG_ND_DEBUG") != nullptr;
    const long long ntask = static_cast<long long>(d_tasks.n);
    DBuf<unsigned long long> dbg;
    if (debug) {
        dbg.alloc((size_t)ntask * 4);
        dbg.zero(st);
        a.dbg = dbg.p;
    }
    void* args[] = {&a};
    PDG_CUDA(cudaLaunchCooperativeKernel((void*)k_nd_solve, grid, kNdBlock, args, smem, st));
    count_launch(1);
    PDG_CHECK_LAUNCH();
    if (debug) {  // per task kind and depth: earliest start, latest end (us from the first start)
        const std::vector<unsigned long long> h = dbg.download(st);
        const std::vector<NdTask> ts = d_tasks.download(st);
        unsigned long long t00 = ~0ull, tend = 0;
        for (long long i = 0; i < ntask; ++i) {
            t00 = std::min(t00, h[4 * i]);
            tend = std::max(tend, h[4 * i + 1]);
        }
        std::fprintf(stderr, "nd solve n=%d fronts=%d depth=%d tasks=%lld grid=%d max/cta=%d vmax=%d arena=%zu (max buf %zu) stages=%d x %u B total %.2f us\n", n,
                     nfront, maxdepth, ntask, grid, max_tasks, vmax, arena_bytes, max_task_buf, stages, stage_bytes, (tend - t00) * 1e-3);
        for (int type = 0; type < 3; ++type)
            for (int d = maxdepth; d >= 0; --d) {
                const int dd = type == 2 ? maxdepth - d : d;
                unsigned long long s0 = ~0ull, e1 = 0, busy = 0, gat = 0, w0 = 0;
                double mb = 0.0;
                int cntk = 0;
                for (long long i = 0; i < ntask; ++i)
                    if (ts[i].type == type && fronts[ts[i].front].depth == dd) {
                        s0 = std::min(s0, h[4 * i]);
                        e1 = std::max(e1, h[4 * i + 1]);
                        busy += h[4 * i + 1] - h[4 * i];
                        gat += h[4 * i + 2] - h[4 * i];
                        w0 += h[4 * i + 3] - h[4 * i + 2];
                        mb += 8e-6 * ts[i].nrows * ts[i].ld;
                        ++cntk;
                    }
                if (cntk)
                    std::fprintf(stderr,
                                 "  %s depth %2d tasks %5d  %7.2f MB  inputs ready %8.2f .. signalled %8.2f  per task: ready->signal %6.2f "
                                 "gather %6.2f  compute %6.2f us\n",
                                 type == 0 ? "gather  " : type == 1 ? "forward " : "backward", dd, cntk, mb,
                                 (s0 - t00) * 1e-3, (e1 - t00) * 1e-3, busy * 1e-3 / cntk, gat * 1e-3 / cntk, w0 * 1e-3 / cntk);
            }
    }
}

}  // namespace pdg
