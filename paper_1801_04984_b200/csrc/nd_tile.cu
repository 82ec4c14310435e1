// Nested-dissection solve, tile-streaming kernel (opt-in, PDG_ND_TILES=1; the default
// is the row-chunk kernel of nd.cu). Same factor and the same dataflow as nd.cuh
// describes: forward [y_S; u_F] = M (b_S - w_C1|S - w_C2|S), backward
// x_S = M^T [y_S; -x_B]. What changes is how a CTA streams and consumes M / M^T:
//
//  * Tiles of complete rows. A front pass (M: (s+b) x s, or M^T: s x (s+b)) is
//    repacked at setup into tiles of rb rows (rb a power of two <= 32, rb x cols
//    x 8 B <= one ring stage). Inside a tile, lane l = r + rb j owns row r and
//    the column pairs c2 = j, j + J, j + 2J, ... (J = 32 / rb), and the tile is
//    stored so that lane l's t-th double2 is element t * 32 + l: every load is
//    one coalesced 512 B warp access, and a row needs only a log2(J)-step
//    butterfly at the end instead of a reduction per row chunk.
//  * Tiles go to the compute warps strictly round robin (tile q of the CTA's
//    stream -> warp q % 8), so the TMA ring drains in order at full rate
//    (tools/ubench/stream_ring.cu: 8 x 16 KB stages, 8 consumer warps stream at
//    the HBM copy rate). No L2 prefetch cursor (it cost bandwidth, measured).
//  * Inputs. Two staging warps prepare, ahead and independently of the
//    dependencies, each task's static inputs in its arena buffer: the output
//    indices and b_S (forward) or the boundary pivot positions (backward). The
//    dependent part (children's updates, y_S, x_B) is gathered by all 256
//    compute threads right after the dependency wait: one round of loads.
//  * Placement. Fronts at depth >= local_depth form subtrees that run on one CTA
//    each (their dependencies stay inside the CTA, in task order); the levels
//    above are split into row ranges balanced over all CTAs.
// Fixed-order sums throughout: repeated solves are bit-identical.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>

#include "llsync.cuh"
#include "nd.cuh"

namespace pdg {

namespace {

constexpr int kTW = 8;                     // compute warps
constexpr int kTGroups = 2;                // gather groups (tasks alternate between them)
constexpr int kTGroupWarps = 2;            // warps per gather group
constexpr int kTGroupThreads = 32 * kTGroupWarps;
constexpr int kTWarpProducer = kTW;
constexpr int kTWarpGather = kTW + 1;
constexpr int kTWarpSignal = kTWarpGather + kTGroups * kTGroupWarps;
constexpr int kTBlock = 32 * (kTWarpSignal + 1);
constexpr int kTLoads = 16;                // gather loads in flight per thread
constexpr int kTMaxRhs = 2;
constexpr int kTBufs = 8;  // staged-barrier slots (tasks between staging and compute)
constexpr unsigned kTHeader = 1024;

size_t a16(size_t v) { return (v + 15) / 16 * 16; }

// arena layout of a task buffer: v [kTMaxRhs][cp] | tail [kTMaxRhs][tail_n] | oix [nrows] | bix [b, backward]
__host__ __device__ inline size_t tb_tail(const NdTileTask& t) { return (size_t)kTMaxRhs * t.cp * 8; }
__host__ __device__ inline size_t tb_oix(const NdTileTask& t) {
    return tb_tail(t) + (((size_t)kTMaxRhs * t.tail_n * 8 + 15) / 16) * 16;
}
__host__ __device__ inline size_t tb_bix(const NdTileTask& t) { return tb_oix(t) + (((size_t)t.nrows * 4 + 15) / 16) * 16; }
__host__ __device__ inline size_t tb_size(const NdTileTask& t) {
    return tb_bix(t) + (t.type == 2 ? (((size_t)t.b * 4 + 15) / 16) * 16 : 0);
}

struct TileArgs {
    const NdTileTask* tasks;
    const int* ctoff;
    const int* toix;
    const int* sdofs;
    const int* bpos;
    const double* tstore;
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
    int n, nrhs, stages, max_tasks;
    unsigned stage_bytes;
    size_t task_bytes;
    const int* stop;
    unsigned long long* dbg;  // optional per task: %globaltimer [deps met, gathered, tiles done, signalled]
    int nodep;                // timing only (PDG_ND_NODEP): no dependency waits (wrong results)
    int fence;                // PDG_ND_FENCE: fence.acq_rel.gpu before each completion release
    unsigned backoff;         // ns between dependency polls (PDG_ND_BACKOFF)
    int nostream;             // timing only (PDG_ND_NOSTREAM): no matrix stream, no products (wrong results)
    int evict_first;          // factor stream with L2 evict_first (default; PDG_ND_EVICT_NORMAL=1 to compare)
    long long pf_shared, pf_local;  // L2 prefetch distance in bytes (PDG_ND_PF_SHARED_KB, PDG_ND_PF_LOCAL_KB)
};

__device__ __forceinline__ unsigned long long t_ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void t_red_release_add(unsigned long long* p, unsigned long long v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// 1D bulk copy with an L2 eviction-priority hint: the factor streams through L2 once per
// solve and must not push out the small dataflow vectors (y, xpos, cb) the gathers read
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                              unsigned long long policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            dev::smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(dev::smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void group_sync(int g) { asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(kTGroupThreads) : "memory"); }

// The dependent inputs of a task into its buffer (after the dependency wait), by NT
// threads: forward v = (b_S - w_C1|S) - w_C2|S and the pass-through tail; backward
// v = [y_S; -x_B]. One round of kTLoads loads per thread in flight.
template <int NT>
__device__ __forceinline__ void gather_dependent(const TileArgs& a, const NdTileTask& T, unsigned char* buf, int t) {
    const int nr = a.nrhs;
    double* v = reinterpret_cast<double*>(buf);
    double* tail = reinterpret_cast<double*>(buf + tb_tail(T));
    const int* bix = reinterpret_cast<const int*>(buf + tb_bix(T));
    if (T.type == 1 && !T.leaf) {
        const double* c0p = a.cb + T.cboff;
        const double* c1p = c0p + (T.s + T.b);
        const int ns = nr * T.s, nt2 = nr * T.tail_n;
        for (int e0 = t; e0 < ns + nt2; e0 += NT * kTLoads) {
            double w0[kTLoads], w1[kTLoads];
            int dst[kTLoads];
#pragma unroll
            for (int u = 0; u < kTLoads; ++u) {
                const int e = e0 + u * NT;
                int k = 0, col = 0;
                dst[u] = -1;
                if (e < ns) {
                    k = e / T.s;
                    col = e - k * T.s;
                    dst[u] = k * T.cp + col;
                } else if (e < ns + nt2) {
                    const int f = e - ns;
                    k = f / T.tail_n;
                    const int ti = f - k * T.tail_n;
                    col = T.tail_lo + ti;
                    dst[u] = -2 - (k * T.tail_n + ti);
                }
                w0[u] = dst[u] != -1 ? __ldcg(c0p + k * a.cbtot + col) : 0.0;
                w1[u] = dst[u] != -1 ? __ldcg(c1p + k * a.cbtot + col) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kTLoads; ++u) {
                if (dst[u] >= 0)
                    v[dst[u]] = (v[dst[u]] - w0[u]) - w1[u];
                else if (dst[u] <= -2)
                    tail[-2 - dst[u]] = w0[u] + w1[u];
            }
        }
    } else if (T.type == 2) {  // [y_S; -x_B]
        const int len = T.s + T.b, tot = nr * len;
        for (int e0 = t; e0 < tot; e0 += NT * kTLoads) {
            double w[kTLoads];
            int dst[kTLoads];
#pragma unroll
            for (int u = 0; u < kTLoads; ++u) {
                const int e = e0 + u * NT;
                dst[u] = -1;
                w[u] = 0.0;
                if (e < tot) {
                    const int k = e / len, c = e - k * len;
                    dst[u] = k * T.cp + c;
                    w[u] = c < T.s ? __ldcg(a.y + (long long)k * a.n + T.sdof + c)
                                   : -__ldcg(a.xpos + (long long)k * a.n + bix[c - T.s]);
                }
            }
#pragma unroll
            for (int u = 0; u < kTLoads; ++u)
                if (dst[u] >= 0) v[dst[u]] = w[u];
        }
    }
}

__device__ __forceinline__ void wait_deps(const TileArgs& a, const NdTileTask& T) {
    // polls back off: many CTAs wait on one counter at the top levels
    if (T.wait0 >= 0) {
        const unsigned long long tgt = a.call * (unsigned long long)T.need0;
        while (t_ld_acquire(a.cnt + T.wait0) < tgt) __nanosleep(a.backoff);
    }
    if (T.wait1 >= 0) {
        const unsigned long long tgt = a.call * (unsigned long long)T.need1;
        while (t_ld_acquire(a.cnt + T.wait1) < tgt) __nanosleep(a.backoff);
    }
}
__device__ __forceinline__ void compute_sync() {
    asm volatile("bar.sync %0, %1;" ::"n"(1 + kTGroups), "n"(32 * kTW) : "memory");
}

__global__ void __launch_bounds__(kTBlock, 1) k_nd_tile_solve(TileArgs a) {
    using namespace dev;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem);  // [32]
    unsigned long long* empty = full + 32;                                   // [32]
    unsigned long long* ready = empty + 32;                                  // [kTBufs] input gathered
    unsigned long long* done = ready + kTBufs;                               // [kTBufs] compute warps done
    volatile int* tasks_done = reinterpret_cast<volatile int*>(done + kTBufs);
    NdTileTask* tsk = reinterpret_cast<NdTileTask*>(smem + kTHeader);
    unsigned char* ring = smem + kTHeader + a.task_bytes;
    unsigned char* arena = ring + (size_t)a.stages * a.stage_bytes;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int t0 = a.ctoff[blockIdx.x], nt = a.ctoff[blockIdx.x + 1] - t0;
    const int nr = a.nrhs;
    if (tid == 0) {
        for (int k = 0; k < a.stages; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], 1);
        }
        for (int k = 0; k < kTBufs; ++k) {
            mbar_init(&ready[k], 1);
            mbar_init(&done[k], kTW);
        }
        *tasks_done = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    {
        static_assert(sizeof(NdTileTask) % 4 == 0, "NdTileTask is copied as ints");
        const int* src = reinterpret_cast<const int*>(a.tasks + t0);
        int* dst = reinterpret_cast<int*>(tsk);
        const int words = nt * static_cast<int>(sizeof(NdTileTask) / 4);
        for (int w = tid; w < words; w += kTBlock) dst[w] = src[w];
    }
    __syncthreads();
    if (a.stop && *a.stop) {  // skipped call: completion counters advance as if every task ran
        for (int i = tid; i < nt; i += kTBlock) atomicAdd(a.cnt + tsk[i].signal, 1ull);
        return;
    }
    if (warp == kTWarpProducer) {  // TMA producer: every tile of every task, in order
        if (lane == 0 && !a.nostream) {
            unsigned long long policy, keep;
            if (a.evict_first)
                asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
            else
                asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(policy));
            // the top levels (the latency-critical turn at the root) stay in L2 across solves
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
            int seq = 0;
            // L2 prefetch cursor (task pi, chunk pc), up to pf_shared / pf_local bytes ahead of the
            // fill: the shared levels wait on dependencies with HBM idle, so their next tiles can
            // be on chip (L2) when the inputs arrive
            int pi = 0, pc = 0;
            long long filled = 0, pref = 0;
            auto prefetch = [&]() {
                while (pi < nt) {
                    const NdTileTask& P = tsk[pi];
                    const long long lim = P.cgather ? a.pf_shared : a.pf_local;
                    if (pc >= P.nchunks) {
                        ++pi;
                        pc = 0;
                        continue;
                    }
                    if (pref - filled >= lim) break;
                    const unsigned bytes = static_cast<unsigned>(min(P.kt, P.ntiles - pc * P.kt) * P.tile_d2) * 16u;
                    if (pref >= filled)
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.tstore + P.src + (size_t)pc * P.kt * P.tile_d2 * 2),
                                     "r"(bytes)
                                     : "memory");
                    pref += bytes;
                    ++pc;
                }
            };
            for (int i = 0; i < nt; ++i) {
                const NdTileTask& T = tsk[i];
                const double* src = a.tstore + T.src;
                for (int c = 0; c < T.nchunks; ++c, ++seq) {  // chunk c: tiles [c kt, min(ntiles, (c + 1) kt))
                    const int k = seq % a.stages;
                    const unsigned bytes = static_cast<unsigned>(min(T.kt, T.ntiles - c * T.kt) * T.tile_d2) * 16u;
                    if (a.pf_shared > 0 || a.pf_local > 0) prefetch();
                    filled += bytes;
                    if (pref < filled) {  // the prefetch cursor never trails the fill
                        pi = i;
                        pc = c + 1;
                        pref = filled;
                    }
                    if (seq >= a.stages) mbar_wait(&empty[k], static_cast<unsigned>(((seq / a.stages) - 1) & 1));
                    mbar_arrive_expect_tx(&full[k], bytes);
                    bulk_g2s_hint(ring + (size_t)k * a.stage_bytes, src + (size_t)c * T.kt * T.tile_d2 * 2, bytes,
                                  &full[k], T.l2keep ? keep : policy);
                }
            }
        }
        return;
    }
    if (warp == kTWarpSignal) {  // signaller: completion counters and buffer release, tasks in order
        if (lane == 0)
            for (int i = 0; i < nt; ++i) {
                mbar_wait(&done[i % kTBufs], static_cast<unsigned>((i / kTBufs) & 1));
                if (a.dbg) a.dbg[(size_t)(t0 + i) * 8 + 2] = globaltimer();
                // the compute warps' outputs reach this thread through the done barrier; the
                // gpu-scope release is cumulative over them (PDG_ND_FENCE: an explicit fence first)
                if (a.fence) asm volatile("fence.acq_rel.gpu;" ::: "memory");
                t_red_release_add(a.cnt + tsk[i].signal, 1ull);
                __threadfence_block();
                *tasks_done = i + 1;
                if (a.dbg) a.dbg[(size_t)(t0 + i) * 8 + 3] = globaltimer();
            }
        return;
    }
    if (warp >= kTWarpGather) {  // gather groups: task j on group j % kTGroups, ahead of the compute
        const int g = (warp - kTWarpGather) / kTGroupWarps;
        const int gt = tid - (kTWarpGather + g * kTGroupWarps) * 32;
        for (int j = g; j < nt; j += kTGroups) {
            const NdTileTask& T = tsk[j];
            // the buffer space (fdep) and the barrier slot (j - kTBufs) are free once those tasks are done
            const int need = max(T.fdep, j - kTBufs) + 1;
            while (*tasks_done < need) __nanosleep(32);
            __threadfence_block();
            if (a.dbg && gt == 0) a.dbg[(size_t)(t0 + j) * 8 + 4] = globaltimer();
            unsigned char* buf = arena + T.boff;
            double* v = reinterpret_cast<double*>(buf);
            double* tail = reinterpret_cast<double*>(buf + tb_tail(T));
            int* oix = reinterpret_cast<int*>(buf + tb_oix(T));
            int* bix = reinterpret_cast<int*>(buf + tb_bix(T));
            // ---- static inputs (no dependency): output indices, b_S / boundary positions ----
            for (int r = gt; r < T.nrows; r += kTGroupThreads) oix[r] = __ldg(a.toix + T.oix_off + r);
            if (T.type == 1) {  // b_S, zero padding, zero second rhs when nrhs = 1
                const int tot = kTMaxRhs * T.cp;
                for (int c0 = gt; c0 < tot; c0 += kTGroupThreads * kTLoads) {
                    double xv[kTLoads];
#pragma unroll
                    for (int u = 0; u < kTLoads; ++u) {
                        const int c = c0 + u * kTGroupThreads, k = c / T.cp, cc = c - k * T.cp;
                        xv[u] = (c < tot && k < nr && cc < T.s) ? a.b[k * a.ldb + __ldg(a.sdofs + T.sdof + cc)] : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < kTLoads; ++u)
                        if (c0 + u * kTGroupThreads < tot) v[c0 + u * kTGroupThreads] = xv[u];
                }
            } else {
                for (int c = gt; c < T.b; c += kTGroupThreads) bix[c] = __ldg(a.bpos + T.bdof + c);
                for (int k = 0; k < kTMaxRhs; ++k)  // padding columns, and the whole unused rhs
                    for (int c = (k < nr ? T.ncols : 0) + gt; c < T.cp; c += kTGroupThreads) v[k * T.cp + c] = 0.0;
            }
            // ---- the dependency wait ----
            if (gt == 0 && !a.nodep && !T.cgather) wait_deps(a, T);
            if (a.dbg && gt == 0 && !T.cgather) a.dbg[(size_t)(t0 + j) * 8 + 5] = globaltimer();
            group_sync(g);  // b_S written and the dependencies met, for every thread of the group
            // ---- dependent inputs (shared-level tasks: by the compute warps, see below) ----
            if (!T.cgather) gather_dependent<kTGroupThreads>(a, T, buf, gt);
            group_sync(g);
            if (gt == 0) {
                if (a.dbg && !T.cgather) a.dbg[(size_t)(t0 + j) * 8] = globaltimer();
                mbar_arrive(&ready[j % kTBufs]);
            }
        }
        return;
    }
    // ---- compute warps: no CTA-wide barrier; a warp moves on as soon as the next input is ready ----
    int seq = 0;
    for (int i = 0; i < nt; ++i) {
        const NdTileTask& T = tsk[i];
        unsigned char* buf = arena + T.boff;
        const double* v = reinterpret_cast<const double*>(buf);
        const double* tail = reinterpret_cast<const double*>(buf + tb_tail(T));
        const int* oix = reinterpret_cast<const int*>(buf + tb_oix(T));
        const int first = a.nostream ? kTW : (warp - seq % kTW + kTW) % kTW;
        // every warp waits for every task's input, chunks or not: keeps all warps within one
        // phase of the ready / done barriers (a warp skipping tasks could alias a phase)
        mbar_wait(&ready[i % kTBufs], static_cast<unsigned>((i / kTBufs) & 1));
        if (T.cgather) {  // shared levels: all compute threads gather the dependent inputs (one round)
            if (tid == 0 && !a.nodep) wait_deps(a, T);
            if (a.dbg && tid == 0) a.dbg[(size_t)(t0 + i) * 8 + 5] = globaltimer();
            compute_sync();
            gather_dependent<32 * kTW>(a, T, buf, tid);
            compute_sync();
            if (a.dbg && tid == 0) a.dbg[(size_t)(t0 + i) * 8] = globaltimer();
        }
        if (a.dbg && lane == 0 && first == 0) a.dbg[(size_t)(t0 + i) * 8 + 1] = globaltimer();
        if (first < T.nchunks) {
            const int rb = T.rb, J = 32 / rb, jl = lane / rb, rl = lane - jl * rb;
            const int nslab = T.tile_d2 >> 5;
            const double2* v0 = reinterpret_cast<const double2*>(v);
            const double2* v1 = reinterpret_cast<const double2*>(v + T.cp);
            for (int c = first; c < T.nchunks; c += kTW) {
                const int sq = seq + c, slot = sq % a.stages;
                // the slot's previous chunk (sq - stages) consumed before waiting on this one's
                // phase (2 stages is a multiple of kTW: that wait is always on a single phase)
                if (sq >= a.stages) mbar_wait(&empty[slot], static_cast<unsigned>(((sq / a.stages) - 1) & 1));
                mbar_wait(&full[slot], static_cast<unsigned>((sq / a.stages) & 1));
                const int q1 = min(T.ntiles, (c + 1) * T.kt);
                for (int q = c * T.kt; q < q1; ++q) {
                    const double2* tile = reinterpret_cast<const double2*>(ring + (size_t)slot * a.stage_bytes) +
                                          (size_t)(q - c * T.kt) * T.tile_d2 + lane;
                    double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0, q0 = 0.0, qq1 = 0.0, q2 = 0.0, q3 = 0.0;
                    int t = 0;
                    for (; t + 1 < nslab; t += 2) {
                        const double2 m0 = tile[t * 32], m1 = tile[(t + 1) * 32];
                        const double2 a0 = v0[t * J + jl], b0 = v1[t * J + jl];
                        const double2 a1 = v0[(t + 1) * J + jl], b1 = v1[(t + 1) * J + jl];
                        p0 = fma(m0.x, a0.x, p0);
                        p1 = fma(m0.y, a0.y, p1);
                        q0 = fma(m0.x, b0.x, q0);
                        qq1 = fma(m0.y, b0.y, qq1);
                        p2 = fma(m1.x, a1.x, p2);
                        p3 = fma(m1.y, a1.y, p3);
                        q2 = fma(m1.x, b1.x, q2);
                        q3 = fma(m1.y, b1.y, q3);
                    }
                    if (t < nslab) {
                        const double2 m0 = tile[t * 32];
                        const double2 a0 = v0[t * J + jl], b0 = v1[t * J + jl];
                        p0 = fma(m0.x, a0.x, p0);
                        p1 = fma(m0.y, a0.y, p1);
                        q0 = fma(m0.x, b0.x, q0);
                        qq1 = fma(m0.y, b0.y, qq1);
                    }
                    if (q == q1 - 1) {  // the chunk's data is in registers: release the slot
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&empty[slot]);
                    }
                    double s0 = (p0 + p1) + (p2 + p3), s1 = (q0 + qq1) + (q2 + q3);
                    for (int o = rb; o < 32; o <<= 1) {
                        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
                        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
                    }
                    const int row = q * rb + rl;
                    if (jl == 0 && row < T.nrows) {
                        const int gr = T.r0 + row;
                        if (T.type == 2) {
                            a.xpos[T.sdof + gr] = s0;
                            a.x[oix[row]] = s0;
                            if (nr > 1) {
                                a.xpos[(long long)a.n + T.sdof + gr] = s1;
                                a.x[a.ldx + oix[row]] = s1;
                            }
                        } else if (gr < T.s) {
                            a.y[T.sdof + gr] = s0;
                            if (nr > 1) a.y[(long long)a.n + T.sdof + gr] = s1;
                        } else {  // update vector entry (+ the pass-through), into the parent's slot
                            const int ti = gr - T.tail_lo;
                            a.cb[oix[row]] = s0 + (T.leaf ? 0.0 : tail[ti]);
                            if (nr > 1) a.cb[a.cbtot + oix[row]] = s1 + (T.leaf ? 0.0 : tail[T.tail_n + ti]);
                        }
                    }
                }
            }
        }
        seq += T.nchunks;
        __syncwarp();
        if (lane == 0) mbar_arrive(&done[i % kTBufs]);  // this warp's outputs of task i written (or it had none)
    }
}

// ---- level-synchronous solve (PDG_ND_LEVELS): one launch per tree level and pass ----
// All fronts of a level are independent: every block takes units (a front's row range),
// gathers the front's input vector into shared memory (all 256 threads, one round of
// loads), and its 8 warps stream the unit's tiles straight from global memory (coalesced
// 512 B warp loads, the lane-per-row layout above). The levels are chained with
// programmatic dependent launch: a level's blocks start (and prefetch their tiles into L2)
// while the previous level runs, then wait (griddepcontrol.wait) for its results.
constexpr int kLvlThreads = 256;
// level unit buffer: the task buffer (tb_size) plus, forward, the b_S gather indices
__host__ __device__ inline size_t lvl_sidx(const NdTileTask& t) { return tb_size(t); }
__host__ __device__ inline size_t lvl_size(const NdTileTask& t) {
    return tb_size(t) + (t.type == 1 ? (((size_t)t.s * 4 + 15) / 16) * 16 : 0);
}

// prefetch: 0 none, 1 L2 prefetch of the unit's tiles, 2 the tiles themselves into shared
// memory by TMA bulk copies (stage_bytes = the staging region), issued before the wait
template <bool STAGED>
__global__ void __launch_bounds__(kLvlThreads) k_nd_level(TileArgs a, int u0, int u1, int prefetch, int lvl) {
    extern __shared__ __align__(128) unsigned char lsm[];
    __shared__ NdTileTask Ts;
    __shared__ __align__(8) unsigned long long tbar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nr = a.nrhs;
    constexpr bool staged = STAGED;
    unsigned char* stage = lsm;  // staged tiles (prefetch 2)
    bool waited = false;
    unsigned phase = 0;
    if (staged && tid == 0) {
        dev::mbar_init(&tbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int u = u0 + blockIdx.x; u < u1; u += gridDim.x) {
        if (tid < (int)(sizeof(NdTileTask) / 4))
            reinterpret_cast<int*>(&Ts)[tid] = __ldg(reinterpret_cast<const int*>(a.tasks + u) + tid);
        __syncthreads();
        const NdTileTask& T = Ts;
        unsigned char* buf = lsm + (staged ? a.stage_bytes : 0);
        double* v = reinterpret_cast<double*>(buf);
        double* tail = reinterpret_cast<double*>(buf + tb_tail(T));
        int* oix = reinterpret_cast<int*>(buf + tb_oix(T));
        int* bix = reinterpret_cast<int*>(buf + tb_bix(T));
        int* sidx = reinterpret_cast<int*>(buf + lvl_sidx(T));
        const long long tbytes = (long long)T.ntiles * T.tile_d2 * 16;
        if (staged && tid == 0) {  // the unit's tiles (static) into shared memory, in flight during the wait
            dev::mbar_arrive_expect_tx(&tbar, static_cast<unsigned>(tbytes));
            for (long long off = 0; off < tbytes; off += 32768)
                dev::bulk_g2s(stage + off, reinterpret_cast<const char*>(a.tstore + T.src) + off,
                              static_cast<unsigned>(min(32768LL, tbytes - off)), &tbar);
        }
        // ---- static data (before the dependency wait): the unit's tiles into L2, the index lists ----
        if (prefetch == 1) {
            const long long bytes = (long long)T.ntiles * T.tile_d2 * 16;
            for (long long off = (long long)tid * 16384; off < bytes; off += (long long)kLvlThreads * 16384) {
                const unsigned nb = static_cast<unsigned>(min(16384LL, bytes - off));
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<const char*>(a.tstore + T.src) + off),
                             "r"(nb)
                             : "memory");
            }
        }
        for (int r = tid; r < T.nrows; r += kLvlThreads) oix[r] = __ldg(a.toix + T.oix_off + r);
        if (T.type == 1)
            for (int c = tid; c < T.s; c += kLvlThreads) sidx[c] = __ldg(a.sdofs + T.sdof + c);
        else
            for (int c = tid; c < T.b; c += kLvlThreads) bix[c] = __ldg(a.bpos + T.bdof + c);
        if (!waited) {  // the previous level's results (and b) are visible past this point
            asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
            asm volatile("griddepcontrol.wait;" ::: "memory");
            waited = true;
        }
        __syncthreads();
        if (a.stop && *a.stop) {  // speculative GMRES step after the cycle ended
            if (staged) dev::mbar_wait(&tbar, phase);  // no bulk copy may outlive the CTA
            return;
        }
        if (a.dbg && tid == 0) {  // PDG_ND_DEBUG: per level [first start past the wait, last end, launch seen]
            atomicMin(a.dbg + 3 * lvl, dev::globaltimer());
        }
        // ---- the input vector in one round of loads ----
        if (T.type == 1) {
            const double* c0p = a.cb + T.cboff;
            const double* c1p = c0p + (T.s + T.b);
            const bool inner = !T.leaf;
            const int tot = kTMaxRhs * T.cp, nt2 = nr * T.tail_n;
            for (int e0 = tid; e0 < tot + nt2; e0 += kLvlThreads * 8) {
                double w0[8], w1[8], bv[8];
                int dst[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int e = e0 + q * kLvlThreads;
                    int k = 0, col = 0;
                    dst[q] = -1;
                    bv[q] = 0.0;
                    if (e < tot) {
                        k = e / T.cp;
                        col = e - k * T.cp;
                        dst[q] = e;
                        if (k < nr && col < T.s) bv[q] = a.b[k * a.ldb + sidx[col]];
                    } else if (e < tot + nt2) {
                        const int f = e - tot;
                        k = f / T.tail_n;
                        const int ti = f - k * T.tail_n;
                        col = T.tail_lo + ti;
                        dst[q] = -2 - (k * T.tail_n + ti);
                    }
                    const bool ld = inner && ((dst[q] >= 0 && k < nr && col < T.s) || dst[q] <= -2);
                    w0[q] = ld ? __ldcg(c0p + k * a.cbtot + col) : 0.0;
                    w1[q] = ld ? __ldcg(c1p + k * a.cbtot + col) : 0.0;
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (dst[q] >= 0)
                        v[dst[q]] = inner ? (bv[q] - w0[q]) - w1[q] : bv[q];
                    else if (dst[q] <= -2)
                        tail[-2 - dst[q]] = w0[q] + w1[q];
                }
            }
        } else {
            const int len = T.s + T.b, tot = kTMaxRhs * T.cp;
            for (int e0 = tid; e0 < tot; e0 += kLvlThreads * 8) {
                double w[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int e = e0 + q * kLvlThreads, k = e / T.cp, c = e - k * T.cp;
                    w[q] = 0.0;
                    if (e < tot && k < nr && c < len)
                        w[q] = c < T.s ? __ldcg(a.y + (long long)k * a.n + T.sdof + c)
                                       : -__ldcg(a.xpos + (long long)k * a.n + bix[c - T.s]);
                }
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (e0 + q * kLvlThreads < tot) v[e0 + q * kLvlThreads] = w[q];
            }
        }
        __syncthreads();
        const int rb = T.rb, J = 32 / rb, jl = lane / rb, rl = lane - jl * rb;
        const int nslab = T.tile_d2 >> 5;
        const double2* v0 = reinterpret_cast<const double2*>(v);
        const double2* v1 = reinterpret_cast<const double2*>(v + T.cp);
        if (staged) {
            dev::mbar_wait(&tbar, phase);
            phase ^= 1u;
        }
        const double2* tiles = staged ? reinterpret_cast<const double2*>(stage)
                                      : reinterpret_cast<const double2*>(a.tstore + T.src);
        for (int q = warp; q < T.ntiles; q += kLvlThreads / 32) {
            const double2* tile = tiles + (size_t)q * T.tile_d2 + lane;
            double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0, q0 = 0.0, qq1 = 0.0, q2 = 0.0, q3 = 0.0;
            auto ld = [&](const double2* p_) {
                if constexpr (STAGED)
                    return *p_;
                else
                    return __ldcs(p_);
            };
            int t = 0;
            for (; t + 3 < nslab; t += 4) {
                const double2 m0 = ld(tile + t * 32), m1 = ld(tile + (t + 1) * 32);
                const double2 m2 = ld(tile + (t + 2) * 32), m3 = ld(tile + (t + 3) * 32);
                const double2 a0 = v0[t * J + jl], b0 = v1[t * J + jl], a1 = v0[(t + 1) * J + jl], b1 = v1[(t + 1) * J + jl];
                const double2 a2 = v0[(t + 2) * J + jl], b2 = v1[(t + 2) * J + jl], a3 = v0[(t + 3) * J + jl],
                              b3 = v1[(t + 3) * J + jl];
                p0 = fma(m0.x, a0.x, p0);
                p1 = fma(m0.y, a0.y, p1);
                q0 = fma(m0.x, b0.x, q0);
                qq1 = fma(m0.y, b0.y, qq1);
                p2 = fma(m1.x, a1.x, p2);
                p3 = fma(m1.y, a1.y, p3);
                q2 = fma(m1.x, b1.x, q2);
                q3 = fma(m1.y, b1.y, q3);
                p0 = fma(m2.x, a2.x, p0);
                p1 = fma(m2.y, a2.y, p1);
                q0 = fma(m2.x, b2.x, q0);
                qq1 = fma(m2.y, b2.y, qq1);
                p2 = fma(m3.x, a3.x, p2);
                p3 = fma(m3.y, a3.y, p3);
                q2 = fma(m3.x, b3.x, q2);
                q3 = fma(m3.y, b3.y, q3);
            }
            for (; t < nslab; ++t) {
                const double2 m0 = ld(tile + t * 32);
                const double2 a0 = v0[t * J + jl], b0 = v1[t * J + jl];
                p0 = fma(m0.x, a0.x, p0);
                p1 = fma(m0.y, a0.y, p1);
                q0 = fma(m0.x, b0.x, q0);
                qq1 = fma(m0.y, b0.y, qq1);
            }
            double s0 = (p0 + p1) + (p2 + p3), s1 = (q0 + qq1) + (q2 + q3);
            for (int o = rb; o < 32; o <<= 1) {
                s0 += __shfl_xor_sync(0xffffffffu, s0, o);
                s1 += __shfl_xor_sync(0xffffffffu, s1, o);
            }
            const int row = q * rb + rl;
            if (jl == 0 && row < T.nrows) {
                const int gr = T.r0 + row;
                if (T.type == 2) {
                    a.xpos[T.sdof + gr] = s0;
                    a.x[oix[row]] = s0;
                    if (nr > 1) {
                        a.xpos[(long long)a.n + T.sdof + gr] = s1;
                        a.x[a.ldx + oix[row]] = s1;
                    }
                } else if (gr < T.s) {
                    a.y[T.sdof + gr] = s0;
                    if (nr > 1) a.y[(long long)a.n + T.sdof + gr] = s1;
                } else {
                    const int ti = gr - T.tail_lo;
                    a.cb[oix[row]] = s0 + (T.leaf ? 0.0 : tail[ti]);
                    if (nr > 1) a.cb[a.cbtot + oix[row]] = s1 + (T.leaf ? 0.0 : tail[T.tail_n + ti]);
                }
            }
        }
        __syncthreads();  // the buffers are reused by the next unit
        if (a.dbg && tid == 0) atomicMax(a.dbg + 3 * lvl + 1, dev::globaltimer());
    }
    if (!waited) {
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
}

// tile store from the row-major M / M^T store: one block per tile
struct TilePack {
    long long dst;  // doubles
    long long src;  // doubles: first row of the tile in the row-major store
    int ld, ncols, rows, rb, tile_d2;
};
__global__ void k_nd_tile_pack(const TilePack* __restrict__ jobs, const double* __restrict__ store, double* __restrict__ out) {
    const TilePack J = jobs[blockIdx.x];
    const int jj = 32 / J.rb;
    double2* o = reinterpret_cast<double2*>(out + J.dst);
    for (int e = threadIdx.x; e < J.tile_d2; e += blockDim.x) {
        const int t = e >> 5, l = e & 31, jl = l / J.rb, r = l - jl * J.rb;
        const int c = 2 * (t * jj + jl);
        double2 m = make_double2(0.0, 0.0);
        if (r < J.rows) {
            const double* row = store + J.src + (long long)r * J.ld;
            if (c < J.ncols) m.x = row[c];
            if (c + 1 < J.ncols) m.y = row[c + 1];
        }
        o[e] = m;
    }
}

}  // namespace

bool nd_levels_default() {
    const char* e = std::getenv("PDG_ND_LEVELS");
    return e && std::atoi(e) > 0;
}

bool nd_tile_default() {
    // opt-in (PDG_ND_TILES=1): measured no faster than the row-chunk kernel at config 1
    const char* e = std::getenv("PDG_ND_TILES");
    return (e && std::atoi(e) > 0) || nd_levels_default();
}

void NdChol::build_tiles(const std::vector<std::vector<int>>& children, const std::vector<int>& parent,
                         const std::vector<int>& hs, const std::vector<int>& hbp, const std::vector<int>& hcbdst,
                         cudaStream_t st) {
    const int nf = nfront;
    int dev = 0, nsm = 0;
    PDG_CUDA(cudaGetDevice(&dev));
    PDG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    tgrid = nsm;
    // ring: 4 x 32 KB stages (large bulk copies keep the per-SM stream near the HBM share;
    // 2 stages must be a multiple of the compute warps); tiles of <= 16 KB packed into chunks
    tstages = 4;
    if (const char* e = std::getenv("PDG_ND_STAGES")) tstages = std::min(32, std::max(kTW / 2, std::atoi(e)));
    tstages = (tstages + kTW / 2 - 1) / (kTW / 2) * (kTW / 2);
    unsigned tile_cap = 16384;
    tstage_bytes = 32768;
    if (const char* e = std::getenv("PDG_ND_STAGE_KB")) tstage_bytes = 1024u * std::max(16, std::atoi(e));
    if (const char* e = std::getenv("PDG_ND_TILE_KB")) tile_cap = 1024u * std::max(4, std::atoi(e));
    int cmax = 0;
    for (const auto& F : fronts) cmax = std::max(cmax, F.s + F.b);
    const long long wide = ((long long)(cmax + 63) / 64 * 64) * 8;  // one row of the widest pass
    tile_cap = static_cast<unsigned>(std::max<long long>(tile_cap, wide));
    tstage_bytes = std::max(tstage_bytes, tile_cap);
    require(levels || hybrid || tstage_bytes <= 65536, "nested dissection: front too wide for the tile ring");
    // subtree mapping (see the file comment)
    int local_depth = maxdepth + 1;
    {
        std::vector<int> per_depth(maxdepth + 1, 0);
        for (const auto& F : fronts) per_depth[F.depth]++;
        for (int d = maxdepth; d >= 0; --d)
            if (per_depth[d] <= tgrid) {
                local_depth = d;
                break;
            }
        if (const char* e = std::getenv("PDG_ND_LOCAL_DEPTH")) {
            const int v = std::atoi(e);
            local_depth = v < 0 ? maxdepth + 1 : std::min(v, maxdepth + 1);
        }
    }
    std::vector<int> cta_of(nf, -1);
    {
        std::vector<int> roots;
        for (int k = 0; k < nf; ++k)
            if (fronts[k].depth == local_depth) roots.push_back(k);
        const int nr = static_cast<int>(roots.size());
        for (int j = 0; j < nr; ++j) cta_of[roots[j]] = static_cast<int>((long long)j * tgrid / std::max(nr, 1));
        for (int d = local_depth + 1; d <= maxdepth; ++d)
            for (int k = 0; k < nf; ++k)
                if (fronts[k].depth == d && parent[k] >= 0) cta_of[k] = cta_of[parent[k]];
    }
    // levels whose tiles are loaded with L2 evict_last (kept in L2 across solves)
    int l2keep_depth = 1;
    if (const char* e = std::getenv("PDG_ND_L2KEEP_DEPTH")) l2keep_depth = std::atoi(e);
    // tile geometry of a pass with `cols` columns: rows per tile and padded columns
    auto geometry = [&](int cols, int& rb, int& cp) {
        rb = 32;
        for (;;) {
            const int J = 32 / rb;
            cp = (cols + 2 * J - 1) / (2 * J) * (2 * J);
            if ((long long)rb * cp * 8 <= tile_cap || rb == 1) break;
            rb >>= 1;
        }
        require((long long)rb * cp * 8 <= tile_cap, "nested dissection: tile larger than a ring stage");
    };
    std::vector<int> ntask_of(3 * nf, 0);
    std::vector<std::vector<NdTileTask>> per_cta(tgrid);
    std::vector<int> oix;
    std::vector<TilePack> packs;
    long long toff = 0;
    auto make_tasks = [&](int k, int type, int rows_per_task) {
        const NdFront& F = fronts[k];
        const int rows = type == 1 ? F.s + F.b : F.s;
        const int cols = type == 1 ? F.s : F.s + F.b;
        const int ld = type == 1 ? F.ldm : F.ldt;
        const long long base = type == 1 ? F.moff : F.mtoff;
        int rb, cp;
        geometry(cols, rb, cp);
        const int J = 32 / rb;
        const int tile_d2 = cp / (2 * J) * 32;
        const int cap = std::max(rb, (rows_per_task + rb - 1) / rb * rb);
        const int kt = std::max(1, static_cast<int>(tstage_bytes / (16u * tile_d2)));
        std::vector<NdTileTask> out;
        for (int r0 = 0; r0 < rows; r0 += cap) {
            NdTileTask t{};
            t.type = type;
            t.front = k;
            t.r0 = r0;
            t.nrows = std::min(cap, rows - r0);
            t.cp = cp;
            t.ncols = cols;
            t.rb = rb;
            t.ntiles = (t.nrows + rb - 1) / rb;
            t.tile_d2 = tile_d2;
            t.kt = kt;
            t.nchunks = (t.ntiles + kt - 1) / kt;
            t.s = F.s;
            t.b = F.b;
            t.sdof = F.sdof;
            t.bdof = F.bdof;
            t.cboff = F.cboff;
            t.leaf = children[k].empty() ? 1 : 0;
            t.wait0 = t.wait1 = -1;
            t.signal = 3 * k + type;
            t.src = toff;
            for (int q = 0; q < t.ntiles; ++q) {
                TilePack p{};
                p.dst = toff;
                p.src = base + (long long)(r0 + q * rb) * ld;
                p.ld = ld;
                p.ncols = cols;
                p.rows = std::min(rb, t.nrows - q * rb);
                p.rb = rb;
                p.tile_d2 = tile_d2;
                packs.push_back(p);
                toff += 2LL * tile_d2;
            }
            t.oix_off = static_cast<int>(oix.size());
            for (int r = 0; r < t.nrows; ++r) {
                const int gr = r0 + r;
                oix.push_back(type == 2 ? hs[F.sdof + gr] : (gr >= F.s ? hcbdst[F.bdof + gr - F.s] : 0));
            }
            // pass-through rows of a non-leaf forward task: its own boundary rows
            t.tail_lo = std::max(r0, F.s);
            t.tail_n = (type == 1 && !t.leaf) ? std::max(0, r0 + t.nrows - t.tail_lo) : 0;
            out.push_back(t);
            ntask_of[3 * k + type]++;
        }
        return out;
    };
    auto level_bytes = [&](int type, int depth) {
        double by = 0.0;
        for (const auto& F : fronts)
            if (F.depth == depth) by += 8.0 * (double)(F.s + F.b) * F.s;
        (void)type;
        return by;
    };
    // task lists: local forward (deepest first), shared forward, shared backward, local backward
    auto place_level = [&](int type, int depth) {
        std::vector<NdTileTask> ts;
        const bool local = depth >= local_depth;
        const double want = level_bytes(type, depth) / tgrid;
        for (int k = 0; k < nf; ++k) {
            if (fronts[k].depth != depth) continue;
            const NdFront& F = fronts[k];
            const int cols = type == 1 ? F.s : F.s + F.b;
            const int rows = type == 1 ? F.s + F.b : F.s;
            const int rpt = local ? rows : std::max(1, static_cast<int>(std::ceil(want / (8.0 * std::max(cols, 1)))));
            std::vector<NdTileTask> v = make_tasks(k, type, rpt);
            for (auto& t : v) {
                t.cgather = local ? 0 : 1;
                t.l2keep = depth <= l2keep_depth ? 1 : 0;
            }
            if (local)
                for (auto& t : v) per_cta[cta_of[k]].push_back(t);
            else
                ts.insert(ts.end(), v.begin(), v.end());
        }
        if (!local) {  // contiguous byte-balanced ranges over the CTAs
            double wsum = 0.0;
            for (const auto& t : ts) wsum += 8.0 * t.nrows * t.cp + 2048.0;
            double acc = 0.0;
            for (const auto& t : ts) {
                const double w = 8.0 * t.nrows * t.cp + 2048.0;
                int q = static_cast<int>((acc + 0.5 * w) / wsum * tgrid);
                q = std::min(std::max(q, 0), tgrid - 1);
                per_cta[q].push_back(t);
                acc += w;
            }
        }
    };
    if (levels || hybrid) {  // level-synchronous units: fwd levels deepest first, then bwd levels
        std::vector<NdTileTask> units;
        lvl_off.clear();
        lvl_smem.clear();
        int min_rows = 8;
        if (const char* e = std::getenv("PDG_ND_LVL_MINROWS")) min_rows = std::max(1, std::atoi(e));
        double upb = 2.0;  // units per CTA slot of the grid, for the levels large enough to split
        if (const char* e = std::getenv("PDG_ND_LVL_UPB")) upb = std::max(0.25, std::atof(e));
        // PDG_ND_LVL_PF: 1 (default) L2 prefetch of a unit's tiles before the dependency wait;
        // 2 the tiles staged in shared memory by TMA bulk copies (units capped to the staging
        // region; measured slower at config 1: 352 vs 276 us); 0 none
        lvl_pf = std::getenv("PDG_ND_LVL_PF") ? std::atoi(std::getenv("PDG_ND_LVL_PF")) : 1;
        long long lvl_stage = lvl_pf == 2 ? 96 * 1024 : (1LL << 40);  // staging region of a unit's tiles
        if (const char* e = std::getenv("PDG_ND_LVL_STAGE_KB")) lvl_stage = 1024LL * std::max(16, std::atoi(e));
        long long stage_max = 0;
        auto add_level = [&](int type, int depth) {
            const double want = std::min(level_bytes(type, depth) / (upb * tgrid), (double)lvl_stage);
            size_t smax = 0;
            lvl_off.push_back(static_cast<int>(units.size()));
            for (int k = 0; k < nf; ++k) {
                if (fronts[k].depth != depth) continue;
                const NdFront& F = fronts[k];
                const int cols = type == 1 ? F.s : F.s + F.b;
                const int rows = type == 1 ? F.s + F.b : F.s;
                int rpt = std::max(min_rows, static_cast<int>(std::ceil(want / (8.0 * std::max(cols, 1)))));
                // staged tiles: a unit's tiles must fit the staging region
                const int rb_cols = std::max(1, cols);
                while (rpt > 1 && (double)rpt * rb_cols * 8.0 > lvl_stage * 0.98) rpt = (rpt + 1) / 2;
                for (auto& t : make_tasks(k, type, std::min(rows, rpt))) {
                    smax = std::max(smax, lvl_size(t));
                    stage_max = std::max<long long>(stage_max, (long long)t.ntiles * t.tile_d2 * 16);
                    units.push_back(t);
                }
            }
            lvl_smem.push_back(a16(smax));
        };
        const int dtop = lvl_max_depth >= 0 ? std::min(lvl_max_depth, maxdepth) : maxdepth;
        for (int d = dtop; d >= lvl_min_depth; --d) add_level(1, d);
        for (int d = lvl_min_depth; d <= dtop; ++d) add_level(2, d);
        lvl_off.push_back(static_cast<int>(units.size()));
        lvl_stage_bytes = static_cast<unsigned>((stage_max + 127) / 128 * 128);
        size_t smax = 0;
        for (size_t v : lvl_smem) smax = std::max(smax, v);
        lvl_staged = lvl_pf == 2 && smax + lvl_stage_bytes <= 226 * 1024;  // else tiles come from global memory
        require(smax <= 226 * 1024, "nested dissection: level unit buffer exceeds shared memory");
        tstore.alloc((size_t)std::max<long long>(toff, 1));
        {
            DBuf<TilePack> dp;
            dp.upload(packs, st);
            const long long np = static_cast<long long>(packs.size());
            for (long long o = 0; o < np; o += 65535) {
                const unsigned g = static_cast<unsigned>(std::min<long long>(65535, np - o));
                k_nd_tile_pack<<<g, 256, 0, st>>>(dp.p + o, store.p, tstore.p);
                PDG_CHECK_LAUNCH();
            }
            PDG_CUDA(cudaStreamSynchronize(st));
        }
        tile_bytes = 8.0 * (double)toff;
        d_ttasks.upload(units, st);
        d_toix.upload(oix, st);
        PDG_CUDA(cudaFuncSetAttribute(k_nd_level<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
        PDG_CUDA(cudaFuncSetAttribute(k_nd_level<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
        PDG_CUDA(cudaStreamSynchronize(st));
        (void)hbp;
        (void)cta_of;
        return;
    }
    for (int d = maxdepth; d >= 0; --d) place_level(1, d);
    for (int d = 0; d <= maxdepth; ++d) place_level(2, d);
    // dependencies: forward after both children's forward, backward after the parent's backward
    for (auto& v : per_cta)
        for (auto& t : v) {
            if (t.type == 1) {
                const auto& ch = children[t.front];
                if (ch.size() > 0) {
                    t.wait0 = 3 * ch[0] + 1;
                    t.need0 = ntask_of[3 * ch[0] + 1];
                }
                if (ch.size() > 1) {
                    t.wait1 = 3 * ch[1] + 1;
                    t.need1 = ntask_of[3 * ch[1] + 1];
                }
            } else {
                const int p = parent[t.front];
                t.wait0 = p >= 0 ? 3 * p + 2 : 3 * t.front + 1;
                t.need0 = p >= 0 ? ntask_of[3 * p + 2] : ntask_of[3 * t.front + 1];
            }
        }
    // completion counters one 128 B line apart: the pollers of one counter do not contend
    // with the completions of its neighbours
    constexpr int kCntStride = 16;
    for (auto& v : per_cta)
        for (auto& t : v) {
            t.signal *= kCntStride;
            if (t.wait0 >= 0) t.wait0 *= kCntStride;
            if (t.wait1 >= 0) t.wait1 *= kCntStride;
        }
    counters.alloc((size_t)3 * nf * kCntStride);
    counters.zero(st);
    // shared memory: header, task list, ring, arena (FIFO buffers placed here)
    tmax_tasks = 0;
    size_t max_buf = 0;
    for (auto& v : per_cta) {
        tmax_tasks = std::max(tmax_tasks, static_cast<int>(v.size()));
        for (auto& t : v) max_buf = std::max(max_buf, tb_size(t));
    }
    ttask_bytes = a16((size_t)tmax_tasks * sizeof(NdTileTask));
    const size_t limit = 227 * 1024;
    const size_t fixed = kTHeader + ttask_bytes + (size_t)tstages * tstage_bytes;
    require(fixed + 2 * max_buf <= limit, "nested dissection: tile solve does not fit in shared memory (" +
                                              std::to_string(fixed) + " + 2 x " + std::to_string(max_buf) + ")");
    tarena = (limit - fixed) / 128 * 128;
    tsmem = fixed + tarena;
    for (auto& v : per_cta) {
        size_t head = 0;
        int prev_dep = -1;
        for (int j = 0; j < static_cast<int>(v.size()); ++j) {
            const size_t sz = (tb_size(v[j]) + 127) / 128 * 128;
            if (head + sz > tarena) head = 0;
            v[j].boff = static_cast<int>(head);
            int dep = -1;
            for (int i = j - 1; i >= 0; --i) {
                const size_t lo = v[i].boff, hi = lo + (tb_size(v[i]) + 127) / 128 * 128;
                if (lo < head + sz && head < hi) {
                    dep = i;
                    break;
                }
            }
            v[j].fdep = prev_dep = std::max(dep, prev_dep);
            head += sz;
        }
    }
    std::vector<NdTileTask> all;
    std::vector<int> hct(tgrid + 1, 0);
    for (int q = 0; q < tgrid; ++q) {
        all.insert(all.end(), per_cta[q].begin(), per_cta[q].end());
        hct[q + 1] = static_cast<int>(all.size());
    }
    // repack the factor into tiles
    tstore.alloc((size_t)std::max<long long>(toff, 1));
    {
        DBuf<TilePack> dp;
        dp.upload(packs, st);
        const long long np = static_cast<long long>(packs.size());
        for (long long o = 0; o < np; o += 65535) {
            const unsigned g = static_cast<unsigned>(std::min<long long>(65535, np - o));
            k_nd_tile_pack<<<g, 256, 0, st>>>(dp.p + o, store.p, tstore.p);
            PDG_CHECK_LAUNCH();
        }
        PDG_CUDA(cudaStreamSynchronize(st));
    }
    tile_bytes = 8.0 * (double)toff;
    d_ttasks.upload(all, st);
    tctoff.upload(hct, st);
    d_toix.upload(oix, st);
    // the attribute is per device: set it on every build (cheap)
    // the attribute is per device and per function, shared by every instance: the full limit
    PDG_CUDA(cudaFuncSetAttribute(k_nd_tile_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(limit)));
    int per_sm = 0;
    PDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_nd_tile_solve, kTBlock, tsmem));
    require(per_sm >= 1 && tgrid <= per_sm * nsm, "nested dissection: tile solve grid not co-resident");
    (void)hbp;
    PDG_CUDA(cudaStreamSynchronize(st));
}

void NdChol::solve_levels(const double* b, long long ldb, double* x, long long ldx, int nrhs, cudaStream_t st) {
    solve_levels_range(b, ldb, x, ldx, nrhs, 0, static_cast<int>(lvl_smem.size()), st);
}

// level kernels l0..l1-1 (the forward levels are the first half of the list, the backward the second)
void NdChol::solve_levels_range(const double* b, long long ldb, double* x, long long ldx, int nrhs, int l0, int l1,
                                cudaStream_t st) {
    TileArgs a{};
    a.tasks = d_ttasks.p;
    a.toix = d_toix.p;
    a.sdofs = sdofs.p;
    a.bpos = bpos.p;
    a.tstore = tstore.p;
    a.b = b;
    a.ldb = ldb;
    a.x = x;
    a.ldx = ldx;
    a.y = y.p;
    a.xpos = xpos.p;
    a.cb = cbuf.p;
    a.cbtot = cbtot;
    a.n = n;
    a.nrhs = nrhs;
    a.stop = guard;
    const int pf = lvl_pf == 2 && !lvl_staged ? 1 : lvl_pf;
    a.stage_bytes = pf == 2 ? lvl_stage_bytes : 0;
    static const int bpsm = std::getenv("PDG_ND_LVL_BLOCKS") ? std::max(1, std::atoi(std::getenv("PDG_ND_LVL_BLOCKS"))) : 8;
    static const int use_pdl = !(std::getenv("PDG_ND_LVL_PDL") && std::atoi(std::getenv("PDG_ND_LVL_PDL")) == 0);
    const int nl = static_cast<int>(lvl_smem.size());
    const bool dbg_on = std::getenv("PDG_ND_DEBUG") != nullptr;
    DBuf<unsigned long long> dbg;
    if (dbg_on) {
        std::vector<unsigned long long> init(3 * nl, 0ull);
        for (int l = 0; l < nl; ++l) init[3 * l] = ~0ull;
        dbg.upload(init, st);
        a.dbg = dbg.p;
    }
    for (int l = l0; l < l1; ++l) {
        int u0 = lvl_off[l], u1 = lvl_off[l + 1];
        if (u1 <= u0) continue;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(std::min(u1 - u0, bpsm * tgrid)));
        cfg.blockDim = dim3(kLvlThreads);
        cfg.dynamicSmemBytes = lvl_smem[l] + a.stage_bytes;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = use_pdl ? 1 : 0;
        int p = pf;
        if (p == 2)
            PDG_CUDA(cudaLaunchKernelEx(&cfg, k_nd_level<true>, a, u0, u1, p, l));
        else
            PDG_CUDA(cudaLaunchKernelEx(&cfg, k_nd_level<false>, a, u0, u1, p, l));
        count_launch(1);
    }
    PDG_CHECK_LAUNCH();
    if (dbg_on) {
        const std::vector<unsigned long long> h = dbg.download(st);
        unsigned long long t00 = ~0ull;
        for (int l = l0; l < l1; ++l) t00 = std::min(t00, h[3 * l]);
        std::fprintf(stderr, "nd level solve n=%d levels=%d (%d..%d)\n", n, nl, l0, l1 - 1);
        for (int l = l0; l < l1; ++l) {
            double mb = 0.0;
            const std::vector<NdTileTask> ts = d_ttasks.download(st);
            for (int u = lvl_off[l]; u < lvl_off[l + 1]; ++u) mb += 16e-6 * ts[u].ntiles * ts[u].tile_d2;
            std::fprintf(stderr, "  level %2d units %5d %7.2f MB  start %8.2f  end %8.2f  (%6.2f us)\n", l,
                         lvl_off[l + 1] - lvl_off[l], mb, (h[3 * l] - t00) * 1e-3, (h[3 * l + 1] - t00) * 1e-3,
                         (h[3 * l + 1] - h[3 * l]) * 1e-3);
        }
    }
}

void NdChol::solve_tiles(const double* b, long long ldb, double* x, long long ldx, int nrhs, cudaStream_t st) {
    TileArgs a{};
    a.tasks = d_ttasks.p;
    a.ctoff = tctoff.p;
    a.toix = d_toix.p;
    a.sdofs = sdofs.p;
    a.bpos = bpos.p;
    a.tstore = tstore.p;
    a.b = b;
    a.ldb = ldb;
    a.x = x;
    a.ldx = ldx;
    a.y = y.p;
    a.xpos = xpos.p;
    a.cb = cbuf.p;
    a.cnt = counters.p;
    a.call = call;
    a.cbtot = cbtot;
    a.n = n;
    a.nrhs = nrhs;
    a.stages = tstages;
    a.max_tasks = tmax_tasks;
    a.stage_bytes = tstage_bytes;
    a.task_bytes = ttask_bytes;
    a.stop = guard;
    a.nodep = std::getenv("PDG_ND_NODEP") != nullptr;
    a.fence = std::getenv("PDG_ND_FENCE") != nullptr;
    a.backoff = 64;
    a.nostream = std::getenv("PDG_ND_NOSTREAM") != nullptr;
    a.evict_first = std::getenv("PDG_ND_EVICT_NORMAL") == nullptr;
    a.pf_shared = 256 * 1024;
    a.pf_local = 0;
    if (const char* e = std::getenv("PDG_ND_PF_SHARED_KB")) a.pf_shared = 1024LL * std::max(0, std::atoi(e));
    if (const char* e = std::getenv("PDG_ND_PF_LOCAL_KB")) a.pf_local = 1024LL * std::max(0, std::atoi(e));
    if (const char* e = std::getenv("PDG_ND_BACKOFF")) a.backoff = static_cast<unsigned>(std::max(0, std::atoi(e)));
    const bool debug = std::getenv("PDG_ND_DEBUG") != nullptr;
    const long long ntask = static_cast<long long>(d_ttasks.n);
    DBuf<unsigned long long> dbg;
    if (debug) {
        dbg.alloc((size_t)ntask * 8);
        dbg.zero(st);
        a.dbg = dbg.p;
    }
    void* args[] = {&a};
    PDG_CUDA(cudaLaunchCooperativeKernel((void*)k_nd_tile_solve, tgrid, kTBlock, args, tsmem, st));
    count_launch(1);
    PDG_CHECK_LAUNCH();
    if (debug) {
        const std::vector<unsigned long long> h = dbg.download(st);
        const std::vector<NdTileTask> ts = d_ttasks.download(st);
        unsigned long long t00 = ~0ull, tend = 0;
        for (long long i = 0; i < ntask; ++i) {
            t00 = std::min(t00, h[8 * i + 4]);
            tend = std::max(tend, h[8 * i + 3]);
        }
        std::fprintf(stderr,
                     "nd solve n=%d fronts=%d depth=%d tasks=%lld grid=%d max/cta=%d stages=%d x %u B arena=%zu tile store %.1f MB "
                     "total %.2f us\n",
                     n, nfront, maxdepth, ntask, tgrid, tmax_tasks, tstages, tstage_bytes, tarena, tile_bytes * 1e-6,
                     (tend - t00) * 1e-3);
        std::fprintf(stderr, "  (per task: start = buffer free; deps = dependencies met; ready = inputs gathered)\n");
        for (int type = 1; type < 3; ++type)
            for (int d = maxdepth; d >= 0; --d) {
                const int dd = type == 2 ? maxdepth - d : d;
                unsigned long long s0 = ~0ull, dm = ~0ull, r0 = ~0ull, e1 = 0, wdep = 0, gat = 0, comp = 0, sig = 0;
                double mb = 0.0;
                int cntk = 0;
                for (long long i = 0; i < ntask; ++i)
                    if (ts[i].type == type && fronts[ts[i].front].depth == dd) {
                        const unsigned long long* q = &h[8 * i];
                        s0 = std::min(s0, q[4]);
                        dm = std::min(dm, q[5]);
                        r0 = std::min(r0, q[0]);
                        e1 = std::max(e1, q[3]);
                        wdep += q[5] - q[4];
                        gat += q[0] - q[5];
                        comp += q[2] - q[1];
                        sig += q[3] - q[2];
                        mb += 16e-6 * ts[i].ntiles * ts[i].tile_d2;
                        ++cntk;
                    }
                if (cntk)
                    std::fprintf(stderr,
                                 "  %s d%2d tasks %5d %7.2f MB  first start %7.2f deps %7.2f ready %7.2f  last signal %7.2f | "
                                 "avg start->deps %5.2f deps->ready %5.2f compute %5.2f done->signal %5.2f us\n",
                                 type == 1 ? "fwd" : "bwd", dd, cntk, mb, (s0 - t00) * 1e-3, (dm - t00) * 1e-3,
                                 (r0 - t00) * 1e-3, (e1 - t00) * 1e-3, wdep * 1e-3 / cntk, gat * 1e-3 / cntk,
                                 comp * 1e-3 / cntk, sig * 1e-3 / cntk);
            }
    }
}

}  // namespace pdg
