// Streaming mode of the nested-dissection solve (NdChol::stream): for factors whose
// fronts are too wide for the shared-memory dataflow kernels (nd.cu, nd_tile.cu) -- the
// 3D meshes of BASELINE config 2, where the top separator of 32^3 cells has 24,576 dofs
// and the factor is ~80 GB. Same math as the other solve paths (the exact inner solves of
// fixed_stress.hpp:109-139):
//   forward   [y_S; u_F] = M (b_S - w_C1|S - w_C2|S),  w_F = u_F + w_C1|B + w_C2|B
//   backward  x_S = M^T [y_S; -x_B]
// One launch per tree level and pass (stream order carries the dependencies; at these
// sizes a level streams 1-15 GB, so launch gaps are noise). A CTA takes a unit = 64 rows
// of one front's M (or M^T), read straight from the row-major factor store with 16-byte
// streaming loads, 8 rows per warp in flight at once; the front's input vector is formed
// on the fly (right-hand side minus the children's update vectors, or [y_S; -x_B]) and
// staged through shared memory in tiles of 2048 columns shared by the CTA's 64 rows, so
// its L2 traffic is 1/64 of the factor traffic. The zero triangle of L_SS^{-1} is skipped
// (per unit a column range). Sums run in a fixed order: repeats are bit-identical.
// HBM-bound: algorithmic bytes = the nonzero part of the factor once per pass.
#include <algorithm>
#include <cstdlib>

#include "nd.cuh"

namespace pdg {

namespace {

constexpr int kSRows = 64;     // rows per unit (8 warps x 8 rows)
constexpr int kSTile = 2048;   // columns per shared-memory tile
constexpr int kSThreads = 256;

struct StreamArgs {
    const NdStreamUnit* units;
    const int* sdofs;
    const int* bpos;
    const int* cbdst;
    const double* store;
    const float* store32;  // fast mode: the factor stored in fp32 (store is null)
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

// 16-byte packets of the factor store: 2 fp64 or (fast mode) 4 fp32 entries; sums in fp64
template <typename T>
struct Pkt;
template <>
struct Pkt<double> {
    using V = double2;
    static constexpr int N = 2;
    static __device__ __forceinline__ double mac(const V& m, const double* v, double acc) {
        const double2 w = *reinterpret_cast<const double2*>(v);
        return fma(m.y, w.y, fma(m.x, w.x, acc));
    }
};
template <>
struct Pkt<float> {
    using V = float4;
    static constexpr int N = 4;
    static __device__ __forceinline__ double mac(const V& m, const double* v, double acc) {
        const double2 w0 = *reinterpret_cast<const double2*>(v), w1 = *reinterpret_cast<const double2*>(v + 2);
        return fma((double)m.w, w1.y, fma((double)m.z, w1.x, fma((double)m.y, w0.y, fma((double)m.x, w0.x, acc))));
    }
};

// RPW rows per warp: a unit has up to 8 * RPW rows (64 by default; 32 or 16 on levels with few
// units, where more CTAs keep more bytes in flight)
template <int NR, int RPW, typename T>
__global__ void __launch_bounds__(kSThreads, 4) k_nd_stream(StreamArgs a, int u0) {
    using P = Pkt<T>;
    using V = typename P::V;
    constexpr int PN = P::N;
    if (a.stop && *a.stop) return;  // speculative GMRES step after the cycle ended
    __shared__ double vs[NR][kSTile];
    __shared__ NdStreamUnit Us;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid < (int)(sizeof(NdStreamUnit) / 4))
        reinterpret_cast<int*>(&Us)[tid] = __ldg(reinterpret_cast<const int*>(a.units + u0 + blockIdx.x) + tid);
    __syncthreads();
    const NdStreamUnit& U = Us;
    const int fwd = U.type == 1;
    const int sb = U.s + U.b;
    double acc[RPW][NR];
#pragma unroll
    for (int j = 0; j < RPW; ++j)
#pragma unroll
        for (int k = 0; k < NR; ++k) acc[j][k] = 0.0;
    const int rw = warp * RPW;  // this warp's first row within the unit
    const T* store = sizeof(T) == 8 ? reinterpret_cast<const T*>(a.store) : reinterpret_cast<const T*>(a.store32);
    const T* rowp = store + U.src + (long long)(U.r0 + rw) * U.ld;
    for (int c0 = U.cbeg; c0 < U.ncols; c0 += kSTile) {
        const int nc = min(kSTile, U.ncols - c0);
        // ---- the input vector tile ----
        for (int c = tid; c < ((nc + PN - 1) & ~(PN - 1)); c += kSThreads) {
            const int gc = c0 + c;
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                double v = 0.0;
                if (c < nc) {
                    if (fwd) {
                        const double* cbk = a.cb + k * a.cbtot + U.cboff;
                        v = (a.b[k * a.ldb + __ldg(a.sdofs + U.sdof + gc)] - __ldcg(cbk + gc)) - __ldcg(cbk + sb + gc);
                    } else {
                        v = gc < U.s ? __ldcg(a.y + (long long)k * a.n + U.sdof + gc)
                                     : -__ldcg(a.xpos + (long long)k * a.n + __ldg(a.bpos + U.bdof + gc - U.s));
                    }
                }
                vs[k][c] = v;
            }
        }
        __syncthreads();
        // ---- RPW rows per warp against the tile ----
        const int np = (nc + PN - 1) / PN;
        const int nrw = min(RPW, U.nrows - rw);  // rows of this warp (<= 0: none)
        if (nrw == RPW) {
            constexpr int UN = 8 / RPW;  // 8 16-byte loads in flight per lane
            int p = lane;
            if constexpr (UN > 1)
            for (; p + 32 * (UN - 1) < np; p += 32 * UN) {
                V m[UN][RPW];
#pragma unroll
                for (int q = 0; q < UN; ++q)
#pragma unroll
                    for (int j = 0; j < RPW; ++j)
                        m[q][j] = __ldcs(reinterpret_cast<const V*>(rowp + (long long)j * U.ld + c0) + p + 32 * q);
#pragma unroll
                for (int q = 0; q < UN; ++q)
#pragma unroll
                    for (int k = 0; k < NR; ++k) {
#pragma unroll
                        for (int j = 0; j < RPW; ++j) acc[j][k] = P::mac(m[q][j], &vs[k][PN * (p + 32 * q)], acc[j][k]);
                    }
            }
            for (; p < np; p += 32) {
                V m[RPW];
#pragma unroll
                for (int j = 0; j < RPW; ++j) m[j] = __ldcs(reinterpret_cast<const V*>(rowp + (long long)j * U.ld + c0) + p);
#pragma unroll
                for (int k = 0; k < NR; ++k) {
#pragma unroll
                    for (int j = 0; j < RPW; ++j) acc[j][k] = P::mac(m[j], &vs[k][PN * p], acc[j][k]);
                }
            }
        } else if (nrw > 0) {
            for (int p = lane; p < np; p += 32) {
#pragma unroll
                for (int j = 0; j < RPW; ++j) {
                    if (j < nrw) {
                        const V mv = __ldcs(reinterpret_cast<const V*>(rowp + (long long)j * U.ld + c0) + p);
#pragma unroll
                        for (int k = 0; k < NR; ++k) acc[j][k] = P::mac(mv, &vs[k][PN * p], acc[j][k]);
                    }
                }
            }
        }
        __syncthreads();
    }
    // ---- row sums (fixed butterfly) and outputs ----
#pragma unroll
    for (int j = 0; j < RPW; ++j)
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            double s = acc[j][k];
            for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            acc[j][k] = s;
        }
    if (lane < RPW && rw + lane < U.nrows) {
        const int gr = U.r0 + rw + lane;
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < RPW; ++j)
                if (j == lane) s = acc[j][k];
            if (!fwd) {
                a.xpos[(long long)k * a.n + U.sdof + gr] = s;
                a.x[k * a.ldx + __ldg(a.sdofs + U.sdof + gr)] = s;
            } else if (gr < U.s) {
                a.y[(long long)k * a.n + U.sdof + gr] = s;
            } else {  // update vector entry plus the children's pass-through, into the parent's slot
                const double* cbk = a.cb + k * a.cbtot + U.cboff;
                const double tail = __ldcg(cbk + gr) + __ldcg(cbk + sb + gr);
                a.cb[k * a.cbtot + __ldg(a.cbdst + U.bdof + gr - U.s)] = s + tail;
            }
        }
    }
}

}  // namespace

// Units per (pass, depth): forward levels deepest first, then backward levels root first.
void NdChol::build_stream(cudaStream_t st) {
    std::vector<NdStreamUnit> units;
    double read_bytes = 0.0;
    stream_off.clear();
    stream_rpw.clear();
    const int want = std::getenv("PDG_ND_STREAM_UNITS") ? std::atoi(std::getenv("PDG_ND_STREAM_UNITS")) : 3000;
    auto add_level = [&](int type, int depth) {
        stream_off.push_back(static_cast<int>(units.size()));
        // rows per unit: 64, or 32 / 16 while the level has fewer than `want` units
        long long rows_tot = 0;
        for (int k = 0; k < nfront; ++k)
            if (fronts[k].depth == depth) rows_tot += type == 1 ? fronts[k].s + fronts[k].b : fronts[k].s;
        int rpu = kSRows;
        while (rpu > 16 && rows_tot / rpu < want) rpu /= 2;
        stream_rpw.push_back(rpu / 8);
        for (int k = 0; k < nfront; ++k) {
            const NdFront& F = fronts[k];
            if (F.depth != depth) continue;
            const int rows = type == 1 ? F.s + F.b : F.s;
            for (int r0 = 0; r0 < rows; r0 += rpu) {
                NdStreamUnit u{};
                u.src = type == 1 ? F.moff : F.mtoff;
                u.type = type;
                u.r0 = r0;
                u.nrows = std::min(rpu, rows - r0);
                // L_SS^{-1} is lower triangular: a forward row r < s has entries in columns <= r, a
                // backward row r (of L_SS^{-T} | G^T) in columns >= r; the exact zeros are not read
                u.ncols = type == 1 ? (r0 + u.nrows <= F.s ? r0 + u.nrows : F.s) : F.s + F.b;
                u.cbeg = type == 1 ? 0 : (fp32 ? (r0 & ~3) : (r0 & ~1));
                read_bytes += (fp32 ? 4.0 : 8.0) * u.nrows * (u.ncols - u.cbeg);
                u.ld = type == 1 ? F.ldm : F.ldt;
                u.s = F.s;
                u.b = F.b;
                u.sdof = F.sdof;
                u.bdof = F.bdof;
                u.cboff = F.cboff;
                units.push_back(u);
            }
        }
    };
    for (int d = maxdepth; d >= 0; --d) add_level(1, d);
    for (int d = 0; d <= maxdepth; ++d) add_level(2, d);
    stream_off.push_back(static_cast<int>(units.size()));
    factor_bytes = read_bytes;  // what a solve streams: the nonzero parts of M and M^T once each
    d_sunits.upload(units, st);
    PDG_CUDA(cudaStreamSynchronize(st));
}

void NdChol::solve_stream(const double* b, long long ldb, double* x, long long ldx, int nrhs, cudaStream_t st) {
    StreamArgs a{d_sunits.p, sdofs.p, bpos.p, cbdst.p, store.p, store32.p, b, ldb, x, ldx, y.p, xpos.p, cbuf.p, cbtot, n, guard};
    const int nl = static_cast<int>(stream_off.size()) - 1;
    auto launch = [&](auto tag, int nu, int u0, int rpw) {
        using T = decltype(tag);
        if (nrhs == 1) {
            if (rpw == 8) k_nd_stream<1, 8, T><<<nu, kSThreads, 0, st>>>(a, u0);
            else if (rpw == 4) k_nd_stream<1, 4, T><<<nu, kSThreads, 0, st>>>(a, u0);
            else k_nd_stream<1, 2, T><<<nu, kSThreads, 0, st>>>(a, u0);
        } else {
            if (rpw == 8) k_nd_stream<2, 8, T><<<nu, kSThreads, 0, st>>>(a, u0);
            else if (rpw == 4) k_nd_stream<2, 4, T><<<nu, kSThreads, 0, st>>>(a, u0);
            else k_nd_stream<2, 2, T><<<nu, kSThreads, 0, st>>>(a, u0);
        }
    };
    for (int l = 0; l < nl; ++l) {
        const int u0 = stream_off[l], nu = stream_off[l + 1] - u0;
        if (nu == 0) continue;
        if (fp32)
            launch(float{}, nu, u0, stream_rpw[l]);
        else
            launch(double{}, nu, u0, stream_rpw[l]);
        count_launch(1);
    }
    PDG_CHECK_LAUNCH();
}

}  // namespace pdg
