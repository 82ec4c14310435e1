// Build and order-fixed SpMV of the canonical assembled space-time operator.
//
// Canonical operator (the matrix the reference's direct block path forms at
// slab.hpp:146-153, mat(bi,bj) = T(bi,bj) D + [bi==bj] tau K), layout
// [u_0 q_0 p_0 | u_1 q_1 p_1]. Entry values:
//   u-row  : tau*a (u_i), tau*((-b)*e) (p_i)
//   q-row  : tau*mq (q_i), tau*bv (p_i)
//   p-row  : for j: theta_ij*((-b)*e) (u_j), [j==i] tau*bv (q_i), theta_ij*((-(1/M))*m_p) (p_j)
#include <cstdlib>
#include <cub/cub.cuh>

#include "ops.cuh"
#include "spacetime_op.cuh"

namespace pdg {

namespace {

struct Theta {
    double t[4];
    double w[2];  // tau * kappa_i per component (fixed_stress.hpp:50; kappa = 1 in the slab solver)
};

// ---- U class ---------------------------------------------------------------
__global__ void k_u_count(int n_cells, const int* __restrict__ a_off, const int* __restrict__ e_off, int m,
                          long long* cnt) {
    for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < (long long)m * n_cells;
         g += (long long)gridDim.x * blockDim.x) {
        const int c = static_cast<int>(g % n_cells);
        const int r = 8 * c;
        cnt[g] = (a_off[r + 1] - a_off[r]) + (e_off[r + 1] - e_off[r]);
    }
}

__global__ void k_u_fill(int n_cells, int m, int nt, int nu, int nq, Theta th, double mb, const int* __restrict__ a_off,
                         const int* __restrict__ a_idx, const double* __restrict__ a_val, const int* __restrict__ e_off,
                         const int* __restrict__ e_idx, const double* __restrict__ e_val, const long long* __restrict__ u_off,
                         int* u_col, double* u_val, int* err) {
    const long long total = (long long)m * n_cells * 8;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
        const long long g = t >> 3;
        const int l = static_cast<int>(t & 7);
        const int i = static_cast<int>(g / n_cells);
        const int c = static_cast<int>(g % n_cells);
        const int r = 8 * c + l, r0 = 8 * c;
        const int la = a_off[r + 1] - a_off[r], le = e_off[r + 1] - e_off[r];
        if (la != a_off[r0 + 1] - a_off[r0] || le != e_off[r0 + 1] - e_off[r0]) {
            atomicOr(err, 1);
            continue;
        }
        long long k = u_off[g];
        for (int q = 0; q < la; ++q, ++k) {
            const int col = a_idx[a_off[r] + q];
            if (col != a_idx[a_off[r0] + q]) atomicOr(err, 2);
            u_val[k * 8 + l] = __dmul_rn(th.w[i], a_val[a_off[r] + q]);
            if (l == 0) u_col[k] = i * nt + col;
        }
        for (int q = 0; q < le; ++q, ++k) {
            const int col = e_idx[e_off[r] + q];
            if (col != e_idx[e_off[r0] + q]) atomicOr(err, 2);
            u_val[k * 8 + l] = __dmul_rn(th.w[i], __dmul_rn(mb, e_val[e_off[r] + q]));
            if (l == 0) u_col[k] = i * nt + nu + nq + col;
        }
    }
}

// ---- S class (q- and p-rows, SELL-32) ----------------------------------------
__device__ __forceinline__ int s_row_len(long long s, int m, int nq, int np, Theta th, const int* mq_off, const int* b_off,
                                         const int* et_off, const int* bt_off) {
    const int i = static_cast<int>(s / (nq + np));
    const int loc = static_cast<int>(s % (nq + np));
    if (loc < nq) return (mq_off[loc + 1] - mq_off[loc]) + (b_off[loc + 1] - b_off[loc]);
    const int c = loc - nq;
    int len = bt_off[c + 1] - bt_off[c];
    for (int j = 0; j < m; ++j)
        if (th.t[i * m + j] != 0.0) len += (et_off[c + 1] - et_off[c]) + 1;
    return len;
}

__global__ void k_s_len(long long s_rows, int m, int nq, int np, Theta th, const int* mq_off, const int* b_off,
                        const int* et_off, const int* bt_off, int* s_len) {
    for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < s_rows; s += (long long)gridDim.x * blockDim.x)
        s_len[s] = s_row_len(s, m, nq, np, th, mq_off, b_off, et_off, bt_off);
}

__global__ void k_s_slice_width(long long s_rows, long long n_slices, const int* s_len, long long* w) {
    for (long long sl = blockIdx.x * (long long)blockDim.x + threadIdx.x; sl < n_slices; sl += (long long)gridDim.x * blockDim.x) {
        int mx = 0;
        for (int l = 0; l < 32; ++l) {
            const long long s = sl * 32 + l;
            if (s < s_rows) mx = max(mx, s_len[s]);
        }
        w[sl] = mx;
    }
}

__global__ void k_s_fill(long long s_rows, int m, int nt, int nu, int nq, int np, double tau, double mb, double minv, Theta th,
                         const int* mq_off, const int* mq_idx, const double* mq_val, const int* b_off, const int* b_idx,
                         const double* b_val, const int* et_off, const int* et_idx, const double* et_val, const int* bt_off,
                         const int* bt_idx, const double* bt_val, const double* m_p, const long long* s_off, int* s_col,
                         double* s_val) {
    for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < s_rows; s += (long long)gridDim.x * blockDim.x) {
        const long long sl = s >> 5;
        const int lane = static_cast<int>(s & 31);
        long long k = s_off[sl];
        const int i = static_cast<int>(s / (nq + np));
        const int loc = static_cast<int>(s % (nq + np));
        auto put = [&](int col, double v) {
            s_col[k * 32 + lane] = col;
            s_val[k * 32 + lane] = v;
            ++k;
        };
        if (loc < nq) {
            const int f = loc;
            for (int q = mq_off[f]; q < mq_off[f + 1]; ++q) put(i * nt + nu + mq_idx[q], __dmul_rn(th.w[i], mq_val[q]));
            for (int q = b_off[f]; q < b_off[f + 1]; ++q) put(i * nt + nu + nq + b_idx[q], __dmul_rn(th.w[i], b_val[q]));
        } else {
            const int c = loc - nq;
            for (int j = 0; j < m; ++j) {
                const double t = th.t[i * m + j];
                if (t != 0.0)
                    for (int q = et_off[c]; q < et_off[c + 1]; ++q)
                        put(j * nt + et_idx[q], __dmul_rn(t, __dmul_rn(mb, et_val[q])));
                if (j == i)
                    for (int q = bt_off[c]; q < bt_off[c + 1]; ++q)
                        put(i * nt + nu + bt_idx[q], __dmul_rn(th.w[i], bt_val[q]));
                if (t != 0.0) put(j * nt + nu + nq + c, __dmul_rn(t, __dmul_rn(minv, m_p[c])));
            }
        }
        // pad the slice with explicit zeros (never read: the kernel stops at s_len)
        const long long end = s_off[sl + 1];
        for (; k < end; ++k) {
            s_col[k * 32 + lane] = 0;
            s_val[k * 32 + lane] = 0.0;
        }
    }
}

// ---- SpMV ---------------------------------------------------------------------
// Blocks [0, gu) run the U class (one thread per (group,row)), the remaining
// blocks the S class (one thread per row).
constexpr int kSpmvBlock = 256;
constexpr int kSpmvMaxDots = 8;  // fused Gram-Schmidt pass-1 dots: up to 8 basis vectors

// DOTS (the GMRES operator application, north_star "SpMV fused with the GMRES dot
// products"): y is also copied to y2 (the Gram-Schmidt work vector) and every block
// writes its partial sums of V_j . y over the rows it produced, j < ncols <= 8
// (partial[block][j], block-order summed by the Arnoldi kernel). y itself is computed
// exactly as without DOTS (bit-identical).
template <bool DOTS>
__global__ void __launch_bounds__(kSpmvBlock) k_spmv(long long u_threads, int u2, long long s_rows, int gu, int n_cells, int nt,
                                                     int nu, int nq, int np, const long long* __restrict__ u_off,
                                                     const int* __restrict__ u_col, const double* __restrict__ u_val,
                                                     const long long* __restrict__ s_off, const int* __restrict__ s_len,
                                                     const int* __restrict__ s_col, const double* __restrict__ s_val,
                                                     const double* __restrict__ x, double* __restrict__ y,
                                                     const int* __restrict__ stop, const double* __restrict__ V, int ncols,
                                                     long long nrows, double* __restrict__ y2, double* __restrict__ partial) {
    if (stop && *stop) return;
    double acc[kSpmvMaxDots];
#pragma unroll
    for (int q = 0; q < kSpmvMaxDots; ++q) acc[q] = 0.0;
    auto dots = [&](long long row, double v) {
        if (DOTS) {
            if (y2) y2[row] = v;
#pragma unroll
            for (int q = 0; q < kSpmvMaxDots; ++q)
                if (q < ncols) acc[q] += __ldg(&V[(long long)q * nrows + row]) * v;
        }
    };
    if (static_cast<int>(blockIdx.x) < gu) {
        const long long stride = (long long)gu * blockDim.x;
        if (!u2) {  // one row per thread (large operators: more independent streams in flight)
            for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < u_threads; t += stride) {
                const long long g = t >> 3;
                const int l = static_cast<int>(t & 7);
                const long long b = __ldg(&u_off[g]), e = __ldg(&u_off[g + 1]);
                double s = 0.0;
#pragma unroll 8
                for (long long k = b; k < e; ++k) {
                    const double v = __ldcs(&u_val[k * 8 + l]);
                    const double xv = __ldg(&x[__ldg(&u_col[k])]);
                    s = __dadd_rn(s, __dmul_rn(v, xv));
                }
                const int i = static_cast<int>(g / n_cells);
                const int c = static_cast<int>(g - (long long)i * n_cells);
                const long long row = (long long)i * nt + 8 * c + l;
                y[row] = s;
                dots(row, s);
            }
        } else {
            // two rows (2j, 2j+1) of a group per thread (small operators: the grid fits one wave):
            // one column index and one x load serve both, values as one 16-byte load; each row
            // still summed alone in stored order
            const double2* __restrict__ uv2 = reinterpret_cast<const double2*>(u_val);
            for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < u_threads; t += stride) {
                const long long g = t >> 2;
                const int j = static_cast<int>(t & 3);
                const long long b = __ldg(&u_off[g]), e = __ldg(&u_off[g + 1]);
                double s0 = 0.0, s1 = 0.0;
#pragma unroll 8
                for (long long k = b; k < e; ++k) {
                    const double2 v = __ldcs(&uv2[k * 4 + j]);
                    const double xv = __ldg(&x[__ldg(&u_col[k])]);
                    s0 = __dadd_rn(s0, __dmul_rn(v.x, xv));
                    s1 = __dadd_rn(s1, __dmul_rn(v.y, xv));
                }
                const int i = static_cast<int>(g / n_cells);
                const int c = static_cast<int>(g - (long long)i * n_cells);
                const long long row = (long long)i * nt + 8 * c + 2 * j;
                y[row] = s0;
                y[row + 1] = s1;
                dots(row, s0);
                dots(row + 1, s1);
            }
        }
    } else {
        const int bid = blockIdx.x - gu;
        const long long stride = (long long)(gridDim.x - gu) * blockDim.x;
        for (long long srow = bid * (long long)blockDim.x + threadIdx.x; srow < s_rows; srow += stride) {
            const long long b = __ldg(&s_off[srow >> 5]);
            const int lane = static_cast<int>(srow & 31);
            const int len = __ldg(&s_len[srow]);
            double s = 0.0;
#pragma unroll 4
            for (int k = 0; k < len; ++k) {
                const long long pos = (b + k) * 32 + lane;
                const double v = __ldcs(&s_val[pos]);
                const double xv = __ldg(&x[__ldcs(&s_col[pos])]);
                s = __dadd_rn(s, __dmul_rn(v, xv));
            }
            const int i = static_cast<int>(srow / (nq + np));
            const int loc = static_cast<int>(srow - (long long)i * (nq + np));
            const long long row = (long long)i * nt + nu + loc;
            y[row] = s;
            dots(row, s);
        }
    }
    if (DOTS) {  // block partials, fixed order: warp butterflies, then the warps in order
        __shared__ double sh[kSpmvMaxDots][kSpmvBlock / 32];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
        for (int q = 0; q < kSpmvMaxDots; ++q)
            for (int o = 16; o; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < kSpmvMaxDots; ++q) sh[q][warp] = acc[q];
        __syncthreads();
        if (threadIdx.x < ncols) {
            double t = 0.0;
            for (int w = 0; w < kSpmvBlock / 32; ++w) t += sh[threadIdx.x][w];
            partial[(long long)blockIdx.x * ncols + threadIdx.x] = t;
        }
    }
}

// Owned-row test of an S-class row for the strip of cell rows [r0, r1):
// flux rows by face row (horizontal faces level j -> row min(j, ny-1), vertical
// faces column-major -> their row, mesh.hpp:59-60), pressure rows by cell row.
__device__ __forceinline__ bool s_row_owned(long long srow, int nq, int np, int nx, int ny, int r0, int r1) {
    const int loc = static_cast<int>(srow % (nq + np));
    int row;
    if (loc < nq) {
        const int nh = nx * (ny + 1);
        row = loc < nh ? min(loc / nx, ny - 1) : (loc - nh) % ny;
    } else {
        row = (loc - nq) / nx;
    }
    return row >= r0 && row < r1;
}

// k_spmv restricted to a strip: U groups of the strip's cells (every component),
// the listed S slices, writes masked to owned rows.
__global__ void __launch_bounds__(kSpmvBlock) k_spmv_strip(long long u_threads, int cell0, int ncells_strip, int gu,
                                                           long long n_slices, const long long* __restrict__ slices,
                                                           long long s_rows,
                                                           int n_cells, int nt, int nu, int nq, int np, int nx, int ny,
                                                           int r0, int r1, const long long* __restrict__ u_off,
                                                           const int* __restrict__ u_col, const double* __restrict__ u_val,
                                                           const long long* __restrict__ s_off, const int* __restrict__ s_len,
                                                           const int* __restrict__ s_col, const double* __restrict__ s_val,
                                                           const double* __restrict__ x, double* __restrict__ y,
                                                     const int* __restrict__ stop) {
    if (stop && *stop) return;
    if (static_cast<int>(blockIdx.x) < gu) {
        const long long stride = (long long)gu * blockDim.x;
        for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < u_threads; t += stride) {
            const long long gl = t >> 3;  // local group: component-major over the strip's cells
            const int l = static_cast<int>(t & 7);
            const int i = static_cast<int>(gl / ncells_strip);
            const int c = cell0 + static_cast<int>(gl % ncells_strip);
            const long long g = (long long)i * n_cells + c;
            const long long b = __ldg(&u_off[g]), e = __ldg(&u_off[g + 1]);
            double s = 0.0;
#pragma unroll 8
            for (long long k = b; k < e; ++k) {
                const double v = __ldcs(&u_val[k * 8 + l]);
                const double xv = __ldg(&x[__ldg(&u_col[k])]);
                s = __dadd_rn(s, __dmul_rn(v, xv));
            }
            y[(long long)i * nt + 8 * c + l] = s;
        }
    } else {
        const int bid = blockIdx.x - gu;
        const long long stride = (long long)(gridDim.x - gu) * blockDim.x;
        for (long long t = bid * (long long)blockDim.x + threadIdx.x; t < n_slices * 32; t += stride) {
            const long long sl = __ldg(&slices[t >> 5]);
            const int lane = static_cast<int>(t & 31);
            const long long srow = sl * 32 + lane;
            if (srow >= s_rows) continue;
            const long long b = __ldg(&s_off[sl]);
            const int len = __ldg(&s_len[srow]);
            double s = 0.0;
#pragma unroll 4
            for (int k = 0; k < len; ++k) {
                const long long pos = (b + k) * 32 + lane;
                const double v = __ldcs(&s_val[pos]);
                const double xv = __ldg(&x[__ldcs(&s_col[pos])]);
                s = __dadd_rn(s, __dmul_rn(v, xv));
            }
            if (s_row_owned(srow, nq, np, nx, ny, r0, r1)) {
                const int i = static_cast<int>(srow / (nq + np));
                const int loc = static_cast<int>(srow - (long long)i * (nq + np));
                y[(long long)i * nt + nu + loc] = s;
            }
        }
    }
}

}  // namespace

long long scan_ll(const long long* in, long long* out, long long n, cudaStream_t st) {
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n + 1, st);
    DBuf<unsigned char> buf(tmp + 1);
    cub::DeviceScan::ExclusiveSum(buf.p, tmp, in, out, n + 1, st);
    long long total = 0;
    PDG_CUDA(cudaMemcpyAsync(&total, out + n, sizeof(long long), cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    return total;
}

void SpaceTimeOp::build(const SpatialOps& ops, int m_, const double* theta, double tau, cudaStream_t st,
                        const double* kappa) {
    require(m_ == 1 || m_ == 2, "space-time block: m must be 1 or 2");
    m = m_;
    n_u = ops.n_u;
    n_q = ops.n_q;
    n_p = ops.n_p;
    n_cells = ops.n_p;
    nt = ops.n_total();
    rows = (long long)m * nt;
    Theta th{};
    for (int k = 0; k < m * m; ++k) th.t[k] = theta[k];
    for (int i = 0; i < m; ++i) th.w[i] = kappa ? tau * kappa[i] : tau;
    const double mb = -ops.biot_b, minv = -ops.inv_m;
    // U groups: 8 consecutive displacement rows sharing one column list (a 2D cell, or a third
    // of a 3D cell's 24 rows)
    require(ops.n_u % 8 == 0 && (ops.n_u == 8 * ops.n_p || ops.n_u == 24 * ops.n_p),
            "space-time block: n_u must be 8 or 24 times n_cells");
    n_ug = ops.n_u / 8;
    u_groups = (long long)m * n_ug;
    s_rows = (long long)m * (n_q + n_p);
    s_slices = (s_rows + 31) / 32;
    if (ops.n_u == 8 * ops.n_p && build_kp(ops, th.t, th.w, st)) return;

    // U class
    DBuf<long long> cnt(u_groups + 1);
    cnt.zero(st);
    k_u_count<<<grid_for(u_groups, 256), 256, 0, st>>>(n_ug, ops.A.off.p, ops.E.off.p, m, cnt.p);
    PDG_CHECK_LAUNCH();
    u_off.alloc(u_groups + 1);
    u_entries = scan_ll(cnt.p, u_off.p, u_groups, st);
    u_col.alloc(u_entries);
    u_val.alloc(8 * u_entries);
    DBuf<int> err(1);
    err.zero(st);
    k_u_fill<<<grid_for(u_groups * 8, 256), 256, 0, st>>>(n_ug, m, nt, n_u, n_q, th, mb, ops.A.off.p, ops.A.idx.p,
                                                           ops.A.val.p, ops.E.off.p, ops.E.idx.p, ops.E.val.p, u_off.p,
                                                           u_col.p, u_val.p, err.p);
    PDG_CHECK_LAUNCH();

    // S class
    s_len.alloc(s_rows);
    k_s_len<<<grid_for(s_rows, 256), 256, 0, st>>>(s_rows, m, n_q, n_p, th, ops.M_q.off.p, ops.B.off.p, ops.Et.off.p,
                                                    ops.Bt.off.p, s_len.p);
    PDG_CHECK_LAUNCH();
    DBuf<long long> w(s_slices + 1);
    w.zero(st);
    k_s_slice_width<<<grid_for(s_slices, 256), 256, 0, st>>>(s_rows, s_slices, s_len.p, w.p);
    PDG_CHECK_LAUNCH();
    s_off.alloc(s_slices + 1);
    s_slots = scan_ll(w.p, s_off.p, s_slices, st);
    s_col.alloc(32 * s_slots);
    s_val.alloc(32 * s_slots);
    k_s_fill<<<grid_for(s_rows, 256), 256, 0, st>>>(s_rows, m, nt, n_u, n_q, n_p, tau, mb, minv, th, ops.M_q.off.p,
                                                     ops.M_q.idx.p, ops.M_q.val.p, ops.B.off.p, ops.B.idx.p, ops.B.val.p,
                                                     ops.Et.off.p, ops.Et.idx.p, ops.Et.val.p, ops.Bt.off.p, ops.Bt.idx.p,
                                                     ops.Bt.val.p, ops.m_p.p, s_off.p, s_col.p, s_val.p);
    PDG_CHECK_LAUNCH();
    int herr = 0;
    PDG_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    require(herr == 0, "space-time block: displacement rows of a cell do not share one column pattern");
    // nnz of the canonical operator
    std::vector<int> lens = s_len.download(st);
    long long snnz = 0;
    for (int v : lens) snnz += v;
    nnz = 8 * u_entries + snnz;
}

void SpaceTimeOp::apply(const double* x, double* y, cudaStream_t st) const {
    ProfScope prof(PROF_SPMV, st, 8.0 * (double)(nnz + 2 * rows));
    if (kp) {
        kp_launch(x, y, nullptr, nullptr, 0, nullptr, false, st);
        return;
    }
    int u2 = rows <= (2LL << 20);  // two U rows per thread up to 2M rows (256^2 dG(1) and below)
    if (const char* e = std::getenv("PDG_SPMV_ROWS")) u2 = std::atoi(e) == 2;  // test override: 1 | 2
    const long long u_threads = u_groups * (u2 ? 4 : 8);
    const int gu = static_cast<int>(std::min<long long>((u_threads + kSpmvBlock - 1) / kSpmvBlock, (long long)num_sms() * 16));
    const int gs = static_cast<int>(std::min<long long>((s_rows + kSpmvBlock - 1) / kSpmvBlock, (long long)num_sms() * 16));
    k_spmv<false><<<gu + gs, kSpmvBlock, 0, st>>>(u_threads, u2, s_rows, gu, n_ug, nt, n_u, n_q, n_p, u_off.p, u_col.p,
                                                  u_val.p, s_off.p, s_len.p, s_col.p, s_val.p, x, y, guard, nullptr, 0, rows,
                                                  nullptr, nullptr);
    count_launch();
    PDG_CHECK_LAUNCH();
}

int SpaceTimeOp::dots_grid() const {
    if (kp) return kp_grid(false);
    int u2 = rows <= (2LL << 20);
    if (const char* e = std::getenv("PDG_SPMV_ROWS")) u2 = std::atoi(e) == 2;
    const long long u_threads = u_groups * (u2 ? 4 : 8);
    const int gu = static_cast<int>(std::min<long long>((u_threads + kSpmvBlock - 1) / kSpmvBlock, (long long)num_sms() * 16));
    const int gs = static_cast<int>(std::min<long long>((s_rows + kSpmvBlock - 1) / kSpmvBlock, (long long)num_sms() * 16));
    return gu + gs;
}

void SpaceTimeOp::apply_dots(const double* x, double* y, double* y2, const double* V, int ncols, double* partial,
                             cudaStream_t st) const {
    require(ncols >= 1 && ncols <= kSpmvMaxDots, "space-time block: fused dots need 1..8 basis vectors");
    ProfScope prof(PROF_SPMV, st, 8.0 * (double)(nnz + 2 * rows));
    if (kp) {
        kp_launch(x, y, y2, V, ncols, partial, false, st);
        return;
    }
    int u2 = rows <= (2LL << 20);
    if (const char* e = std::getenv("PDG_SPMV_ROWS")) u2 = std::atoi(e) == 2;
    const long long u_threads = u_groups * (u2 ? 4 : 8);
    const int gu = static_cast<int>(std::min<long long>((u_threads + kSpmvBlock - 1) / kSpmvBlock, (long long)num_sms() * 16));
    const int gs = static_cast<int>(std::min<long long>((s_rows + kSpmvBlock - 1) / kSpmvBlock, (long long)num_sms() * 16));
    k_spmv<true><<<gu + gs, kSpmvBlock, 0, st>>>(u_threads, u2, s_rows, gu, n_ug, nt, n_u, n_q, n_p, u_off.p, u_col.p,
                                                 u_val.p, s_off.p, s_len.p, s_col.p, s_val.p, x, y, guard, V, ncols, rows,
                                                 y2, partial);
    count_launch();
    PDG_CHECK_LAUNCH();
}

void SpaceTimeOp::set_strip(int nx, int ny, int r0, int r1, cudaStream_t st) {
    require(nx > 0 && ny > 0 && (long long)nx * ny == n_cells && n_u == 8 * n_p,
            "space-time block: strip mesh does not match the operator (strips are 2D only)");
    require(0 <= r0 && r0 < r1 && r1 <= ny, "space-time block: bad strip rows");
    strip_nx = nx;
    strip_ny = ny;
    strip_r0 = r0;
    strip_r1 = r1;
    const int nh = nx * (ny + 1);
    if (kp) {  // QK slices holding an owned face
        std::vector<long long> sl;
        for (long long s = 0; s < qk_slices; ++s) {
            bool any = false;
            for (int l = 0; l < 32 && !any; ++l) {
                const long long f = s * 32 + l;
                if (f >= n_q) break;
                const int row = f < nh ? std::min(static_cast<int>(f) / nx, ny - 1) : static_cast<int>((f - nh) % ny);
                any = row >= r0 && row < r1;
            }
            if (any) sl.push_back(s);
        }
        strip_qslices.upload(sl, st);
        strip_qslices.n = sl.size();
        PDG_CUDA(cudaStreamSynchronize(st));
        return;
    }
    // S slices holding an owned row (host scan of the row -> owner rule)
    auto owned = [&](long long srow) {
        const int loc = static_cast<int>(srow % (n_q + n_p));
        int row;
        if (loc < n_q)
            row = loc < nh ? std::min(loc / nx, ny - 1) : (loc - nh) % ny;
        else
            row = (loc - n_q) / nx;
        return row >= r0 && row < r1;
    };
    std::vector<long long> sl;
    for (long long s = 0; s < s_slices; ++s) {
        bool any = false;
        for (int l = 0; l < 32 && !any; ++l) {
            const long long srow = s * 32 + l;
            any = srow < s_rows && owned(srow);
        }
        if (any) sl.push_back(s);
    }
    strip_slices.upload(sl, st);
    strip_slices.n = sl.size();
    PDG_CUDA(cudaStreamSynchronize(st));
}

void SpaceTimeOp::apply_strip(const double* x, double* y, cudaStream_t st) const {
    require(strip_nx > 0, "space-time block: no strip set");
    if (kp) {
        ProfScope prof(PROF_SPMV, st, 0.0);
        kp_launch(x, y, nullptr, nullptr, 0, nullptr, true, st);
        return;
    }
    const int cell0 = strip_r0 * strip_nx, ncs = (strip_r1 - strip_r0) * strip_nx;
    const long long u_threads = (long long)m * ncs * 8;
    const long long ns = static_cast<long long>(strip_slices.n);
    const int gu = static_cast<int>(std::min<long long>((u_threads + kSpmvBlock - 1) / kSpmvBlock, (long long)num_sms() * 16));
    const int gs = static_cast<int>(
        std::max<long long>(1, std::min<long long>((ns * 32 + kSpmvBlock - 1) / kSpmvBlock, (long long)num_sms() * 16)));
    ProfScope prof(PROF_SPMV, st, 0.0);
    k_spmv_strip<<<gu + gs, kSpmvBlock, 0, st>>>(u_threads, cell0, ncs, gu, ns, strip_slices.p, s_rows, n_cells, nt, n_u, n_q,
                                                 n_p, strip_nx, strip_ny, strip_r0, strip_r1, u_off.p, u_col.p, u_val.p,
                                                 s_off.p, s_len.p, s_col.p, s_val.p, x, y, guard);
    count_launch();
    PDG_CHECK_LAUNCH();
}

void SpaceTimeOp::to_csr(std::vector<long long>& off, std::vector<int>& idx, std::vector<double>& val,
                         cudaStream_t st) const {
    if (kp) {
        kp_to_csr(off, idx, val, st);
        return;
    }
    const auto uo = u_off.download(st);
    const auto uc = u_col.download(st);
    const auto uv = u_val.download(st);
    const auto so = s_off.download(st);
    const auto sl = s_len.download(st);
    const auto sc = s_col.download(st);
    const auto sv = s_val.download(st);
    std::vector<int> len(rows, 0);
    for (long long g = 0; g < u_groups; ++g) {
        const int i = static_cast<int>(g / n_ug), c = static_cast<int>(g % n_ug);
        for (int l = 0; l < 8; ++l) len[(long long)i * nt + 8 * c + l] = static_cast<int>(uo[g + 1] - uo[g]);
    }
    for (long long s = 0; s < s_rows; ++s) {
        const int i = static_cast<int>(s / (n_q + n_p)), loc = static_cast<int>(s % (n_q + n_p));
        len[(long long)i * nt + n_u + loc] = sl[s];
    }
    off.assign(rows + 1, 0);
    for (long long r = 0; r < rows; ++r) off[r + 1] = off[r] + len[r];
    idx.resize(off[rows]);
    val.resize(off[rows]);
    for (long long g = 0; g < u_groups; ++g) {
        const int i = static_cast<int>(g / n_ug), c = static_cast<int>(g % n_ug);
        for (int l = 0; l < 8; ++l) {
            long long o = off[(long long)i * nt + 8 * c + l];
            for (long long k = uo[g]; k < uo[g + 1]; ++k, ++o) {
                idx[o] = uc[k];
                val[o] = uv[k * 8 + l];
            }
        }
    }
    for (long long s = 0; s < s_rows; ++s) {
        const int i = static_cast<int>(s / (n_q + n_p)), loc = static_cast<int>(s % (n_q + n_p));
        long long o = off[(long long)i * nt + n_u + loc];
        const long long b = so[s >> 5];
        const int lane = static_cast<int>(s & 31);
        for (int k = 0; k < sl[s]; ++k, ++o) {
            idx[o] = sc[(b + k) * 32 + lane];
            val[o] = sv[(b + k) * 32 + lane];
        }
    }
}

}  // namespace pdg
