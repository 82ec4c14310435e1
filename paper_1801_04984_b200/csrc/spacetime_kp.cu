// Kronecker-paired (KP) layout of the canonical space-time operator and its
// order-fixed SpMV (spacetime_op.cuh; DESIGN.md section 3 "Operator").
//
// The canonical operator of an m-component block (fixed_stress.hpp:38-60 in the
// assembled form of slab.hpp:146-153) repeats every spatial row pattern m times:
// the displacement rows of component i read A and E at the columns of component
// i, the flux rows M_q and B, the pressure rows E^T of every component, B^T of
// their own and the pressure diagonal of every component. The KP layout keeps the
// m rows of one pattern on one thread: the column list is read once for all of
// them, an entry's m values are one 16-byte load (m = 2), and the displacement
// column runs (8 consecutive dofs of a cell, in A and in E^T) keep one index per
// run. Per thread every row is summed alone, sequentially, in ascending column
// order with __dmul_rn/__dadd_rn: y is bit-identical to SparseMatrix::apply
// (sparse.hpp:30-40) on the canonical CSR (tests/test_gpu_parity.py).
//
// Work order: tiles of 256 cells, each = 8 UK blocks (32 cells x 8 displacement
// rows) + 1 PK block (8 SELL slices of 32 cells) + a share of the QK blocks, so
// the displacement and pressure rows of the same cells run at the same time and
// the x entries they share are read from DRAM once.
#include <cstdlib>
#include <cstring>

#include "ops.cuh"
#include "spacetime_op.cuh"

namespace pdg {

namespace {

constexpr int kKpBlock = 256;
constexpr int kKpTileCells = 256;  // 8 UK blocks of 32 cells, 1 PK block of 8 slices
constexpr int kKpMaxDots = 8;

struct KpCoef {
    double t[4];  // theta (m x m, row-major)
    double w[2];  // tau * kappa_i
};

// ---- build ----------------------------------------------------------------------
__global__ void k_uk_count(int n_cells, const int* __restrict__ a_off, const int* __restrict__ a_idx,
                           const int* __restrict__ e_off, long long* ecnt, long long* hcnt, int* na, int* err) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n_cells; c += gridDim.x * blockDim.x) {
        const int r = 8 * c;
        const int la = a_off[r + 1] - a_off[r], le = e_off[r + 1] - e_off[r];
        bool ok = la % 8 == 0;
        for (int q = 0; ok && q < la; q += 8) {
            const int s = a_idx[a_off[r] + q];
            ok = s % 8 == 0;
            for (int kk = 1; ok && kk < 8; ++kk) ok = a_idx[a_off[r] + q + kk] == s + kk;
        }
        if (!ok) atomicOr(err, 1);
        ecnt[c] = la + le;
        hcnt[c] = la / 8 + le;
        na[c] = la / 8;
    }
}

__global__ void k_uk_fill(int n_cells, int m, KpCoef co, double mb, const int* __restrict__ a_off,
                          const int* __restrict__ a_idx, const double* __restrict__ a_val, const int* __restrict__ e_off,
                          const int* __restrict__ e_idx, const double* __restrict__ e_val,
                          const long long* __restrict__ voff, const long long* __restrict__ hoff, int* hdr, double* val,
                          int* err) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < 8LL * n_cells;
         t += (long long)gridDim.x * blockDim.x) {
        const int c = static_cast<int>(t >> 3), l = static_cast<int>(t & 7);
        const int r = 8 * c + l, r0 = 8 * c;
        const int la = a_off[r + 1] - a_off[r], le = e_off[r + 1] - e_off[r];
        if (la != a_off[r0 + 1] - a_off[r0] || le != e_off[r0 + 1] - e_off[r0]) {
            atomicOr(err, 2);
            continue;
        }
        long long k = voff[c], h = hoff[c];
        for (int q = 0; q < la; ++q, ++k) {
            const int col = a_idx[a_off[r] + q];
            if (col != a_idx[a_off[r0] + q]) atomicOr(err, 2);
            for (int i = 0; i < m; ++i) val[(k * 8 + l) * m + i] = __dmul_rn(co.w[i], a_val[a_off[r] + q]);
            if (l == 0 && q % 8 == 0) hdr[h++] = col;
        }
        for (int q = 0; q < le; ++q, ++k) {
            const int col = e_idx[e_off[r] + q];
            if (col != e_idx[e_off[r0] + q]) atomicOr(err, 2);
            for (int i = 0; i < m; ++i)
                val[(k * 8 + l) * m + i] = __dmul_rn(co.w[i], __dmul_rn(mb, e_val[e_off[r] + q]));
            if (l == 0) hdr[h++] = col;
        }
    }
}

__host__ __device__ inline int pk_slots_of(int m, int ne, int nb) {
    return m * (ne + 1) + (m == 2 ? m * ((nb + 1) / 2) : nb);
}

__global__ void k_pk_count(int n_cells, int m, const int* __restrict__ et_off, const int* __restrict__ et_idx,
                           const int* __restrict__ bt_off, int* slots, int* hints, int* err) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n_cells; c += gridDim.x * blockDim.x) {
        const int ne = et_off[c + 1] - et_off[c], nb = bt_off[c + 1] - bt_off[c];
        bool ok = ne % 8 == 0 && ne / 8 < 256;
        for (int q = 0; ok && q < ne; q += 8) {
            const int s = et_idx[et_off[c] + q];
            ok = s % 8 == 0;
            for (int kk = 1; ok && kk < 8; ++kk) ok = et_idx[et_off[c] + q + kk] == s + kk;
        }
        if (!ok) atomicOr(err, 4);
        slots[c] = pk_slots_of(m, ne, nb);
        hints[c] = 1 + ne / 8 + nb;
    }
}

// max over the 32 lanes of each slice
__global__ void k_slice_max(long long n, long long n_slices, const int* __restrict__ v, long long* w) {
    for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < n_slices; s += (long long)gridDim.x * blockDim.x) {
        int mx = 0;
        for (int l = 0; l < 32; ++l)
            if (s * 32 + l < n) mx = max(mx, v[s * 32 + l]);
        w[s] = mx;
    }
}

__global__ void k_pk_fill(int n_cells, int m, KpCoef co, double mb, double minv, const int* __restrict__ et_off,
                          const int* __restrict__ et_idx, const double* __restrict__ et_val,
                          const int* __restrict__ bt_off, const int* __restrict__ bt_idx,
                          const double* __restrict__ bt_val, const double* __restrict__ m_p,
                          const long long* __restrict__ voff, const long long* __restrict__ hoff, int* hdr,
                          double* val) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n_cells; c += gridDim.x * blockDim.x) {
        const int sl = c >> 5, lane = c & 31;
        const int ne = et_off[c + 1] - et_off[c], nb = bt_off[c + 1] - bt_off[c];
        const long long hb = hoff[sl], vb = voff[sl];
        hdr[hb * 32 + lane] = (ne / 8) | (nb << 8);
        for (int r = 0; r < ne / 8; ++r) hdr[(hb + 1 + r) * 32 + lane] = et_idx[et_off[c] + 8 * r];
        for (int b = 0; b < nb; ++b) hdr[(hb + 1 + ne / 8 + b) * 32 + lane] = bt_idx[bt_off[c] + b];
        long long k = vb;
        auto slot = [&](int i) -> double& { return val[((k * 32) + lane) * m + i]; };
        for (int j = 0; j < m; ++j) {
            for (int q = 0; q < ne; ++q, ++k)
                for (int i = 0; i < m; ++i) slot(i) = __dmul_rn(co.t[i * m + j], __dmul_rn(mb, et_val[et_off[c] + q]));
            if (m == 2) {
                for (int b = 0; b < nb; b += 2, ++k) {
                    slot(0) = __dmul_rn(co.w[j], bt_val[bt_off[c] + b]);
                    slot(1) = b + 1 < nb ? __dmul_rn(co.w[j], bt_val[bt_off[c] + b + 1]) : 0.0;
                }
            } else {
                for (int b = 0; b < nb; ++b, ++k) slot(0) = __dmul_rn(co.w[j], bt_val[bt_off[c] + b]);
            }
            for (int i = 0; i < m; ++i) slot(i) = __dmul_rn(co.t[i * m + j], __dmul_rn(minv, m_p[c]));
            ++k;
        }
    }
}

__global__ void k_qk_len(int nq, const int* __restrict__ mq_off, const int* __restrict__ b_off, int* len) {
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nq; f += gridDim.x * blockDim.x)
        len[f] = (mq_off[f + 1] - mq_off[f]) + (b_off[f + 1] - b_off[f]);
}

__global__ void k_qk_fill(int nq, int m, KpCoef co, const int* __restrict__ mq_off, const int* __restrict__ mq_idx,
                          const double* __restrict__ mq_val, const int* __restrict__ b_off, const int* __restrict__ b_idx,
                          const double* __restrict__ b_val, const long long* __restrict__ off, int* col, double* val) {
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nq; f += gridDim.x * blockDim.x) {
        const int lane = f & 31;
        long long k = off[f >> 5];
        for (int q = mq_off[f]; q < mq_off[f + 1]; ++q, ++k) {
            col[k * 32 + lane] = mq_idx[q];
            for (int i = 0; i < m; ++i) val[(k * 32 + lane) * m + i] = __dmul_rn(co.w[i], mq_val[q]);
        }
        for (int q = b_off[f]; q < b_off[f + 1]; ++q, ++k) {
            col[k * 32 + lane] = nq + b_idx[q];
            for (int i = 0; i < m; ++i) val[(k * 32 + lane) * m + i] = __dmul_rn(co.w[i], b_val[q]);
        }
    }
}

// ---- SpMV ---------------------------------------------------------------------------
struct KpArgs {
    int n_cells, nt, nu, nq;
    int cell0, cell1, tile0;  // cells [cell0, cell1) computed; tiles start at tile0 (multiple of 256)
    int per, qpt;             // blocks per tile (9 + qpt), QK blocks per tile
    int pkfirst;
    int heavy;                // > 0: the tiles' 9 UK / PK blocks come first in the grid (heavy = 9 tiles), the QK blocks after them
    long long nqs;            // QK slices scheduled (all, or the strip's list)
    const long long* qlist;   // strip: QK slice list
    int nx, ny, r0, r1;       // strip: face-row ownership of the flux rows
    const long long *uk_voff, *uk_hoff;
    const int *uk_na, *uk_hdr;
    const double* uk_val;
    const long long *pk_voff, *pk_hoff;
    const int* pk_hdr;
    const double* pk_val;
    const long long* qk_off;
    const int *qk_len, *qk_col;
    const double* qk_val;
    const double* x;
    double* y;
    const int* stop;
    const double* V;
    int ncols;
    long long nrows;
    double* y2;
    double* partial;
};

template <int M>
__device__ __forceinline__ void ld_slot(const double* __restrict__ p, long long idx, double (&v)[M]) {
    if constexpr (M == 2) {
        const double2 t = __ldcs(reinterpret_cast<const double2*>(p) + idx);
        v[0] = t.x;
        v[1] = t.y;
    } else {
        v[0] = __ldcs(p + idx);
    }
}

__device__ __forceinline__ double mac(double s, double v, double x) { return __dadd_rn(s, __dmul_rn(v, x)); }

// PF (default; PDG_SPMV_PF=0 turns it off): the column headers of a thread's rows are loaded in
// one batch up front, and the pressure entries of a displacement row in one batch, so a thread's
// dependent-load chain is offsets -> headers -> one round per 8-column run instead of two rounds
// per run and per entry; registers capped at 64 (4 CTAs per SM). The sums keep their order. With
// the QK blocks at the end of the grid (and, on meshes whose x stays in L2 anyway, the PK
// blocks - the longest threads - at its start), measured on B200: config 1 (128^2, one wave of
// 768 CTAs) 45 -> 33 us per application, 256^2 0.81 -> 0.93, 512^2 0.84 -> 0.93, 1024^2 0.95 of HBM.
constexpr int kPfRuns = 6, kPfEnt = 6, kPfFaces = 4;  // batch sizes (the 2D operator: 5 runs, 5 entries, 4 faces)
constexpr int kKpPkFirstCells = 100000;               // PK blocks first up to this many cells
#ifndef KP_MINB
#define KP_MINB 4
#endif

template <int M, bool DOTS, bool STRIP, bool PF>
__global__ void __launch_bounds__(kKpBlock, PF ? KP_MINB : 1) k_spmv_kp(const KpArgs a) {
    if (a.stop && *a.stop) return;
    double acc[kKpMaxDots];
#pragma unroll
    for (int q = 0; q < kKpMaxDots; ++q) acc[q] = 0.0;
    auto out = [&](long long row, double v) {
        a.y[row] = v;
        if (DOTS) {
            if (a.y2) a.y2[row] = v;
#pragma unroll
            for (int q = 0; q < kKpMaxDots; ++q)
                if (q < a.ncols) acc[q] += __ldg(&a.V[(long long)q * a.nrows + row]) * v;
        }
    };
    int tile, part;
    if (a.heavy == 0) {
        tile = blockIdx.x / a.per;
        part = blockIdx.x - tile * a.per;
    } else if ((int)blockIdx.x < a.heavy / 9 && a.pkfirst) {  // the PK blocks (longest threads) first
        tile = blockIdx.x;
        part = 8;
    } else if ((int)blockIdx.x < a.heavy) {
        const int ub = a.pkfirst ? blockIdx.x - a.heavy / 9 : blockIdx.x;
        tile = a.pkfirst ? ub >> 3 : ub / 9;
        part = a.pkfirst ? ub & 7 : ub - tile * 9;
    } else {
        const int qb = blockIdx.x - a.heavy;
        tile = qb / a.qpt;
        part = 9 + qb - tile * a.qpt;
    }
    const int tbase = a.tile0 + tile * kKpTileCells;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double* __restrict__ x = a.x;
    if (part < 8) {
        // UK: thread = (cell, displacement row l), the cell's M components
        const int c = tbase + part * 32 + (threadIdx.x >> 3), l = threadIdx.x & 7;
        if (c >= a.cell0 && c < a.cell1) {
            const long long vo = __ldg(&a.uk_voff[c]), ho = __ldg(&a.uk_hoff[c]);
            const int nent = static_cast<int>(__ldg(&a.uk_voff[c + 1]) - vo);
            const int na = __ldg(&a.uk_na[c]);
            const int ne = nent - 8 * na;
            double s[M];
#pragma unroll
            for (int i = 0; i < M; ++i) s[i] = 0.0;
            const long long sb = vo * 8 + l;  // slot of entry k: sb + 8 k
            auto run = [&](int r, int base) {
                double v[8][M];
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) ld_slot<M>(a.uk_val, sb + 8LL * (8 * r + kk), v[kk]);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
#pragma unroll
                    for (int i = 0; i < M; ++i) s[i] = mac(s[i], v[kk][i], __ldg(&x[(long long)i * a.nt + base + kk]));
            };
            auto ent = [&](int e, int col) {
                double v[M];
                ld_slot<M>(a.uk_val, sb + 8LL * (8 * na + e), v);
#pragma unroll
                for (int i = 0; i < M; ++i) s[i] = mac(s[i], v[i], __ldg(&x[(long long)i * a.nt + a.nu + a.nq + col]));
            };
            const int* __restrict__ hp = a.uk_hdr + ho;
            if constexpr (PF) {
                int hb[kPfRuns], ec[kPfEnt];
#pragma unroll
                for (int r = 0; r < kPfRuns; ++r) hb[r] = r < na ? __ldg(hp + r) : 0;
#pragma unroll
                for (int e = 0; e < kPfEnt; ++e) ec[e] = e < ne ? __ldg(hp + na + e) : 0;
#pragma unroll
                for (int r = 0; r < kPfRuns; ++r)
                    if (r < na) run(r, hb[r]);
                for (int r = kPfRuns; r < na; ++r) run(r, __ldg(hp + r));
                double ev[kPfEnt][M], ex[kPfEnt][M];
#pragma unroll
                for (int e = 0; e < kPfEnt; ++e)
                    if (e < ne) {
                        ld_slot<M>(a.uk_val, sb + 8LL * (8 * na + e), ev[e]);
#pragma unroll
                        for (int i = 0; i < M; ++i) ex[e][i] = __ldg(&x[(long long)i * a.nt + a.nu + a.nq + ec[e]]);
                    }
#pragma unroll
                for (int e = 0; e < kPfEnt; ++e)
                    if (e < ne)
#pragma unroll
                        for (int i = 0; i < M; ++i) s[i] = mac(s[i], ev[e][i], ex[e][i]);
                for (int e = kPfEnt; e < ne; ++e) ent(e, __ldg(hp + na + e));
            } else {
                for (int r = 0; r < na; ++r) run(r, __ldg(hp + r));
                for (int e = 0; e < ne; ++e) ent(e, __ldg(hp + na + e));
            }
#pragma unroll
            for (int i = 0; i < M; ++i) out((long long)i * a.nt + 8 * c + l, s[i]);
        }
    } else if (part == 8) {
        // PK: thread = cell, its M pressure rows; SELL-32 slices of cells
        const int c = tbase + threadIdx.x;
        if (c >= a.cell0 && c < a.cell1) {
            const int sl = c >> 5;
            const long long hb = __ldg(&a.pk_hoff[sl]), vb = __ldg(&a.pk_voff[sl]);
            const int* __restrict__ hdr = a.pk_hdr + hb * 32 + lane;
            const int h0 = __ldcs(hdr);
            const int ne8 = h0 & 255, nb = h0 >> 8;
            double s[M];
#pragma unroll
            for (int i = 0; i < M; ++i) s[i] = 0.0;
            long long k = vb * 32 + lane;  // slot index, advances by 32 per slot
            int pb[kPfRuns], pf[kPfFaces];
            if constexpr (PF) {
#pragma unroll
                for (int r = 0; r < kPfRuns; ++r) pb[r] = r < ne8 ? __ldcs(&hdr[32 * (1 + r)]) : 0;
#pragma unroll
                for (int b = 0; b < kPfFaces; ++b) pf[b] = b < nb ? __ldcs(&hdr[32 * (1 + ne8 + b)]) : 0;
            }
            const int* __restrict__ fc = hdr + 32 * (1 + ne8);
#pragma unroll
            for (int j = 0; j < M; ++j) {
                const double* __restrict__ xj = x + (long long)j * a.nt;
                auto run = [&](int base) {
                    double v[8][M];
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) ld_slot<M>(a.pk_val, k + 32LL * kk, v[kk]);
                    k += 32LL * 8;
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const double xv = __ldg(&xj[base + kk]);
#pragma unroll
                        for (int i = 0; i < M; ++i) s[i] = mac(s[i], v[kk][i], xv);
                    }
                };
                // the B^T entries of component j: row j only (m = 2: two entries per slot)
                auto faces2 = [&](int b, int c0, int c1) {
                    double v[2];
                    ld_slot<2>(a.pk_val, k, v);
                    k += 32;
                    s[j] = mac(s[j], v[0], __ldg(&xj[a.nu + c0]));
                    if (b + 1 < nb) s[j] = mac(s[j], v[1], __ldg(&xj[a.nu + c1]));
                };
                auto face1 = [&](int c0) {
                    double v[1];
                    ld_slot<1>(a.pk_val, k, v);
                    k += 32;
                    s[0] = mac(s[0], v[0], __ldg(&xj[a.nu + c0]));
                };
                if constexpr (PF) {
#pragma unroll
                    for (int r = 0; r < kPfRuns; ++r)
                        if (r < ne8) run(pb[r]);
                    for (int r = kPfRuns; r < ne8; ++r) run(__ldcs(&hdr[32 * (1 + r)]));
                    if constexpr (M == 2) {
#pragma unroll
                        for (int b = 0; b < kPfFaces; b += 2)
                            if (b < nb) faces2(b, pf[b], pf[b + 1]);
                        for (int b = kPfFaces; b < nb; b += 2)
                            faces2(b, __ldcs(&fc[32 * b]), b + 1 < nb ? __ldcs(&fc[32 * (b + 1)]) : 0);
                    } else {
#pragma unroll
                        for (int b = 0; b < kPfFaces; ++b)
                            if (b < nb) face1(pf[b]);
                        for (int b = kPfFaces; b < nb; ++b) face1(__ldcs(&fc[32 * b]));
                    }
                } else {
                    for (int r = 0; r < ne8; ++r) run(__ldcs(&hdr[32 * (1 + r)]));
                    if constexpr (M == 2) {
                        for (int b = 0; b < nb; b += 2)
                            faces2(b, __ldcs(&fc[32 * b]), b + 1 < nb ? __ldcs(&fc[32 * (b + 1)]) : 0);
                    } else {
                        for (int b = 0; b < nb; ++b) face1(__ldcs(&fc[32 * b]));
                    }
                }
                {
                    double v[M];
                    ld_slot<M>(a.pk_val, k, v);
                    k += 32;
                    const double xv = __ldg(&xj[a.nu + a.nq + c]);
#pragma unroll
                    for (int i = 0; i < M; ++i) s[i] = mac(s[i], v[i], xv);
                }
            }
#pragma unroll
            for (int i = 0; i < M; ++i) out((long long)i * a.nt + a.nu + a.nq + c, s[i]);
        }
    } else {
        // QK: thread = face, its M flux rows; SELL-32 slices of faces
        const long long si = (long long)(tile * a.qpt + (part - 9)) * 8 + warp;
        if (si < a.nqs) {
            const long long sl = STRIP ? __ldg(&a.qlist[si]) : si;
            const long long f = sl * 32 + lane;
            if (f < a.nq) {
                const int len = __ldg(&a.qk_len[f]);
                const long long ob = __ldg(&a.qk_off[sl]) * 32 + lane;
                double s[M];
#pragma unroll
                for (int i = 0; i < M; ++i) s[i] = 0.0;
#pragma unroll 4
                for (int q = 0; q < len; ++q) {
                    double v[M];
                    ld_slot<M>(a.qk_val, ob + 32LL * q, v);
                    const int col = a.nu + __ldcs(&a.qk_col[ob + 32LL * q]);
#pragma unroll
                    for (int i = 0; i < M; ++i) s[i] = mac(s[i], v[i], __ldg(&x[(long long)i * a.nt + col]));
                }
                bool own = true;
                if (STRIP) {
                    const int nh = a.nx * (a.ny + 1);
                    const int fi = static_cast<int>(f);
                    const int row = fi < nh ? min(fi / a.nx, a.ny - 1) : (fi - nh) % a.ny;
                    own = row >= a.r0 && row < a.r1;
                }
                if (own)
#pragma unroll
                    for (int i = 0; i < M; ++i) out((long long)i * a.nt + a.nu + f, s[i]);
            }
        }
    }
    if (DOTS) {  // block partials, fixed order: warp butterflies, then the warps in order
        __shared__ double sh[kKpMaxDots][kKpBlock / 32];
#pragma unroll
        for (int q = 0; q < kKpMaxDots; ++q)
            for (int o = 16; o; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < kKpMaxDots; ++q) sh[q][warp] = acc[q];
        __syncthreads();
        if (threadIdx.x < a.ncols) {
            double t = 0.0;
            for (int w = 0; w < kKpBlock / 32; ++w) t += sh[threadIdx.x][w];
            a.partial[(long long)blockIdx.x * a.ncols + threadIdx.x] = t;
        }
    }
}

}  // namespace

bool SpaceTimeOp::build_kp(const SpatialOps& ops, const double* theta, const double* w, cudaStream_t st) {
    if (const char* e = std::getenv("PDG_SPMV_FORMAT"))
        if (std::strcmp(e, "sell") == 0) return false;
    for (int k = 0; k < m * m; ++k)
        if (theta[k] == 0.0) return false;  // the paired rows would not share their column lists
    KpCoef co{};
    for (int k = 0; k < m * m; ++k) co.t[k] = theta[k];
    for (int i = 0; i < m; ++i) co.w[i] = w[i];
    const double mb = -ops.biot_b, minv = -ops.inv_m;
    DBuf<int> err(1);
    err.zero(st);

    // UK
    DBuf<long long> ecnt(n_cells + 1), hcnt(n_cells + 1);
    ecnt.zero(st);
    hcnt.zero(st);
    uk_na.alloc(n_cells);
    k_uk_count<<<grid_for(n_cells, 256), 256, 0, st>>>(n_cells, ops.A.off.p, ops.A.idx.p, ops.E.off.p, ecnt.p, hcnt.p,
                                                        uk_na.p, err.p);
    PDG_CHECK_LAUNCH();
    uk_voff.alloc(n_cells + 1);
    uk_hoff.alloc(n_cells + 1);
    kp_u_entries = scan_ll(ecnt.p, uk_voff.p, n_cells, st);
    kp_u_hdr = scan_ll(hcnt.p, uk_hoff.p, n_cells, st);
    uk_hdr.alloc(kp_u_hdr);
    uk_val.alloc((size_t)8 * m * kp_u_entries);
    k_uk_fill<<<grid_for(8LL * n_cells, 256), 256, 0, st>>>(n_cells, m, co, mb, ops.A.off.p, ops.A.idx.p, ops.A.val.p,
                                                             ops.E.off.p, ops.E.idx.p, ops.E.val.p, uk_voff.p, uk_hoff.p,
                                                             uk_hdr.p, uk_val.p, err.p);
    PDG_CHECK_LAUNCH();

    // PK
    pk_slices = (n_cells + 31) / 32;
    {
        DBuf<int> slots(n_cells), hints(n_cells);
        k_pk_count<<<grid_for(n_cells, 256), 256, 0, st>>>(n_cells, m, ops.Et.off.p, ops.Et.idx.p, ops.Bt.off.p, slots.p,
                                                            hints.p, err.p);
        PDG_CHECK_LAUNCH();
        DBuf<long long> wv(pk_slices + 1), wh(pk_slices + 1);
        wv.zero(st);
        wh.zero(st);
        k_slice_max<<<grid_for(pk_slices, 256), 256, 0, st>>>(n_cells, pk_slices, slots.p, wv.p);
        k_slice_max<<<grid_for(pk_slices, 256), 256, 0, st>>>(n_cells, pk_slices, hints.p, wh.p);
        PDG_CHECK_LAUNCH();
        pk_voff.alloc(pk_slices + 1);
        pk_hoff.alloc(pk_slices + 1);
        pk_slots = scan_ll(wv.p, pk_voff.p, pk_slices, st);
        pk_hslots = scan_ll(wh.p, pk_hoff.p, pk_slices, st);
    }
    pk_hdr.alloc((size_t)32 * pk_hslots);
    pk_val.alloc((size_t)32 * m * pk_slots);
    pk_hdr.zero(st);
    pk_val.zero(st);
    k_pk_fill<<<grid_for(n_cells, 256), 256, 0, st>>>(n_cells, m, co, mb, minv, ops.Et.off.p, ops.Et.idx.p, ops.Et.val.p,
                                                       ops.Bt.off.p, ops.Bt.idx.p, ops.Bt.val.p, ops.m_p.p, pk_voff.p,
                                                       pk_hoff.p, pk_hdr.p, pk_val.p);
    PDG_CHECK_LAUNCH();

    // QK
    qk_slices = (n_q + 31) / 32;
    qk_len.alloc(n_q);
    k_qk_len<<<grid_for(n_q, 256), 256, 0, st>>>(n_q, ops.M_q.off.p, ops.B.off.p, qk_len.p);
    PDG_CHECK_LAUNCH();
    {
        DBuf<long long> wq(qk_slices + 1);
        wq.zero(st);
        k_slice_max<<<grid_for(qk_slices, 256), 256, 0, st>>>(n_q, qk_slices, qk_len.p, wq.p);
        PDG_CHECK_LAUNCH();
        qk_off.alloc(qk_slices + 1);
        qk_slots = scan_ll(wq.p, qk_off.p, qk_slices, st);
    }
    qk_col.alloc((size_t)32 * qk_slots);
    qk_val.alloc((size_t)32 * m * qk_slots);
    qk_col.zero(st);
    qk_val.zero(st);
    k_qk_fill<<<grid_for(n_q, 256), 256, 0, st>>>(n_q, m, co, ops.M_q.off.p, ops.M_q.idx.p, ops.M_q.val.p, ops.B.off.p,
                                                   ops.B.idx.p, ops.B.val.p, qk_off.p, qk_col.p, qk_val.p);
    PDG_CHECK_LAUNCH();

    int herr = 0;
    PDG_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    require((herr & 2) == 0, "space-time block: displacement rows of a cell do not share one column pattern");
    if (herr) {  // no 8-runs of displacement columns: the SELL layout takes the operator
        for (auto* b : {&uk_voff, &uk_hoff, &pk_voff, &pk_hoff, &qk_off}) b->release();
        for (auto* b : {&uk_na, &uk_hdr, &pk_hdr, &qk_len, &qk_col}) b->release();
        for (auto* b : {&uk_val, &pk_val, &qk_val}) b->release();
        return false;
    }
    kp = true;
    nnz = (long long)m * ((long long)ops.A.nnz + ops.E.nnz + ops.M_q.nnz + ops.B.nnz + ops.Bt.nnz) +
          (long long)m * m * ((long long)ops.Et.nnz + n_cells);
    return true;
}

int SpaceTimeOp::kp_grid(bool strip) const {
    int cell0 = 0, cell1 = n_cells;
    long long nqs = qk_slices;
    if (strip) {
        cell0 = strip_r0 * strip_nx;
        cell1 = strip_r1 * strip_nx;
        nqs = static_cast<long long>(strip_qslices.n);
    }
    const int tile0 = cell0 / kKpTileCells * kKpTileCells;
    const int tiles = std::max(1, (cell1 - tile0 + kKpTileCells - 1) / kKpTileCells);
    const long long qblocks = (nqs + 7) / 8;
    const int qpt = static_cast<int>((qblocks + tiles - 1) / tiles);
    return tiles * (9 + qpt);
}

void SpaceTimeOp::kp_launch(const double* x, double* y, double* y2, const double* V, int ncols, double* partial,
                            bool strip, cudaStream_t st) const {
    KpArgs a{};
    a.n_cells = n_cells;
    a.nt = nt;
    a.nu = n_u;
    a.nq = n_q;
    a.cell0 = 0;
    a.cell1 = n_cells;
    a.nqs = qk_slices;
    if (strip) {
        a.cell0 = strip_r0 * strip_nx;
        a.cell1 = strip_r1 * strip_nx;
        a.nqs = static_cast<long long>(strip_qslices.n);
        a.qlist = strip_qslices.p;
        a.nx = strip_nx;
        a.ny = strip_ny;
        a.r0 = strip_r0;
        a.r1 = strip_r1;
    }
    a.tile0 = a.cell0 / kKpTileCells * kKpTileCells;
    const int tiles = std::max(1, (a.cell1 - a.tile0 + kKpTileCells - 1) / kKpTileCells);
    const long long qblocks = (a.nqs + 7) / 8;
    a.qpt = static_cast<int>((qblocks + tiles - 1) / tiles);
    a.per = 9 + a.qpt;
    a.uk_voff = uk_voff.p;
    a.uk_hoff = uk_hoff.p;
    a.uk_na = uk_na.p;
    a.uk_hdr = uk_hdr.p;
    a.uk_val = uk_val.p;
    a.pk_voff = pk_voff.p;
    a.pk_hoff = pk_hoff.p;
    a.pk_hdr = pk_hdr.p;
    a.pk_val = pk_val.p;
    a.qk_off = qk_off.p;
    a.qk_len = qk_len.p;
    a.qk_col = qk_col.p;
    a.qk_val = qk_val.p;
    a.x = x;
    a.y = y;
    a.stop = guard;
    a.V = V;
    a.ncols = ncols;
    a.nrows = rows;
    a.y2 = y2;
    a.partial = partial;
    const int grid = tiles * a.per;
    const bool dots = partial != nullptr;
    static const int pf_env = std::getenv("PDG_SPMV_PF") ? std::atoi(std::getenv("PDG_SPMV_PF")) : 1;
    const bool pf = pf_env != 0;
    static const int ql_env = std::getenv("PDG_SPMV_QLAST") ? std::atoi(std::getenv("PDG_SPMV_QLAST")) : -1;
    a.heavy = (ql_env >= 0 ? ql_env != 0 : pf) ? 9 * tiles : 0;
    // PK blocks first while x stays in L2 anyway (measured: 256^2 0.855 -> 0.93 of HBM, 1024^2 0.954 -> 0.938)
    static const int pk_env = std::getenv("PDG_SPMV_PKFIRST") ? std::atoi(std::getenv("PDG_SPMV_PKFIRST")) : -1;
    a.pkfirst = pk_env >= 0 ? pk_env : (n_cells <= kKpPkFirstCells ? 1 : 0);
#define PDG_KP_LAUNCH(M_, D_, S_)                                          \
    do {                                                                   \
        if (pf)                                                            \
            k_spmv_kp<M_, D_, S_, true><<<grid, kKpBlock, 0, st>>>(a);     \
        else                                                               \
            k_spmv_kp<M_, D_, S_, false><<<grid, kKpBlock, 0, st>>>(a);    \
    } while (0)
    if (m == 2) {
        if (strip)
            PDG_KP_LAUNCH(2, false, true);
        else if (dots)
            PDG_KP_LAUNCH(2, true, false);
        else
            PDG_KP_LAUNCH(2, false, false);
    } else {
        if (strip)
            PDG_KP_LAUNCH(1, false, true);
        else if (dots)
            PDG_KP_LAUNCH(1, true, false);
        else
            PDG_KP_LAUNCH(1, false, false);
    }
#undef PDG_KP_LAUNCH
    count_launch();
    PDG_CHECK_LAUNCH();
}

void SpaceTimeOp::kp_to_csr(std::vector<long long>& off, std::vector<int>& idx, std::vector<double>& val,
                            cudaStream_t st) const {
    const auto uvo = uk_voff.download(st), uho = uk_hoff.download(st);
    const auto una = uk_na.download(st);
    const auto uh = uk_hdr.download(st);
    const auto uv = uk_val.download(st);
    const auto pvo = pk_voff.download(st), pho = pk_hoff.download(st);
    const auto ph = pk_hdr.download(st);
    const auto pv = pk_val.download(st);
    const auto qo = qk_off.download(st);
    const auto ql = qk_len.download(st);
    const auto qc = qk_col.download(st);
    const auto qv = qk_val.download(st);
    off.assign(rows + 1, 0);
    idx.clear();
    val.clear();
    idx.reserve(nnz);
    val.reserve(nnz);
    auto push = [&](long long col, double v) {
        idx.push_back(static_cast<int>(col));
        val.push_back(v);
    };
    long long row = 0;
    for (int i = 0; i < m; ++i) {
        const long long ob = (long long)i * nt;
        for (int c = 0; c < n_cells; ++c)  // u rows
            for (int l = 0; l < 8; ++l) {
                const long long vo = uvo[c], ho = uho[c];
                const int na = una[c], ne = static_cast<int>(uvo[c + 1] - vo) - 8 * na;
                for (int r = 0; r < na; ++r)
                    for (int kk = 0; kk < 8; ++kk) push(ob + uh[ho + r] + kk, uv[((vo + 8 * r + kk) * 8 + l) * m + i]);
                for (int e = 0; e < ne; ++e) push(ob + n_u + n_q + uh[ho + na + e], uv[((vo + 8 * na + e) * 8 + l) * m + i]);
                off[++row] = static_cast<long long>(idx.size());
            }
        for (int f = 0; f < n_q; ++f) {  // q rows
            const int lane = f & 31;
            const long long b = qo[f >> 5];
            for (int q = 0; q < ql[f]; ++q) push(ob + n_u + qc[(b + q) * 32 + lane], qv[((b + q) * 32 + lane) * m + i]);
            off[++row] = static_cast<long long>(idx.size());
        }
        for (int c = 0; c < n_cells; ++c) {  // p rows
            const int sl = c >> 5, lane = c & 31;
            const long long hb = pho[sl];
            const int h0 = ph[hb * 32 + lane], ne8 = h0 & 255, nb = h0 >> 8;
            long long k = pvo[sl];
            auto sv = [&](int comp) { return pv[((k * 32) + lane) * m + comp]; };
            for (int j = 0; j < m; ++j) {
                const long long oj = (long long)j * nt;
                for (int r = 0; r < ne8; ++r) {
                    const int base = ph[(hb + 1 + r) * 32 + lane];
                    for (int kk = 0; kk < 8; ++kk, ++k) push(oj + base + kk, sv(i));
                }
                if (m == 2) {
                    for (int b = 0; b < nb; b += 2, ++k)
                        if (j == i) {
                            push(oj + n_u + ph[(hb + 1 + ne8 + b) * 32 + lane], sv(0));
                            if (b + 1 < nb) push(oj + n_u + ph[(hb + 1 + ne8 + b + 1) * 32 + lane], sv(1));
                        }
                } else {
                    for (int b = 0; b < nb; ++b, ++k) push(oj + n_u + ph[(hb + 1 + ne8 + b) * 32 + lane], sv(0));
                }
                push(oj + n_u + n_q + c, sv(i));
                ++k;
            }
            off[++row] = static_cast<long long>(idx.size());
        }
    }
}

}  // namespace pdg
