// On-device assembly of the spatial operators (assemble_operators,
// assembly.hpp:177-395) and of the constant-data right-hand side
// (assemble_rhs, assembly.hpp:467-563) on the structured nx x ny mesh.
//
// One thread block per cell builds the cell's 8 displacement rows of A and E
// directly at their final CSR positions. The reference assembles triplets and
// merges duplicates in push order (sparse.hpp:83-110): an entry is
//   0.0 + (cell term) + sum over the cell's faces in ascending face index
//   (S, N, W, E) of one contribution per face quadrature point,
// and this kernel accumulates exactly that sequence, with the reference's
// expression association (this file is compiled with --fmad=false), so the
// device CSR is bit-identical to the reference's.
#include <cub/cub.cuh>

#include "ops.cuh"
#include "timebasis.hpp"

namespace pdg {

namespace {

struct Geo {
    int nx, ny;
    double hx, hy, lam, mu, eta, gamma, kperm;
    double g2p[2], g2w[2], g6p[6], g6w[6];
    int disp_dir[4][2];  // dirichlet flags per tag (left,right,bottom,top) per component
    double disp_data[4][2];
    int flow_kind[4];
    double flow_data[4];
};

// face ids of the structured mesh (mesh.hpp:59-60)
__device__ __forceinline__ int hface(const Geo& g, int i, int j) { return j * g.nx + i; }
__device__ __forceinline__ int vface(const Geo& g, int i, int j) { return g.nx * (g.ny + 1) + i * g.ny + j; }

struct FaceInfo {
    bool vertical, boundary;
    int cm, cp;  // cell_minus, cell_plus (-1)
    double nx, ny, measure, x0, y0;
    int tag;  // 0 interior, 1 left, 2 right, 3 bottom, 4 top
};

__device__ FaceInfo face_info(const Geo& g, int f) {
    FaceInfo F;
    const int nh = g.nx * (g.ny + 1);
    if (f < nh) {
        const int i = f % g.nx, j = f / g.nx;
        F.vertical = false;
        F.measure = g.hx;
        F.x0 = i * g.hx;
        F.y0 = j * g.hy;
        F.nx = 0.0;
        if (j == 0) {
            F.cm = i;
            F.cp = -1;
            F.ny = -1.0;
            F.tag = 3;
        } else if (j == g.ny) {
            F.cm = (g.ny - 1) * g.nx + i;
            F.cp = -1;
            F.ny = 1.0;
            F.tag = 4;
        } else {
            F.cm = (j - 1) * g.nx + i;
            F.cp = j * g.nx + i;
            F.ny = 1.0;
            F.tag = 0;
        }
    } else {
        const int k = f - nh, i = k / g.ny, j = k % g.ny;
        F.vertical = true;
        F.measure = g.hy;
        F.x0 = i * g.hx;
        F.y0 = j * g.hy;
        F.ny = 0.0;
        if (i == 0) {
            F.cm = j * g.nx;
            F.cp = -1;
            F.nx = -1.0;
            F.tag = 1;
        } else if (i == g.nx) {
            F.cm = j * g.nx + g.nx - 1;
            F.cp = -1;
            F.nx = 1.0;
            F.tag = 2;
        } else {
            F.cm = j * g.nx + i - 1;
            F.cp = j * g.nx + i;
            F.nx = 1.0;
            F.tag = 0;
        }
    }
    F.boundary = F.cp < 0;
    return F;
}

__device__ __forceinline__ double shp(int a, double xi, double eta) {
    switch (a) {
        case 0: return (1.0 - xi) * (1.0 - eta);
        case 1: return xi * (1.0 - eta);
        case 2: return (1.0 - xi) * eta;
        default: return xi * eta;
    }
}
__device__ __forceinline__ double dxi(int a, double eta) {
    switch (a) {
        case 0: return -(1.0 - eta);
        case 1: return 1.0 - eta;
        case 2: return -eta;
        default: return eta;
    }
}
__device__ __forceinline__ double deta(int a, double xi) {
    switch (a) {
        case 0: return -(1.0 - xi);
        case 1: return -xi;
        case 2: return 1.0 - xi;
        default: return xi;
    }
}

// traction of basis (node a, comp) (assembly.hpp:101-116)
__device__ __forceinline__ void traction(const Geo& g, int a, int comp, double xi, double eta, double nx, double ny,
                                         double& t0, double& t1) {
    const double g0 = dxi(a, eta) / g.hx, g1 = deta(a, xi) / g.hy;
    double sxx, syy, sxy;
    if (comp == 0) {
        sxx = (2.0 * g.mu + g.lam) * g0;
        syy = g.lam * g0;
        sxy = g.mu * g1;
    } else {
        sxx = g.lam * g1;
        syy = (2.0 * g.mu + g.lam) * g1;
        sxy = g.mu * g0;
    }
    t0 = sxx * nx + sxy * ny;
    t1 = sxy * nx + syy * ny;
}

// reference point of cell c on face F at arclength s (face_trace + face_ref_point)
__device__ __forceinline__ void ref_point(const Geo& g, const FaceInfo& F, int c, double s, double& xi, double& eta) {
    const double cx0 = (c % g.nx) * g.hx, cy0 = (c / g.nx) * g.hy;
    if (F.vertical) {
        const bool left = fabs(F.x0 - cx0) < 1e-12 * (g.hx + 1.0);
        xi = left ? 0.0 : 1.0;
        eta = s;
    } else {
        const bool bottom = fabs(F.y0 - cy0) < 1e-12 * (g.hy + 1.0);
        xi = s;
        eta = bottom ? 0.0 : 1.0;
    }
}

__device__ __forceinline__ double sipg(const Geo& g, const FaceInfo& F) {
    double h = 0.0;
    int cnt = 0;
    h += F.vertical ? g.hx : g.hy;
    ++cnt;
    if (F.cp >= 0) {
        h += F.vertical ? g.hx : g.hy;
        ++cnt;
    }
    h /= cnt;
    return g.gamma * (g.lam + 2.0 * g.mu) / h;
}

// interior-face SIPG contribution at quadrature point qk, test (s1,l1), trial (s2,l2)
__device__ double face_term(const Geo& g, const FaceInfo& F, int qk, int s1, int l1, int s2, int l2) {
    const double s = g.g2p[qk];
    const double w = g.g2w[qk] * F.measure;
    const int cells[2] = {F.cm, F.cp};
    const double sgn[2] = {1.0, -1.0};
    double xi1, eta1, xi2, eta2;
    ref_point(g, F, cells[s1], s, xi1, eta1);
    ref_point(g, F, cells[s2], s, xi2, eta2);
    const int a1 = l1 / 2, c1 = l1 % 2, a2 = l2 / 2, c2 = l2 % 2;
    const double n1 = shp(a1, xi1, eta1), n2 = shp(a2, xi2, eta2);
    const double v10 = c1 == 0 ? n1 : 0.0, v11 = c1 == 1 ? n1 : 0.0;
    const double v20 = c2 == 0 ? n2 : 0.0, v21 = c2 == 1 ? n2 : 0.0;
    double t10, t11, t20, t21;
    traction(g, a1, c1, xi1, eta1, F.nx, F.ny, t10, t11);
    traction(g, a2, c2, xi2, eta2, F.nx, F.ny, t20, t21);
    const double gamma_f = sipg(g, F);
    const double cons = -0.5 * (t20 * v10 + t21 * v11) * sgn[s1];
    const double symm = -0.5 * (t10 * v20 + t11 * v21) * sgn[s2];
    const double pen = gamma_f * sgn[s1] * sgn[s2] * (v10 * v20 + v11 * v21);
    return w * (cons + symm + pen);
}

// Nitsche boundary contribution (assembly.hpp:343-368)
__device__ double nitsche_term(const Geo& g, const FaceInfo& F, int qk, int l1, int l2) {
    const double s = g.g2p[qk];
    const double w = g.g2w[qk] * F.measure;
    double xi, eta;
    ref_point(g, F, F.cm, s, xi, eta);
    const int* dir = g.disp_dir[F.tag - 1];
    const int a1 = l1 / 2, c1 = l1 % 2, a2 = l2 / 2, c2 = l2 % 2;
    const double n1 = shp(a1, xi, eta), n2 = shp(a2, xi, eta);
    const double v10 = c1 == 0 ? n1 : 0.0, v11 = c1 == 1 ? n1 : 0.0;
    const double v20 = c2 == 0 ? n2 : 0.0, v21 = c2 == 1 ? n2 : 0.0;
    const double m10 = dir[0] ? v10 : 0.0, m11 = dir[1] ? v11 : 0.0;
    const double m20 = dir[0] ? v20 : 0.0, m21 = dir[1] ? v21 : 0.0;
    double t10, t11, t20, t21;
    traction(g, a1, c1, xi, eta, F.nx, F.ny, t10, t11);
    traction(g, a2, c2, xi, eta, F.nx, F.ny, t20, t21);
    const double gamma_f = sipg(g, F);
    const double cons = -(t20 * m10 + t21 * m11);
    const double symm = -(t10 * m20 + t11 * m21);
    const double pen = gamma_f * (m10 * m20 + m11 * m21);
    return w * (cons + symm + pen);
}

__device__ __forceinline__ bool has_dirichlet(const Geo& g, const FaceInfo& F) {
    return F.boundary && (g.disp_dir[F.tag - 1][0] || g.disp_dir[F.tag - 1][1]);
}

// neighbour list of cell c in ascending cell index: S, W, self, E, N
__device__ int neighbours(const Geo& g, int c, int* nb, int* nbface) {
    const int i = c % g.nx, j = c / g.nx;
    int k = 0;
    if (j > 0) {
        nb[k] = c - g.nx;
        nbface[k++] = hface(g, i, j);
    }
    if (i > 0) {
        nb[k] = c - 1;
        nbface[k++] = vface(g, i, j);
    }
    nb[k] = c;
    nbface[k++] = -1;
    if (i < g.nx - 1) {
        nb[k] = c + 1;
        nbface[k++] = vface(g, i + 1, j);
    }
    if (j < g.ny - 1) {
        nb[k] = c + g.nx;
        nbface[k++] = hface(g, i, j + 1);
    }
    return k;
}

__global__ void k_row_lengths(Geo g, int* a_len, int* e_len) {
    const int n = g.nx * g.ny;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
        int nb[5], nf[5];
        const int k = neighbours(g, c, nb, nf);
        for (int l = 0; l < 8; ++l) {
            a_len[8 * c + l] = 8 * k;
            e_len[8 * c + l] = k;
        }
    }
}

// One block (64 threads) per cell: thread (l1, l2) writes A(8c+l1, 8nb+l2) for
// every neighbour nb; threads with l2 == 0 also write the E row 8c+l1.
__global__ void __launch_bounds__(64) k_assemble_cell(Geo g, const int* __restrict__ a_off, int* a_idx, double* a_val,
                                                     const int* __restrict__ e_off, int* e_idx, double* e_val) {
    const int c = blockIdx.x;
    const int l1 = threadIdx.x / 8, l2 = threadIdx.x % 8;
    const int i = c % g.nx, j = c / g.nx;
    const double area = g.hx * g.hy;
    // cell faces in ascending face index: S, N, W, E
    const int cf[4] = {hface(g, i, j), hface(g, i, j + 1), vface(g, i, j), vface(g, i + 1, j)};
    // ---- volume term ke(l1,l2) and div_int(l1) (assembly.hpp:210-229)
    const int L1 = l1 > l2 ? l1 : l2, L2 = l1 > l2 ? l2 : l1;
    double ke = 0.0, div = 0.0;
    for (int qi = 0; qi < 2; ++qi)
        for (int qj = 0; qj < 2; ++qj) {
            const double xi = g.g2p[qi], eta = g.g2p[qj];
            const double w = g.g2w[qi] * g.g2w[qj] * area;
            double e1[3], e2[3];
            {
                const int a = L1 / 2, comp = L1 % 2;
                const double g0 = dxi(a, eta) / g.hx, g1 = deta(a, xi) / g.hy;
                if (comp == 0) {
                    e1[0] = g0; e1[1] = 0.0; e1[2] = 0.5 * g1;
                } else {
                    e1[0] = 0.0; e1[1] = g1; e1[2] = 0.5 * g0;
                }
            }
            {
                const int a = L2 / 2, comp = L2 % 2;
                const double g0 = dxi(a, eta) / g.hx, g1 = deta(a, xi) / g.hy;
                if (comp == 0) {
                    e2[0] = g0; e2[1] = 0.0; e2[2] = 0.5 * g1;
                } else {
                    e2[0] = 0.0; e2[1] = g1; e2[2] = 0.5 * g0;
                }
            }
            const double v = 2.0 * g.mu * (e1[0] * e2[0] + e1[1] * e2[1] + 2.0 * e1[2] * e2[2]) +
                             g.lam * (e1[0] + e1[1]) * (e2[0] + e2[1]);
            ke += w * v;
            if (l2 == 0) {
                const int a = l1 / 2, comp = l1 % 2;
                const double g0 = dxi(a, eta) / g.hx, g1 = deta(a, xi) / g.hy;
                const double ex = comp == 0 ? g0 : 0.0, ey = comp == 0 ? 0.0 : g1;
                div += w * (ex + ey);
            }
        }
    int nb[5], nf[5];
    const int k = neighbours(g, c, nb, nf);
    const int rowA = 8 * c + l1;
    for (int q = 0; q < k; ++q) {
        double s = 0.0;
        if (nb[q] == c) {
            s += ke;
            for (int t = 0; t < 4; ++t) {
                const FaceInfo F = face_info(g, cf[t]);
                if (!F.boundary) {
                    const int side = (F.cm == c) ? 0 : 1;
                    for (int qk = 0; qk < 2; ++qk) s += face_term(g, F, qk, side, l1, side, l2);
                } else if (has_dirichlet(g, F)) {
                    for (int qk = 0; qk < 2; ++qk) s += nitsche_term(g, F, qk, l1, l2);
                }
            }
        } else {
            const FaceInfo F = face_info(g, nf[q]);
            const int s1 = (F.cm == c) ? 0 : 1;
            for (int qk = 0; qk < 2; ++qk) s += face_term(g, F, qk, s1, l1, 1 - s1, l2);
        }
        const int pos = a_off[rowA] + 8 * q + l2;
        a_idx[pos] = 8 * nb[q] + l2;
        a_val[pos] = s;
    }
    if (l2 != 0) return;
    // ---- E row (assembly.hpp:233, :329-332, :369-372)
    const int a1 = l1 / 2, c1 = l1 % 2;
    for (int q = 0; q < k; ++q) {
        double s = 0.0;
        auto face_e = [&](const FaceInfo& F, int qk) {
            const double sq = g.g2p[qk];
            double xi, eta;
            ref_point(g, F, c, sq, xi, eta);
            const double nv = shp(a1, xi, eta);
            const double v0 = c1 == 0 ? nv : 0.0, v1 = c1 == 1 ? nv : 0.0;
            return F.nx * v0 + F.ny * v1;
        };
        if (nb[q] == c) {
            s += div;
            for (int t = 0; t < 4; ++t) {
                const FaceInfo F = face_info(g, cf[t]);
                if (!F.boundary) {
                    const double ss1 = (F.cm == c) ? 1.0 : -1.0;
                    for (int qk = 0; qk < 2; ++qk) {
                        const double w = g.g2w[qk] * F.measure;
                        s += -0.5 * w * ss1 * face_e(F, qk);
                    }
                } else if (has_dirichlet(g, F)) {
                    const int ncmp = F.vertical ? 0 : 1;
                    if (g.disp_dir[F.tag - 1][ncmp])
                        for (int qk = 0; qk < 2; ++qk) {
                            const double w = g.g2w[qk] * F.measure;
                            s += -w * face_e(F, qk);
                        }
                }
            }
        } else {
            const FaceInfo F = face_info(g, nf[q]);
            const double ss1 = (F.cm == c) ? 1.0 : -1.0;
            for (int qk = 0; qk < 2; ++qk) {
                const double w = g.g2w[qk] * F.measure;
                s += -0.5 * w * ss1 * face_e(F, qk);
            }
        }
        const int pos = e_off[rowA] + q;
        e_idx[pos] = nb[q];
        e_val[pos] = s;
    }
}

// Flux rows (M_q, B) and pressure mass, one thread per face (assembly.hpp:236-279).
__global__ void k_flux_lengths(Geo g, int nq, const signed char* qc, int* mq_len, int* b_len) {
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nq; f += gridDim.x * blockDim.x) {
        const FaceInfo F = face_info(g, f);
        if (qc[f]) {
            mq_len[f] = 1;
            b_len[f] = 0;
            continue;
        }
        // diagonal + one opposite face per adjacent cell (if that face is free)
        int n = 1, nb = 0;
        for (int side = 0; side < 2; ++side) {
            const int c = side ? F.cp : F.cm;
            if (c < 0) continue;
            ++nb;
            const int i = c % g.nx, j = c / g.nx;
            int opp;
            if (F.vertical)
                opp = (f == vface(g, i, j)) ? vface(g, i + 1, j) : vface(g, i, j);
            else
                opp = (f == hface(g, i, j)) ? hface(g, i, j + 1) : hface(g, i, j);
            if (!qc[opp]) ++n;
        }
        mq_len[f] = n;
        b_len[f] = nb;
    }
}

__device__ __forceinline__ double axis_sign(const FaceInfo& F) { return F.vertical ? F.nx : F.ny; }

__global__ void k_flux_fill(Geo g, int nq, const double* __restrict__ kcells, const signed char* qc, const int* mq_off,
                            int* mq_idx, double* mq_val, const int* b_off, int* b_idx, double* b_val) {
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nq; f += gridDim.x * blockDim.x) {
        const FaceInfo F = face_info(g, f);
        if (qc[f]) {
            mq_idx[mq_off[f]] = f;
            mq_val[mq_off[f]] = 1.0;
            continue;
        }
        const double area = g.hx * g.hy;
        // entries: (opp_minus?), f, (opp_plus?) in ascending face order; the
        // diagonal sums d3 of cell_minus then cell_plus (ascending cell index).
        int cols[3];
        double vals[3];
        int n = 0;
        double diag = 0.0;
        int opp_c[2] = {-1, -1};
        double cross_c[2] = {0.0, 0.0};
        for (int side = 0; side < 2; ++side) {
            const int c = side ? F.cp : F.cm;
            if (c < 0) continue;
            const int i = c % g.nx, j = c / g.nx;
            const double keff = g.eta / (kcells ? kcells[c] : g.kperm);
            const double d3 = keff * area / 3.0, d6 = keff * area / 6.0;
            int f0, f1;
            if (F.vertical) {
                f0 = vface(g, i, j);
                f1 = vface(g, i + 1, j);
            } else {
                f0 = hface(g, i, j);
                f1 = hface(g, i, j + 1);
            }
            const double cross = d6 * axis_sign(face_info(g, f0)) * axis_sign(face_info(g, f1));
            diag += d3;
            const int opp = (f == f0) ? f1 : f0;
            if (!qc[opp]) {
                opp_c[side] = opp;
                cross_c[side] = cross;
            }
        }
        // ascending: the lower opposite face, f, the higher opposite face
        int lo = -1, hi = -1;
        double vlo = 0.0, vhi = 0.0;
        for (int side = 0; side < 2; ++side) {
            if (opp_c[side] < 0) continue;
            if (opp_c[side] < f) {
                lo = opp_c[side];
                vlo = cross_c[side];
            } else {
                hi = opp_c[side];
                vhi = cross_c[side];
            }
        }
        if (lo >= 0) {
            cols[n] = lo;
            vals[n++] = vlo;
        }
        cols[n] = f;
        vals[n++] = diag;
        if (hi >= 0) {
            cols[n] = hi;
            vals[n++] = vhi;
        }
        for (int q = 0; q < n; ++q) {
            mq_idx[mq_off[f] + q] = cols[q];
            mq_val[mq_off[f] + q] = vals[q];
        }
        // B row: adjacent cells ascending, value -s_out * |F|
        int q = 0;
        for (int side = 0; side < 2; ++side) {
            const int c = side ? F.cp : F.cm;
            if (c < 0) continue;
            const double sout = F.boundary ? 1.0 : (c == F.cm ? 1.0 : -1.0);
            b_idx[b_off[f] + q] = c;
            b_val[b_off[f] + q] = -sout * F.measure;
            ++q;
        }
    }
}

__global__ void k_qc(Geo g, int nq, signed char* qc) {
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nq; f += gridDim.x * blockDim.x) {
        const FaceInfo F = face_info(g, f);
        qc[f] = (F.boundary && g.flow_kind[F.tag - 1] == 1) ? 1 : 0;
    }
}

__global__ void k_mp(Geo g, int n, double* mp) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) mp[c] = g.hx * g.hy;
}

// assemble_rhs for constant boundary data (no volume data): one thread per
// (cell, local dof) accumulates the cell's boundary faces in ascending face
// order, 6-point rule (assembly.hpp:515-555).
__global__ void k_rhs_u(Geo g, double* u) {
    const int n = g.nx * g.ny;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < 8LL * n; t += (long long)gridDim.x * blockDim.x) {
        const int c = static_cast<int>(t / 8), l = static_cast<int>(t % 8);
        const int i = c % g.nx, j = c / g.nx;
        if (i > 0 && i < g.nx - 1 && j > 0 && j < g.ny - 1) {  // interior cell: no boundary face
            u[t] = 0.0;
            continue;
        }
        const int cf[4] = {hface(g, i, j), hface(g, i, j + 1), vface(g, i, j), vface(g, i + 1, j)};
        const int a = l / 2, comp = l % 2;
        double r = 0.0;
        for (int q = 0; q < 4; ++q) {
            const FaceInfo F = face_info(g, cf[q]);
            if (!F.boundary) continue;
            const int tag = F.tag - 1;
            const int* dir = g.disp_dir[tag];
            const double gamma_f = sipg(g, F);
            const double tn0 = dir[0] ? 0.0 : g.disp_data[tag][0], tn1 = dir[1] ? 0.0 : g.disp_data[tag][1];
            // dirichlet_data only exists for fixed(); rollers carry traction data
            const bool fixed = dir[0] && dir[1];
            const double ud0 = fixed ? g.disp_data[tag][0] : 0.0, ud1 = fixed ? g.disp_data[tag][1] : 0.0;
            const double mud0 = dir[0] ? ud0 : 0.0, mud1 = dir[1] ? ud1 : 0.0;
            const double tnc = comp == 0 ? tn0 : tn1, mudc = comp == 0 ? mud0 : mud1;
            for (int qk = 0; qk < 6; ++qk) {
                const double s = g.g6p[qk];
                const double w = g.g6w[qk] * F.measure;
                double xi, eta;
                ref_point(g, F, c, s, xi, eta);
                const double nv = shp(a, xi, eta);
                if (!dir[comp]) r += w * nv * tnc;
                if (dir[comp]) r += w * gamma_f * nv * mudc;
                double tv0, tv1;
                traction(g, a, comp, xi, eta, F.nx, F.ny, tv0, tv1);
                r -= w * (tv0 * mud0 + tv1 * mud1);
            }
        }
        u[t] = r + 0.0;  // + rhs_ref_u (zero: no reference-state fields)
    }
}

__global__ void k_rhs_qp(Geo g, int nq, int np, const signed char* qc, double* q, double* p) {
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nq; f += gridDim.x * blockDim.x) {
        const FaceInfo F = face_info(g, f);
        double r = 0.0;
        if (F.boundary) {
            const int tag = F.tag - 1;
            if (g.flow_kind[tag] == 0) {
                for (int qk = 0; qk < 6; ++qk) {
                    const double w = g.g6w[qk] * F.measure;
                    r -= w * g.flow_data[tag];
                }
            }  // no-flow faces: essential value 0
        }
        q[f] = r;
    }
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < np; c += gridDim.x * blockDim.x) p[c] = 0.0;
}

// ---- assemble_rhs with sampled data (assembly.hpp:467-563 in full: VolumeData and time- /
// space-dependent boundary functions). The host evaluates its fields at the quadrature points
// (6 x 6 Gauss per cell, xi outer; 6 Gauss per boundary face) and the kernels accumulate in the
// reference's order: per dof the volume points (i, j) in order, then the cell's boundary
// faces in ascending face index; per flux row the adjacent cells in ascending index, then the
// boundary term, then the eliminated couplings (mq_bc, b_bc) in push order.
struct Samples {
    const double* momentum;   // [cell][36][2] or null
    const double* darcy;      // [cell][36][2] or null
    const double* mass;       // [cell][36] or null
    const double* traction;   // [bface][6][2]
    const double* dirichlet;  // [bface][6][2]
    const double* flow;       // [bface][6]
};

// index of boundary face f in the ascending list of boundary faces
__device__ __forceinline__ int bface_index(const Geo& g, int f) {
    const int nh = g.nx * (g.ny + 1);
    if (f < g.nx) return f;
    if (f < nh) return g.nx + (f - g.ny * g.nx);
    if (f < nh + g.ny) return 2 * g.nx + (f - nh);
    return 2 * g.nx + g.ny + (f - nh - g.nx * g.ny);
}

__global__ void k_rhs_u_s(Geo g, Samples sm, double* u) {
    const int n = g.nx * g.ny;
    const double area = g.hx * g.hy;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < 8LL * n; t += (long long)gridDim.x * blockDim.x) {
        const int c = static_cast<int>(t / 8), l = static_cast<int>(t % 8);
        const int i = c % g.nx, j = c / g.nx;
        const int cf[4] = {hface(g, i, j), hface(g, i, j + 1), vface(g, i, j), vface(g, i + 1, j)};
        const int a = l / 2, comp = l % 2;
        double r = 0.0;
        if (sm.momentum)
            for (int qi = 0; qi < 6; ++qi)
                for (int qj = 0; qj < 6; ++qj) {
                    const double w = g.g6w[qi] * g.g6w[qj] * area;
                    const double nv = shp(a, g.g6p[qi], g.g6p[qj]);
                    r += w * nv * sm.momentum[((long long)c * 36 + qi * 6 + qj) * 2 + comp];
                }
        for (int q = 0; q < 4; ++q) {
            const FaceInfo F = face_info(g, cf[q]);
            if (!F.boundary) continue;
            const int* dir = g.disp_dir[F.tag - 1];
            const double gamma_f = sipg(g, F);
            const long long bf = bface_index(g, cf[q]);
            for (int qk = 0; qk < 6; ++qk) {
                const double s = g.g6p[qk];
                const double w = g.g6w[qk] * F.measure;
                double xi, eta;
                ref_point(g, F, c, s, xi, eta);
                const double tn0 = sm.traction[(bf * 6 + qk) * 2], tn1 = sm.traction[(bf * 6 + qk) * 2 + 1];
                const double ud0 = sm.dirichlet[(bf * 6 + qk) * 2], ud1 = sm.dirichlet[(bf * 6 + qk) * 2 + 1];
                const double mud0 = dir[0] ? ud0 : 0.0, mud1 = dir[1] ? ud1 : 0.0;
                const double nv = shp(a, xi, eta);
                if (!dir[comp]) r += w * nv * (comp == 0 ? tn0 : tn1);
                if (dir[comp]) r += w * gamma_f * nv * (comp == 0 ? mud0 : mud1);
                double tv0, tv1;
                traction(g, a, comp, xi, eta, F.nx, F.ny, tv0, tv1);
                r -= w * (tv0 * mud0 + tv1 * mud1);
            }
        }
        u[t] = r + 0.0;
    }
}

// prescribed normal-flux values of the constrained faces: q_values[f] = sum_k (w_k / |F|) data_k
__global__ void k_rhs_qvalues(Geo g, int nq, const signed char* qc, Samples sm, double* qv) {
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nq; f += gridDim.x * blockDim.x) {
        double v = 0.0;
        if (qc[f]) {
            const FaceInfo F = face_info(g, f);
            const long long bf = bface_index(g, f);
            for (int qk = 0; qk < 6; ++qk) {
                const double w = g.g6w[qk] * F.measure;
                v += w / F.measure * sm.flow[bf * 6 + qk];
            }
        }
        qv[f] = v;
    }
}

__global__ void k_rhs_qp_s(Geo g, int nq, int np, const double* __restrict__ kcells, const signed char* qc, Samples sm,
                           const double* __restrict__ qv, double* q, double* p) {
    const double area = g.hx * g.hy;
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nq; f += gridDim.x * blockDim.x) {
        const FaceInfo F = face_info(g, f);
        if (qc[f]) {  // essential value (assembly.hpp:554)
            q[f] = qv[f];
            continue;
        }
        double r = 0.0;
        if (sm.darcy)
            for (int side = 0; side < 2; ++side) {
                const int c = side ? F.cp : F.cm;
                if (c < 0) continue;
                const int i = c % g.nx, j = c / g.nx;
                // local face of c: W, E (vertical) or S, N (horizontal), and its normal sign
                const bool low = F.vertical ? (f == vface(g, i, j)) : (f == hface(g, i, j));
                const double sg = F.vertical ? F.nx : F.ny;
                for (int qi = 0; qi < 6; ++qi)
                    for (int qj = 0; qj < 6; ++qj) {
                        const double xi = g.g6p[qi], eta = g.g6p[qj];
                        const double w = g.g6w[qi] * g.g6w[qj] * area;
                        const double t = F.vertical ? xi : eta;
                        const double wf = low ? sg * (1.0 - t) : sg * t;
                        r += w * wf * sm.darcy[((long long)c * 36 + qi * 6 + qj) * 2 + (F.vertical ? 0 : 1)];
                    }
            }
        if (F.boundary) {  // pressure condition (assembly.hpp:549-550)
            const long long bf = bface_index(g, f);
            for (int qk = 0; qk < 6; ++qk) {
                const double w = g.g6w[qk] * F.measure;
                r -= w * sm.flow[bf * 6 + qk];
            }
        }
        // eliminated couplings to constrained faces (mq_bc, assembly.hpp:250-258, :556)
        for (int side = 0; side < 2; ++side) {
            const int c = side ? F.cp : F.cm;
            if (c < 0) continue;
            const int i = c % g.nx, j = c / g.nx;
            int f0, f1;
            if (F.vertical) {
                f0 = vface(g, i, j);
                f1 = vface(g, i + 1, j);
            } else {
                f0 = hface(g, i, j);
                f1 = hface(g, i, j + 1);
            }
            const int opp = (f == f0) ? f1 : f0;
            if (!qc[opp]) continue;
            const double keff = g.eta / (kcells ? kcells[c] : g.kperm);
            const double d6 = keff * area / 6.0;
            const double cross = d6 * axis_sign(face_info(g, f0)) * axis_sign(face_info(g, f1));
            r -= cross * qv[opp];
        }
        q[f] = r;
    }
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < np; c += gridDim.x * blockDim.x) {
        double r = 0.0;
        if (sm.mass)
            for (int qi = 0; qi < 6; ++qi)
                for (int qj = 0; qj < 6; ++qj) {
                    const double w = g.g6w[qi] * g.g6w[qj] * area;
                    r -= w * sm.mass[(long long)c * 36 + qi * 6 + qj];
                }
        // b_bc (assembly.hpp:270-273, :557): the cell's constrained faces in the order W, E, S, N
        const int i = c % g.nx, j = c / g.nx;
        const int cfo[4] = {vface(g, i, j), vface(g, i + 1, j), hface(g, i, j), hface(g, i, j + 1)};
        for (int k = 0; k < 4; ++k) {
            const int f = cfo[k];
            if (!qc[f]) continue;
            const FaceInfo F = face_info(g, f);
            const double sout = F.boundary ? 1.0 : (c == F.cm ? 1.0 : -1.0);
            const double v = -sout * F.measure;
            r -= v * qv[f];
        }
        p[c] = r;
    }
}

Geo make_geo(const pdg_problem& p) {
    Geo g{};
    g.nx = p.nx;
    g.ny = p.ny;
    g.hx = p.lx / p.nx;
    g.hy = p.ly / p.ny;
    g.lam = p.lambda;
    g.mu = p.mu;
    g.eta = p.eta;
    g.gamma = p.penalty;
    g.kperm = p.k_perm;
    std::vector<double> pts, wts;
    tc_gauss(2, pts, wts);
    for (int k = 0; k < 2; ++k) {
        g.g2p[k] = pts[k];
        g.g2w[k] = wts[k];
    }
    tc_gauss(6, pts, wts);
    for (int k = 0; k < 6; ++k) {
        g.g6p[k] = pts[k];
        g.g6w[k] = wts[k];
    }
    for (int s = 0; s < 4; ++s) {
        const int kind = p.disp_kind[s];
        require(kind >= 0 && kind <= 3, "pdg_problem: bad displacement kind");
        g.disp_dir[s][0] = (kind == 0 || kind == 2);
        g.disp_dir[s][1] = (kind == 0 || kind == 3);
        g.disp_data[s][0] = p.disp_data[s][0];
        g.disp_data[s][1] = p.disp_data[s][1];
        require(p.flow_kind[s] == 0 || p.flow_kind[s] == 1, "pdg_problem: bad flow kind");
        g.flow_kind[s] = p.flow_kind[s];
        g.flow_data[s] = p.flow_data[s];
    }
    return g;
}

void scan_offsets(const int* len, int* off, int n, cudaStream_t st) {
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, len, off, n + 1, st);
    DBuf<unsigned char> buf(tmp + 1);
    cub::DeviceScan::ExclusiveSum(buf.p, tmp, len, off, n + 1, st);
}

int last_offset(const int* off, int n, cudaStream_t st) {
    int v = 0;
    PDG_CUDA(cudaMemcpyAsync(&v, off + n, sizeof(int), cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    return v;
}

}  // namespace

void assemble_ops_device(SpatialOps& s, const pdg_problem& p, cudaStream_t st) {
    require(p.nx >= 1 && p.ny >= 1, "build_mesh: cell counts must be positive");
    require(p.lx > 0.0 && p.ly > 0.0, "build_mesh: edge lengths must be positive");
    require(p.penalty > 0.0, "assemble_operators: penalty must be positive");
    require(p.mu > 0.0, "material: mu must be positive");
    require(p.eta > 0.0, "material: eta must be positive");
    require(p.biot_m > 0.0, "material: Biot modulus M must be positive");
    require(p.biot_b > 0.0 && p.biot_b <= 1.0, "material: Biot coefficient b must lie in (0, 1]");
    require(p.k_perm > 0.0, "material: permeability must be positive");
    require(8LL * p.nx * p.ny * 45 < (1LL << 31), "pdg_ops_assemble: mesh too large for int32 CSR offsets");
    const Geo g = make_geo(p);
    s.nx = p.nx;
    s.ny = p.ny;
    const int n = p.nx * p.ny;
    s.n_u = 8 * n;
    s.n_p = n;
    s.n_q = p.nx * (p.ny + 1) + (p.nx + 1) * p.ny;
    s.biot_b = p.biot_b;
    s.inv_m = 1.0 / p.biot_m;
    s.k_dr = p.lambda + 2.0 * p.mu / 2;
    s.has_problem = true;
    s.prob = p;
    DBuf<double> kc;
    if (p.k_perm_cells) {
        s.k_cells.assign(p.k_perm_cells, p.k_perm_cells + n);
        for (double k : s.k_cells) require(k > 0.0, "material: per-cell permeability must be positive");
        kc.upload(s.k_cells, st);
    }
    s.prob.k_perm_cells = nullptr;
    // A, E
    DBuf<int> alen(s.n_u + 1), elen(s.n_u + 1);
    k_row_lengths<<<grid_for(n, 256), 256, 0, st>>>(g, alen.p, elen.p);
    PDG_CHECK_LAUNCH();
    s.A.rows = s.A.cols = s.n_u;
    s.E.rows = s.n_u;
    s.E.cols = s.n_p;
    s.A.off.alloc(s.n_u + 1);
    s.E.off.alloc(s.n_u + 1);
    scan_offsets(alen.p, s.A.off.p, s.n_u, st);
    scan_offsets(elen.p, s.E.off.p, s.n_u, st);
    s.A.nnz = last_offset(s.A.off.p, s.n_u, st);
    s.E.nnz = last_offset(s.E.off.p, s.n_u, st);
    s.A.idx.alloc(s.A.nnz);
    s.A.val.alloc(s.A.nnz);
    s.E.idx.alloc(s.E.nnz);
    s.E.val.alloc(s.E.nnz);
    k_assemble_cell<<<n, 64, 0, st>>>(g, s.A.off.p, s.A.idx.p, s.A.val.p, s.E.off.p, s.E.idx.p, s.E.val.p);
    PDG_CHECK_LAUNCH();
    // flux blocks
    s.q_constrained.alloc(s.n_q);
    k_qc<<<grid_for(s.n_q, 256), 256, 0, st>>>(g, s.n_q, s.q_constrained.p);
    DBuf<int> mql(s.n_q + 1), bl(s.n_q + 1);
    k_flux_lengths<<<grid_for(s.n_q, 256), 256, 0, st>>>(g, s.n_q, s.q_constrained.p, mql.p, bl.p);
    PDG_CHECK_LAUNCH();
    s.M_q.rows = s.M_q.cols = s.n_q;
    s.B.rows = s.n_q;
    s.B.cols = s.n_p;
    s.M_q.off.alloc(s.n_q + 1);
    s.B.off.alloc(s.n_q + 1);
    scan_offsets(mql.p, s.M_q.off.p, s.n_q, st);
    scan_offsets(bl.p, s.B.off.p, s.n_q, st);
    s.M_q.nnz = last_offset(s.M_q.off.p, s.n_q, st);
    s.B.nnz = last_offset(s.B.off.p, s.n_q, st);
    s.M_q.idx.alloc(s.M_q.nnz);
    s.M_q.val.alloc(s.M_q.nnz);
    s.B.idx.alloc(s.B.nnz);
    s.B.val.alloc(s.B.nnz);
    k_flux_fill<<<grid_for(s.n_q, 256), 256, 0, st>>>(g, s.n_q, kc.n ? kc.p : nullptr, s.q_constrained.p, s.M_q.off.p,
                                                       s.M_q.idx.p, s.M_q.val.p, s.B.off.p, s.B.idx.p, s.B.val.p);
    PDG_CHECK_LAUNCH();
    s.m_p.alloc(s.n_p);
    k_mp<<<grid_for(n, 256), 256, 0, st>>>(g, n, s.m_p.p);
    PDG_CHECK_LAUNCH();
    PDG_CUDA(cudaStreamSynchronize(st));
}

void assemble_rhs_sampled_device(const SpatialOps& s, const pdg_rhs_samples& h, double* u, double* q, double* p,
                                 cudaStream_t st) {
    if (s.nz > 0) return assemble_rhs_sampled_device3(s, h, u, q, p, st);
    require(h.traction && h.dirichlet && h.flow, "pdg_ops_rhs_sampled: boundary samples must be given");
    const Geo g = make_geo(s.prob);
    const size_t nc = (size_t)s.n_p, nbf = 2 * ((size_t)s.nx + s.ny);
    DBuf<double> mom, dar, mas, tra, dir, flo, kc, qv(s.n_q);
    Samples sm{};
    if (h.momentum) {
        mom.upload(h.momentum, nc * 72, st);
        sm.momentum = mom.p;
    }
    if (h.darcy) {
        dar.upload(h.darcy, nc * 72, st);
        sm.darcy = dar.p;
    }
    if (h.mass) {
        mas.upload(h.mass, nc * 36, st);
        sm.mass = mas.p;
    }
    tra.upload(h.traction, nbf * 12, st);
    dir.upload(h.dirichlet, nbf * 12, st);
    flo.upload(h.flow, nbf * 6, st);
    sm.traction = tra.p;
    sm.dirichlet = dir.p;
    sm.flow = flo.p;
    if (!s.k_cells.empty()) kc.upload(s.k_cells, st);
    k_rhs_u_s<<<grid_for(8LL * s.n_p, 256), 256, 0, st>>>(g, sm, u);
    k_rhs_qvalues<<<grid_for(s.n_q, 256), 256, 0, st>>>(g, s.n_q, s.q_constrained.p, sm, qv.p);
    k_rhs_qp_s<<<grid_for(std::max(s.n_q, s.n_p), 256), 256, 0, st>>>(g, s.n_q, s.n_p, kc.n ? kc.p : nullptr,
                                                                       s.q_constrained.p, sm, qv.p, q, p);
    count_launch(3);
    PDG_CHECK_LAUNCH();
    PDG_CUDA(cudaStreamSynchronize(st));  // the staging buffers are released at scope exit
}

void assemble_rhs_device(const SpatialOps& s, double t, double* u, double* q, double* p, cudaStream_t st) {
    if (s.nz > 0) return assemble_rhs_device3(s, t, u, q, p, st);
    (void)t;  // constant boundary data: time-independent
    const Geo g = make_geo(s.prob);
    k_rhs_u<<<grid_for(8LL * s.n_p, 256), 256, 0, st>>>(g, u);
    k_rhs_qp<<<grid_for(std::max(s.n_q, s.n_p), 256), 256, 0, st>>>(g, s.n_q, s.n_p, s.q_constrained.p, q, p);
    count_launch(2);
    PDG_CHECK_LAUNCH();
}

}  // namespace pdg
