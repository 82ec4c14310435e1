// On-device assembly of the spatial operators and of the constant-data right-hand
// side on a structured nx x ny x nz mesh of hexahedra: the 3D extension of
// assembly.cu (BASELINE configs 2 and 4). The reference is 2D only
// (/root/reference/SPEC.md:14), so this generalises assemble_operators
// (assembly.hpp:177-395) and assemble_rhs (assembly.hpp:467-563) dimension by
// dimension: discontinuous trilinear displacement with SIPG (24 dofs per cell),
// one normal-velocity flux dof per face, piecewise constant pressure.
//
// Numbering (the 2D conventions of mesh.hpp:42-67 / dofs.hpp:28-46 extended):
//   cell c = (k ny + j) nx + i; faces by normal axis, highest axis first:
//   z-normal f = (k ny + j) nx + i, y-normal nzf + (j nz + k) nx + i,
//   x-normal nzf + nyf + (i nz + k) ny + j; node a = 4 az + 2 ay + ax,
//   u dof = 24 c + 3 a + comp; tags 1 xlo 2 xhi 3 ylo 4 yhi 5 zlo 6 zhi.
//
// One thread block per cell builds the cell's 24 rows of A and E at their final
// CSR positions. As in 2D an entry is
//   0.0 + (cell term) + sum over the cell's faces in ascending face index
//   (zlo, zhi, ylo, yhi, xlo, xhi) of one contribution per face quadrature point
//   (2 x 2 Gauss, first tangential axis outer),
// accumulated in exactly that order with the expression association of the CPU
// restatement oracle/refcpu/fem3d.hpp (this file is compiled with --fmad=false):
// the device CSR is bit-identical to it (tests/test_gpu_3d.py).
#include <cub/cub.cuh>

#include "ops.cuh"
#include "timebasis.hpp"

namespace pdg {

namespace {

struct Geo3 {
    int nx, ny, nz;
    double h[3], lam, mu, eta, gamma, kperm;
    double g2p[2], g2w[2], g6p[6], g6w[6];
    int disp_dir[6][3];  // dirichlet flags per tag (xlo..zhi) per component
    double disp_data[6][3];
    int flow_kind[6];
    double flow_data[6];
};

__device__ __forceinline__ int nzf(const Geo3& g) { return g.nx * g.ny * (g.nz + 1); }
__device__ __forceinline__ int nyf(const Geo3& g) { return g.nx * (g.ny + 1) * g.nz; }
__device__ __forceinline__ int zface(const Geo3& g, int i, int j, int k) { return (k * g.ny + j) * g.nx + i; }
__device__ __forceinline__ int yface(const Geo3& g, int i, int j, int k) { return nzf(g) + (j * g.nz + k) * g.nx + i; }
__device__ __forceinline__ int xface(const Geo3& g, int i, int j, int k) {
    return nzf(g) + nyf(g) + (i * g.nz + k) * g.ny + j;
}
__device__ __forceinline__ int cell_id(const Geo3& g, int i, int j, int k) { return (k * g.ny + j) * g.nx + i; }

struct Face3 {
    int axis, idx;  // normal axis, plane index along it
    int cm, cp;     // cell_minus, cell_plus (-1)
    double n[3], measure;
    int tag;
    bool boundary;
};

__device__ Face3 face_info(const Geo3& g, int f) {
    Face3 F;
    int i, j, k;
    const int a = nzf(g), b = nyf(g);
    if (f < a) {
        F.axis = 2;
        k = f / (g.nx * g.ny);
        j = (f / g.nx) % g.ny;
        i = f % g.nx;
        F.idx = k;
        F.measure = g.h[0] * g.h[1];
    } else if (f < a + b) {
        const int q = f - a;
        F.axis = 1;
        j = q / (g.nz * g.nx);
        k = (q / g.nx) % g.nz;
        i = q % g.nx;
        F.idx = j;
        F.measure = g.h[0] * g.h[2];
    } else {
        const int q = f - a - b;
        F.axis = 0;
        i = q / (g.nz * g.ny);
        k = (q / g.ny) % g.nz;
        j = q % g.ny;
        F.idx = i;
        F.measure = g.h[1] * g.h[2];
    }
    const int nax = F.axis == 0 ? g.nx : F.axis == 1 ? g.ny : g.nz;
    const int di = F.axis == 0, dj = F.axis == 1, dk = F.axis == 2;
    F.n[0] = F.n[1] = F.n[2] = 0.0;
    if (F.idx == 0) {
        F.cm = cell_id(g, i, j, k);
        F.cp = -1;
        F.n[F.axis] = -1.0;
        F.tag = 1 + 2 * F.axis;
    } else if (F.idx == nax) {
        F.cm = cell_id(g, i - di, j - dj, k - dk);
        F.cp = -1;
        F.n[F.axis] = 1.0;
        F.tag = 2 + 2 * F.axis;
    } else {
        F.cm = cell_id(g, i - di, j - dj, k - dk);
        F.cp = cell_id(g, i, j, k);
        F.n[F.axis] = 1.0;
        F.tag = 0;
    }
    F.boundary = F.cp < 0;
    return F;
}

__device__ __forceinline__ double lin(int b, double t) { return b ? t : 1.0 - t; }
__device__ __forceinline__ double dlin(int b) { return b ? 1.0 : -1.0; }
__device__ __forceinline__ double shp(int a, const double* r) {
    return lin(a & 1, r[0]) * lin((a >> 1) & 1, r[1]) * lin(a >> 2, r[2]);
}
__device__ __forceinline__ void grad(const Geo3& g, int a, const double* r, double* gr) {
    const int ax = a & 1, ay = (a >> 1) & 1, az = a >> 2;
    gr[0] = dlin(ax) * lin(ay, r[1]) * lin(az, r[2]) / g.h[0];
    gr[1] = lin(ax, r[0]) * dlin(ay) * lin(az, r[2]) / g.h[1];
    gr[2] = lin(ax, r[0]) * lin(ay, r[1]) * dlin(az) / g.h[2];
}
// strain of basis (a, comp): {xx, yy, zz, xy, xz, yz}
__device__ __forceinline__ void strain(const Geo3& g, int a, int comp, const double* r, double* e) {
    double gr[3];
    grad(g, a, r, gr);
    if (comp == 0) {
        e[0] = gr[0]; e[1] = 0.0; e[2] = 0.0; e[3] = 0.5 * gr[1]; e[4] = 0.5 * gr[2]; e[5] = 0.0;
    } else if (comp == 1) {
        e[0] = 0.0; e[1] = gr[1]; e[2] = 0.0; e[3] = 0.5 * gr[0]; e[4] = 0.0; e[5] = 0.5 * gr[2];
    } else {
        e[0] = 0.0; e[1] = 0.0; e[2] = gr[2]; e[3] = 0.0; e[4] = 0.5 * gr[0]; e[5] = 0.5 * gr[1];
    }
}
// sigma(basis) n, sigma = 2 mu eps + lambda tr(eps) I
__device__ __forceinline__ void traction(const Geo3& g, int a, int comp, const double* r, const double* n, double* t) {
    double gr[3];
    grad(g, a, r, gr);
    const double lam = g.lam, mu = g.mu;
    double sxx, syy, szz, sxy, sxz, syz;
    if (comp == 0) {
        sxx = (2.0 * mu + lam) * gr[0];
        syy = lam * gr[0];
        szz = lam * gr[0];
        sxy = mu * gr[1];
        sxz = mu * gr[2];
        syz = 0.0;
    } else if (comp == 1) {
        sxx = lam * gr[1];
        syy = (2.0 * mu + lam) * gr[1];
        szz = lam * gr[1];
        sxy = mu * gr[0];
        sxz = 0.0;
        syz = mu * gr[2];
    } else {
        sxx = lam * gr[2];
        syy = lam * gr[2];
        szz = (2.0 * mu + lam) * gr[2];
        sxy = 0.0;
        sxz = mu * gr[0];
        syz = mu * gr[1];
    }
    t[0] = sxx * n[0] + sxy * n[1] + sxz * n[2];
    t[1] = sxy * n[0] + syy * n[1] + syz * n[2];
    t[2] = sxz * n[0] + syz * n[1] + szz * n[2];
}
__device__ __forceinline__ double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

// reference point of cell c on face F at tangential coordinates (s1, s2)
__device__ __forceinline__ void ref_point(const Geo3& g, const Face3& F, int c, double s1, double s2, double* r) {
    const int ci[3] = {c % g.nx, (c / g.nx) % g.ny, c / (g.nx * g.ny)};
    const double fixed = F.idx == ci[F.axis] ? 0.0 : 1.0;
    if (F.axis == 0) {
        r[0] = fixed; r[1] = s1; r[2] = s2;
    } else if (F.axis == 1) {
        r[0] = s1; r[1] = fixed; r[2] = s2;
    } else {
        r[0] = s1; r[1] = s2; r[2] = fixed;
    }
}

__device__ __forceinline__ double sipg(const Geo3& g, const Face3& F) {
    double h = 0.0;
    int cnt = 0;
    h += g.h[F.axis];
    ++cnt;
    if (F.cp >= 0) {
        h += g.h[F.axis];
        ++cnt;
    }
    h /= cnt;
    return g.gamma * (g.lam + 2.0 * g.mu) / h;
}

__device__ __forceinline__ void basis_vec(int comp, double nv, double* v) {
    v[0] = comp == 0 ? nv : 0.0;
    v[1] = comp == 1 ? nv : 0.0;
    v[2] = comp == 2 ? nv : 0.0;
}

// interior-face SIPG contribution at quadrature point (qa, qb), test (s1,l1), trial (s2,l2)
__device__ double face_term(const Geo3& g, const Face3& F, int qa, int qb, int s1, int l1, int s2, int l2) {
    const double w = g.g2w[qa] * g.g2w[qb] * F.measure;
    const int cells[2] = {F.cm, F.cp};
    const double sgn[2] = {1.0, -1.0};
    double r1[3], r2[3];
    ref_point(g, F, cells[s1], g.g2p[qa], g.g2p[qb], r1);
    ref_point(g, F, cells[s2], g.g2p[qa], g.g2p[qb], r2);
    const int a1 = l1 / 3, c1 = l1 % 3, a2 = l2 / 3, c2 = l2 % 3;
    double v1[3], v2[3], t1[3], t2[3];
    basis_vec(c1, shp(a1, r1), v1);
    basis_vec(c2, shp(a2, r2), v2);
    traction(g, a1, c1, r1, F.n, t1);
    traction(g, a2, c2, r2, F.n, t2);
    const double gamma_f = sipg(g, F);
    const double cons = -0.5 * dot3(t2, v1) * sgn[s1];
    const double symm = -0.5 * dot3(t1, v2) * sgn[s2];
    const double pen = gamma_f * sgn[s1] * sgn[s2] * dot3(v1, v2);
    return w * (cons + symm + pen);
}

// Nitsche boundary contribution (the 3D form of assembly.hpp:343-368)
__device__ double nitsche_term(const Geo3& g, const Face3& F, int qa, int qb, int l1, int l2) {
    const double w = g.g2w[qa] * g.g2w[qb] * F.measure;
    double r[3];
    ref_point(g, F, F.cm, g.g2p[qa], g.g2p[qb], r);
    const int* dir = g.disp_dir[F.tag - 1];
    const int a1 = l1 / 3, c1 = l1 % 3, a2 = l2 / 3, c2 = l2 % 3;
    double v1[3], v2[3], t1[3], t2[3];
    basis_vec(c1, shp(a1, r), v1);
    basis_vec(c2, shp(a2, r), v2);
    traction(g, a1, c1, r, F.n, t1);
    traction(g, a2, c2, r, F.n, t2);
    double m1[3], m2[3];
    for (int d = 0; d < 3; ++d) {
        m1[d] = dir[d] ? v1[d] : 0.0;
        m2[d] = dir[d] ? v2[d] : 0.0;
    }
    const double gamma_f = sipg(g, F);
    const double cons = -dot3(t2, m1);
    const double symm = -dot3(t1, m2);
    const double pen = gamma_f * dot3(m1, m2);
    return w * (cons + symm + pen);
}

__device__ __forceinline__ bool has_dirichlet(const Geo3& g, const Face3& F) {
    return F.boundary && (g.disp_dir[F.tag - 1][0] || g.disp_dir[F.tag - 1][1] || g.disp_dir[F.tag - 1][2]);
}

// neighbour list of cell c in ascending cell index: k-1, j-1, i-1, self, i+1, j+1, k+1
__device__ int neighbours(const Geo3& g, int c, int* nb, int* nbface) {
    const int i = c % g.nx, j = (c / g.nx) % g.ny, k = c / (g.nx * g.ny);
    int n = 0;
    if (k > 0) {
        nb[n] = c - g.nx * g.ny;
        nbface[n++] = zface(g, i, j, k);
    }
    if (j > 0) {
        nb[n] = c - g.nx;
        nbface[n++] = yface(g, i, j, k);
    }
    if (i > 0) {
        nb[n] = c - 1;
        nbface[n++] = xface(g, i, j, k);
    }
    nb[n] = c;
    nbface[n++] = -1;
    if (i < g.nx - 1) {
        nb[n] = c + 1;
        nbface[n++] = xface(g, i + 1, j, k);
    }
    if (j < g.ny - 1) {
        nb[n] = c + g.nx;
        nbface[n++] = yface(g, i, j + 1, k);
    }
    if (k < g.nz - 1) {
        nb[n] = c + g.nx * g.ny;
        nbface[n++] = zface(g, i, j, k + 1);
    }
    return n;
}

// the cell's faces in ascending face index: zlo, zhi, ylo, yhi, xlo, xhi
__device__ __forceinline__ void cell_faces_asc(const Geo3& g, int c, int* cf) {
    const int i = c % g.nx, j = (c / g.nx) % g.ny, k = c / (g.nx * g.ny);
    cf[0] = zface(g, i, j, k);
    cf[1] = zface(g, i, j, k + 1);
    cf[2] = yface(g, i, j, k);
    cf[3] = yface(g, i, j + 1, k);
    cf[4] = xface(g, i, j, k);
    cf[5] = xface(g, i + 1, j, k);
}

__global__ void k_row_lengths3(Geo3 g, int* a_len, int* e_len) {
    const int n = g.nx * g.ny * g.nz;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
        int nb[7], nf[7];
        const int k = neighbours(g, c, nb, nf);
        for (int l = 0; l < 24; ++l) {
            a_len[24 * c + l] = 24 * k;
            e_len[24 * c + l] = k;
        }
    }
}

// One block (576 threads) per cell: thread (l1, l2) writes A(24c+l1, 24nb+l2) for every
// neighbour nb; threads with l2 == 0 also write the E row 24c+l1.
__global__ void __launch_bounds__(576) k_assemble_cell3(Geo3 g, const int* __restrict__ a_off, int* a_idx, double* a_val,
                                                       const int* __restrict__ e_off, int* e_idx, double* e_val) {
    const int c = blockIdx.x;
    const int l1 = threadIdx.x / 24, l2 = threadIdx.x % 24;
    const double vol = g.h[0] * g.h[1] * g.h[2];
    int cf[6];
    cell_faces_asc(g, c, cf);
    // ---- volume term ke(l1,l2) and div_int(l1): 2 x 2 x 2 Gauss, lower triangle mirrored
    const int L1 = l1 > l2 ? l1 : l2, L2 = l1 > l2 ? l2 : l1;
    double ke = 0.0, div = 0.0;
    for (int qi = 0; qi < 2; ++qi)
        for (int qj = 0; qj < 2; ++qj)
            for (int qk = 0; qk < 2; ++qk) {
                const double r[3] = {g.g2p[qi], g.g2p[qj], g.g2p[qk]};
                const double w = g.g2w[qi] * g.g2w[qj] * g.g2w[qk] * vol;
                double e1[6], e2[6];
                strain(g, L1 / 3, L1 % 3, r, e1);
                strain(g, L2 / 3, L2 % 3, r, e2);
                const double v = 2.0 * g.mu *
                                     (e1[0] * e2[0] + e1[1] * e2[1] + e1[2] * e2[2] + 2.0 * e1[3] * e2[3] +
                                      2.0 * e1[4] * e2[4] + 2.0 * e1[5] * e2[5]) +
                                 g.lam * (e1[0] + e1[1] + e1[2]) * (e2[0] + e2[1] + e2[2]);
                ke += w * v;
                if (l2 == 0) {
                    double e[6];
                    strain(g, l1 / 3, l1 % 3, r, e);
                    div += w * (e[0] + e[1] + e[2]);
                }
            }
    int nb[7], nf[7];
    const int k = neighbours(g, c, nb, nf);
    const int rowA = 24 * c + l1;
    for (int q = 0; q < k; ++q) {
        double s = 0.0;
        if (nb[q] == c) {
            s += ke;
            for (int t = 0; t < 6; ++t) {
                const Face3 F = face_info(g, cf[t]);
                if (!F.boundary) {
                    const int side = (F.cm == c) ? 0 : 1;
                    for (int qa = 0; qa < 2; ++qa)
                        for (int qb = 0; qb < 2; ++qb) s += face_term(g, F, qa, qb, side, l1, side, l2);
                } else if (has_dirichlet(g, F)) {
                    for (int qa = 0; qa < 2; ++qa)
                        for (int qb = 0; qb < 2; ++qb) s += nitsche_term(g, F, qa, qb, l1, l2);
                }
            }
        } else {
            const Face3 F = face_info(g, nf[q]);
            const int s1 = (F.cm == c) ? 0 : 1;
            for (int qa = 0; qa < 2; ++qa)
                for (int qb = 0; qb < 2; ++qb) s += face_term(g, F, qa, qb, s1, l1, 1 - s1, l2);
        }
        const int pos = a_off[rowA] + 24 * q + l2;
        a_idx[pos] = 24 * nb[q] + l2;
        a_val[pos] = s;
    }
    if (l2 != 0) return;
    // ---- E row: div term, then -1/2 {p} n . [[v]] per interior face and the Nitsche term
    const int a1 = l1 / 3, c1 = l1 % 3;
    auto face_e = [&](const Face3& F, int qa, int qb) {
        double r[3], v[3];
        ref_point(g, F, c, g.g2p[qa], g.g2p[qb], r);
        basis_vec(c1, shp(a1, r), v);
        return F.n[0] * v[0] + F.n[1] * v[1] + F.n[2] * v[2];
    };
    for (int q = 0; q < k; ++q) {
        double s = 0.0;
        if (nb[q] == c) {
            s += div;
            for (int t = 0; t < 6; ++t) {
                const Face3 F = face_info(g, cf[t]);
                if (!F.boundary) {
                    const double ss1 = (F.cm == c) ? 1.0 : -1.0;
                    for (int qa = 0; qa < 2; ++qa)
                        for (int qb = 0; qb < 2; ++qb) {
                            const double w = g.g2w[qa] * g.g2w[qb] * F.measure;
                            s += -0.5 * w * ss1 * face_e(F, qa, qb);
                        }
                } else if (has_dirichlet(g, F)) {
                    if (g.disp_dir[F.tag - 1][F.axis])
                        for (int qa = 0; qa < 2; ++qa)
                            for (int qb = 0; qb < 2; ++qb) {
                                const double w = g.g2w[qa] * g.g2w[qb] * F.measure;
                                s += -w * face_e(F, qa, qb);
                            }
                }
            }
        } else {
            const Face3 F = face_info(g, nf[q]);
            const double ss1 = (F.cm == c) ? 1.0 : -1.0;
            for (int qa = 0; qa < 2; ++qa)
                for (int qb = 0; qb < 2; ++qb) {
                    const double w = g.g2w[qa] * g.g2w[qb] * F.measure;
                    s += -0.5 * w * ss1 * face_e(F, qa, qb);
                }
        }
        const int pos = e_off[rowA] + q;
        e_idx[pos] = nb[q];
        e_val[pos] = s;
    }
}

// the two faces of cell c along `axis` (low, high)
__device__ __forceinline__ void axis_faces(const Geo3& g, int c, int axis, int& f0, int& f1) {
    const int i = c % g.nx, j = (c / g.nx) % g.ny, k = c / (g.nx * g.ny);
    if (axis == 0) {
        f0 = xface(g, i, j, k);
        f1 = xface(g, i + 1, j, k);
    } else if (axis == 1) {
        f0 = yface(g, i, j, k);
        f1 = yface(g, i, j + 1, k);
    } else {
        f0 = zface(g, i, j, k);
        f1 = zface(g, i, j, k + 1);
    }
}

__global__ void k_flux_lengths3(Geo3 g, int nq, const signed char* qc, int* mq_len, int* b_len) {
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nq; f += gridDim.x * blockDim.x) {
        const Face3 F = face_info(g, f);
        if (qc[f]) {
            mq_len[f] = 1;
            b_len[f] = 0;
            continue;
        }
        int n = 1, nb = 0;
        for (int side = 0; side < 2; ++side) {
            const int c = side ? F.cp : F.cm;
            if (c < 0) continue;
            ++nb;
            int f0, f1;
            axis_faces(g, c, F.axis, f0, f1);
            const int opp = (f == f0) ? f1 : f0;
            if (!qc[opp]) ++n;
        }
        mq_len[f] = n;
        b_len[f] = nb;
    }
}

__global__ void k_flux_fill3(Geo3 g, int nq, const double* __restrict__ kcells, const signed char* qc, const int* mq_off,
                             int* mq_idx, double* mq_val, const int* b_off, int* b_idx, double* b_val) {
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nq; f += gridDim.x * blockDim.x) {
        const Face3 F = face_info(g, f);
        if (qc[f]) {
            mq_idx[mq_off[f]] = f;
            mq_val[mq_off[f]] = 1.0;
            continue;
        }
        const double vol = g.h[0] * g.h[1] * g.h[2];
        // entries: (opp_minus?), f, (opp_plus?) in ascending face order; the diagonal sums
        // d3 of cell_minus then cell_plus (ascending cell index)
        double diag = 0.0;
        int opp_c[2] = {-1, -1};
        double cross_c[2] = {0.0, 0.0};
        for (int side = 0; side < 2; ++side) {
            const int c = side ? F.cp : F.cm;
            if (c < 0) continue;
            const double keff = g.eta / (kcells ? kcells[c] : g.kperm);
            const double d3 = keff * vol / 3.0, d6 = keff * vol / 6.0;
            int f0, f1;
            axis_faces(g, c, F.axis, f0, f1);
            const Face3 F0 = face_info(g, f0), F1 = face_info(g, f1);
            const double cross = d6 * F0.n[F.axis] * F1.n[F.axis];
            diag += d3;
            const int opp = (f == f0) ? f1 : f0;
            if (!qc[opp]) {
                opp_c[side] = opp;
                cross_c[side] = cross;
            }
        }
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
        int n = mq_off[f];
        if (lo >= 0) {
            mq_idx[n] = lo;
            mq_val[n++] = vlo;
        }
        mq_idx[n] = f;
        mq_val[n++] = diag;
        if (hi >= 0) {
            mq_idx[n] = hi;
            mq_val[n++] = vhi;
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

__global__ void k_qc3(Geo3 g, int nq, signed char* qc) {
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nq; f += gridDim.x * blockDim.x) {
        const Face3 F = face_info(g, f);
        qc[f] = (F.boundary && g.flow_kind[F.tag - 1] == 1) ? 1 : 0;
    }
}

__global__ void k_mp3(Geo3 g, int n, double* mp) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) mp[c] = g.h[0] * g.h[1] * g.h[2];
}

// assemble_rhs for constant boundary data (no volume data): one thread per (cell, local dof)
// accumulates the cell's boundary faces in ascending face order, 6 x 6 Gauss points.
__global__ void k_rhs_u3(Geo3 g, double* u) {
    const int n = g.nx * g.ny * g.nz;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < 24LL * n; t += (long long)gridDim.x * blockDim.x) {
        const int c = static_cast<int>(t / 24), l = static_cast<int>(t % 24);
        int cf[6];
        cell_faces_asc(g, c, cf);
        const int a = l / 3, comp = l % 3;
        double r = 0.0;
        for (int q = 0; q < 6; ++q) {
            const Face3 F = face_info(g, cf[q]);
            if (!F.boundary) continue;
            const int tag = F.tag - 1;
            const int* dir = g.disp_dir[tag];
            const double gamma_f = sipg(g, F);
            // dirichlet data only exists for fixed(); rollers and traction faces carry traction data
            const bool fixed = dir[0] && dir[1] && dir[2];
            double tn[3], mud[3];
            for (int d = 0; d < 3; ++d) {
                tn[d] = fixed ? 0.0 : g.disp_data[tag][d];
                mud[d] = (fixed && dir[d]) ? g.disp_data[tag][d] : 0.0;
            }
            for (int qa = 0; qa < 6; ++qa)
                for (int qb = 0; qb < 6; ++qb) {
                    const double w = g.g6w[qa] * g.g6w[qb] * F.measure;
                    double rp[3], tv[3];
                    ref_point(g, F, c, g.g6p[qa], g.g6p[qb], rp);
                    const double nv = shp(a, rp);
                    if (!dir[comp]) r += w * nv * tn[comp];
                    if (dir[comp]) r += w * gamma_f * nv * mud[comp];
                    traction(g, a, comp, rp, F.n, tv);
                    r -= w * dot3(tv, mud);
                }
        }
        u[t] = r + 0.0;  // + rhs_ref_u (zero: no reference-state fields)
    }
}

__global__ void k_rhs_qp3(Geo3 g, int nq, int np, double* q, double* p) {
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nq; f += gridDim.x * blockDim.x) {
        const Face3 F = face_info(g, f);
        double r = 0.0;
        if (F.boundary) {
            const int tag = F.tag - 1;
            if (g.flow_kind[tag] == 0) {
                for (int qa = 0; qa < 6; ++qa)
                    for (int qb = 0; qb < 6; ++qb) {
                        const double w = g.g6w[qa] * g.g6w[qb] * F.measure;
                        r -= w * g.flow_data[tag];
                    }
            }  // no-flow faces: essential value 0
        }
        q[f] = r;
    }
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < np; c += gridDim.x * blockDim.x) p[c] = 0.0;
}

// ---- assemble_rhs with sampled data in 3D (the 3D form of assembly.hpp:467-563 in full; the
// oracle's assemble_rhs3_sampled): volume sources at the 6 x 6 x 6 Gauss points per cell (xi
// outermost), boundary data at the 6 x 6 points per boundary face (ascending face index, first
// tangential axis outer); accumulation order as in assembly.cu's 2D kernels.
struct Samples3 {
    const double* momentum;   // [cell][216][3] or null
    const double* darcy;      // [cell][216][3] or null
    const double* mass;       // [cell][216] or null
    const double* traction;   // [bface][36][3]
    const double* dirichlet;  // [bface][36][3]
    const double* flow;       // [bface][36]
};

__device__ __forceinline__ int bface_index3(const Geo3& g, int f) {
    const int nxy = g.nx * g.ny, nxz = g.nx * g.nz, nyz = g.ny * g.nz, a = nzf(g), b = nyf(g);
    if (f < nxy) return f;
    if (f < a) return nxy + (f - g.nz * nxy);
    if (f < a + nxz) return 2 * nxy + (f - a);
    if (f < a + b) return 2 * nxy + nxz + (f - a - g.ny * nxz);
    if (f < a + b + nyz) return 2 * nxy + 2 * nxz + (f - a - b);
    return 2 * nxy + 2 * nxz + nyz + (f - a - b - g.nx * nyz);
}

__global__ void k_rhs_u_s3(Geo3 g, Samples3 sm, double* u) {
    const int n = g.nx * g.ny * g.nz;
    const double vol = g.h[0] * g.h[1] * g.h[2];
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < 24LL * n; t += (long long)gridDim.x * blockDim.x) {
        const int c = static_cast<int>(t / 24), l = static_cast<int>(t % 24);
        int cf[6];
        cell_faces_asc(g, c, cf);
        const int a = l / 3, comp = l % 3;
        double r = 0.0;
        if (sm.momentum)
            for (int qi = 0; qi < 6; ++qi)
                for (int qj = 0; qj < 6; ++qj)
                    for (int qk = 0; qk < 6; ++qk) {
                        const double ref[3] = {g.g6p[qi], g.g6p[qj], g.g6p[qk]};
                        const double w = g.g6w[qi] * g.g6w[qj] * g.g6w[qk] * vol;
                        r += w * shp(a, ref) * sm.momentum[((long long)c * 216 + (qi * 6 + qj) * 6 + qk) * 3 + comp];
                    }
        for (int q = 0; q < 6; ++q) {
            const Face3 F = face_info(g, cf[q]);
            if (!F.boundary) continue;
            const int* dir = g.disp_dir[F.tag - 1];
            const double gamma_f = sipg(g, F);
            const long long bf = bface_index3(g, cf[q]);
            for (int qa = 0; qa < 6; ++qa)
                for (int qb = 0; qb < 6; ++qb) {
                    const double w = g.g6w[qa] * g.g6w[qb] * F.measure;
                    const long long sp = (bf * 36 + qa * 6 + qb) * 3;
                    double rp[3], tv[3], mud[3];
                    ref_point(g, F, c, g.g6p[qa], g.g6p[qb], rp);
                    for (int d = 0; d < 3; ++d) mud[d] = dir[d] ? sm.dirichlet[sp + d] : 0.0;
                    const double nv = shp(a, rp);
                    if (!dir[comp]) r += w * nv * sm.traction[sp + comp];
                    if (dir[comp]) r += w * gamma_f * nv * mud[comp];
                    traction(g, a, comp, rp, F.n, tv);
                    r -= w * dot3(tv, mud);
                }
        }
        u[t] = r + 0.0;
    }
}

__global__ void k_rhs_qvalues3(Geo3 g, int nq, const signed char* qc, Samples3 sm, double* qv) {
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nq; f += gridDim.x * blockDim.x) {
        double v = 0.0;
        if (qc[f]) {
            const Face3 F = face_info(g, f);
            const long long bf = bface_index3(g, f);
            for (int qa = 0; qa < 6; ++qa)
                for (int qb = 0; qb < 6; ++qb) {
                    const double w = g.g6w[qa] * g.g6w[qb] * F.measure;
                    v += w / F.measure * sm.flow[bf * 36 + qa * 6 + qb];
                }
        }
        qv[f] = v;
    }
}

__global__ void k_rhs_qp_s3(Geo3 g, int nq, int np, const double* __restrict__ kcells, const signed char* qc, Samples3 sm,
                            const double* __restrict__ qv, double* q, double* p) {
    const double vol = g.h[0] * g.h[1] * g.h[2];
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nq; f += gridDim.x * blockDim.x) {
        const Face3 F = face_info(g, f);
        if (qc[f]) {
            q[f] = qv[f];
            continue;
        }
        double r = 0.0;
        if (sm.darcy)
            for (int side = 0; side < 2; ++side) {
                const int c = side ? F.cp : F.cm;
                if (c < 0) continue;
                int f0, f1;
                axis_faces(g, c, F.axis, f0, f1);
                const bool low = f == f0;
                const double sg = F.n[F.axis];
                for (int qi = 0; qi < 6; ++qi)
                    for (int qj = 0; qj < 6; ++qj)
                        for (int qk = 0; qk < 6; ++qk) {
                            const double ref[3] = {g.g6p[qi], g.g6p[qj], g.g6p[qk]};
                            const double w = g.g6w[qi] * g.g6w[qj] * g.g6w[qk] * vol;
                            const double wf = low ? sg * (1.0 - ref[F.axis]) : sg * ref[F.axis];
                            r += w * wf * sm.darcy[((long long)c * 216 + (qi * 6 + qj) * 6 + qk) * 3 + F.axis];
                        }
            }
        if (F.boundary) {
            const long long bf = bface_index3(g, f);
            for (int qa = 0; qa < 6; ++qa)
                for (int qb = 0; qb < 6; ++qb) {
                    const double w = g.g6w[qa] * g.g6w[qb] * F.measure;
                    r -= w * sm.flow[bf * 36 + qa * 6 + qb];
                }
        }
        for (int side = 0; side < 2; ++side) {  // eliminated couplings to constrained faces (mq_bc)
            const int c = side ? F.cp : F.cm;
            if (c < 0) continue;
            int f0, f1;
            axis_faces(g, c, F.axis, f0, f1);
            const int opp = (f == f0) ? f1 : f0;
            if (!qc[opp]) continue;
            const double keff = g.eta / (kcells ? kcells[c] : g.kperm);
            const double d6 = keff * vol / 6.0;
            const Face3 F0 = face_info(g, f0), F1 = face_info(g, f1);
            const double cross = d6 * F0.n[F.axis] * F1.n[F.axis];
            r -= cross * qv[opp];
        }
        q[f] = r;
    }
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < np; c += gridDim.x * blockDim.x) {
        double r = 0.0;
        if (sm.mass)
            for (int qi = 0; qi < 6; ++qi)
                for (int qj = 0; qj < 6; ++qj)
                    for (int qk = 0; qk < 6; ++qk) {
                        const double w = g.g6w[qi] * g.g6w[qj] * g.g6w[qk] * vol;
                        r -= w * sm.mass[(long long)c * 216 + (qi * 6 + qj) * 6 + qk];
                    }
        // b_bc: the cell's constrained faces in the order xlo, xhi, ylo, yhi, zlo, zhi
        for (int axis = 0; axis < 3; ++axis) {
            int ff[2];
            axis_faces(g, c, axis, ff[0], ff[1]);
            for (int e = 0; e < 2; ++e) {
                if (!qc[ff[e]]) continue;
                const Face3 F = face_info(g, ff[e]);
                const double sout = F.boundary ? 1.0 : (c == F.cm ? 1.0 : -1.0);
                const double v = -sout * F.measure;
                r -= v * qv[ff[e]];
            }
        }
        p[c] = r;
    }
}

Geo3 make_geo3(const pdg_problem3& p) {
    Geo3 g{};
    g.nx = p.nx;
    g.ny = p.ny;
    g.nz = p.nz;
    g.h[0] = p.lx / p.nx;
    g.h[1] = p.ly / p.ny;
    g.h[2] = p.lz / p.nz;
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
    for (int s = 0; s < 6; ++s) {
        const int kind = p.disp_kind[s];
        require(kind >= 0 && kind <= 4, "pdg_problem3: bad displacement kind");
        g.disp_dir[s][0] = (kind == 0 || kind == 2);
        g.disp_dir[s][1] = (kind == 0 || kind == 3);
        g.disp_dir[s][2] = (kind == 0 || kind == 4);
        for (int d = 0; d < 3; ++d) g.disp_data[s][d] = p.disp_data[s][d];
        require(p.flow_kind[s] == 0 || p.flow_kind[s] == 1, "pdg_problem3: bad flow kind");
        g.flow_kind[s] = p.flow_kind[s];
        g.flow_data[s] = p.flow_data[s];
    }
    return g;
}

void scan_offsets3(const int* len, int* off, int n, cudaStream_t st) {
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, len, off, n + 1, st);
    DBuf<unsigned char> buf(tmp + 1);
    cub::DeviceScan::ExclusiveSum(buf.p, tmp, len, off, n + 1, st);
}

int last_offset3(const int* off, int n, cudaStream_t st) {
    int v = 0;
    PDG_CUDA(cudaMemcpyAsync(&v, off + n, sizeof(int), cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    return v;
}

}  // namespace

void assemble_ops_device3(SpatialOps& s, const pdg_problem3& p, cudaStream_t st) {
    require(p.nx >= 1 && p.ny >= 1 && p.nz >= 1, "build_mesh: cell counts must be positive");
    require(p.lx > 0.0 && p.ly > 0.0 && p.lz > 0.0, "build_mesh: edge lengths must be positive");
    require(p.penalty > 0.0, "assemble_operators: penalty must be positive");
    require(p.mu > 0.0, "material: mu must be positive");
    require(p.eta > 0.0, "material: eta must be positive");
    require(p.biot_m > 0.0, "material: Biot modulus M must be positive");
    require(p.biot_b > 0.0 && p.biot_b <= 1.0, "material: Biot coefficient b must lie in (0, 1]");
    require(p.k_perm > 0.0, "material: permeability must be positive");
    require(24LL * p.nx * p.ny * p.nz * 168 < (1LL << 31), "pdg_ops_assemble3: mesh too large for int32 CSR offsets");
    const Geo3 g = make_geo3(p);
    s.nx = p.nx;
    s.ny = p.ny;
    s.nz = p.nz;
    const int n = p.nx * p.ny * p.nz;
    s.n_u = 24 * n;
    s.n_p = n;
    s.n_q = p.nx * p.ny * (p.nz + 1) + p.nx * (p.ny + 1) * p.nz + (p.nx + 1) * p.ny * p.nz;
    s.biot_b = p.biot_b;
    s.inv_m = 1.0 / p.biot_m;
    s.k_dr = p.lambda + 2.0 * p.mu / 3;  // lambda + 2 mu / d, d = 3
    s.has_problem = true;
    s.prob3 = p;
    DBuf<double> kc;
    if (p.k_perm_cells) {
        s.k_cells.assign(p.k_perm_cells, p.k_perm_cells + n);
        for (double k : s.k_cells) require(k > 0.0, "material: per-cell permeability must be positive");
        kc.upload(s.k_cells, st);
    }
    s.prob3.k_perm_cells = nullptr;
    // A, E
    DBuf<int> alen(s.n_u + 1), elen(s.n_u + 1);
    k_row_lengths3<<<grid_for(n, 256), 256, 0, st>>>(g, alen.p, elen.p);
    PDG_CHECK_LAUNCH();
    s.A.rows = s.A.cols = s.n_u;
    s.E.rows = s.n_u;
    s.E.cols = s.n_p;
    s.A.off.alloc(s.n_u + 1);
    s.E.off.alloc(s.n_u + 1);
    scan_offsets3(alen.p, s.A.off.p, s.n_u, st);
    scan_offsets3(elen.p, s.E.off.p, s.n_u, st);
    s.A.nnz = last_offset3(s.A.off.p, s.n_u, st);
    s.E.nnz = last_offset3(s.E.off.p, s.n_u, st);
    s.A.idx.alloc(s.A.nnz);
    s.A.val.alloc(s.A.nnz);
    s.E.idx.alloc(s.E.nnz);
    s.E.val.alloc(s.E.nnz);
    k_assemble_cell3<<<n, 576, 0, st>>>(g, s.A.off.p, s.A.idx.p, s.A.val.p, s.E.off.p, s.E.idx.p, s.E.val.p);
    PDG_CHECK_LAUNCH();
    // flux blocks
    s.q_constrained.alloc(s.n_q);
    k_qc3<<<grid_for(s.n_q, 256), 256, 0, st>>>(g, s.n_q, s.q_constrained.p);
    DBuf<int> mql(s.n_q + 1), bl(s.n_q + 1);
    k_flux_lengths3<<<grid_for(s.n_q, 256), 256, 0, st>>>(g, s.n_q, s.q_constrained.p, mql.p, bl.p);
    PDG_CHECK_LAUNCH();
    s.M_q.rows = s.M_q.cols = s.n_q;
    s.B.rows = s.n_q;
    s.B.cols = s.n_p;
    s.M_q.off.alloc(s.n_q + 1);
    s.B.off.alloc(s.n_q + 1);
    scan_offsets3(mql.p, s.M_q.off.p, s.n_q, st);
    scan_offsets3(bl.p, s.B.off.p, s.n_q, st);
    s.M_q.nnz = last_offset3(s.M_q.off.p, s.n_q, st);
    s.B.nnz = last_offset3(s.B.off.p, s.n_q, st);
    s.M_q.idx.alloc(s.M_q.nnz);
    s.M_q.val.alloc(s.M_q.nnz);
    s.B.idx.alloc(s.B.nnz);
    s.B.val.alloc(s.B.nnz);
    k_flux_fill3<<<grid_for(s.n_q, 256), 256, 0, st>>>(g, s.n_q, kc.n ? kc.p : nullptr, s.q_constrained.p, s.M_q.off.p,
                                                        s.M_q.idx.p, s.M_q.val.p, s.B.off.p, s.B.idx.p, s.B.val.p);
    PDG_CHECK_LAUNCH();
    s.m_p.alloc(s.n_p);
    k_mp3<<<grid_for(n, 256), 256, 0, st>>>(g, n, s.m_p.p);
    PDG_CHECK_LAUNCH();
    PDG_CUDA(cudaStreamSynchronize(st));
}

void assemble_rhs_sampled_device3(const SpatialOps& s, const pdg_rhs_samples& h, double* u, double* q, double* p,
                                  cudaStream_t st) {
    require(h.traction && h.dirichlet && h.flow, "pdg_ops_rhs_sampled: boundary samples must be given");
    const Geo3 g = make_geo3(s.prob3);
    const size_t nc = (size_t)s.n_p;
    const size_t nbf = 2 * ((size_t)s.nx * s.ny + (size_t)s.nx * s.nz + (size_t)s.ny * s.nz);
    DBuf<double> mom, dar, mas, tra, dir, flo, kc, qv(s.n_q);
    Samples3 sm{};
    if (h.momentum) {
        mom.upload(h.momentum, nc * 648, st);
        sm.momentum = mom.p;
    }
    if (h.darcy) {
        dar.upload(h.darcy, nc * 648, st);
        sm.darcy = dar.p;
    }
    if (h.mass) {
        mas.upload(h.mass, nc * 216, st);
        sm.mass = mas.p;
    }
    tra.upload(h.traction, nbf * 108, st);
    dir.upload(h.dirichlet, nbf * 108, st);
    flo.upload(h.flow, nbf * 36, st);
    sm.traction = tra.p;
    sm.dirichlet = dir.p;
    sm.flow = flo.p;
    if (!s.k_cells.empty()) kc.upload(s.k_cells, st);
    k_rhs_u_s3<<<grid_for(24LL * s.n_p, 256), 256, 0, st>>>(g, sm, u);
    k_rhs_qvalues3<<<grid_for(s.n_q, 256), 256, 0, st>>>(g, s.n_q, s.q_constrained.p, sm, qv.p);
    k_rhs_qp_s3<<<grid_for(std::max(s.n_q, s.n_p), 256), 256, 0, st>>>(g, s.n_q, s.n_p, kc.n ? kc.p : nullptr,
                                                                        s.q_constrained.p, sm, qv.p, q, p);
    count_launch(3);
    PDG_CHECK_LAUNCH();
    PDG_CUDA(cudaStreamSynchronize(st));  // the staging buffers are released at scope exit
}

void assemble_rhs_device3(const SpatialOps& s, double t, double* u, double* q, double* p, cudaStream_t st) {
    (void)t;  // constant boundary data: time-independent
    const Geo3 g = make_geo3(s.prob3);
    k_rhs_u3<<<grid_for(24LL * s.n_p, 256), 256, 0, st>>>(g, u);
    k_rhs_qp3<<<grid_for(std::max(s.n_q, s.n_p), 256), 256, 0, st>>>(g, s.n_q, s.n_p, q, p);
    count_launch(2);
    PDG_CHECK_LAUNCH();
}

}  // namespace pdg
