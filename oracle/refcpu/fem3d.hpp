// ORACLE / TEST INFRASTRUCTURE ONLY. Not part of the product.
//
// 3D extension of the CPU restatement (BASELINE configs 2 and 4). The reference
// is 2D only (material.hpp:44 dim = 2), so there is
// NO reference arithmetic to follow here: PARITY UNPINNED. This file generalises
// fem.hpp's restatement of assembly.hpp:177-563 dimension by dimension (the same
// element pair on hexahedra: discontinuous trilinear displacement with SIPG,
// lowest-order Raviart-Thomas flux as one normal-velocity dof per face, piecewise
// constant pressure), keeps the reference's conventions (push order: cell term,
// then faces in ascending face index, one push per face quadrature point;
// eliminated no-flux faces; Nitsche Dirichlet faces) and is validated by its own
// properties in tests/test_oracle3d.py (symmetry, rigid-body and patch tests,
// divergence identities, RT0 exactness, agreement of the 2D code on extruded
// data). The device assembly (csrc/assembly3d.cu) is checked bit for bit against
// this file.
//
// Conventions (the 2D ones of mesh.hpp:42-67 / dofs.hpp:28-46, extended):
//   cell  c = (k ny + j) nx + i
//   faces by normal axis, highest axis first (2D: horizontal faces, then vertical):
//     z-normal (k = 0..nz)  f = (k ny + j) nx + i
//     y-normal (j = 0..ny)  f = nzf + (j nz + k) nx + i
//     x-normal (i = 0..nx)  f = nzf + nyf + (i nz + k) ny + j
//   cell faces in the order xlo, xhi, ylo, yhi, zlo, zhi (2D: W, E, S, N)
//   tags: 0 interior, 1 xlo, 2 xhi, 3 ylo, 4 yhi, 5 zlo, 6 zhi
//   nodes a = 4 az + 2 ay + ax; u dof = 24 c + 3 a + comp; q dof = face; p dof = cell
#pragma once

#include "fem.hpp"

namespace refcpu {

struct Cell3 {
    double x0, y0, z0, hx, hy, hz;
    double volume() const { return hx * hy * hz; }
    double h(int axis) const { return axis == 0 ? hx : axis == 1 ? hy : hz; }
};

struct Face3 {
    int axis;  // normal axis 0 x, 1 y, 2 z
    int cell_minus, cell_plus;
    double n[3];
    double measure;
    int tag;
    int idx;  // index of the face plane along its axis (0..n_axis)
    bool is_boundary() const { return cell_plus < 0; }
};

struct Mesh3 {
    int nx = 0, ny = 0, nz = 0;
    double lx = 0, ly = 0, lz = 0;
    std::vector<Cell3> cells;
    std::vector<Face3> faces;
    int n_cells() const { return nx * ny * nz; }
    int n_faces() const { return static_cast<int>(faces.size()); }
    int nzf() const { return nx * ny * (nz + 1); }
    int nyf() const { return nx * (ny + 1) * nz; }
    int cell_index(int i, int j, int k) const { return (k * ny + j) * nx + i; }
    int z_face(int i, int j, int k) const { return (k * ny + j) * nx + i; }
    int y_face(int i, int j, int k) const { return nzf() + (j * nz + k) * nx + i; }
    int x_face(int i, int j, int k) const { return nzf() + nyf() + (i * nz + k) * ny + j; }
    std::array<int, 6> cell_faces(int c) const {
        const int i = c % nx, j = (c / nx) % ny, k = c / (nx * ny);
        return {x_face(i, j, k), x_face(i + 1, j, k), y_face(i, j, k), y_face(i, j + 1, k), z_face(i, j, k),
                z_face(i, j, k + 1)};
    }
};

inline Mesh3 build_mesh3(int nx, int ny, int nz, double lx, double ly, double lz) {
    if (nx < 1 || ny < 1 || nz < 1) throw std::invalid_argument("build_mesh: cell counts must be positive");
    if (!(lx > 0.0) || !(ly > 0.0) || !(lz > 0.0)) throw std::invalid_argument("build_mesh: edge lengths must be positive");
    Mesh3 m;
    m.nx = nx;
    m.ny = ny;
    m.nz = nz;
    m.lx = lx;
    m.ly = ly;
    m.lz = lz;
    const double hx = lx / nx, hy = ly / ny, hz = lz / nz;
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) m.cells.push_back({i * hx, j * hy, k * hz, hx, hy, hz});
    auto make = [&](int axis, int idx, int nax, int c_lo, int c_hi, double measure) {
        Face3 f{};
        f.axis = axis;
        f.idx = idx;
        f.measure = measure;
        f.n[0] = f.n[1] = f.n[2] = 0.0;
        if (idx == 0) {
            f.cell_minus = c_hi;
            f.cell_plus = -1;
            f.n[axis] = -1.0;
            f.tag = 1 + 2 * axis;
        } else if (idx == nax) {
            f.cell_minus = c_lo;
            f.cell_plus = -1;
            f.n[axis] = 1.0;
            f.tag = 2 + 2 * axis;
        } else {
            f.cell_minus = c_lo;
            f.cell_plus = c_hi;
            f.n[axis] = 1.0;
            f.tag = 0;
        }
        m.faces.push_back(f);
    };
    for (int k = 0; k <= nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i)
                make(2, k, nz, k > 0 ? m.cell_index(i, j, k - 1) : -1, k < nz ? m.cell_index(i, j, k) : -1, hx * hy);
    for (int j = 0; j <= ny; ++j)
        for (int k = 0; k < nz; ++k)
            for (int i = 0; i < nx; ++i)
                make(1, j, ny, j > 0 ? m.cell_index(i, j - 1, k) : -1, j < ny ? m.cell_index(i, j, k) : -1, hx * hz);
    for (int i = 0; i <= nx; ++i)
        for (int k = 0; k < nz; ++k)
            for (int j = 0; j < ny; ++j)
                make(0, i, nx, i > 0 ? m.cell_index(i - 1, j, k) : -1, i < nx ? m.cell_index(i, j, k) : -1, hy * hz);
    return m;
}

inline double face_outward_sign3(const Mesh3& mesh, int f, int c) {
    const Face3& face = mesh.faces[f];
    if (face.cell_plus < 0) return 1.0;
    return c == face.cell_minus ? 1.0 : -1.0;
}

using VectorField3T = std::function<std::array<double, 3>(double, double, double, double)>;
using ScalarField3T = std::function<double(double, double, double, double)>;

struct DisplacementBC3 {
    std::array<bool, 3> dirichlet = {false, false, false};
    std::array<double, 3> dirichlet_data = {0.0, 0.0, 0.0};  // constant data only
    std::array<double, 3> traction_data = {0.0, 0.0, 0.0};
};
struct FlowBC3 {
    bool no_flow = false;
    double pressure = 0.0;
};
struct BoundarySpec3 {
    std::array<DisplacementBC3, 6> displacement;  // slot = tag - 1
    std::array<FlowBC3, 6> flow;
};

namespace shapes3 {
inline double l(int b, double t) { return b ? t : 1.0 - t; }
inline double dl(int b) { return b ? 1.0 : -1.0; }
inline double n(int a, double xi, double eta, double zeta) {
    return l(a & 1, xi) * l((a >> 1) & 1, eta) * l(a >> 2, zeta);
}
inline std::array<double, 3> grad(const Cell3& c, int a, double xi, double eta, double zeta) {
    const int ax = a & 1, ay = (a >> 1) & 1, az = a >> 2;
    return {dl(ax) * l(ay, eta) * l(az, zeta) / c.hx, l(ax, xi) * dl(ay) * l(az, zeta) / c.hy,
            l(ax, xi) * l(ay, eta) * dl(az) / c.hz};
}
// strain of basis (a, comp): {xx, yy, zz, xy, xz, yz}
inline std::array<double, 6> strain(const Cell3& c, int a, int comp, double xi, double eta, double zeta) {
    const auto g = grad(c, a, xi, eta, zeta);
    if (comp == 0) return {g[0], 0.0, 0.0, 0.5 * g[1], 0.5 * g[2], 0.0};
    if (comp == 1) return {0.0, g[1], 0.0, 0.5 * g[0], 0.0, 0.5 * g[2]};
    return {0.0, 0.0, g[2], 0.0, 0.5 * g[0], 0.5 * g[1]};
}
// sigma(basis) n with sigma = 2 mu eps + lambda tr(eps) I
inline std::array<double, 3> traction(const Cell3& c, const MaterialParameters& m, int a, int comp, double xi,
                                      double eta, double zeta, const double* nrm) {
    const auto g = grad(c, a, xi, eta, zeta);
    const double lam = m.lambda_lame, mu = m.mu_lame;
    double sxx, syy, szz, sxy, sxz, syz;
    if (comp == 0) {
        sxx = (2.0 * mu + lam) * g[0];
        syy = lam * g[0];
        szz = lam * g[0];
        sxy = mu * g[1];
        sxz = mu * g[2];
        syz = 0.0;
    } else if (comp == 1) {
        sxx = lam * g[1];
        syy = (2.0 * mu + lam) * g[1];
        szz = lam * g[1];
        sxy = mu * g[0];
        sxz = 0.0;
        syz = mu * g[2];
    } else {
        sxx = lam * g[2];
        syy = lam * g[2];
        szz = (2.0 * mu + lam) * g[2];
        sxy = 0.0;
        sxz = mu * g[0];
        syz = mu * g[1];
    }
    return {sxx * nrm[0] + sxy * nrm[1] + sxz * nrm[2], sxy * nrm[0] + syy * nrm[1] + syz * nrm[2],
            sxz * nrm[0] + syz * nrm[1] + szz * nrm[2]};
}
}  // namespace shapes3

// reference point of `cell` on face f at tangential coordinates (s1, s2) along the
// two remaining axes in ascending axis order
inline std::array<double, 3> face_ref_point3(const Mesh3& mesh, int f, int cell, double s1, double s2) {
    const Face3& face = mesh.faces[f];
    const int nx = mesh.nx, ny = mesh.ny;
    const int ci[3] = {cell % nx, (cell / nx) % ny, cell / (nx * ny)};
    const double fixed = face.idx == ci[face.axis] ? 0.0 : 1.0;
    if (face.axis == 0) return {fixed, s1, s2};
    if (face.axis == 1) return {s1, fixed, s2};
    return {s1, s2, fixed};
}

inline double sipg_face_coefficient3(const Mesh3& mesh, const MaterialParameters& mat, double gamma, int face) {
    const Face3& f = mesh.faces[face];
    double h = 0.0;
    int cnt = 0;
    for (int c : {f.cell_minus, f.cell_plus}) {
        if (c < 0) continue;
        h += mesh.cells[c].h(f.axis);
        ++cnt;
    }
    h /= cnt;
    return gamma * (mat.lambda_lame + 2.0 * mat.mu_lame) / h;
}

inline MaterialParameters material_from_lame3(double lambda, double mu, double k_perm, double eta, double biot_m,
                                              double biot_b) {
    MaterialParameters m;
    m.lambda_lame = lambda;
    m.mu_lame = mu;
    m.k_perm = k_perm;
    m.eta = eta;
    m.biot_m = biot_m;
    m.k_dr = lambda + 2.0 * mu / 3;  // lambda + 2 mu / d, d = 3 (material.hpp:63-66 with dim = 3)
    m.biot_b = biot_b;
    if (!(mu > 0.0)) throw std::invalid_argument("material: mu must be positive");
    if (!(eta > 0.0)) throw std::invalid_argument("material: eta must be positive");
    if (!(biot_m > 0.0)) throw std::invalid_argument("material: Biot modulus M must be positive");
    if (!(biot_b > 0.0) || biot_b > 1.0) throw std::invalid_argument("material: Biot coefficient b must lie in (0, 1]");
    if (!(k_perm > 0.0)) throw std::invalid_argument("material: permeability must be positive");
    return m;
}

inline double dot3(const std::array<double, 3>& a, const std::array<double, 3>& b) {
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

// 3D analogue of assemble_operators (fem.hpp; assembly.hpp:177-395)
inline SpatialOperators assemble_operators3(const Mesh3& mesh, const MaterialParameters& mat, double penalty_gamma,
                                            const BoundarySpec3& bc) {
    if (!(penalty_gamma > 0.0)) throw std::invalid_argument("assemble_operators: penalty must be positive");
    for (double k : mat.k_perm_cells)
        if (!(k > 0.0)) throw std::invalid_argument("material: per-cell permeability must be positive");
    SpatialOperators ops;
    ops.penalty = penalty_gamma;
    ops.mat = mat;
    ops.n_u = 24 * mesh.n_cells();
    ops.n_q = mesh.n_faces();
    ops.n_p = mesh.n_cells();
    const QuadratureRule g2 = gauss_legendre(2);

    ops.q_constrained.assign(ops.n_q, 0);
    for (int f = 0; f < mesh.n_faces(); ++f) {
        const Face3& face = mesh.faces[f];
        if (face.is_boundary() && bc.flow[face.tag - 1].no_flow) ops.q_constrained[f] = 1;
    }

    std::vector<Triplet> ta, tmq, tb, te, tmp;
    const size_t nc = static_cast<size_t>(mesh.n_cells());
    ta.reserve(nc * 576 + static_cast<size_t>(mesh.n_faces()) * 4 * 2304);
    te.reserve(nc * 24 + static_cast<size_t>(mesh.n_faces()) * 4 * 96);

    // ---- cell contributions
    for (int c = 0; c < mesh.n_cells(); ++c) {
        const Cell3& cell = mesh.cells[c];
        const double vol = cell.volume();
        const double lam = mat.lambda_lame, mu = mat.mu_lame;
        double ke[24][24] = {};
        double div_int[24] = {};
        for (size_t qi = 0; qi < 2; ++qi)
            for (size_t qj = 0; qj < 2; ++qj)
                for (size_t qk = 0; qk < 2; ++qk) {
                    const double xi = g2.points[qi], eta = g2.points[qj], zeta = g2.points[qk];
                    const double w = g2.weights[qi] * g2.weights[qj] * g2.weights[qk] * vol;
                    std::array<std::array<double, 6>, 24> eps;
                    for (int l = 0; l < 24; ++l) eps[l] = shapes3::strain(cell, l / 3, l % 3, xi, eta, zeta);
                    for (int l1 = 0; l1 < 24; ++l1) {
                        for (int l2 = 0; l2 <= l1; ++l2) {
                            const auto &e1 = eps[l1], &e2 = eps[l2];
                            const double v = 2.0 * mu *
                                                 (e1[0] * e2[0] + e1[1] * e2[1] + e1[2] * e2[2] + 2.0 * e1[3] * e2[3] +
                                                  2.0 * e1[4] * e2[4] + 2.0 * e1[5] * e2[5]) +
                                             lam * (e1[0] + e1[1] + e1[2]) * (e2[0] + e2[1] + e2[2]);
                            ke[l1][l2] += w * v;
                            if (l2 != l1) ke[l2][l1] += w * v;
                        }
                        div_int[l1] += w * (eps[l1][0] + eps[l1][1] + eps[l1][2]);
                    }
                }
        for (int l1 = 0; l1 < 24; ++l1) {
            for (int l2 = 0; l2 < 24; ++l2) ta.push_back({24 * c + l1, 24 * c + l2, ke[l1][l2]});
            te.push_back({24 * c + l1, c, div_int[l1]});
        }

        const auto cf = mesh.cell_faces(c);
        const double keff = mat.eta / mat.permeability(c);
        std::array<double, 6> sgn{};
        for (int k = 0; k < 6; ++k) {
            const Face3& f = mesh.faces[cf[k]];
            sgn[k] = f.n[f.axis];
        }
        const double d3 = keff * vol / 3.0, d6 = keff * vol / 6.0;
        for (int pair = 0; pair < 3; ++pair) {
            const int f0 = cf[2 * pair], f1 = cf[2 * pair + 1];
            const double cross = d6 * sgn[2 * pair] * sgn[2 * pair + 1];
            auto push_mq = [&](int r, int cc, double v) {
                const bool rc = ops.q_constrained[r], cc_c = ops.q_constrained[cc];
                if (rc) return;
                if (cc_c)
                    ops.mq_bc.push_back({r, cc, v});
                else
                    tmq.push_back({r, cc, v});
            };
            push_mq(f0, f0, d3);
            push_mq(f1, f1, d3);
            push_mq(f0, f1, cross);
            push_mq(f1, f0, cross);
        }
        for (int k = 0; k < 6; ++k) {
            const int f = cf[k];
            const double sout = face_outward_sign3(mesh, f, c);
            const double v = -sout * mesh.faces[f].measure;
            if (ops.q_constrained[f])
                ops.b_bc.push_back({f, c, v});
            else
                tb.push_back({f, c, v});
        }
        tmp.push_back({c, c, vol});
    }
    for (int f = 0; f < ops.n_q; ++f)
        if (ops.q_constrained[f]) tmq.push_back({f, f, 1.0});

    // ---- face contributions (2 x 2 Gauss points per face, first tangential axis outer)
    for (int f = 0; f < mesh.n_faces(); ++f) {
        const Face3& face = mesh.faces[f];
        const double gamma_f = sipg_face_coefficient3(mesh, mat, penalty_gamma, f);
        if (!face.is_boundary()) {
            const std::array<int, 2> cells = {face.cell_minus, face.cell_plus};
            const std::array<double, 2> side_sign = {1.0, -1.0};
            for (size_t qa = 0; qa < 2; ++qa)
                for (size_t qb = 0; qb < 2; ++qb) {
                    const double w = g2.weights[qa] * g2.weights[qb] * face.measure;
                    std::array<std::array<std::array<double, 3>, 24>, 2> val{}, trac{};
                    for (int side = 0; side < 2; ++side) {
                        const Cell3& cell = mesh.cells[cells[side]];
                        const auto rp = face_ref_point3(mesh, f, cells[side], g2.points[qa], g2.points[qb]);
                        for (int l = 0; l < 24; ++l) {
                            const int a = l / 3, comp = l % 3;
                            const double nv = shapes3::n(a, rp[0], rp[1], rp[2]);
                            val[side][l] = {comp == 0 ? nv : 0.0, comp == 1 ? nv : 0.0, comp == 2 ? nv : 0.0};
                            trac[side][l] = shapes3::traction(cell, mat, a, comp, rp[0], rp[1], rp[2], face.n);
                        }
                    }
                    for (int s1 = 0; s1 < 2; ++s1)
                        for (int l1 = 0; l1 < 24; ++l1) {
                            const int gi = 24 * cells[s1] + l1;
                            for (int s2 = 0; s2 < 2; ++s2)
                                for (int l2 = 0; l2 < 24; ++l2) {
                                    const int gj = 24 * cells[s2] + l2;
                                    const double cons = -0.5 * dot3(trac[s2][l2], val[s1][l1]) * side_sign[s1];
                                    const double symm = -0.5 * dot3(trac[s1][l1], val[s2][l2]) * side_sign[s2];
                                    const double pen =
                                        gamma_f * side_sign[s1] * side_sign[s2] * dot3(val[s1][l1], val[s2][l2]);
                                    ta.push_back({gi, gj, w * (cons + symm + pen)});
                                }
                            const double nv = face.n[0] * val[s1][l1][0] + face.n[1] * val[s1][l1][1] +
                                              face.n[2] * val[s1][l1][2];
                            for (int pc = 0; pc < 2; ++pc) te.push_back({gi, cells[pc], -0.5 * w * side_sign[s1] * nv});
                        }
                }
        } else {
            const int c = face.cell_minus;
            const Cell3& cell = mesh.cells[c];
            const DisplacementBC3& dbc = bc.displacement[face.tag - 1];
            if (!dbc.dirichlet[0] && !dbc.dirichlet[1] && !dbc.dirichlet[2]) continue;
            const int ncmp = face.axis;
            for (size_t qa = 0; qa < 2; ++qa)
                for (size_t qb = 0; qb < 2; ++qb) {
                    const double w = g2.weights[qa] * g2.weights[qb] * face.measure;
                    const auto rp = face_ref_point3(mesh, f, c, g2.points[qa], g2.points[qb]);
                    std::array<std::array<double, 3>, 24> val{}, trac{};
                    for (int l = 0; l < 24; ++l) {
                        const int a = l / 3, comp = l % 3;
                        const double nv = shapes3::n(a, rp[0], rp[1], rp[2]);
                        val[l] = {comp == 0 ? nv : 0.0, comp == 1 ? nv : 0.0, comp == 2 ? nv : 0.0};
                        trac[l] = shapes3::traction(cell, mat, a, comp, rp[0], rp[1], rp[2], face.n);
                    }
                    auto mask = [&](const std::array<double, 3>& v) {
                        return std::array<double, 3>{dbc.dirichlet[0] ? v[0] : 0.0, dbc.dirichlet[1] ? v[1] : 0.0,
                                                     dbc.dirichlet[2] ? v[2] : 0.0};
                    };
                    for (int l1 = 0; l1 < 24; ++l1) {
                        const int gi = 24 * c + l1;
                        const auto mv1 = mask(val[l1]);
                        for (int l2 = 0; l2 < 24; ++l2) {
                            const int gj = 24 * c + l2;
                            const auto mv2 = mask(val[l2]);
                            const double cons = -dot3(trac[l2], mv1);
                            const double symm = -dot3(trac[l1], mv2);
                            const double pen = gamma_f * dot3(mv1, mv2);
                            ta.push_back({gi, gj, w * (cons + symm + pen)});
                        }
                        if (dbc.dirichlet[ncmp]) {
                            const double nv =
                                face.n[0] * val[l1][0] + face.n[1] * val[l1][1] + face.n[2] * val[l1][2];
                            te.push_back({gi, c, -w * nv});
                        }
                    }
                }
        }
    }

    ops.A = csr_from_triplets(ops.n_u, ops.n_u, ta);
    ops.M_q = csr_from_triplets(ops.n_q, ops.n_q, tmq);
    ops.B = csr_from_triplets(ops.n_q, ops.n_p, tb);
    ops.E = csr_from_triplets(ops.n_u, ops.n_p, te);
    ops.M_p = csr_from_triplets(ops.n_p, ops.n_p, tmp);
    ops.m_p_diag.resize(ops.n_p);
    for (int c = 0; c < ops.n_p; ++c) ops.m_p_diag[c] = mesh.cells[c].volume();
    ops.rhs_ref_u.assign(ops.n_u, 0.0);
    // faces grouped by z level (z faces of level k, then the y and x faces of cell layer k):
    // the banded ordering of the flux Schur complement (solver.hpp FlowSchurSolver)
    for (int k = 0; k <= mesh.nz; ++k) {
        for (int j = 0; j < mesh.ny; ++j)
            for (int i = 0; i < mesh.nx; ++i) ops.face_band_perm.push_back(mesh.z_face(i, j, k));
        if (k == mesh.nz) break;
        for (int j = 0; j <= mesh.ny; ++j)
            for (int i = 0; i < mesh.nx; ++i) ops.face_band_perm.push_back(mesh.y_face(i, j, k));
        for (int i = 0; i <= mesh.nx; ++i)
            for (int j = 0; j < mesh.ny; ++j) ops.face_band_perm.push_back(mesh.x_face(i, j, k));
    }
    return ops;
}

// 3D analogue of assemble_rhs (assembly.hpp:467-563) for constant boundary data and no
// volume data: 6 x 6 Gauss points per boundary face.
inline FieldVecs assemble_rhs3(const Mesh3& mesh, const MaterialParameters& mat, const SpatialOperators& ops,
                               const BoundarySpec3& bc, double /*t*/) {
    FieldVecs r;
    r.u.assign(ops.n_u, 0.0);
    r.q.assign(ops.n_q, 0.0);
    r.p.assign(ops.n_p, 0.0);
    const QuadratureRule gq = gauss_legendre(kDataQuadOrder);
    Vec q_values(ops.n_q, 0.0);
    for (int f = 0; f < mesh.n_faces(); ++f) {
        const Face3& face = mesh.faces[f];
        if (!face.is_boundary()) continue;
        const int c = face.cell_minus;
        const Cell3& cell = mesh.cells[c];
        const DisplacementBC3& dbc = bc.displacement[face.tag - 1];
        const FlowBC3& fbc = bc.flow[face.tag - 1];
        const double gamma_f = sipg_face_coefficient3(mesh, mat, ops.penalty, f);
        for (size_t qa = 0; qa < gq.points.size(); ++qa)
            for (size_t qb = 0; qb < gq.points.size(); ++qb) {
                const double w = gq.weights[qa] * gq.weights[qb] * face.measure;
                const auto rp = face_ref_point3(mesh, f, c, gq.points[qa], gq.points[qb]);
                const std::array<double, 3> tn = dbc.traction_data;
                const std::array<double, 3> mud = {dbc.dirichlet[0] ? dbc.dirichlet_data[0] : 0.0,
                                                   dbc.dirichlet[1] ? dbc.dirichlet_data[1] : 0.0,
                                                   dbc.dirichlet[2] ? dbc.dirichlet_data[2] : 0.0};
                for (int l = 0; l < 24; ++l) {
                    const int a = l / 3, comp = l % 3;
                    const double nv = shapes3::n(a, rp[0], rp[1], rp[2]);
                    const int gi = 24 * c + l;
                    if (!dbc.dirichlet[comp]) r.u[gi] += w * nv * tn[comp];
                    if (dbc.dirichlet[comp]) r.u[gi] += w * gamma_f * nv * mud[comp];
                    const auto tv = shapes3::traction(cell, mat, a, comp, rp[0], rp[1], rp[2], face.n);
                    r.u[gi] -= w * dot3(tv, mud);
                }
                if (!fbc.no_flow) r.q[f] -= w * fbc.pressure;
            }
        if (fbc.no_flow) r.q[f] = q_values[f];
    }
    for (const Triplet& tr : ops.mq_bc) r.q[tr.row] -= tr.value * q_values[tr.col];
    for (const Triplet& tr : ops.b_bc) r.p[tr.col] -= tr.value * q_values[tr.row];
    for (int i = 0; i < ops.n_u; ++i) r.u[i] += ops.rhs_ref_u[i];
    return r;
}

// assemble_rhs3 with sampled data: the 3D analogue of assembly.hpp:467-563 in full (volume
// sources and space- / time-dependent boundary data), the fields given at the quadrature points
// (6 x 6 x 6 Gauss per cell, xi outermost; 6 x 6 per boundary face in ascending face index, first
// tangential axis outer). null = absent field (the volume loop is skipped as in the reference).
struct RhsSamples3 {
    const double* momentum = nullptr;   // [cell][216][3]
    const double* darcy = nullptr;      // [cell][216][3]
    const double* mass = nullptr;       // [cell][216]
    const double* traction = nullptr;   // [bface][36][3]
    const double* dirichlet = nullptr;  // [bface][36][3]
    const double* flow = nullptr;       // [bface][36]  prescribed pressure, or normal flux on no-flow-kind faces
};
inline FieldVecs assemble_rhs3_sampled(const Mesh3& mesh, const MaterialParameters& mat, const SpatialOperators& ops,
                                       const BoundarySpec3& bc, const RhsSamples3& sm) {
    FieldVecs r;
    r.u.assign(ops.n_u, 0.0);
    r.q.assign(ops.n_q, 0.0);
    r.p.assign(ops.n_p, 0.0);
    const QuadratureRule gq = gauss_legendre(kDataQuadOrder);
    if (sm.momentum || sm.darcy || sm.mass) {
        for (int c = 0; c < mesh.n_cells(); ++c) {
            const Cell3& cell = mesh.cells[c];
            const double vol = cell.volume();
            const auto cf = mesh.cell_faces(c);
            std::array<double, 6> sgn{};
            for (int k = 0; k < 6; ++k) {
                const Face3& f = mesh.faces[cf[k]];
                sgn[k] = f.n[f.axis];
            }
            for (size_t i = 0; i < 6; ++i)
                for (size_t j = 0; j < 6; ++j)
                    for (size_t k = 0; k < 6; ++k) {
                        const double ref[3] = {gq.points[i], gq.points[j], gq.points[k]};
                        const double w = gq.weights[i] * gq.weights[j] * gq.weights[k] * vol;
                        const size_t sp = static_cast<size_t>(c) * 216 + (i * 6 + j) * 6 + k;
                        if (sm.momentum)
                            for (int a = 0; a < 8; ++a) {
                                const double nv = shapes3::n(a, ref[0], ref[1], ref[2]);
                                for (int comp = 0; comp < 3; ++comp)
                                    r.u[24 * c + 3 * a + comp] += w * nv * sm.momentum[3 * sp + comp];
                            }
                        if (sm.darcy)
                            for (int axis = 0; axis < 3; ++axis) {
                                const int flo = cf[2 * axis], fhi = cf[2 * axis + 1];
                                const double wl = sgn[2 * axis] * (1.0 - ref[axis]), wh = sgn[2 * axis + 1] * ref[axis];
                                if (!ops.q_constrained[flo]) r.q[flo] += w * wl * sm.darcy[3 * sp + axis];
                                if (!ops.q_constrained[fhi]) r.q[fhi] += w * wh * sm.darcy[3 * sp + axis];
                            }
                        if (sm.mass) r.p[c] -= w * sm.mass[sp];
                    }
        }
    }
    Vec q_values(ops.n_q, 0.0);
    size_t bf = 0;
    for (int f = 0; f < mesh.n_faces(); ++f) {
        const Face3& face = mesh.faces[f];
        if (!face.is_boundary()) continue;
        const int c = face.cell_minus;
        const Cell3& cell = mesh.cells[c];
        const DisplacementBC3& dbc = bc.displacement[face.tag - 1];
        const FlowBC3& fbc = bc.flow[face.tag - 1];
        const double gamma_f = sipg_face_coefficient3(mesh, mat, ops.penalty, f);
        for (size_t qa = 0; qa < 6; ++qa)
            for (size_t qb = 0; qb < 6; ++qb) {
                const double w = gq.weights[qa] * gq.weights[qb] * face.measure;
                const auto rp = face_ref_point3(mesh, f, c, gq.points[qa], gq.points[qb]);
                const size_t sp = bf * 36 + qa * 6 + qb;
                const std::array<double, 3> tn = {sm.traction[3 * sp], sm.traction[3 * sp + 1], sm.traction[3 * sp + 2]};
                const std::array<double, 3> mud = {dbc.dirichlet[0] ? sm.dirichlet[3 * sp] : 0.0,
                                                   dbc.dirichlet[1] ? sm.dirichlet[3 * sp + 1] : 0.0,
                                                   dbc.dirichlet[2] ? sm.dirichlet[3 * sp + 2] : 0.0};
                for (int l = 0; l < 24; ++l) {
                    const int a = l / 3, comp = l % 3;
                    const double nv = shapes3::n(a, rp[0], rp[1], rp[2]);
                    const int gi = 24 * c + l;
                    if (!dbc.dirichlet[comp]) r.u[gi] += w * nv * tn[comp];
                    if (dbc.dirichlet[comp]) r.u[gi] += w * gamma_f * nv * mud[comp];
                    const auto tv = shapes3::traction(cell, mat, a, comp, rp[0], rp[1], rp[2], face.n);
                    r.u[gi] -= w * dot3(tv, mud);
                }
                if (!fbc.no_flow)
                    r.q[f] -= w * sm.flow[sp];
                else
                    q_values[f] += w / face.measure * sm.flow[sp];
            }
        if (fbc.no_flow) r.q[f] = q_values[f];
        ++bf;
    }
    for (const Triplet& tr : ops.mq_bc) r.q[tr.row] -= tr.value * q_values[tr.col];
    for (const Triplet& tr : ops.b_bc) r.p[tr.col] -= tr.value * q_values[tr.row];
    for (int i = 0; i < ops.n_u; ++i) r.u[i] += ops.rhs_ref_u[i];
    return r;
}

// the sample points of assemble_rhs3_sampled
inline void rhs3_sample_points(const Mesh3& mesh, double* cell_xyz, int* bface_ids, double* bface_xyz) {
    const QuadratureRule gq = gauss_legendre(kDataQuadOrder);
    if (cell_xyz)
        for (int c = 0; c < mesh.n_cells(); ++c) {
            const Cell3& cell = mesh.cells[c];
            for (size_t i = 0; i < 6; ++i)
                for (size_t j = 0; j < 6; ++j)
                    for (size_t k = 0; k < 6; ++k) {
                        double* o = cell_xyz + (static_cast<size_t>(c) * 216 + (i * 6 + j) * 6 + k) * 3;
                        o[0] = cell.x0 + gq.points[i] * cell.hx;
                        o[1] = cell.y0 + gq.points[j] * cell.hy;
                        o[2] = cell.z0 + gq.points[k] * cell.hz;
                    }
        }
    size_t bf = 0;
    for (int f = 0; f < mesh.n_faces(); ++f) {
        const Face3& face = mesh.faces[f];
        if (!face.is_boundary()) continue;
        if (bface_ids) bface_ids[bf] = f;
        if (bface_xyz) {
            const Cell3& cell = mesh.cells[face.cell_minus];
            for (size_t qa = 0; qa < 6; ++qa)
                for (size_t qb = 0; qb < 6; ++qb) {
                    const auto rp = face_ref_point3(mesh, f, face.cell_minus, gq.points[qa], gq.points[qb]);
                    double* o = bface_xyz + (bf * 36 + qa * 6 + qb) * 3;
                    o[0] = cell.x0 + rp[0] * cell.hx;
                    o[1] = cell.y0 + rp[1] * cell.hy;
                    o[2] = cell.z0 + rp[2] * cell.hz;
                }
        }
        ++bf;
    }
}

}  // namespace refcpu
