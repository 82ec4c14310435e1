// ORACLE / TEST INFRASTRUCTURE ONLY. Not part of the product.
//
// CPU restatement (Eigen-free, C++17) of the porodg reference's spatial
// discretisation: quadrature, mesh, dof maps, boundary/material data and the
// operator / right-hand-side assembly. Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline leg may load this code, and only as a checker.
//
// Every function cites the reference file:line it follows
// (paths relative to /root/reference/proj/include/porodg/).
// Floating-point expressions are written in the same association order as
// the reference so that, compiled with -ffp-contract=off (the reference's
// Release build has no -march and therefore no FMA, proj/CMakeLists.txt:7-9),
// the assembled matrices are bit-identical to the reference's.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <functional>
#include <limits>
#include <numeric>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace refcpu {

using Vec = std::vector<double>;

class SolverError : public std::runtime_error {  // errors.hpp:10-13
public:
    using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------------------
// quadrature.hpp:9-59
// ---------------------------------------------------------------------------
struct QuadratureRule {
    std::vector<double> points, weights;
};

inline std::pair<double, double> legendre(int n, double x) {  // quadrature.hpp:17-28
    if (n == 0) return {1.0, 0.0};
    double pm = 1.0, p = x;
    for (int k = 2; k <= n; ++k) {
        const double pn = ((2.0 * k - 1.0) * x * p - (k - 1.0) * pm) / k;
        pm = p;
        p = pn;
    }
    const double dp = n * (x * p - pm) / (x * x - 1.0);
    return {p, dp};
}

inline QuadratureRule gauss_legendre(int n) {  // quadrature.hpp:33-54
    if (n < 1) throw std::invalid_argument("gauss_legendre: n must be >= 1");
    QuadratureRule q;
    q.points.resize(n);
    q.weights.resize(n);
    for (int i = 0; i < n; ++i) {
        double x = std::cos(M_PI * (i + 0.75) / (n + 0.5));
        for (int it = 0; it < 100; ++it) {
            const auto pd = legendre(n, x);
            const double dx = pd.first / pd.second;
            x -= dx;
            if (std::abs(dx) < 1e-15) break;
        }
        const auto pd = legendre(n, x);
        const double w = 2.0 / ((1.0 - x * x) * pd.second * pd.second);
        q.points[n - 1 - i] = 0.5 * (x + 1.0);
        q.weights[n - 1 - i] = 0.5 * w;
    }
    return q;
}

constexpr int kDataQuadOrder = 6;  // quadrature.hpp:59

// ---------------------------------------------------------------------------
// mesh.hpp:11-180
// ---------------------------------------------------------------------------
enum class FaceTag { interior = 0, left = 1, right = 2, bottom = 3, top = 4 };
enum class FaceOrientation { horizontal, vertical };

struct Cell {
    double x0, y0, hx, hy;
    double area() const { return hx * hy; }
};

struct Face {
    FaceOrientation orientation;
    int cell_minus, cell_plus;
    double nx, ny, measure;
    FaceTag tag;
    double x0, y0, x1, y1;
    bool is_boundary() const { return cell_plus < 0; }
};

struct Mesh {
    int nx = 0, ny = 0;
    double lx = 0, ly = 0;
    std::vector<Cell> cells;
    std::vector<Face> faces;
    int n_cells() const { return nx * ny; }
    int n_faces() const { return static_cast<int>(faces.size()); }
    int cell_index(int i, int j) const { return j * nx + i; }
    int horizontal_face_index(int i, int j) const { return j * nx + i; }
    int vertical_face_index(int i, int j) const { return nx * (ny + 1) + i * ny + j; }
    std::array<int, 4> cell_faces(int c) const {  // mesh.hpp:63-67, order W,E,S,N
        const int i = c % nx, j = c / nx;
        return {vertical_face_index(i, j), vertical_face_index(i + 1, j), horizontal_face_index(i, j),
                horizontal_face_index(i, j + 1)};
    }
};

inline Mesh build_mesh(int nx, int ny, double lx, double ly) {  // mesh.hpp:73-155
    if (nx < 1 || ny < 1) throw std::invalid_argument("build_mesh: cell counts must be positive");
    if (!(lx > 0.0) || !(ly > 0.0)) throw std::invalid_argument("build_mesh: edge lengths must be positive");
    Mesh m;
    m.nx = nx;
    m.ny = ny;
    m.lx = lx;
    m.ly = ly;
    const double hx = lx / nx, hy = ly / ny;
    m.cells.reserve(static_cast<size_t>(nx) * ny);
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) m.cells.push_back({i * hx, j * hy, hx, hy});
    for (int j = 0; j <= ny; ++j)
        for (int i = 0; i < nx; ++i) {
            Face f;
            f.orientation = FaceOrientation::horizontal;
            f.measure = hx;
            f.x0 = i * hx;
            f.x1 = (i + 1) * hx;
            f.y0 = f.y1 = j * hy;
            if (j == 0) {
                f.cell_minus = m.cell_index(i, 0);
                f.cell_plus = -1;
                f.nx = 0.0;
                f.ny = -1.0;
                f.tag = FaceTag::bottom;
            } else if (j == ny) {
                f.cell_minus = m.cell_index(i, ny - 1);
                f.cell_plus = -1;
                f.nx = 0.0;
                f.ny = 1.0;
                f.tag = FaceTag::top;
            } else {
                f.cell_minus = m.cell_index(i, j - 1);
                f.cell_plus = m.cell_index(i, j);
                f.nx = 0.0;
                f.ny = 1.0;
                f.tag = FaceTag::interior;
            }
            m.faces.push_back(f);
        }
    for (int i = 0; i <= nx; ++i)
        for (int j = 0; j < ny; ++j) {
            Face f;
            f.orientation = FaceOrientation::vertical;
            f.measure = hy;
            f.x0 = f.x1 = i * hx;
            f.y0 = j * hy;
            f.y1 = (j + 1) * hy;
            if (i == 0) {
                f.cell_minus = m.cell_index(0, j);
                f.cell_plus = -1;
                f.nx = -1.0;
                f.ny = 0.0;
                f.tag = FaceTag::left;
            } else if (i == nx) {
                f.cell_minus = m.cell_index(nx - 1, j);
                f.cell_plus = -1;
                f.nx = 1.0;
                f.ny = 0.0;
                f.tag = FaceTag::right;
            } else {
                f.cell_minus = m.cell_index(i - 1, j);
                f.cell_plus = m.cell_index(i, j);
                f.nx = 1.0;
                f.ny = 0.0;
                f.tag = FaceTag::interior;
            }
            m.faces.push_back(f);
        }
    return m;
}

inline double face_outward_sign(const Mesh& mesh, int f, int c) {  // mesh.hpp:176-180
    const Face& face = mesh.faces[f];
    if (face.cell_plus < 0) return 1.0;
    return c == face.cell_minus ? 1.0 : -1.0;
}

// dofs.hpp:28-46 : u dof = 8c + 2a + comp, q dof = face, p dof = cell.
struct DofMaps {
    int n_u = 0, n_q = 0, n_p = 0;
    int u_dof(int c, int a, int comp) const { return 8 * c + 2 * a + comp; }
};
inline DofMaps build_dof_maps(const Mesh& m) {
    DofMaps d;
    d.n_u = 8 * m.n_cells();
    d.n_q = m.n_faces();
    d.n_p = m.n_cells();
    return d;
}

// ---------------------------------------------------------------------------
// boundary.hpp:14-105, material.hpp:21-70
// ---------------------------------------------------------------------------
using ScalarFieldT = std::function<double(double, double, double)>;
using VectorFieldT = std::function<std::array<double, 2>(double, double, double)>;
using ScalarField = std::function<double(double, double)>;
using VectorField = std::function<std::array<double, 2>(double, double)>;

inline double eval_or_zero(const ScalarFieldT& f, double x, double y, double t) { return f ? f(x, y, t) : 0.0; }
inline std::array<double, 2> eval_or_zero(const VectorFieldT& f, double x, double y, double t) {
    return f ? f(x, y, t) : std::array<double, 2>{0.0, 0.0};
}

struct DisplacementBC {  // boundary.hpp:27-56
    std::array<bool, 2> dirichlet = {false, false};
    VectorFieldT dirichlet_data;
    VectorFieldT traction_data;
    static DisplacementBC fixed(VectorFieldT d = {}) {
        DisplacementBC b;
        b.dirichlet = {true, true};
        b.dirichlet_data = std::move(d);
        return b;
    }
    static DisplacementBC traction(VectorFieldT d = {}) {
        DisplacementBC b;
        b.traction_data = std::move(d);
        return b;
    }
    static DisplacementBC roller_x(VectorFieldT t = {}) {
        DisplacementBC b;
        b.dirichlet = {true, false};
        b.traction_data = std::move(t);
        return b;
    }
    static DisplacementBC roller_y(VectorFieldT t = {}) {
        DisplacementBC b;
        b.dirichlet = {false, true};
        b.traction_data = std::move(t);
        return b;
    }
};

struct FlowBC {  // boundary.hpp:61-69
    enum class Kind { pressure, normal_flux };
    Kind kind = Kind::pressure;
    ScalarFieldT data;
    static FlowBC pressure(ScalarFieldT d = {}) { return {Kind::pressure, std::move(d)}; }
    static FlowBC no_flow() { return {Kind::normal_flux, {}}; }
};

struct BoundarySpec {  // boundary.hpp:71-105
    std::array<std::optional<DisplacementBC>, 4> displacement;
    std::array<std::optional<FlowBC>, 4> flow;
    static int slot(FaceTag t) {
        if (t == FaceTag::interior) throw std::invalid_argument("boundary spec: interior tag");
        return static_cast<int>(t) - 1;
    }
    void set_displacement(FaceTag t, DisplacementBC b) { displacement[slot(t)] = std::move(b); }
    void set_flow(FaceTag t, FlowBC b) { flow[slot(t)] = std::move(b); }
    const DisplacementBC& displacement_on(FaceTag t) const { return *displacement[slot(t)]; }
    const FlowBC& flow_on(FaceTag t) const { return *flow[slot(t)]; }
    void validate() const {
        static const char* names[4] = {"left", "right", "bottom", "top"};
        for (int s = 0; s < 4; ++s) {
            if (!displacement[s])
                throw std::invalid_argument(std::string("boundary spec: no displacement condition on ") + names[s]);
            if (!flow[s]) throw std::invalid_argument(std::string("boundary spec: no flow condition on ") + names[s]);
        }
    }
    static BoundarySpec all_fixed_pressure(ScalarFieldT p = {}) {
        BoundarySpec b;
        for (FaceTag t : {FaceTag::left, FaceTag::right, FaceTag::bottom, FaceTag::top}) {
            b.set_displacement(t, DisplacementBC::fixed());
            b.set_flow(t, FlowBC::pressure(p));
        }
        return b;
    }
};

struct MaterialParameters {  // material.hpp:25-70
    double lambda_lame = 1.0, mu_lame = 1.0, k_perm = 1.0;
    std::vector<double> k_perm_cells;
    double eta = 1.0, biot_b = 0.8, biot_m = 10.0, k_dr = 2.0;
    double k_s = std::numeric_limits<double>::infinity();
    double permeability(int c) const { return k_perm_cells.empty() ? k_perm : k_perm_cells[c]; }
    void validate() const {
        if (!(mu_lame > 0.0)) throw std::invalid_argument("material: mu must be positive");
        if (!(eta > 0.0)) throw std::invalid_argument("material: eta must be positive");
        if (!(biot_m > 0.0)) throw std::invalid_argument("material: Biot modulus M must be positive");
        if (!(biot_b > 0.0) || biot_b > 1.0)
            throw std::invalid_argument("material: Biot coefficient b must lie in (0, 1]");
        if (!(k_perm > 0.0)) throw std::invalid_argument("material: permeability must be positive");
        for (double k : k_perm_cells)
            if (!(k > 0.0)) throw std::invalid_argument("material: per-cell permeability must be positive");
        const double kdr_expect = lambda_lame + 2.0 * mu_lame / 2;
        if (std::abs(k_dr - kdr_expect) > 1e-12 * std::max(1.0, std::abs(kdr_expect)))
            throw std::invalid_argument("material: k_dr inconsistent with lambda + 2 mu / d");
    }
};

// problems.hpp:28-50 (material_from_config), b given directly.
inline MaterialParameters material_from_lame(double lambda, double mu, double k_perm, double eta, double biot_m,
                                             double biot_b) {
    MaterialParameters m;
    m.lambda_lame = lambda;
    m.mu_lame = mu;
    m.k_perm = k_perm;
    m.eta = eta;
    m.biot_m = biot_m;
    m.k_dr = lambda + 2.0 * mu / 2;
    m.biot_b = biot_b;
    m.validate();
    return m;
}

// ---------------------------------------------------------------------------
// sparse.hpp:12-110
// ---------------------------------------------------------------------------
struct Triplet {
    int row, col;
    double value;
};

struct SparseMatrix {
    int rows = 0, cols = 0;
    std::vector<int> row_offsets, col_indices;
    std::vector<double> values;
    int nnz() const { return static_cast<int>(values.size()); }

    // sparse.hpp:30-40 : s starts at 0.0, sequential in stored order.
    void apply(const double* x, double* y) const {
        for (int i = 0; i < rows; ++i) {
            double s = 0.0;
            for (int k = row_offsets[i]; k < row_offsets[i + 1]; ++k) s += values[k] * x[col_indices[k]];
            y[i] = s;
        }
    }
    Vec apply(const Vec& x) const {
        if (static_cast<int>(x.size()) != cols) throw std::invalid_argument("spmv: dimension mismatch");
        Vec y(rows);
        apply(x.data(), y.data());
        return y;
    }
    // sparse.hpp:43-50 : scatter in ascending source row.
    Vec apply_transpose(const Vec& x) const {
        if (static_cast<int>(x.size()) != rows) throw std::invalid_argument("spmv_transpose: dimension mismatch");
        Vec y(cols, 0.0);
        for (int i = 0; i < rows; ++i)
            for (int k = row_offsets[i]; k < row_offsets[i + 1]; ++k) y[col_indices[k]] += values[k] * x[i];
        return y;
    }
    double coeff(int i, int j) const {
        for (int k = row_offsets[i]; k < row_offsets[i + 1]; ++k)
            if (col_indices[k] == j) return values[k];
        return 0.0;
    }
    bool well_formed() const {  // sparse.hpp:67-78
        if (static_cast<int>(row_offsets.size()) != rows + 1) return false;
        if (row_offsets.front() != 0 || row_offsets.back() != nnz()) return false;
        for (int i = 0; i < rows; ++i) {
            if (row_offsets[i] > row_offsets[i + 1]) return false;
            for (int k = row_offsets[i] + 1; k < row_offsets[i + 1]; ++k)
                if (col_indices[k - 1] >= col_indices[k]) return false;
        }
        for (int c : col_indices)
            if (c < 0 || c >= cols) return false;
        return true;
    }
    int bandwidth() const {
        int bw = 0;
        for (int i = 0; i < rows; ++i)
            for (int k = row_offsets[i]; k < row_offsets[i + 1]; ++k) bw = std::max(bw, std::abs(i - col_indices[k]));
        return bw;
    }
};

// sparse.hpp:83-110 : stable sort by (row, col), duplicates summed in push
// order starting from 0.0. Implemented as a stable counting sort by row
// followed by a stable per-row sort by column (same result as one
// std::stable_sort on the (row, col) key, without its O(n) extra copy).
inline SparseMatrix csr_from_triplets(int rows, int cols, const std::vector<Triplet>& trips) {
    for (const Triplet& t : trips)
        if (t.row < 0 || t.row >= rows || t.col < 0 || t.col >= cols)
            throw std::invalid_argument("csr_from_triplets: index out of range");
    std::vector<int64_t> start(static_cast<size_t>(rows) + 1, 0);
    for (const Triplet& t : trips) start[t.row + 1]++;
    for (int i = 0; i < rows; ++i) start[i + 1] += start[i];
    std::vector<int64_t> fill(start.begin(), start.end() - 1);
    std::vector<std::pair<int, double>> buf(trips.size());
    for (const Triplet& t : trips) buf[fill[t.row]++] = {t.col, t.value};
    SparseMatrix m;
    m.rows = rows;
    m.cols = cols;
    m.row_offsets.assign(rows + 1, 0);
    m.col_indices.reserve(trips.size());
    m.values.reserve(trips.size());
    for (int r = 0; r < rows; ++r) {
        auto b = buf.begin() + start[r], e = buf.begin() + start[r + 1];
        std::stable_sort(b, e, [](const std::pair<int, double>& a, const std::pair<int, double>& c) {
            return a.first < c.first;
        });
        for (auto it = b; it != e;) {
            const int c = it->first;
            double s = 0.0;
            while (it != e && it->first == c) s += (it++)->second;
            m.col_indices.push_back(c);
            m.values.push_back(s);
            m.row_offsets[r + 1] += 1;
        }
    }
    for (int r = 0; r < rows; ++r) m.row_offsets[r + 1] += m.row_offsets[r];
    return m;
}

// ---------------------------------------------------------------------------
// assembly.hpp:54-118 (shape functions)
// ---------------------------------------------------------------------------
namespace shapes {
inline double n(int a, double xi, double eta) {
    switch (a) {
        case 0: return (1.0 - xi) * (1.0 - eta);
        case 1: return xi * (1.0 - eta);
        case 2: return (1.0 - xi) * eta;
        default: return xi * eta;
    }
}
inline double dn_dxi(int a, double eta) {
    switch (a) {
        case 0: return -(1.0 - eta);
        case 1: return 1.0 - eta;
        case 2: return -eta;
        default: return eta;
    }
}
inline double dn_deta(int a, double xi) {
    switch (a) {
        case 0: return -(1.0 - xi);
        case 1: return -xi;
        case 2: return 1.0 - xi;
        default: return xi;
    }
}
inline std::array<double, 2> grad(const Cell& c, int a, double xi, double eta) {
    return {dn_dxi(a, eta) / c.hx, dn_deta(a, xi) / c.hy};
}
inline std::array<double, 3> strain(const Cell& c, int a, int comp, double xi, double eta) {
    const auto g = grad(c, a, xi, eta);
    if (comp == 0) return {g[0], 0.0, 0.5 * g[1]};
    return {0.0, g[1], 0.5 * g[0]};
}
inline std::array<double, 2> traction(const Cell& c, const MaterialParameters& m, int a, int comp, double xi,
                                      double eta, double nx, double ny) {
    const auto g = grad(c, a, xi, eta);
    const double lam = m.lambda_lame, mu = m.mu_lame;
    double sxx, syy, sxy;
    if (comp == 0) {
        sxx = (2.0 * mu + lam) * g[0];
        syy = lam * g[0];
        sxy = mu * g[1];
    } else {
        sxx = lam * g[1];
        syy = (2.0 * mu + lam) * g[1];
        sxy = mu * g[0];
    }
    return {sxx * nx + sxy * ny, sxy * nx + syy * ny};
}
}  // namespace shapes

struct FaceTrace {  // assembly.hpp:124-145
    std::array<int, 2> nodes;
    bool vertical;
    double fixed_ref;
};
inline FaceTrace face_trace(const Mesh& mesh, int face, int cell) {
    const Face& f = mesh.faces[face];
    const Cell& c = mesh.cells[cell];
    FaceTrace t;
    t.vertical = f.orientation == FaceOrientation::vertical;
    if (t.vertical) {
        const bool left = std::abs(f.x0 - c.x0) < 1e-12 * (c.hx + 1.0);
        t.fixed_ref = left ? 0.0 : 1.0;
        t.nodes = left ? std::array<int, 2>{0, 2} : std::array<int, 2>{1, 3};
    } else {
        const bool bottom = std::abs(f.y0 - c.y0) < 1e-12 * (c.hy + 1.0);
        t.fixed_ref = bottom ? 0.0 : 1.0;
        t.nodes = bottom ? std::array<int, 2>{0, 1} : std::array<int, 2>{2, 3};
    }
    return t;
}
inline std::array<double, 2> face_ref_point(const FaceTrace& t, double s) {
    return t.vertical ? std::array<double, 2>{t.fixed_ref, s} : std::array<double, 2>{s, t.fixed_ref};
}

inline double sipg_face_coefficient(const Mesh& mesh, const MaterialParameters& mat, double gamma,
                                    int face) {  // assembly.hpp:160-172
    const Face& f = mesh.faces[face];
    double h = 0.0;
    int cnt = 0;
    for (int c : {f.cell_minus, f.cell_plus}) {
        if (c < 0) continue;
        h += f.orientation == FaceOrientation::vertical ? mesh.cells[c].hx : mesh.cells[c].hy;
        ++cnt;
    }
    h /= cnt;
    return gamma * (mat.lambda_lame + 2.0 * mat.mu_lame) / h;
}

// assembly.hpp:38-52
struct SpatialOperators {
    SparseMatrix A, M_q, B, E, M_p;
    Vec m_p_diag;
    double penalty = 0.0;
    MaterialParameters mat;
    BoundarySpec bc;
    std::vector<char> q_constrained;
    std::vector<Triplet> mq_bc, b_bc;
    Vec rhs_ref_u;  // A u0 - b E p0 - E sigma_v0 : zero (no reference-state fields in scope)
    // oracle-only: banded ordering of the faces for the sparse-direct flow backend when the
    // mesh is not the 2D structured one (fem3d.hpp); empty = the 2D face-row order
    std::vector<int> face_band_perm;
    int n_u = 0, n_q = 0, n_p = 0;
    int n_total() const { return n_u + n_q + n_p; }
};

// assembly.hpp:177-395. Reference-state fields (u0, p0, sigma0_v) are not in
// the hot-path scope and are taken as zero, so rhs_ref_u = 0.
inline SpatialOperators assemble_operators(const Mesh& mesh, const DofMaps& dofs, const MaterialParameters& mat,
                                           double penalty_gamma, const BoundarySpec& bc) {
    if (!(penalty_gamma > 0.0)) throw std::invalid_argument("assemble_operators: penalty must be positive");
    bc.validate();
    mat.validate();
    SpatialOperators ops;
    ops.penalty = penalty_gamma;
    ops.mat = mat;
    ops.bc = bc;
    ops.n_u = dofs.n_u;
    ops.n_q = dofs.n_q;
    ops.n_p = dofs.n_p;
    const QuadratureRule g2 = gauss_legendre(2);

    ops.q_constrained.assign(dofs.n_q, 0);
    for (int f = 0; f < mesh.n_faces(); ++f) {
        const Face& face = mesh.faces[f];
        if (face.is_boundary() && bc.flow_on(face.tag).kind == FlowBC::Kind::normal_flux) ops.q_constrained[f] = 1;
    }

    std::vector<Triplet> ta, tmq, tb, te, tmp;
    const size_t nc = static_cast<size_t>(mesh.n_cells());
    ta.reserve(nc * 64 + static_cast<size_t>(mesh.n_faces()) * 2 * 256);
    te.reserve(nc * 8 + static_cast<size_t>(mesh.n_faces()) * 64);

    // ---- cell contributions (assembly.hpp:204-277)
    for (int c = 0; c < mesh.n_cells(); ++c) {
        const Cell& cell = mesh.cells[c];
        const double area = cell.area();
        const double lam = mat.lambda_lame, mu = mat.mu_lame;
        double ke[8][8] = {};
        double div_int[8] = {};
        for (size_t qi = 0; qi < g2.points.size(); ++qi)
            for (size_t qj = 0; qj < g2.points.size(); ++qj) {
                const double xi = g2.points[qi], eta = g2.points[qj];
                const double w = g2.weights[qi] * g2.weights[qj] * area;
                std::array<std::array<double, 3>, 8> eps;
                for (int l = 0; l < 8; ++l) eps[l] = shapes::strain(cell, l / 2, l % 2, xi, eta);
                for (int l1 = 0; l1 < 8; ++l1) {
                    for (int l2 = 0; l2 <= l1; ++l2) {
                        const auto &e1 = eps[l1], &e2 = eps[l2];
                        const double v = 2.0 * mu * (e1[0] * e2[0] + e1[1] * e2[1] + 2.0 * e1[2] * e2[2]) +
                                         lam * (e1[0] + e1[1]) * (e2[0] + e2[1]);
                        ke[l1][l2] += w * v;
                        if (l2 != l1) ke[l2][l1] += w * v;
                    }
                    div_int[l1] += w * (eps[l1][0] + eps[l1][1]);
                }
            }
        for (int l1 = 0; l1 < 8; ++l1) {
            for (int l2 = 0; l2 < 8; ++l2) ta.push_back({8 * c + l1, 8 * c + l2, ke[l1][l2]});
            te.push_back({8 * c + l1, c, div_int[l1]});
        }

        const auto cf = mesh.cell_faces(c);
        const double keff = mat.eta / mat.permeability(c);
        std::array<double, 4> sgn{};
        for (int k = 0; k < 4; ++k) {
            const Face& f = mesh.faces[cf[k]];
            sgn[k] = f.orientation == FaceOrientation::vertical ? f.nx : f.ny;
        }
        const double d3 = keff * area / 3.0, d6 = keff * area / 6.0;
        for (int pair = 0; pair < 2; ++pair) {
            const int f0 = cf[2 * pair], f1 = cf[2 * pair + 1];
            const double cross = d6 * sgn[2 * pair] * sgn[2 * pair + 1];
            auto push_mq = [&](int r, int cc, double v) {
                const bool rc = ops.q_constrained[r], cc_c = ops.q_constrained[cc];
                if (rc && r == cc) return;
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
        for (int k = 0; k < 4; ++k) {
            const int f = cf[k];
            const double sout = face_outward_sign(mesh, f, c);
            const double v = -sout * mesh.faces[f].measure;
            if (ops.q_constrained[f])
                ops.b_bc.push_back({f, c, v});
            else
                tb.push_back({f, c, v});
        }
        tmp.push_back({c, c, area});
    }
    for (int f = 0; f < dofs.n_q; ++f)
        if (ops.q_constrained[f]) tmq.push_back({f, f, 1.0});

    // ---- face contributions (assembly.hpp:281-376)
    for (int f = 0; f < mesh.n_faces(); ++f) {
        const Face& face = mesh.faces[f];
        const double gamma_f = sipg_face_coefficient(mesh, mat, penalty_gamma, f);
        const std::array<double, 2> nrm = {face.nx, face.ny};
        if (!face.is_boundary()) {
            const std::array<int, 2> cells = {face.cell_minus, face.cell_plus};
            const std::array<double, 2> side_sign = {1.0, -1.0};
            const std::array<FaceTrace, 2> trs = {face_trace(mesh, f, cells[0]), face_trace(mesh, f, cells[1])};
            for (size_t qk = 0; qk < g2.points.size(); ++qk) {
                const double s = g2.points[qk];
                const double w = g2.weights[qk] * face.measure;
                std::array<std::array<std::array<double, 2>, 8>, 2> val{}, trac{};
                for (int side = 0; side < 2; ++side) {
                    const Cell& cell = mesh.cells[cells[side]];
                    const auto rp = face_ref_point(trs[side], s);
                    for (int l = 0; l < 8; ++l) {
                        const int a = l / 2, comp = l % 2;
                        const double nv = shapes::n(a, rp[0], rp[1]);
                        val[side][l] = {comp == 0 ? nv : 0.0, comp == 1 ? nv : 0.0};
                        trac[side][l] = shapes::traction(cell, mat, a, comp, rp[0], rp[1], nrm[0], nrm[1]);
                    }
                }
                for (int s1 = 0; s1 < 2; ++s1)
                    for (int l1 = 0; l1 < 8; ++l1) {
                        const int gi = 8 * cells[s1] + l1;
                        for (int s2 = 0; s2 < 2; ++s2)
                            for (int l2 = 0; l2 < 8; ++l2) {
                                const int gj = 8 * cells[s2] + l2;
                                const double cons =
                                    -0.5 * (trac[s2][l2][0] * val[s1][l1][0] + trac[s2][l2][1] * val[s1][l1][1]) *
                                    side_sign[s1];
                                const double symm =
                                    -0.5 * (trac[s1][l1][0] * val[s2][l2][0] + trac[s1][l1][1] * val[s2][l2][1]) *
                                    side_sign[s2];
                                const double pen = gamma_f * side_sign[s1] * side_sign[s2] *
                                                   (val[s1][l1][0] * val[s2][l2][0] + val[s1][l1][1] * val[s2][l2][1]);
                                ta.push_back({gi, gj, w * (cons + symm + pen)});
                            }
                        const double nv = nrm[0] * val[s1][l1][0] + nrm[1] * val[s1][l1][1];
                        for (int pc = 0; pc < 2; ++pc) te.push_back({gi, cells[pc], -0.5 * w * side_sign[s1] * nv});
                    }
            }
        } else {
            const int c = face.cell_minus;
            const Cell& cell = mesh.cells[c];
            const DisplacementBC& dbc = bc.displacement_on(face.tag);
            if (!dbc.dirichlet[0] && !dbc.dirichlet[1]) continue;
            const FaceTrace tr = face_trace(mesh, f, c);
            const int ncmp = face.orientation == FaceOrientation::vertical ? 0 : 1;
            for (size_t qk = 0; qk < g2.points.size(); ++qk) {
                const double s = g2.points[qk];
                const double w = g2.weights[qk] * face.measure;
                const auto rp = face_ref_point(tr, s);
                std::array<std::array<double, 2>, 8> val{}, trac{};
                for (int l = 0; l < 8; ++l) {
                    const int a = l / 2, comp = l % 2;
                    const double nv = shapes::n(a, rp[0], rp[1]);
                    val[l] = {comp == 0 ? nv : 0.0, comp == 1 ? nv : 0.0};
                    trac[l] = shapes::traction(cell, mat, a, comp, rp[0], rp[1], nrm[0], nrm[1]);
                }
                auto mask = [&](const std::array<double, 2>& v) {
                    return std::array<double, 2>{dbc.dirichlet[0] ? v[0] : 0.0, dbc.dirichlet[1] ? v[1] : 0.0};
                };
                for (int l1 = 0; l1 < 8; ++l1) {
                    const int gi = 8 * c + l1;
                    const auto mv1 = mask(val[l1]);
                    for (int l2 = 0; l2 < 8; ++l2) {
                        const int gj = 8 * c + l2;
                        const auto mv2 = mask(val[l2]);
                        const double cons = -(trac[l2][0] * mv1[0] + trac[l2][1] * mv1[1]);
                        const double symm = -(trac[l1][0] * mv2[0] + trac[l1][1] * mv2[1]);
                        const double pen = gamma_f * (mv1[0] * mv2[0] + mv1[1] * mv2[1]);
                        ta.push_back({gi, gj, w * (cons + symm + pen)});
                    }
                    if (dbc.dirichlet[ncmp]) {
                        const double nv = nrm[0] * val[l1][0] + nrm[1] * val[l1][1];
                        te.push_back({gi, c, -w * nv});
                    }
                }
            }
        }
    }

    ops.A = csr_from_triplets(dofs.n_u, dofs.n_u, ta);
    ops.M_q = csr_from_triplets(dofs.n_q, dofs.n_q, tmq);
    ops.B = csr_from_triplets(dofs.n_q, dofs.n_p, tb);
    ops.E = csr_from_triplets(dofs.n_u, dofs.n_p, te);
    ops.M_p = csr_from_triplets(dofs.n_p, dofs.n_p, tmp);
    ops.m_p_diag.resize(dofs.n_p);
    for (int c = 0; c < dofs.n_p; ++c) ops.m_p_diag[c] = mesh.cells[c].area();
    ops.rhs_ref_u.assign(dofs.n_u, 0.0);
    return ops;
}

struct VolumeData {  // assembly.hpp:24-28
    VectorFieldT momentum, darcy;
    ScalarFieldT mass;
};

struct FieldVecs {
    Vec u, q, p;
};

// assembly.hpp:467-563
inline FieldVecs assemble_rhs(const Mesh& mesh, const DofMaps& dofs, const MaterialParameters& mat,
                              const SpatialOperators& ops, const VolumeData& data, double t) {
    FieldVecs r;
    r.u.assign(dofs.n_u, 0.0);
    r.q.assign(dofs.n_q, 0.0);
    r.p.assign(dofs.n_p, 0.0);
    const QuadratureRule gq = gauss_legendre(kDataQuadOrder);
    if (data.momentum || data.darcy || data.mass) {
        for (int c = 0; c < mesh.n_cells(); ++c) {
            const Cell& cell = mesh.cells[c];
            const double area = cell.area();
            const auto cf = mesh.cell_faces(c);
            std::array<double, 4> sgn{};
            for (int k = 0; k < 4; ++k) {
                const Face& f = mesh.faces[cf[k]];
                sgn[k] = f.orientation == FaceOrientation::vertical ? f.nx : f.ny;
            }
            for (size_t i = 0; i < gq.points.size(); ++i)
                for (size_t j = 0; j < gq.points.size(); ++j) {
                    const double xi = gq.points[i], eta = gq.points[j];
                    const double w = gq.weights[i] * gq.weights[j] * area;
                    const double x = cell.x0 + xi * cell.hx, y = cell.y0 + eta * cell.hy;
                    if (data.momentum) {
                        const auto fm = data.momentum(x, y, t);
                        for (int a = 0; a < 4; ++a) {
                            const double nv = shapes::n(a, xi, eta);
                            r.u[dofs.u_dof(c, a, 0)] += w * nv * fm[0];
                            r.u[dofs.u_dof(c, a, 1)] += w * nv * fm[1];
                        }
                    }
                    if (data.darcy) {
                        const auto fd = data.darcy(x, y, t);
                        const std::array<double, 2> wx = {sgn[0] * (1.0 - xi), sgn[1] * xi};
                        const std::array<double, 2> wy = {sgn[2] * (1.0 - eta), sgn[3] * eta};
                        if (!ops.q_constrained[cf[0]]) r.q[cf[0]] += w * wx[0] * fd[0];
                        if (!ops.q_constrained[cf[1]]) r.q[cf[1]] += w * wx[1] * fd[0];
                        if (!ops.q_constrained[cf[2]]) r.q[cf[2]] += w * wy[0] * fd[1];
                        if (!ops.q_constrained[cf[3]]) r.q[cf[3]] += w * wy[1] * fd[1];
                    }
                    if (data.mass) r.p[c] -= w * data.mass(x, y, t);
                }
        }
    }
    Vec q_values(dofs.n_q, 0.0);
    for (int f = 0; f < mesh.n_faces(); ++f) {
        const Face& face = mesh.faces[f];
        if (!face.is_boundary()) continue;
        const int c = face.cell_minus;
        const Cell& cell = mesh.cells[c];
        const FaceTrace tr = face_trace(mesh, f, c);
        const DisplacementBC& dbc = ops.bc.displacement_on(face.tag);
        const FlowBC& fbc = ops.bc.flow_on(face.tag);
        const double gamma_f = sipg_face_coefficient(mesh, mat, ops.penalty, f);
        for (size_t qk = 0; qk < gq.points.size(); ++qk) {
            const double s = gq.points[qk];
            const double w = gq.weights[qk] * face.measure;
            const auto rp = face_ref_point(tr, s);
            const double x = face.x0 + s * (face.x1 - face.x0);
            const double y = face.y0 + s * (face.y1 - face.y0);
            const auto tn = eval_or_zero(dbc.traction_data, x, y, t);
            const auto ud = eval_or_zero(dbc.dirichlet_data, x, y, t);
            const std::array<double, 2> mud = {dbc.dirichlet[0] ? ud[0] : 0.0, dbc.dirichlet[1] ? ud[1] : 0.0};
            for (int l = 0; l < 8; ++l) {
                const int a = l / 2, comp = l % 2;
                const double nv = shapes::n(a, rp[0], rp[1]);
                const int gi = dofs.u_dof(c, a, comp);
                if (!dbc.dirichlet[comp]) r.u[gi] += w * nv * tn[comp];
                if (dbc.dirichlet[comp]) r.u[gi] += w * gamma_f * nv * mud[comp];
                const auto tv = shapes::traction(cell, mat, a, comp, rp[0], rp[1], face.nx, face.ny);
                r.u[gi] -= w * (tv[0] * mud[0] + tv[1] * mud[1]);
            }
            if (fbc.kind == FlowBC::Kind::pressure)
                r.q[f] -= w * eval_or_zero(fbc.data, x, y, t);
            else
                q_values[f] += w / face.measure * eval_or_zero(fbc.data, x, y, t);
        }
        if (fbc.kind == FlowBC::Kind::normal_flux) r.q[f] = q_values[f];
    }
    for (const Triplet& tr : ops.mq_bc) r.q[tr.row] -= tr.value * q_values[tr.col];
    for (const Triplet& tr : ops.b_bc) r.p[tr.col] -= tr.value * q_values[tr.row];
    for (int i = 0; i < dofs.n_u; ++i) r.u[i] += ops.rhs_ref_u[i];
    return r;
}

// assembly.hpp:409-413 : D(u,p) = -b E^T u - (1/M) m_p .* p
inline Vec apply_time_derivative_p(const SpatialOperators& ops, const double* u, const double* p) {
    Vec ut(u, u + ops.n_u);
    Vec et = ops.E.apply_transpose(ut);
    const double mb = -ops.mat.biot_b, im = 1.0 / ops.mat.biot_m;
    Vec d(ops.n_p);
    for (int c = 0; c < ops.n_p; ++c) d[c] = mb * et[c] - im * (ops.m_p_diag[c] * p[c]);
    return d;
}

// project_p / project_u (assembly.hpp:415-460) : initial fields for the
// reference's seeded test problems.
inline Vec project_p(const Mesh& mesh, const DofMaps& dofs, const ScalarField& f) {
    Vec v(dofs.n_p, 0.0);
    if (!f) return v;
    const QuadratureRule gq = gauss_legendre(kDataQuadOrder);
    for (int c = 0; c < mesh.n_cells(); ++c) {
        const Cell& cell = mesh.cells[c];
        double s = 0.0;
        for (size_t i = 0; i < gq.points.size(); ++i)
            for (size_t j = 0; j < gq.points.size(); ++j)
                s += gq.weights[i] * gq.weights[j] * f(cell.x0 + gq.points[i] * cell.hx, cell.y0 + gq.points[j] * cell.hy);
        v[c] = s;
    }
    return v;
}

// 4x4 Q1 mass inverse (assembly.hpp:435-438): closed form of the inverse of
// [[4,2,2,1],[2,4,1,2],[2,1,4,2],[1,2,2,4]]/36 is
// 4*[[4,-2,-2,1],[-2,4,1,-2],[-2,1,4,-2],[1,-2,-2,4]].
inline Vec project_u(const Mesh& mesh, const DofMaps& dofs, const VectorField& f) {
    Vec v(dofs.n_u, 0.0);
    if (!f) return v;
    static const double minv[4][4] = {
        {16, -8, -8, 4}, {-8, 16, 4, -8}, {-8, 4, 16, -8}, {4, -8, -8, 16}};
    const QuadratureRule gq = gauss_legendre(kDataQuadOrder);
    for (int c = 0; c < mesh.n_cells(); ++c) {
        const Cell& cell = mesh.cells[c];
        double bx[4] = {}, by[4] = {};
        for (size_t i = 0; i < gq.points.size(); ++i)
            for (size_t j = 0; j < gq.points.size(); ++j) {
                const double xi = gq.points[i], eta = gq.points[j];
                const double w = gq.weights[i] * gq.weights[j];
                const auto uv = f(cell.x0 + xi * cell.hx, cell.y0 + eta * cell.hy);
                for (int a = 0; a < 4; ++a) {
                    const double nv = shapes::n(a, xi, eta);
                    bx[a] += w * nv * uv[0];
                    by[a] += w * nv * uv[1];
                }
            }
        for (int a = 0; a < 4; ++a) {
            double sx = 0.0, sy = 0.0;
            for (int b = 0; b < 4; ++b) {
                sx += minv[a][b] * bx[b];
                sy += minv[a][b] * by[b];
            }
            v[dofs.u_dof(c, a, 0)] = sx;
            v[dofs.u_dof(c, a, 1)] = sy;
        }
    }
    return v;
}

}  // namespace refcpu
