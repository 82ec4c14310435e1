// ORACLE / TEST INFRASTRUCTURE ONLY. Not part of the product.
//
// C ABI over the CPU restatement, loaded by tests/ (ctypes) and by bench.py's
// cpu_baseline / --impl reference legs. The product library never links it.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <random>

#include "solver.hpp"
#include "fem3d.hpp"

using namespace refcpu;

extern "C" {

// Problem description for the structured-rectangle configurations with
// constant boundary data (BASELINE configs, Terzaghi column).
typedef struct {
    int nx, ny;
    double lx, ly;
    double lambda, mu, k_perm, eta, biot_m, biot_b;
    const double* k_perm_cells;  // nullptr or nx*ny values (cell c = j*nx + i)
    double penalty;
    int disp_kind[4];        // per tag left,right,bottom,top: 0 fixed, 1 traction, 2 roller_x, 3 roller_y
    double disp_data[4][2];  // constant Dirichlet value (fixed) or traction vector (others)
    int flow_kind[4];        // 0 pressure, 1 no_flow
    double flow_data[4];     // constant prescribed pressure
} refcpu_problem;

struct Handle {
    Mesh mesh;
    DofMaps dofs;
    SpatialOperators ops;
    VolumeData data;
    std::string err;
    // 3D extension (fem3d.hpp; no reference counterpart): dim == 3 uses mesh3 / bc3
    int dim = 2;
    Mesh3 mesh3;
    BoundarySpec3 bc3;
};

// assemble_rhs of either dimension
static FieldVecs rhs_at(Handle* h, double t) {
    if (h->dim == 3) return assemble_rhs3(h->mesh3, h->ops.mat, h->ops, h->bc3, t);
    return assemble_rhs(h->mesh, h->dofs, h->ops.mat, h->ops, h->data, t);
}

static thread_local std::string g_err;

const char* refcpu_last_error() { return g_err.c_str(); }

#define GUARD_BEGIN try {
#define GUARD_END                        \
    }                                    \
    catch (const SolverError& e) {       \
        g_err = e.what();                \
        return 2;                        \
    }                                    \
    catch (const std::exception& e) {    \
        g_err = e.what();                \
        return 1;                        \
    }                                    \
    return 0;

static BoundarySpec make_bc(const refcpu_problem* p) {
    BoundarySpec bc;
    const FaceTag tags[4] = {FaceTag::left, FaceTag::right, FaceTag::bottom, FaceTag::top};
    for (int s = 0; s < 4; ++s) {
        const double d0 = p->disp_data[s][0], d1 = p->disp_data[s][1];
        VectorFieldT vf;
        if (d0 != 0.0 || d1 != 0.0)
            vf = [d0, d1](double, double, double) { return std::array<double, 2>{d0, d1}; };
        DisplacementBC db;
        switch (p->disp_kind[s]) {
            case 0: db = DisplacementBC::fixed(vf); break;
            case 1: db = DisplacementBC::traction(vf); break;
            case 2: db = DisplacementBC::roller_x(vf); break;
            case 3: db = DisplacementBC::roller_y(vf); break;
            default: throw std::invalid_argument("bad displacement kind");
        }
        bc.set_displacement(tags[s], db);
        if (p->flow_kind[s] == 0) {
            const double pv = p->flow_data[s];
            ScalarFieldT sf;
            if (pv != 0.0) sf = [pv](double, double, double) { return pv; };
            bc.set_flow(tags[s], FlowBC::pressure(sf));
        } else {
            bc.set_flow(tags[s], FlowBC::no_flow());
        }
    }
    return bc;
}

int refcpu_create(const refcpu_problem* p, void** out) {
    GUARD_BEGIN
    auto h = std::make_unique<Handle>();
    h->mesh = build_mesh(p->nx, p->ny, p->lx, p->ly);
    h->dofs = build_dof_maps(h->mesh);
    MaterialParameters mat = material_from_lame(p->lambda, p->mu, p->k_perm, p->eta, p->biot_m, p->biot_b);
    if (p->k_perm_cells) mat.k_perm_cells.assign(p->k_perm_cells, p->k_perm_cells + p->nx * p->ny);
    mat.validate();
    h->ops = assemble_operators(h->mesh, h->dofs, mat, p->penalty, make_bc(p));
    *out = h.release();
    GUARD_END
}

// 3D problem (fem3d.hpp): tags xlo, xhi, ylo, yhi, zlo, zhi; displacement kinds 0 fixed,
// 1 traction, 2 / 3 / 4 roller fixing the x / y / z component; constant data.
typedef struct {
    int nx, ny, nz;
    double lx, ly, lz;
    double lambda, mu, k_perm, eta, biot_m, biot_b;
    const double* k_perm_cells;  // nullptr or nx*ny*nz values (cell c = (k*ny + j)*nx + i)
    double penalty;
    int disp_kind[6];
    double disp_data[6][3];
    int flow_kind[6];  // 0 pressure, 1 no_flow
    double flow_data[6];
} refcpu_problem3;

int refcpu_create3(const refcpu_problem3* p, void** out) {
    GUARD_BEGIN
    auto h = std::make_unique<Handle>();
    h->dim = 3;
    h->mesh3 = build_mesh3(p->nx, p->ny, p->nz, p->lx, p->ly, p->lz);
    MaterialParameters mat = material_from_lame3(p->lambda, p->mu, p->k_perm, p->eta, p->biot_m, p->biot_b);
    if (p->k_perm_cells) mat.k_perm_cells.assign(p->k_perm_cells, p->k_perm_cells + (size_t)p->nx * p->ny * p->nz);
    for (int s = 0; s < 6; ++s) {
        DisplacementBC3& d = h->bc3.displacement[s];
        const int kind = p->disp_kind[s];
        if (kind < 0 || kind > 4) throw std::invalid_argument("bad displacement kind");
        d.dirichlet = {kind == 0 || kind == 2, kind == 0 || kind == 3, kind == 0 || kind == 4};
        for (int k = 0; k < 3; ++k) {
            // dirichlet data only for fixed(); rollers and traction faces carry traction data
            d.dirichlet_data[k] = kind == 0 ? p->disp_data[s][k] : 0.0;
            d.traction_data[k] = kind == 0 ? 0.0 : p->disp_data[s][k];
        }
        if (p->flow_kind[s] != 0 && p->flow_kind[s] != 1) throw std::invalid_argument("bad flow kind");
        h->bc3.flow[s].no_flow = p->flow_kind[s] == 1;
        h->bc3.flow[s].pressure = p->flow_data[s];
    }
    h->ops = assemble_operators3(h->mesh3, mat, p->penalty, h->bc3);
    *out = h.release();
    GUARD_END
}

// Smooth, time-dependent analytic test fields for the full assemble_rhs path (VolumeData and
// boundary functions, assembly.hpp:24-28, boundary.hpp:12-13): kind 0 clears them, kind 1
// installs momentum / Darcy / mass sources and, on every tag, traction, Dirichlet and flow data
// (prescribed pressure, or a nonzero prescribed normal flux on no-flow-kind faces). 2D.
int refcpu_set_test_fields(void* hp, int kind) {
    GUARD_BEGIN
    auto* h = static_cast<Handle*>(hp);
    if (h->dim != 2) throw std::invalid_argument("test fields: 2D only");
    const FaceTag tags[4] = {FaceTag::left, FaceTag::right, FaceTag::bottom, FaceTag::top};
    if (kind == 0) {
        h->data = VolumeData{};
        for (FaceTag t : tags) {
            h->ops.bc.displacement[BoundarySpec::slot(t)]->dirichlet_data = {};
            h->ops.bc.displacement[BoundarySpec::slot(t)]->traction_data = {};
            h->ops.bc.flow[BoundarySpec::slot(t)]->data = {};
        }
    } else {
        h->data.momentum = [](double x, double y, double t) {
            return std::array<double, 2>{std::sin(1.3 * x + 0.7 * y) * (1.0 + 0.5 * t), x * y - 0.3 * t};
        };
        h->data.darcy = [](double x, double y, double t) {
            return std::array<double, 2>{std::cos(2.0 * x) * y + t, 0.25 + x - y * y * t};
        };
        h->data.mass = [](double x, double y, double t) { return std::exp(-t) * (1.0 + x) * std::sin(3.0 * y); };
        int k = 0;
        for (FaceTag t : tags) {
            const double a = 0.1 * (++k);
            h->ops.bc.displacement[BoundarySpec::slot(t)]->dirichlet_data = [a](double x, double y, double tt) {
                return std::array<double, 2>{a * std::sin(x + 2.0 * y + tt), a * (x - y) * (1.0 + tt)};
            };
            h->ops.bc.displacement[BoundarySpec::slot(t)]->traction_data = [a](double x, double y, double tt) {
                return std::array<double, 2>{a + x * tt, -1.0 + a * std::cos(y - tt)};
            };
            h->ops.bc.flow[BoundarySpec::slot(t)]->data = [a](double x, double y, double tt) {
                return a * (1.0 + x * y) + 0.2 * std::sin(tt + x - y);
            };
        }
    }
    GUARD_END
}

// The installed fields evaluated at assemble_rhs's quadrature points at time t (what a host
// binding passes to pdg_ops_rhs_sampled): per cell the 6 x 6 points (xi outer), per boundary
// face in ascending face index the 6 points. vol_present[3]: momentum, darcy, mass set?
int refcpu_sample_rhs_data(void* hp, double t, double* momentum, double* darcy, double* mass, double* traction,
                           double* dirichlet, double* flow, int* vol_present) {
    GUARD_BEGIN
    auto* h = static_cast<Handle*>(hp);
    const Mesh& mesh = h->mesh;
    const QuadratureRule gq = gauss_legendre(kDataQuadOrder);
    vol_present[0] = static_cast<bool>(h->data.momentum);
    vol_present[1] = static_cast<bool>(h->data.darcy);
    vol_present[2] = static_cast<bool>(h->data.mass);
    for (int c = 0; c < mesh.n_cells(); ++c) {
        const Cell& cell = mesh.cells[c];
        for (size_t i = 0; i < 6; ++i)
            for (size_t j = 0; j < 6; ++j) {
                const double x = cell.x0 + gq.points[i] * cell.hx, y = cell.y0 + gq.points[j] * cell.hy;
                const size_t k = static_cast<size_t>(c) * 36 + i * 6 + j;
                const auto fm = eval_or_zero(h->data.momentum, x, y, t), fd = eval_or_zero(h->data.darcy, x, y, t);
                momentum[2 * k] = fm[0];
                momentum[2 * k + 1] = fm[1];
                darcy[2 * k] = fd[0];
                darcy[2 * k + 1] = fd[1];
                mass[k] = eval_or_zero(h->data.mass, x, y, t);
            }
    }
    size_t b = 0;
    for (int f = 0; f < mesh.n_faces(); ++f) {
        const Face& face = mesh.faces[f];
        if (!face.is_boundary()) continue;
        const DisplacementBC& dbc = h->ops.bc.displacement_on(face.tag);
        const FlowBC& fbc = h->ops.bc.flow_on(face.tag);
        for (size_t q = 0; q < 6; ++q) {
            const double s = gq.points[q];
            const double x = face.x0 + s * (face.x1 - face.x0), y = face.y0 + s * (face.y1 - face.y0);
            const auto tn = eval_or_zero(dbc.traction_data, x, y, t), ud = eval_or_zero(dbc.dirichlet_data, x, y, t);
            traction[(b * 6 + q) * 2] = tn[0];
            traction[(b * 6 + q) * 2 + 1] = tn[1];
            dirichlet[(b * 6 + q) * 2] = ud[0];
            dirichlet[(b * 6 + q) * 2 + 1] = ud[1];
            flow[b * 6 + q] = eval_or_zero(fbc.data, x, y, t);
        }
        ++b;
    }
    GUARD_END
}

// 3D: assemble_rhs3_sampled and its sample points (fem3d.hpp). n_bfaces = 2 (nx ny + nx nz + ny nz).
int refcpu_rhs3_sample_points(void* hp, double* cell_xyz, int* bface_ids, double* bface_xyz) {
    GUARD_BEGIN
    auto* h = static_cast<Handle*>(hp);
    if (h->dim != 3) throw std::invalid_argument("rhs3 sample points: 3D only");
    rhs3_sample_points(h->mesh3, cell_xyz, bface_ids, bface_xyz);
    GUARD_END
}
int refcpu_rhs3_sampled(void* hp, const double* momentum, const double* darcy, const double* mass, const double* traction,
                        const double* dirichlet, const double* flow, double* u, double* q, double* p) {
    GUARD_BEGIN
    auto* h = static_cast<Handle*>(hp);
    if (h->dim != 3) throw std::invalid_argument("rhs3 sampled: 3D only");
    RhsSamples3 sm;
    sm.momentum = momentum;
    sm.darcy = darcy;
    sm.mass = mass;
    sm.traction = traction;
    sm.dirichlet = dirichlet;
    sm.flow = flow;
    const FieldVecs r = assemble_rhs3_sampled(h->mesh3, h->ops.mat, h->ops, h->bc3, sm);
    std::memcpy(u, r.u.data(), sizeof(double) * r.u.size());
    std::memcpy(q, r.q.data(), sizeof(double) * r.q.size());
    std::memcpy(p, r.p.data(), sizeof(double) * r.p.size());
    GUARD_END
}

void refcpu_destroy(void* h) { delete static_cast<Handle*>(h); }

// sizes[0..] = n_u, n_q, n_p, nnz(A), nnz(M_q), nnz(B), nnz(E), nnz(M_p)
int refcpu_sizes(void* hp, long long* sizes) {
    GUARD_BEGIN
    auto* h = static_cast<Handle*>(hp);
    sizes[0] = h->ops.n_u;
    sizes[1] = h->ops.n_q;
    sizes[2] = h->ops.n_p;
    sizes[3] = h->ops.A.nnz();
    sizes[4] = h->ops.M_q.nnz();
    sizes[5] = h->ops.B.nnz();
    sizes[6] = h->ops.E.nnz();
    sizes[7] = h->ops.M_p.nnz();
    GUARD_END
}

static const SparseMatrix& pick(Handle* h, int which) {
    switch (which) {
        case 0: return h->ops.A;
        case 1: return h->ops.M_q;
        case 2: return h->ops.B;
        case 3: return h->ops.E;
        case 4: return h->ops.M_p;
    }
    throw std::invalid_argument("bad block id");
}

// Export block `which` (0 A, 1 M_q, 2 B, 3 E, 4 M_p) as CSR.
int refcpu_export_csr(void* hp, int which, int* off, int* idx, double* val) {
    GUARD_BEGIN
    const SparseMatrix& s = pick(static_cast<Handle*>(hp), which);
    std::memcpy(off, s.row_offsets.data(), sizeof(int) * (s.rows + 1));
    std::memcpy(idx, s.col_indices.data(), sizeof(int) * s.nnz());
    std::memcpy(val, s.values.data(), sizeof(double) * s.nnz());
    GUARD_END
}

int refcpu_export_misc(void* hp, double* m_p_diag, signed char* q_constrained, double* b_biot, double* inv_m,
                       double* k_dr) {
    GUARD_BEGIN
    auto* h = static_cast<Handle*>(hp);
    std::memcpy(m_p_diag, h->ops.m_p_diag.data(), sizeof(double) * h->ops.n_p);
    for (int i = 0; i < h->ops.n_q; ++i) q_constrained[i] = h->ops.q_constrained[i];
    *b_biot = h->ops.mat.biot_b;
    *inv_m = 1.0 / h->ops.mat.biot_m;
    *k_dr = h->ops.mat.k_dr;
    GUARD_END
}

// assemble_rhs at time t (constant boundary data; no volume data).
int refcpu_assemble_rhs(void* hp, double t, double* u, double* q, double* p) {
    GUARD_BEGIN
    auto* h = static_cast<Handle*>(hp);
    const FieldVecs r = rhs_at(h, t);
    std::memcpy(u, r.u.data(), sizeof(double) * r.u.size());
    std::memcpy(q, r.q.data(), sizeof(double) * r.q.size());
    std::memcpy(p, r.p.data(), sizeof(double) * r.p.size());
    GUARD_END
}

// Time basis and Schur constants for degree r (r <= 1): out arrays sized
// (r+1), (r+1)^2.
int refcpu_time_constants(int r, double* nodes, double* weights, double* phi0, double* G_hat, double* T, double* Q) {
    GUARD_BEGIN
    const TimeBasis b = time_matrices(r);
    const SchurForm s = real_schur(b);
    const int n = r + 1;
    for (int i = 0; i < n; ++i) {
        nodes[i] = b.nodes[i];
        weights[i] = b.weights[i];
        phi0[i] = b.phi_at0[i];
    }
    for (int i = 0; i < n * n; ++i) {
        G_hat[i] = b.G_hat[i];
        T[i] = s.T[i];
        Q[i] = s.Q[i];
    }
    GUARD_END
}

// dG(r) basis alone (no Schur form): nodes, weights, phi(0) [r+1], G_hat [(r+1)^2].
int refcpu_time_basis(int r, double* nodes, double* weights, double* phi0, double* G_hat) {
    GUARD_BEGIN
    const TimeBasis b = time_matrices(r);
    const int n = r + 1;
    for (int i = 0; i < n; ++i) {
        nodes[i] = b.nodes[i];
        weights[i] = b.weights[i];
        phi0[i] = b.phi_at0[i];
    }
    for (int i = 0; i < n * n; ++i) G_hat[i] = b.G_hat[i];
    GUARD_END
}

// Register the raw (unordered) real Schur form W = Q T Q^T of the (r+1) x (r+1) time operator,
// r >= 2, computed by LAPACK (solver.hpp real_schur).
int refcpu_set_raw_schur(int r, const double* T, const double* Q) {
    GUARD_BEGIN
    const int n = r + 1;
    RawSchur rs;
    rs.T.assign(T, T + n * n);
    rs.Q.assign(Q, Q + n * n);
    raw_schur_registry()[n] = rs;
    GUARD_END
}

// Diagonal blocks of the ordered Schur form of degree r.
int refcpu_schur_blocks(int r, int* n_blocks, int* sizes, int* starts) {
    GUARD_BEGIN
    const SchurForm s = real_schur(time_matrices(r));
    *n_blocks = s.n_blocks();
    for (int g = 0; g < s.n_blocks(); ++g) {
        sizes[g] = s.block_sizes[g];
        starts[g] = s.block_starts[g];
    }
    GUARD_END
}

struct StCsr {
    SparseMatrix s;
};

// Canonical space-time operator for block theta (m x m row-major), tau.
int refcpu_spacetime_build(void* hp, int m, const double* theta, double tau, void** out, long long* rows_nnz) {
    GUARD_BEGIN
    auto* h = static_cast<Handle*>(hp);
    auto st = std::make_unique<StCsr>();
    st->s = build_spacetime_csr(h->ops, std::vector<double>(theta, theta + m * m), m, tau);
    rows_nnz[0] = st->s.rows;
    rows_nnz[1] = st->s.nnz();
    *out = st.release();
    GUARD_END
}
int refcpu_spacetime_export(void* sp, int* off, int* idx, double* val) {
    GUARD_BEGIN
    const SparseMatrix& s = static_cast<StCsr*>(sp)->s;
    std::memcpy(off, s.row_offsets.data(), sizeof(int) * (s.rows + 1));
    std::memcpy(idx, s.col_indices.data(), sizeof(int) * s.nnz());
    std::memcpy(val, s.values.data(), sizeof(double) * s.nnz());
    GUARD_END
}
void refcpu_spacetime_destroy(void* sp) { delete static_cast<StCsr*>(sp); }

// SparseMatrix::apply (sparse.hpp:30-40) on caller-provided CSR; optional
// OpenMP over rows (each row is still summed sequentially, so the result is
// bit-identical for any thread count).
int refcpu_csr_apply(int rows, const long long* off, const int* idx, const double* val, const double* x, double* y,
                     int threads) {
    GUARD_BEGIN
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
    for (int i = 0; i < rows; ++i) {
        double s = 0.0;
        for (long long k = off[i]; k < off[i + 1]; ++k) s += val[k] * x[idx[k]];
        y[i] = s;
    }
    GUARD_END
}

// Block operator apply (fixed_stress.hpp:38-60).
int refcpu_apply_block(void* hp, int m, const double* theta, double tau, const double* x, double* y) {
    GUARD_BEGIN
    auto* h = static_cast<Handle*>(hp);
    apply_block_operator(h->ops, std::vector<double>(theta, theta + m * m), m, tau, x, y);
    GUARD_END
}

// Truncated fixed-stress preconditioner for one time component, lambda.
int refcpu_precondition(void* hp, double lambda, double tau, double stab, int sweeps, int backend, const double* r,
                        double* z) {
    GUARD_BEGIN
    auto* h = static_cast<Handle*>(hp);
    const InnerBackend be = backend ? InnerBackend::banded : InnerBackend::dense;
    if (stab < 0.0) stab = h->ops.mat.biot_b * h->ops.mat.biot_b / h->ops.mat.k_dr;
    FixedStressSolver fs(h->ops, {lambda}, 1, tau, stab, make_a_solver(h->ops, be), be, h->mesh.nx, h->mesh.ny);
    fs.precondition(r, z, sweeps);
    GUARD_END
}

typedef struct {
    double tol;
    int restart, max_iter;
    int sweeps;
    double stab;  // < 0: b^2 / K_dr
    int backend;  // 0 dense LU (reference-exact), 1 banded sparse-direct
    int flexible; // 0 gmres (slab.hpp:227), 1 gmres_flexible
} refcpu_solve_opts;

typedef struct {
    int converged, iterations, history_len;
    double final_rel_res;
    double setup_seconds, solve_seconds;
} refcpu_report;

static SolveOptions to_opts(const refcpu_solve_opts* o) {
    SolveOptions s;
    s.gmres.tol = o->tol;
    s.gmres.restart = o->restart;
    s.gmres.max_iter = o->max_iter;
    s.fs.truncation_sweeps = o->sweeps;
    s.fs.stab = o->stab;
    s.backend = o->backend ? InnerBackend::banded : InnerBackend::dense;
    s.flexible = o->flexible != 0;
    return s;
}

// One GMRES solve of the transformed diagonal block (the hot path,
// slab.hpp:456-473) for degree r's single Schur block and a given rhs.
int refcpu_block_solve(void* hp, int r, double tau, const refcpu_solve_opts* o, const double* rhs, double* x,
                       refcpu_report* rep, double* history, int history_cap) {
    using clk = std::chrono::steady_clock;
    GUARD_BEGIN
    auto* h = static_cast<Handle*>(hp);
    const TimeBasis basis = time_matrices(r);
    const SchurForm schur = real_schur(basis);
    const auto t0 = clk::now();
    SlabSolver solver(h->ops, basis, schur, tau, to_opts(o), h->mesh.nx, h->mesh.ny);
    const auto t1 = clk::now();
    const int m = schur.block_sizes[0];
    Vec b(rhs, rhs + static_cast<size_t>(m) * h->ops.n_total());
    BlockReport br;
    Vec sol;
    try {
        sol = solver.solve_block(0, b, br);
    } catch (const SolverError&) {
        throw;
    }
    const auto t2 = clk::now();
    std::copy(sol.begin(), sol.end(), x);
    rep->converged = br.report.converged;
    rep->iterations = br.report.iterations;
    rep->history_len = static_cast<int>(br.report.residual_history.size());
    rep->final_rel_res = br.report.final_relative_residual;
    rep->setup_seconds = std::chrono::duration<double>(t1 - t0).count();
    rep->solve_seconds = std::chrono::duration<double>(t2 - t1).count();
    for (int i = 0; i < std::min(history_cap, rep->history_len); ++i) history[i] = br.report.residual_history[i];
    GUARD_END
}

// GMRES solve of one transformed diagonal block given its theta (m x m, m <= 2) directly
// (slab.hpp:154-171, :220-234): operator FixedStressSolver(theta), preconditioner
// FixedStressSolver(theta(0,0)) per component. Used for the blocks of r >= 2.
int refcpu_block_solve_theta(void* hp, int m, const double* theta, double tau, const refcpu_solve_opts* o,
                             const double* rhs, double* x, refcpu_report* rep) {
    GUARD_BEGIN
    auto* h = static_cast<Handle*>(hp);
    SchurForm one;
    one.n = m;
    one.T.assign(theta, theta + m * m);
    one.block_sizes = {m};
    one.block_starts = {0};
    const TimeBasis basis = time_matrices(m - 1);  // only its size is read by solve_block
    SlabSolver solver(h->ops, basis, one, tau, to_opts(o), h->mesh.nx, h->mesh.ny);
    Vec b(rhs, rhs + static_cast<size_t>(m) * h->ops.n_total());
    BlockReport br;
    const Vec sol = solver.solve_block(0, b, br);
    std::copy(sol.begin(), sol.end(), x);
    rep->converged = br.report.converged;
    rep->iterations = br.report.iterations;
    rep->history_len = static_cast<int>(br.report.residual_history.size());
    rep->final_rel_res = br.report.final_relative_residual;
    rep->setup_seconds = rep->solve_seconds = 0.0;
    GUARD_END
}

// Monolithic-spectral march (march.hpp:45-79,109-117) over uniform slabs.
// Per slab s: iterations[s], final_res[s], solve_seconds[s]; the end trace
// of the final slab (u, q, p stacked, n_total) in end_state; optionally the
// full per-slab state (all r+1 components, n_slabs*(r+1)*n_total) in states.
int refcpu_march(void* hp, int r, double T, int n_slabs, const refcpu_solve_opts* o, int* iterations,
                 double* final_res, double* solve_seconds, double* setup_seconds, double* end_state, double* states,
                 int max_slabs) {
    using clk = std::chrono::steady_clock;
    GUARD_BEGIN
    auto* h = static_cast<Handle*>(hp);
    const SpatialOperators& ops = h->ops;
    const TimePartition part = uniform_partition(T, n_slabs);
    const TimeBasis basis = time_matrices(r);
    const SchurForm schur = real_schur(basis);
    Vec u_prev(ops.n_u, 0.0), p_prev(ops.n_p, 0.0);
    std::unique_ptr<SlabSolver> spectral;
    double cached_tau = -1.0;
    const int nt = ops.n_total();
    const int run = max_slabs > 0 ? std::min(max_slabs, part.n_slabs()) : part.n_slabs();
    *setup_seconds = 0.0;
    for (int n = 0; n < run; ++n) {
        const double tau = part.slab_length(n), t0 = part.t_begin(n);
        std::vector<FieldVecs> nodal(basis.n_nodes());
        for (int i = 0; i < basis.n_nodes(); ++i)
            nodal[i] = rhs_at(h, t0 + basis.nodes[i] * tau);
        const SlabSystem sys = build_slab_system(ops, basis, tau, nodal, u_prev, p_prev);
        const bool rebuild = cached_tau < 0.0 || std::abs(tau - cached_tau) > 1e-12 * tau;
        try {
            if (rebuild) {
                const auto a = clk::now();
                spectral = std::make_unique<SlabSolver>(ops, basis, schur, tau, to_opts(o), h->mesh.nx, h->mesh.ny);
                *setup_seconds += std::chrono::duration<double>(clk::now() - a).count();
            }
            std::vector<BlockReport> reps;
            const auto a = clk::now();
            const std::vector<FieldVecs> st = spectral->solve(sys, reps);
            solve_seconds[n] = std::chrono::duration<double>(clk::now() - a).count();
            int it = 0;
            double res = 0.0;
            for (const BlockReport& br : reps) {
                it = std::max(it, br.gmres_iterations);
                res = std::max(res, br.report.final_relative_residual);
            }
            iterations[n] = it;
            final_res[n] = res;
            cached_tau = tau;
            u_prev = st.back().u;
            p_prev = st.back().p;
            if (states)
                for (int i = 0; i < basis.n_nodes(); ++i) {
                    double* dst = states + (static_cast<size_t>(n) * basis.n_nodes() + i) * nt;
                    std::copy(st[i].u.begin(), st[i].u.end(), dst);
                    std::copy(st[i].q.begin(), st[i].q.end(), dst + ops.n_u);
                    std::copy(st[i].p.begin(), st[i].p.end(), dst + ops.n_u + ops.n_q);
                }
            if (n == run - 1 && end_state) {
                std::copy(st.back().u.begin(), st.back().u.end(), end_state);
                std::copy(st.back().q.begin(), st.back().q.end(), end_state + ops.n_u);
                std::copy(st.back().p.begin(), st.back().p.end(), end_state + ops.n_u + ops.n_q);
            }
        } catch (const SolverError& e) {
            char buf[64];
            std::snprintf(buf, sizeof(buf), "%f", part.t_end(n));
            throw SolverError("slab " + std::to_string(n) + " (t_n = " + buf + "): " + e.what());
        }
    }
    GUARD_END
}

// Fixed-stress march (march.hpp:80-108): per slab, FixedStressSolver(ops,
// G_hat, weights, tau, stab) iterated to tol on the untransformed slab block
// (fixed_stress.hpp:144-172), warm-started from the previous end trace in every
// component (march.hpp:87-93); rebuilt only when tau changes (march.hpp:72).
// sweeps[n] = BlockReport::fs_sweeps of slab n; states as refcpu_march.
int refcpu_march_fs(void* hp, int r, double T, int n_slabs, double tol, int max_sweeps, double stab, int backend,
                    int* sweeps, double* final_res, double* solve_seconds, double* states, int max_slabs) {
    using clk = std::chrono::steady_clock;
    GUARD_BEGIN
    auto* h = static_cast<Handle*>(hp);
    const SpatialOperators& ops = h->ops;
    const TimePartition part = uniform_partition(T, n_slabs);
    const TimeBasis basis = time_matrices(r);
    const int nn = basis.n_nodes(), nt = ops.n_total();
    FixedStressConfig cfg;
    cfg.tol = tol;
    cfg.max_sweeps = max_sweeps;
    cfg.stab = stab;
    if (!(cfg.tol > 0.0 && cfg.tol < 1.0)) throw std::invalid_argument("fixed-stress: tol must be in (0,1)");
    if (cfg.max_sweeps < 1) throw std::invalid_argument("fixed-stress: sweep counts must be >= 1");
    const double st = cfg.resolve_stab(ops.mat);
    const InnerBackend be = backend ? InnerBackend::banded : InnerBackend::dense;
    std::shared_ptr<InnerSolver> a = make_a_solver(ops, be);
    Vec u_prev(ops.n_u, 0.0), p_prev(ops.n_p, 0.0), trace_prev;
    std::unique_ptr<FixedStressSolver> fs;
    double cached_tau = -1.0;
    const int run = max_slabs > 0 ? std::min(max_slabs, part.n_slabs()) : part.n_slabs();
    for (int n = 0; n < run; ++n) {
        const double tau = part.slab_length(n), t0 = part.t_begin(n);
        std::vector<FieldVecs> nodal(nn);
        for (int i = 0; i < nn; ++i)
            nodal[i] = rhs_at(h, t0 + basis.nodes[i] * tau);
        const SlabSystem sys = build_slab_system(ops, basis, tau, nodal, u_prev, p_prev);
        const bool rebuild = cached_tau < 0.0 || std::abs(tau - cached_tau) > 1e-12 * tau;
        try {
            if (rebuild)
                fs = std::make_unique<FixedStressSolver>(ops, basis.G_hat, nn, tau, st, a, be, h->mesh.nx, h->mesh.ny,
                                                         basis.weights);
            Vec rhs(static_cast<size_t>(nn) * nt);
            for (int i = 0; i < nn; ++i) std::copy(sys.rhs[i].begin(), sys.rhs[i].end(), rhs.begin() + i * nt);
            Vec x0;
            if (!trace_prev.empty()) {
                x0.resize(rhs.size());
                for (int i = 0; i < nn; ++i) std::copy(trace_prev.begin(), trace_prev.end(), x0.begin() + i * nt);
            }
            SolverReport rep;
            const auto a0 = clk::now();
            const Vec x = fs->solve(rhs, cfg, x0, rep);
            if (solve_seconds) solve_seconds[n] = std::chrono::duration<double>(clk::now() - a0).count();
            if (!rep.converged)
                throw SolverError("fixed-stress did not converge (rel res " + std::to_string(rep.final_relative_residual) +
                                  ")");
            sweeps[n] = rep.iterations;
            final_res[n] = rep.final_relative_residual;
            cached_tau = tau;
            const double* end = &x[static_cast<size_t>(nn - 1) * nt];
            u_prev.assign(end, end + ops.n_u);
            p_prev.assign(end + ops.n_u + ops.n_q, end + nt);
            trace_prev.assign(end, end + nt);
            if (states) std::copy(x.begin(), x.end(), states + static_cast<size_t>(n) * nn * nt);
        } catch (const SolverError& e) {
            throw SolverError("slab " + std::to_string(n) + " (t_n = " + std::to_string(part.t_end(n)) + "): " +
                              e.what());
        }
    }
    GUARD_END
}

// Slab right-hand side for a given jump (u_prev, p_prev) and slab start t0:
// out is (r+1)*n_total, stacked per Radau node (slab.hpp:58-87).
int refcpu_slab_rhs(void* hp, int r, double t0, double tau, const double* u_prev, const double* p_prev, double* out) {
    GUARD_BEGIN
    auto* h = static_cast<Handle*>(hp);
    const TimeBasis basis = time_matrices(r);
    std::vector<FieldVecs> nodal(basis.n_nodes());
    for (int i = 0; i < basis.n_nodes(); ++i)
        nodal[i] = rhs_at(h, t0 + basis.nodes[i] * tau);
    const SlabSystem sys = build_slab_system(h->ops, basis, tau, nodal, Vec(u_prev, u_prev + h->ops.n_u),
                                             Vec(p_prev, p_prev + h->ops.n_p));
    for (int i = 0; i < basis.n_nodes(); ++i) std::copy(sys.rhs[i].begin(), sys.rhs[i].end(), out + i * h->ops.n_total());
    GUARD_END
}

// Forward transform of the slab rhs into the Schur basis for degree r (single
// block): shat_i = sum_j Q(j,i) R_j / w_j (slab.hpp:186-188).
int refcpu_schur_forward(void* hp, int r, const double* R, double* shat) {
    GUARD_BEGIN
    auto* h = static_cast<Handle*>(hp);
    const TimeBasis basis = time_matrices(r);
    const SchurForm s = real_schur(basis);
    const int n = r + 1, nt = h->ops.n_total();
    for (int i = 0; i < n; ++i) {
        for (int k = 0; k < nt; ++k) shat[i * nt + k] = 0.0;
        for (int j = 0; j < n; ++j)
            for (int k = 0; k < nt; ++k) shat[i * nt + k] += s.q(j, i) * (R[j * nt + k] / basis.weights[j]);
    }
    GUARD_END
}

// local_mass_residual (slab.hpp:292-318) of a slab state: rhs and state are
// (r+1)*n_total, stacked per Radau node; residual is n_p.
int refcpu_mass_residual(void* hp, int r, double tau, const double* rhs, const double* state, double* residual,
                         double* scale) {
    GUARD_BEGIN
    auto* h = static_cast<Handle*>(hp);
    const TimeBasis basis = time_matrices(r);
    const int n = basis.n_nodes(), nt = h->ops.n_total();
    std::vector<Vec> R(n);
    std::vector<const double*> comps(n);
    for (int i = 0; i < n; ++i) {
        R[i].assign(rhs + (long long)i * nt, rhs + (long long)(i + 1) * nt);
        comps[i] = state + (long long)i * nt;
    }
    const MassResidual mr = local_mass_residual(h->ops, basis, tau, R, comps);
    std::copy(mr.residual.begin(), mr.residual.end(), residual);
    *scale = mr.scale;
    GUARD_END
}

// gauss_legendre(n) on [0, 1] (quadrature.hpp:33-54)
int refcpu_gauss(int n, double* pts, double* wts) {
    GUARD_BEGIN
    const QuadratureRule g = gauss_legendre(n);
    for (int i = 0; i < n; ++i) {
        pts[i] = g.points[i];
        wts[i] = g.weights[i];
    }
    GUARD_END
}

// Seeded generators:
//   uniform x_i = -1 + 2 * ((mt19937_64() >> 11) * 2^-53)
//   normal z = sqrt(-2 ln u1) cos(2 pi u2), u1 = ((g>>11)+1) 2^-53, u2 = (g>>11) 2^-53
void refcpu_uniform(unsigned long long seed, long long n, double* out) {
    std::mt19937_64 g(seed);
    for (long long i = 0; i < n; ++i) out[i] = -1.0 + 2.0 * (static_cast<double>(g() >> 11) * 0x1.0p-53);
}
void refcpu_lognormal(unsigned long long seed, long long n, double sigma, double* out) {
    std::mt19937_64 g(seed);
    for (long long i = 0; i < n; ++i) {
        const double u1 = (static_cast<double>(g() >> 11) + 1.0) * 0x1.0p-53;
        const double u2 = static_cast<double>(g() >> 11) * 0x1.0p-53;
        out[i] = std::exp(sigma * (std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2)));
    }
}

}  // extern "C"
