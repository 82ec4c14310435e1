// The reference-side binding (integration/porodg_gpu_slab.hpp) on BASELINE config 0
// (16^2, dG(0)), first slab: reference-shaped operators (here downloaded from the
// device assembly, which is bit-identical to assemble_operators) go through
// pdg_ops_upload with the mesh inferred, and the slab solve through the binding must
// equal the solve on the device-assembled operators bit for bit.
#include <cstdio>
#include <cstring>
#include <vector>

#include "porodg_mock.hpp"
#include "../../integration/porodg_gpu_slab.hpp"

int main() {
    using namespace porodg_b200;
    pdg_problem p{};
    p.nx = p.ny = 16;
    p.lx = p.ly = 1.0;
    p.lambda = 1e4 * 0.3 / ((1.3) * (1.0 - 0.6));
    p.mu = 1e4 / 2.6;
    p.k_perm = 1.0;
    p.eta = 1.0;
    p.biot_m = 1e3;
    p.biot_b = 0.9;
    p.penalty = 10.0;
    const int disp[4] = {1, 1, 0, 1}, flow[4] = {1, 1, 1, 0};
    for (int s = 0; s < 4; ++s) {
        p.disp_kind[s] = disp[s];
        p.flow_kind[s] = flow[s];
    }
    p.disp_data[3][1] = -1.0;
    try {
        Context ctx(0);
        SpatialOperators dev_ops(ctx, p);
        long long sz[7];
        check(pdg_ops_sizes(dev_ops.get(), sz));
        // reference-shaped SpatialOperators
        porodg::SpatialOperators ref;
        ref.n_u = static_cast<int>(sz[0]);
        ref.n_q = static_cast<int>(sz[1]);
        ref.n_p = static_cast<int>(sz[2]);
        porodg::SparseMatrix* mats[4] = {&ref.A, &ref.M_q, &ref.B, &ref.E};
        const int rows[4] = {ref.n_u, ref.n_q, ref.n_q, ref.n_u}, cols[4] = {ref.n_u, ref.n_q, ref.n_p, ref.n_p};
        for (int w = 0; w < 4; ++w) {
            porodg::SparseMatrix& m = *mats[w];
            m.rows = rows[w];
            m.cols = cols[w];
            m.row_offsets.resize(m.rows + 1);
            m.col_indices.resize(static_cast<size_t>(sz[3 + w]));
            m.values.resize(static_cast<size_t>(sz[3 + w]));
            check(pdg_ops_download(dev_ops.get(), w, m.row_offsets.data(), m.col_indices.data(), m.values.data()));
        }
        ref.m_p_diag = porodg::VectorXd(ref.n_p);
        for (int c = 0; c < ref.n_p; ++c) ref.m_p_diag.v[c] = (p.lx / p.nx) * (p.ly / p.ny);
        ref.q_constrained.assign(ref.n_q, 0);
        ref.mat.biot_b = p.biot_b;
        ref.mat.biot_m = p.biot_m;
        ref.mat.k_dr = p.lambda + p.mu;
        // the slab system R_0 = tau b(t_1) (zero initial state)
        const double tau = 0.1;
        std::vector<double> u(ref.n_u), q(ref.n_q), pr(ref.n_p);
        check(pdg_ops_rhs(dev_ops.get(), 0.1, u.data(), q.data(), pr.data()));
        porodg::SlabSystem sys;
        sys.ops = &ref;
        sys.tau = tau;
        porodg::VectorXd r0(ref.n_total());
        int k = 0;
        for (double v : u) r0.v[k++] = tau * v;
        for (double v : q) r0.v[k++] = tau * v;
        for (double v : pr) r0.v[k++] = tau * v;
        sys.rhs.push_back(r0);
        porodg::TimeBasis basis;
        basis.r = 0;
        porodg::SolveOptions opt;
        opt.gmres.restart = 50;
        // through the binding
        GpuSlabBackend<porodg::SpatialOperators> backend(ref, basis, tau, opt);
        auto [state, reports] =
            backend.solve<porodg::SlabState, porodg::BlockReport>(sys, porodg::unstack_fields);
        // directly on the device-assembled operators
        SolveOptions g;
        g.gmres.restart = 50;
        SlabSolver direct(dev_ops, 0, tau, g);
        auto [x, rep] = direct.solve(r0.v);
        std::vector<double> y;
        y.insert(y.end(), state.comps[0].u.v.begin(), state.comps[0].u.v.end());
        y.insert(y.end(), state.comps[0].q.v.begin(), state.comps[0].q.v.end());
        y.insert(y.end(), state.comps[0].p.v.begin(), state.comps[0].p.v.end());
        const bool same = y.size() == x.size() && std::memcmp(y.data(), x.data(), sizeof(double) * x.size()) == 0;
        int dims[2] = {0, 0};
        const pdg_csr B = csr_view(ref.B);
        check(pdg_mesh_dims_from_operators(&B, ref.n_q, dims));
        std::printf("mesh %dx%d iterations %d (direct %d) history %zu bitwise %d\n", dims[0], dims[1],
                    reports[0].gmres_iterations, rep.iterations, reports[0].report.residual_history.size(), same ? 1 : 0);
        return same ? 0 : 1;
    } catch (const std::exception& e) {
        std::printf("error: %s\n", e.what());
        return 2;
    }
}
