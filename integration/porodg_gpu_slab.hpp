// Reference-side binding of the GPU slab solve: the
// backend of porodg::SlabSolver for BlockSolverKind::gmres_fs_gpu. It uses only
// the reference's own types and member names (paths relative to
// proj/include/porodg/):
//   SpatialOperators  assembly.hpp:38-52   (A, M_q, B, E: SparseMatrix rows/cols/
//                                           row_offsets/col_indices/values; m_p_diag,
//                                           q_constrained, mat.biot_b/biot_m/k_dr)
//   TimeBasis         time_basis.hpp:104-114 (r)
//   SlabSystem        slab.hpp:31-40         (tau, rhs: one stacked (u,q,p) per node)
//   SlabState         slab.hpp:22-26         (comps, via unstack_fields, slab.hpp:50-56)
//   BlockReport       slab.hpp:113-119
//   SolveOptions      slab.hpp:123-127       (gmres, fs.truncation_sweeps, fs.stab)
// The structured mesh is recovered from the operators (pdg_ops_upload with
// nx = ny = 0, pdg_mesh_dims_from_operators), so the reference's SlabSolver
// constructor needs nothing beyond what it already receives.
#pragma once

#include <algorithm>
#include <memory>
#include <utility>
#include <vector>

#include "porodg_b200.hpp"

namespace porodg_b200 {

template <class RefOps>
class GpuSlabBackend {
public:
    template <class RefBasis, class RefSolveOptions>
    GpuSlabBackend(const RefOps& ops, const RefBasis& basis, double tau, const RefSolveOptions& opt, int device = 0)
        : ref_(&ops), r_(basis.r) {
        ctx_ = std::make_unique<Context>(device);
        ops_ = std::make_unique<SpatialOperators>(*ctx_, 0, 0, ops);  // mesh inferred from the operators
        SolveOptions g;
        g.gmres.tol = opt.gmres.tol;
        g.gmres.restart = opt.gmres.restart;
        g.gmres.max_iter = opt.gmres.max_iter;
        g.truncation_sweeps = opt.fs.truncation_sweeps;
        g.stab = opt.fs.stab;
        slab_ = std::make_unique<SlabSolver>(*ops_, r_, tau, g);
    }

    // slab.hpp:179-255 on the GPU: Schur transform, GMRES on the transformed block,
    // back-transform. Returns the state and one BlockReport (the r <= 1 single block).
    template <class RefState, class RefReport, class RefSystem, class Unstack>
    std::pair<RefState, std::vector<RefReport>> solve(const RefSystem& sys, Unstack unstack) const {
        using Vec = typename std::decay<decltype(sys.rhs[0])>::type;
        const long long nt = ref_->n_total(), n = r_ + 1;
        std::vector<double> rhs(static_cast<size_t>(n * nt));
        for (long long i = 0; i < n; ++i) std::copy(sys.rhs[i].data(), sys.rhs[i].data() + nt, rhs.begin() + i * nt);
        auto [x, rep] = slab_->solve(rhs);  // throws SolverError with the reference's message text
        RefState st;
        st.comps.resize(static_cast<size_t>(n));
        for (long long i = 0; i < n; ++i) {
            Vec xi(static_cast<int>(nt));
            std::copy(x.begin() + i * nt, x.begin() + (i + 1) * nt, xi.data());
            st.comps[i] = unstack(*ref_, xi);
        }
        RefReport br;
        br.block_index = 0;
        br.block_size = static_cast<int>(n);
        br.gmres_iterations = rep.iterations;
        br.fs_sweeps = fs_sweeps_;
        br.report.converged = rep.converged;
        br.report.iterations = rep.iterations;
        br.report.residual_history = rep.residual_history;
        br.report.final_relative_residual = rep.final_relative_residual;
        return {std::move(st), std::vector<RefReport>{std::move(br)}};
    }

    void set_fs_sweeps(int s) { fs_sweeps_ = s; }

private:
    const RefOps* ref_;
    int r_ = 0, fs_sweeps_ = 1;
    std::unique_ptr<Context> ctx_;
    std::unique_ptr<SpatialOperators> ops_;
    std::unique_ptr<SlabSolver> slab_;
};

}  // namespace porodg_b200
