// One transformed diagonal slab block on the device: canonical space-time
// operator, truncated fixed-stress preconditioner and right-preconditioned
// GMRES (slab.hpp:154-171, :220-234; fixed_stress.hpp:109-181; gmres.hpp:40-139).
#pragma once

#include <memory>

#include "blocktri.cuh"
#include "nd.cuh"
#include "ops.cuh"
#include "spacetime_op.cuh"

namespace pdg {

// Shared exact displacement solve (the reference shares one DenseLu of A
// across all blocks, slab.hpp:155 / fixed_stress.hpp:89-94).
struct ASolver {
    BlockTriChol chol;  // twisted block-tridiagonal (PDG_A_SOLVER=local|general)
    NdChol nd;          // nested dissection (PDG_A_SOLVER=nd)
    bool use_nd = false;
    void solve(const double* b, long long ldb, double* x, long long ldx, int nrhs, cudaStream_t st) {
        if (use_nd)
            nd.solve(b, ldb, x, ldx, nrhs, st);
        else
            chol.solve(b, ldb, x, ldx, nrhs, st);
    }
};
// fp32_factor: fast mode (pdg_gmres_opts.mode 1), honoured by the streaming nested-dissection solve only
std::shared_ptr<ASolver> make_a_solver(const SpatialOps& ops, int max_rhs, cudaStream_t st, bool fp32_factor = false);
HCsr csr_download(const DCsr& a, cudaStream_t st);
// flux Schur complement S_q = w M_q - w^2 B D^{-1} B^T (host CSR, face order), dinv = D^{-1}
HCsr flow_schur_host(const SpatialOps& o, double w, const std::vector<double>& dinv, cudaStream_t st);
// face centres (mesh.hpp:59-60 numbering) in cell units: the nested-dissection coordinates
void face_coords(int nx, int ny, std::vector<double>& cx, std::vector<double>& cy);
int nd_leaf_dofs(int dflt, const char* var = "PDG_ND_LEAF");

// FixedStressSolver(lambda) :: precondition for each of the m components.
struct FixedStressPre {
    const SpatialOps* ops = nullptr;
    int m = 1, sweeps = 1;
    double tau = 0, lambda = 0, stab = 0, w = 0;
    std::shared_ptr<ASolver> a;
    BlockTriChol flow;  // S_q = w M_q - w^2 B D^{-1} B^T in face-row order
    NdChol flow_nd;     // the same S_q by nested dissection (PDG_FLOW_SOLVER=nd)
    bool flow_use_nd = false;
    DBuf<double> dinv;  // 1 / (-(lambda (1/M + stab)) m_p)
    DBuf<double> rq, fp, mech, xold;
    const int* guard = nullptr;  // skip the sweep's kernels once *guard != 0 (speculative GMRES steps)
    void setup(const SpatialOps& ops, int m, double tau, double lambda, double stab, int sweeps,
               std::shared_ptr<ASolver> a, cudaStream_t st);
    void apply(const double* r, double* z, cudaStream_t st);
    void sweep_once(const double* xprev, const double* r, double* z, cudaStream_t st);

    // Coupled form (the fixed-stress march's untransformed slab block, march.hpp:83-84):
    // full Theta = G_hat and kappa = Radau weights, m <= 2. The pressure block
    // -Theta (x) (1/M + stab) M_p is eliminated per cell, the flux Schur complement
    // W (x) M_q + (W Theta^{-1} W) (x) B D^{-1} B^T couples the components and is
    // not symmetric: twisted block LU in face-row blocks holding both components.
    bool coupled = false;
    double th[4] = {0, 0, 0, 0}, thinv[4] = {0, 0, 0, 0}, wc[2] = {0, 0};
    DBuf<double> dinvc, qtmp;
    void setup_coupled(const SpatialOps& ops, int m, double tau, const double* theta, const double* kappa, double stab,
                       std::shared_ptr<ASolver> a, cudaStream_t st);
};

struct Gmres {
    long long n = 0;
    int restart = 50;
    DBuf<double> V, Z, w, x, r, cand, t, y_dev, h_dev, partial, norm_dev;
    DBuf<double> AZ, r0;  // flexible: op(z_j) and the cycle's initial residual (Arnoldi-relation residual)
    DBuf<double> spmv_part;  // first Gram-Schmidt pass partials from the fused SpMV epilogue [block][<= 8]
    int spmv_blocks = 0;
    double* h_host = nullptr;  // pinned
    // device-driven steps (flexible candidate): Hessenberg columns, Givens state (cs, sn, g),
    // step state
    DBuf<double> Hd, givens, lstate;
    void* h_slots = nullptr;  // pinned LoopState per step
    cudaEvent_t evs[2] = {nullptr, nullptr};
    void setup(long long n, int restart, bool keep_z, cudaStream_t st);
    ~Gmres();
};

struct Block {
    Ctx* ctx = nullptr;
    const SpatialOps* ops = nullptr;
    int m = 1;
    double tau = 0, lambda = 0;
    std::vector<double> theta;
    pdg_gmres_opts opts{};
    SpaceTimeOp op;
    FixedStressPre pre;
    Gmres kr;
    DBuf<double> io_in, io_out;  // host-boundary staging
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    long long rows() const { return (long long)m * ops->n_total(); }
    void create(const SpatialOps& ops, int m, const double* theta, double tau, double lambda,
                const pdg_gmres_opts& o, std::shared_ptr<ASolver> a);
    // GMRES solve, device pointers, on ctx->stream. Throws Error(PDG_NOT_CONVERGED) like slab.hpp:228-230.
    void solve(const double* b, double* x, pdg_report* rep, int block_index = 0);
    ~Block();
};

// FixedStressSolver::solve (fixed_stress.hpp:144-172) on the untransformed
// slab block of the fixed-stress march (march.hpp:80-108): Theta = G_hat,
// kappa = the Radau weights. Sweeps from x0 until the true residual of the
// coupled block drops below tol ||rhs||. Device path for dG(0) (one component).
struct FsSolver {
    Ctx* ctx = nullptr;
    const SpatialOps* ops = nullptr;
    int m = 1;
    double tau = 0;
    SpaceTimeOp op;
    FixedStressPre pre;
    Gmres red;  // reduction buffers
    DBuf<double> xa, xb, t, r;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    void create(const SpatialOps& ops, int r, double tau, double stab, std::shared_ptr<ASolver> a);
    // x0 may be null (zero initial guess). Throws Error(PDG_NOT_CONVERGED) like march.hpp:95-97.
    void solve(const double* rhs, const double* x0, double* x_out, double tol, int max_sweeps, pdg_report* rep);
    ~FsSolver();
};

}  // namespace pdg
