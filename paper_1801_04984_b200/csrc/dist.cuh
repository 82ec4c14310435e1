// Multi-GPU slab block solve (one process per GPU; DESIGN.md section 6,
// SURVEY.md 8(e)). Ranks own strips of cell rows; every rank holds the whole
// assembled operators (setup) and owns the rows of its strip.
//
//  * Comm: the library's communicator. NCCL (ncclAllGather, grouped
//    ncclSend/ncclRecv on the rank's stream) in production; a host-staged
//    backend driven by caller callbacks (e.g. torch.distributed gloo) lets
//    several ranks share one GPU in the tests without any kernel waiting on
//    another rank's kernel.
//  * Operator (fixed_stress.hpp:38-60, canonical assembled form): the strip's
//    rows of the space-time SpMV after a halo exchange of the x entries they
//    read (one cell row of neighbours); every row summed as on one GPU.
//  * Krylov reductions (gmres.hpp:94-103): per-rank partial dots, all-gathered
//    and summed in rank order, so every rank holds bit-identical Hessenberg
//    columns and takes the same decisions.
//  * Exact inner solves (fixed_stress.hpp:109-139) across the strips by
//    substructuring: the first block row of every strip but the first is a
//    separator; each rank factors its strip interior with the nested-dissection
//    Cholesky (nd.cuh), keeps the spikes W = K_II^{-1} K_IS of its two
//    separators, and the separator Schur complement (ordered sum of the ranks'
//    contributions) is factored redundantly; per solve: interior solve, one
//    all-gather of the separator right-hand sides, separator solve, x_I = y_I - W x_S.
#pragma once

#include <memory>
#include <vector>

#include "block.cuh"
#include "porodg_b200.h"

namespace pdg {

struct Comm {
    int rank = 0, nranks = 1;
    virtual ~Comm() = default;
    // recv[r * count + j] = (send of rank r)[j]; device buffers on stream st
    virtual void allgather(const double* send, double* recv, size_t count, cudaStream_t st) = 0;
    // one round: to peers[i] send sbuf[i] (scount[i] doubles), from peers[i] receive rbuf[i] (rcount[i])
    virtual void exchange(const std::vector<int>& peers, const std::vector<const double*>& sbuf,
                          const std::vector<size_t>& scount, const std::vector<double*>& rbuf,
                          const std::vector<size_t>& rcount, cudaStream_t st) = 0;
};
std::unique_ptr<Comm> make_nccl_comm(int nranks, int rank, const unsigned char* id, int device);
std::unique_ptr<Comm> make_host_comm(int nranks, int rank, pdg_host_allgather_fn ag, pdg_host_exchange_fn ex, void* user);
void nccl_unique_id(unsigned char* id);

// Point-to-point halo of a full-length global-numbering buffer holding ncomp
// components at a stride: per peer, the global indices sent and received.
struct Halo {
    std::vector<int> peers;
    std::vector<DBuf<long long>> sidx, ridx;
    std::vector<DBuf<double>> sbuf, rbuf;
    int ncomp = 1;
    long long stride = 0;
    void build(const std::vector<int>& peers, const std::vector<std::vector<long long>>& send,
               const std::vector<std::vector<long long>>& recv, int ncomp, long long stride, cudaStream_t st);
    void run(Comm& c, double* x, cudaStream_t st);
};

// Exact SPD solve of K (block tridiagonal in `blocks` strips) across the ranks.
struct DistSub {
    int P = 1, rank = 0, n = 0;
    int ni = 0;                    // interior dofs of this rank
    DBuf<long long> I_d, Stop_d;   // global indices of the interior / own separator dofs
    std::vector<long long> so;     // separator offsets (P - 1 separators), so[P-1] = ns
    int ns = 0, s_top = 0, s_bot = 0, t_top = -1, t_bot = -1;
    NdChol nd;
    DBuf<double> Wt, Wb;           // spikes, n_I x s col-major
    DCsr Ast, Asb;                 // K_SI of the own and the next separator (rows s, local interior columns)
    DBuf<double> Sfac;             // separator Schur complement, Cholesky factor (ns x ns, lower)
    DBuf<double> bI, yI, g, gsum, gall, work;
    DBuf<int> info;
    int lwork = 0;
    std::unique_ptr<LaHandles> la;
    void setup(Comm& c, const HCsr& K, const std::vector<int>& block_of, const std::vector<std::pair<int, int>>& parts,
               const std::vector<int>& node_of, const std::vector<double>& cx, const std::vector<double>& cy, int prof,
               cudaStream_t st);
    // x[own] = K^{-1} b for the owned entries (interior + own separator); b, x full length n,
    // nrhs <= 2 at stride ld; b needs only the owned entries
    void solve(Comm& c, const double* b, double* x, long long ld, int nrhs, cudaStream_t st);
};

struct DistBlock {
    Ctx* ctx = nullptr;
    const SpatialOps* ops = nullptr;
    Comm* comm = nullptr;
    int m = 1, P = 1, rank = 0, r0 = 0, r1 = 0;
    double tau = 0, lambda = 0, w = 0, stab = 0;
    pdg_gmres_opts opts{};
    std::vector<std::pair<int, int>> strips;
    long long nglob = 0, nown = 0;
    DBuf<long long> own_rows;  // global rows of the m-component operator owned here (ascending)
    std::vector<long long> own_rows_h;
    SpaceTimeOp op;
    Halo xhalo;                // x entries of the operator rows
    DBuf<double> xf, yf;       // full-length operator buffers
    // preconditioner (per component: u | q | p global numbering), owned index lists
    DBuf<int> oc, of, ou;      // owned cells, faces, displacement dofs
    int noc = 0, nof = 0, nou = 0;
    Halo hfp, hq, hp;          // fp (cells) for B rows, q (faces) for B^T rows, p (cells) for E rows
    DBuf<double> dinv, fp, rq, qf, pf, mech, uf, rfull, zfull;
    DistSub flow, mech_solver;
    // GMRES
    DBuf<double> V, Z, wv, x, r, cand, t, ydev, dots, dsum, gbuf, part;
    double* hhost = nullptr;
    void create(const SpatialOps& o, Comm* c, int m, const double* theta, double tau, double lambda,
                const pdg_gmres_opts& op, cudaStream_t st);
    void apply(const double* x_own, double* y_own, cudaStream_t st);        // operator rows owned
    void precondition(const double* r_own, double* z_own, cudaStream_t st);  // fixed-stress sweep
    void solve(const double* b_own, double* x_own, pdg_report* rep);
    ~DistBlock();

  private:
    double dot_sum(const double* a, const double* b, cudaStream_t st);
    void multidot_dev(const double* Vb, int ncols, const double* wv_, double* out, cudaStream_t st);
};

}  // namespace pdg
