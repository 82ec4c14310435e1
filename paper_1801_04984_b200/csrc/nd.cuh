// Nested-dissection multifrontal Cholesky with a level-synchronous persistent
// solve: the exact SPD inner solves of the fixed-stress preconditioner
// (fixed_stress.hpp:109-139 applies DenseLu solves, dense.hpp:14-45, of A and of
// the flow block) at O(n log n) factor storage instead of the block-tridiagonal
// O(n w^2), and with O(log n) dependent phases per solve instead of O(ny).
//
// Ordering: geometric nested dissection of the node graph (a node = the dofs of
// one cell or one face): a region is cut by the line of nodes at a coordinate
// value near the median of its longer extent, provided removing that line
// disconnects the two sides (checked on the graph). Each separator is one front
// F with pivots S (its dofs) and boundary B (the ancestor dofs adjacent to the
// region it separates).
//
// Factor (setup, cuSOLVER/cuBLAS on dense fronts, multifrontal extend-add):
//   [L_SS; L_BS] of the front, update F_BB - L_BS L_BS^T to the parent;
//   stored per front as  M  = [L_SS^{-1}; L_BS L_SS^{-1}]   ((s+b) x s, row-major)
//                  and   M^T                               (s x (s+b), row-major).
// Solve (one persistent cooperative kernel, a dataflow without grid barriers):
//   forward   [y_S; u_F] = M (b_S - w_C1|S - w_C2|S)  once both children's forward
//             tasks are done, with the update vector w_F = u_F + w_C1|B + w_C2|B
//             (the children's updates passing through F to its ancestors);
//   backward  x_S = M^T [y_S; -x_B]      once the parent's backward tasks are done.
// Tasks are row chunks placed statically on the CTAs in a topological order;
// each CTA streams the matrix rows of its tasks into a shared-memory ring by
// cp.async.bulk (TMA) several tasks ahead of the dataflow, and completion
// counters (monotone across calls) carry the dependencies. Sums are in a fixed
// order (bit-identical repeats).
#pragma once

#include <string>
#include <vector>

#include "common.cuh"

namespace pdg {

struct LaHandles;

struct NdFront {
    int s, b;             // pivots, boundary dofs
    int sdof, bdof;       // offsets into the S / B dof lists
    int cboff, depth;     // contribution buffer (2 child slots of s + b), tree depth
    long long moff, mtoff;  // M and M^T in the store
    int ldm, ldt;         // row strides (even)
};

// One unit of the solve dataflow: rows [r0, r0 + nrows) of M (forward) or M^T
// (backward) at store + src (row stride ld) times the front's gathered input. A
// task starts when the counters wait0 / wait1 reach call * need0 / need1 and
// bumps counter `signal` when done.
struct NdTask {
    long long src;
    int type;  // 1 forward, 2 backward
    int front, r0, nrows, ld, ncols;
    int s, b, sdof, bdof, cboff;
    int wait0, wait1, need0, need1, signal;
    int leaf;  // no children: forward input is b_S alone, no pass-through updates
    // task buffer in the CTA's shared-memory arena (FIFO, placed on the host): byte offset,
    // stride between the right-hand sides of v (doubles), and the newest earlier task of this
    // CTA whose buffer must be released first (-1: none)
    int boff, vmt, fdep;
    int pad_;
};

// One task of the tile-streaming solve (nd_tile.cu): rows [r0, r0 + nrows) of a
// front pass (type 1: M, type 2: M^T), ntiles tiles of rb complete rows each at
// tstore + src, the row output indices at toix + oix_off, the task buffer at byte
// boff of the CTA's arena (free once CTA-local task fdep is done).
struct NdTileTask {
    long long src;
    int type, front, r0, nrows, cp, ncols, rb, ntiles, tile_d2, kt, nchunks;  // kt tiles per ring chunk
    int s, b, sdof, bdof, cboff, leaf;
    int wait0, wait1, need0, need1, signal;
    int oix_off, boff, fdep, tail_lo, tail_n;
    int cgather;  // the compute warps gather the dependent inputs (shared levels)
    int l2keep;   // tiles loaded with L2 evict_last (top levels)
};
// One unit of the streaming solve (nd_stream.cu): rows [r0, r0 + nrows) of a front's M
// (type 1, forward) or M^T (type 2, backward) at store + src, row stride ld.
struct NdStreamUnit {
    long long src;
    int type, r0, nrows, ncols, ld;
    int s, b, sdof, bdof, cboff;
    int cbeg;  // first column read (even); columns [cbeg, ncols)
};
bool nd_tile_default();
bool nd_levels_default();
bool nd_hybrid_default(int prof_phase);
int nd_top_default(int prof_phase);
int nd_top_cap();

struct NdChol {
    int n = 0, max_rhs = 0, nfront = 0, maxdepth = 0;
    int grid = 0, stages = 3, vmax = 0, max_tasks = 0, smem_tasks = 0, pf = 16;
    unsigned stage_bytes = 24576;
    unsigned long long call = 0;
    size_t smem = 0, arena_bytes = 0, max_task_buf = 0;
    int prof_phase = PROF_A_SOLVE;
    double factor_bytes = 0.0;  // bytes of M and M^T read per solve
    const int* guard = nullptr;  // skip solves on the device once *guard != 0 (speculative GMRES steps)
    long long cbtot = 0;
    // y, xpos in pivot-position order; cbuf: per front, the two children's update vectors
    // scattered to the front's local positions ([child][s + b], per right-hand side)
    DBuf<double> store, y, xpos, cbuf;
    DBuf<int> sdofs, bpos, cbdst, ctoff;  // bpos: pivot position of each boundary dof; cbdst: its slot in the parent's cbuf
    DBuf<unsigned long long> counters;          // [front][-, forward, backward] completed tasks
    DBuf<NdTask> d_tasks;
    std::vector<NdFront> fronts;

    // SPD matrix in host CSR (full symmetric pattern, natural numbering);
    // node_of[dof] groups dofs into graph nodes with coordinates (cx, cy[, cz]).
    void factor(int n, const std::vector<int>& off, const std::vector<int>& idx, const std::vector<double>& val,
                const std::vector<int>& node_of, const std::vector<double>& cx, const std::vector<double>& cy,
                int leaf_dofs, int max_rhs, cudaStream_t st, const std::vector<double>* cz = nullptr);
    // x = A^{-1} b, nrhs <= max_rhs columns at strides ldb / ldx
    void solve(const double* b, long long ldb, double* x, long long ldx, int nrhs, cudaStream_t st);

    // tile-streaming solve (nd_tile.cu, default)
    bool tiles = false;
    int tgrid = 0, tstages = 8, tmax_tasks = 0;
    unsigned tstage_bytes = 32768;
    size_t ttask_bytes = 0, tarena = 0, tsmem = 0;
    double tile_bytes = 0.0;  // bytes of the tile store (the factor plus tile padding)
    DBuf<double> tstore;
    DBuf<NdTileTask> d_ttasks;
    DBuf<int> tctoff, d_toix;
    void build_tiles(const std::vector<std::vector<int>>& children, const std::vector<int>& parent,
                     const std::vector<int>& hs, const std::vector<int>& hbp, const std::vector<int>& hcbdst,
                     cudaStream_t st);
    void solve_tiles(const double* b, long long ldb, double* x, long long ldx, int nrhs, cudaStream_t st);
    // level-synchronous solve (PDG_ND_LEVELS): per level and pass a unit range and its buffer size
    bool levels = false;
    std::string fallback_reason;  // why the chunk kernel's schedule did not fit (levels used instead)
    std::vector<int> lvl_off;
    std::vector<size_t> lvl_smem;
    unsigned lvl_stage_bytes = 0;  // TMA staging region for a unit's tiles
    bool lvl_staged = false;
    int lvl_pf = 1;
    void solve_levels(const double* b, long long ldb, double* x, long long ldx, int nrhs, cudaStream_t st);
    // hybrid (PDG_ND_HYBRID): chunk kernel on the local subtrees (forward, backward schedules),
    // level kernels on the levels 0..hybrid_top in between
    bool hybrid = false;
    int hybrid_top = -1, lvl_max_depth = -1;  // lvl_max_depth >= 0: level units only up to that depth
    DBuf<NdTask> d_tasks_b;
    DBuf<int> ctoff_b;
    void launch_chunks(const NdTask* tasks, const int* cto, const double* b, long long ldb, double* x, long long ldx,
                       int nrhs, cudaStream_t st);
    // dense top (PDG_ND_TOP): the fronts of depth <= top_depth (pivot positions [top0, n)) are
    // not solved front by front; their Schur complement inverse G = S_TT^{-1} (= (A^{-1})_TT)
    // is applied as one GEMV between the forward and backward passes of the fronts below
    int top_depth = -1, ntop = 0, top0 = 0, ldg = 0;
    int lvl_min_depth = 0;       // level kernels for depths lvl_min_depth..lvl_max_depth
    bool split = false;          // two chunk launches (forward, backward) around the top / levels
    DBuf<double> gtop, ctop;     // G (ntop x ldg, row-major), the top right-hand sides [rhs][ldg]
    DBuf<int> top_coff, top_clist;  // per top position: the contribution-buffer entries to subtract
    void build_top(const std::vector<int>& hbp, const std::vector<std::vector<int>>& children,
                   const std::vector<long long>& fo, const double* dense, LaHandles& la, cudaStream_t st);
    void solve_top(const double* b, long long ldb, double* x, long long ldx, int nrhs, cudaStream_t st);
    void solve_levels_range(const double* b, long long ldb, double* x, long long ldx, int nrhs, int l0, int l1,
                            cudaStream_t st);
    // streaming mode (nd_stream.cu): fronts too wide for the shared-memory kernels, or dense
    // fronts too large to hold all at once (3D). Numeric factorization in postorder with one
    // front matrix alive per pending update; one level kernel per depth and pass on the
    // row-major store. PDG_ND_STREAM=1/0 forces / forbids it.
    bool stream = false;
    // fast mode (pdg_gmres_opts.mode 1): the streamed factor stored in fp32 (half the bytes); the
    // factorization and all sums stay fp64. fp32 = fp32_req && stream.
    bool fp32_req = false, fp32 = false;
    DBuf<float> store32;
    std::vector<int> stream_off, stream_rpw;  // per level: first unit, rows per warp (8 | 4 | 2)
    DBuf<NdStreamUnit> d_sunits;
    void build_stream(cudaStream_t st);
    void solve_stream(const double* b, long long ldb, double* x, long long ldx, int nrhs, cudaStream_t st);
    double alg_bytes(int nrhs) const { return factor_bytes + 16.0 * n * nrhs; }
};

}  // namespace pdg
