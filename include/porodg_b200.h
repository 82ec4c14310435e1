/*
 * porodg_b200 -- C ABI of the B200-native (sm_100a) solver for the porodg
 * reference's hot path: the preconditioned GMRES solve of one transformed
 * dG(r)-in-time Biot slab block.
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/proj/include/porodg/):
 *
 *   pdg_ops_upload / pdg_ops_assemble
 *       SpatialOperators produced by assemble_operators  (assembly.hpp:38-52, :177-395)
 *   pdg_block_create
 *       SlabSolver ctor, BlockSolverKind::gmres_fs branch (slab.hpp:154-171):
 *       the shared A factorisation (slab.hpp:155), the block operator
 *       FixedStressSolver(T_gg) and the per-component preconditioner
 *       FixedStressSolver(lambda = T_gg(0,0)) (slab.hpp:161-169)
 *   pdg_block_solve
 *       gmres(op, pre, rhs, opt.gmres) for one diagonal Schur block
 *       (slab.hpp:220-234 -> gmres.hpp:145-150 -> gmres_impl gmres.hpp:40-139)
 *   pdg_block_apply
 *       FixedStressSolver::apply_block -> apply_block_operator (fixed_stress.hpp:38-60,104-106),
 *       evaluated on the canonical assembled space-time operator
 *   pdg_block_precondition
 *       FixedStressSolver::precondition (fixed_stress.hpp:177-181) per time component
 *   pdg_slab_create / pdg_slab_solve
 *       SlabSolver::solve (slab.hpp:179-255): Schur transform, block solve, back-transform
 *   pdg_spmv_csr
 *       SparseMatrix::apply (sparse.hpp:30-40), order-fixed (bit-identical)
 *
 * Conventions: plain pointers and sizes, caller-owned HOST buffers (copied
 * inside the call) unless a function name ends in _device. _device functions
 * run on the context's own non-blocking stream, which no other stream orders:
 * their device inputs must be complete when the call is made (synchronize the
 * stream that produced them), and their outputs are complete when it returns.
 * Every function
 * returns a pdg_status; the message of the last failure on the calling
 * thread is pdg_last_error(). Handles are not thread-safe; destroy order is
 * block/slab -> ops -> ctx.
 */
#ifndef PORODG_B200_H
#define PORODG_B200_H

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PDG_OK = 0,
    PDG_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    PDG_NOT_CONVERGED = 2,    /* SolverError (GMRES budget, singular factor) */
    PDG_CUDA_ERROR = 3,
    PDG_NCCL_ERROR = 4,
    PDG_OUT_OF_MEMORY = 5
} pdg_status;

typedef struct pdg_ctx pdg_ctx;
typedef struct pdg_ops pdg_ops;
typedef struct pdg_block pdg_block;
typedef struct pdg_slab pdg_slab;

/* CSR view (SparseMatrix, sparse.hpp:20-27): int32 offsets and indices. */
typedef struct {
    int rows, cols, nnz;
    const int* row_offsets;  /* rows + 1 */
    const int* col_indices;  /* nnz, strictly increasing per row */
    const double* values;    /* nnz */
} pdg_csr;

/* Structured mesh + material + constant boundary data (mesh.hpp:73,
 * material.hpp:25, boundary.hpp:27-69) for on-device assembly. */
typedef struct {
    int nx, ny;
    double lx, ly;
    double lambda, mu, k_perm, eta, biot_m, biot_b;
    const double* k_perm_cells; /* NULL or nx*ny values, cell c = j*nx + i */
    double penalty;             /* SIPG gamma (problems.hpp:273 default 10) */
    int disp_kind[4];           /* tags left,right,bottom,top: 0 fixed 1 traction 2 roller_x 3 roller_y */
    double disp_data[4][2];     /* constant Dirichlet value / traction vector */
    int flow_kind[4];           /* 0 pressure, 1 no_flow */
    double flow_data[4];        /* constant boundary pressure */
} pdg_problem;

/* 3D extension (BASELINE configs 2 and 4; the reference is 2D only): structured
 * nx x ny x nz mesh of hexahedra with the reference's element pair generalised (discontinuous
 * trilinear SIPG displacement, 24 dofs per cell; one normal-velocity flux dof per face; constant
 * pressure per cell). Cell c = (k ny + j) nx + i; boundary tags xlo, xhi, ylo, yhi, zlo, zhi. */
typedef struct {
    int nx, ny, nz;
    double lx, ly, lz;
    double lambda, mu, k_perm, eta, biot_m, biot_b;
    const double* k_perm_cells; /* NULL or nx*ny*nz values */
    double penalty;
    int disp_kind[6];           /* 0 fixed 1 traction 2 roller_x 3 roller_y 4 roller_z */
    double disp_data[6][3];     /* constant Dirichlet value / traction vector */
    int flow_kind[6];           /* 0 pressure, 1 no_flow */
    double flow_data[6];        /* constant boundary pressure */
} pdg_problem3;

/* GmresOptions (gmres.hpp:24-28) + FixedStressConfig (fixed_stress.hpp:17-22). */
typedef struct {
    double tol;     /* relative true residual, default 1e-10 */
    int restart;    /* default 100 in the reference, 50 in the BASELINE configs */
    int max_iter;   /* default 400 */
    int sweeps;     /* truncated fixed-stress sweeps per preconditioner call, default 1 */
    double stab;    /* < 0: b^2 / K_dr (fixed_stress.hpp:23-27) */
    int candidate;  /* 0: x + P(V y) as gmres.hpp:116 (reference); 1: x + Z y (gmres_flexible, gmres.hpp:113-114) */
    int mode;       /* 0 parity (default): exact fp64 inner solves, as the reference's sparse-direct LU.
                     * 1 fast (SURVEY 8(b) SolveOptions mode): the displacement factor of the streaming
                     * nested-dissection solve (3D meshes) is STORED in fp32 - half the bytes of the
                     * HBM-bound solve; sums stay fp64 and GMRES still iterates to the fp64 true-residual
                     * tolerance, so the solution meets the same acceptance test while the iterates differ
                     * from the reference's at the 1e-7 level of the preconditioner. No effect on 2D. */
} pdg_gmres_opts;

/* SolverReport (gmres.hpp:15-20) plus timings. */
typedef struct {
    int converged;
    int iterations;
    double final_rel_res;
    double* history;   /* caller buffer for the true-residual history, may be NULL */
    int history_cap;
    int history_len;
    double device_ms;  /* device time of the solve (CUDA events on the block's stream) */
    int kernel_launches;
} pdg_report;

const char* pdg_last_error(void);
const char* pdg_version(void);

int pdg_ctx_create(int device, pdg_ctx** out);
/* One context per listed device (pdg_ctx_create(const int* devices, int n, ...)):
 * out[i] is the context of devices[i]. The multi-GPU solve itself is one process (or host
 * thread) per GPU: each binds its context to a pdg_comm (below). On failure nothing is kept. */
int pdg_ctx_create_devices(const int* devices, int n, pdg_ctx** out);
void pdg_ctx_destroy(pdg_ctx* ctx);

/* Structured-mesh dimensions (mesh.hpp:42-60) of reference-assembled operators, from
 * n_p = nx ny, n_q = nx (ny + 1) + ny (nx + 1) and the cell pair of the first interior
 * face row of B (which root is nx). dims = {nx, ny}. */
int pdg_mesh_dims_from_operators(const pdg_csr* B, int n_q, int dims[2]);
/* Upload reference-assembled operators (SpatialOperators) from host CSR.
 * nx = ny = 0: infer the mesh with pdg_mesh_dims_from_operators. */
int pdg_ops_upload(pdg_ctx* ctx, int nx, int ny, const pdg_csr* A, const pdg_csr* M_q, const pdg_csr* B,
                   const pdg_csr* E, const double* m_p_diag, const signed char* q_constrained, double biot_b,
                   double inv_m, double k_dr, pdg_ops** out);
/* Assemble the operators on the device (one thread block per cell / face). */
int pdg_ops_assemble(pdg_ctx* ctx, const pdg_problem* problem, pdg_ops** out);
/* 3D: assemble on the device / upload host CSR blocks of an nx x ny x nz mesh (n_u = 24 n_p;
 * the dimensions locate cells and faces for the nested-dissection orderings). Every handle
 * built on such operators (pdg_block, pdg_slab, pdg_op, pdg_fs for r = 0) works unchanged;
 * strips (pdg_op_set_strip, pdg_dblock) are 2D only. */
int pdg_ops_assemble3(pdg_ctx* ctx, const pdg_problem3* problem, pdg_ops** out);
int pdg_ops_upload3(pdg_ctx* ctx, int nx, int ny, int nz, const pdg_csr* A, const pdg_csr* M_q, const pdg_csr* B,
                    const pdg_csr* E, const double* m_p_diag, const signed char* q_constrained, double biot_b,
                    double inv_m, double k_dr, pdg_ops** out);
/* Sizes: n_u, n_q, n_p, nnz(A), nnz(M_q), nnz(B), nnz(E). */
int pdg_ops_sizes(const pdg_ops* ops, long long sizes[7]);
/* Download block `which` (0 A, 1 M_q, 2 B, 3 E) as CSR into caller buffers. */
int pdg_ops_download(const pdg_ops* ops, int which, int* row_offsets, int* col_indices, double* values);
/* assemble_rhs (assembly.hpp:467-563) for constant boundary data at time t. */
int pdg_ops_rhs(const pdg_ops* ops, double t, double* u, double* q, double* p);
/* assemble_rhs in full (assembly.hpp:467-563): VolumeData (assembly.hpp:24-28) and time- / space-
 * dependent boundary functions (boundary.hpp:12-13). std::function callbacks cannot cross the ABI,
 * so the caller evaluates its fields at the quadrature points for the time t it wants and passes
 * the samples (host arrays); the device accumulates them in the reference's order (bit-identical).
 * Sample points (pdg_rhs_sample_points returns them): per cell c the 6 x 6 Gauss points
 * (x0 + g_i hx, y0 + g_j hy), index c*36 + i*6 + j; per boundary face, in ascending face index
 * (bottom row, top row, left column, right column: 2 nx + 2 ny faces), the 6 Gauss points
 * x0 + g_k (x1 - x0). momentum / darcy / mass may be NULL (absent field, assembly.hpp:485);
 * traction / dirichlet / flow hold eval_or_zero of the face's traction_data, dirichlet_data and
 * flow data (prescribed pressure, or prescribed normal flux on no-flow-kind faces).
 * 3D operators (pdg_ops_assemble3): the same call with 6 x 6 x 6 points per cell, index
 * c*216 + (i*6 + j)*6 + k, vectors of 3 components ([n_cells][216][3], mass [n_cells][216]), and
 * 6 x 6 points per boundary face in ascending face index (first tangential axis outer):
 * [n_bfaces][36][3], flow [n_bfaces][36], n_bfaces = 2 (nx ny + nx nz + ny nz). */
typedef struct {
    const double* momentum;  /* [n_cells][36][2] */
    const double* darcy;     /* [n_cells][36][2] */
    const double* mass;      /* [n_cells][36] */
    const double* traction;  /* [n_bfaces][6][2] */
    const double* dirichlet; /* [n_bfaces][6][2] */
    const double* flow;      /* [n_bfaces][6] */
} pdg_rhs_samples;
/* cell_xy [n_cells][36][2], bface_ids [2 nx + 2 ny], bface_xy [n_bfaces][6][2] (any may be NULL);
 * 3D: [n_cells][216][3], [n_bfaces], [n_bfaces][36][3] */
int pdg_rhs_sample_points(const pdg_ops* ops, double* cell_xy, int* bface_ids, double* bface_xy);
int pdg_ops_rhs_sampled(const pdg_ops* ops, const pdg_rhs_samples* samples, double* u, double* q, double* p);
void pdg_ops_destroy(pdg_ops* ops);

/* One transformed diagonal block: theta is m x m row-major (T_gg), lambda_pre
 * the preconditioner's time weight (T_gg(0,0)). */
int pdg_block_create(pdg_ops* ops, int m, const double* theta, double tau, double lambda_pre,
                     const pdg_gmres_opts* opts, pdg_block** out);
int pdg_block_rows(const pdg_block* blk, long long* rows, long long* nnz);
/* x = GMRES solution of (Theta (x) D + tau K) x = rhs. Host buffers of m * n_total doubles. */
int pdg_block_solve(pdg_block* blk, const double* rhs, double* x, pdg_report* rep);
/* Same with device pointers (no host copies). */
int pdg_block_solve_device(pdg_block* blk, const double* rhs_dev, double* x_dev, pdg_report* rep);
/* y = op(x); mode 0: order-fixed canonical operator (bit-defined). */
int pdg_block_apply(pdg_block* blk, int mode, const double* x, double* y);
int pdg_block_apply_device(pdg_block* blk, int mode, const double* x_dev, double* y_dev, int repeats, float* ms);
/* z = precondition(r) for all m components (slab.hpp:221-226). */
int pdg_block_precondition(pdg_block* blk, const double* r, double* z);
/* Download the canonical space-time CSR (rows+1 offsets as int64). */
int pdg_block_download_csr(const pdg_block* blk, long long* row_offsets, int* col_indices, double* values);
void pdg_block_destroy(pdg_block* blk);

/* The canonical space-time operator alone (no preconditioner / factorisation):
 * the object of the SpMV bandwidth sweep (BASELINE config 3). */
typedef struct pdg_op pdg_op;
int pdg_op_create(pdg_ops* ops, int m, const double* theta, double tau, pdg_op** out);
int pdg_op_rows(const pdg_op* op, long long* rows, long long* nnz);
/* y = op(x) `repeats` times on device buffers; per-launch times (ms) into times_ms[repeats] if not NULL. */
int pdg_op_apply_device(pdg_op* op, const double* x_dev, double* y_dev, int repeats, float* times_ms);
int pdg_op_download_csr(const pdg_op* op, long long* row_offsets, int* col_indices, double* values);
/* Multi-GPU row partitioning: this rank owns the strip of cell rows
 * [r0, r1) of the nx x ny mesh (u and p rows of its cells, q rows of its face rows:
 * horizontal faces of level j belong to row min(j, ny-1), vertical faces to their
 * row). apply_strip writes only the owned rows of y; x must hold the owned entries
 * and the one-cell-row halo (global numbering). Bit-identical per row to apply. */
int pdg_op_set_strip(pdg_op* op, int nx, int ny, int r0, int r1);
int pdg_op_apply_strip_device(pdg_op* op, const double* x_dev, double* y_dev, int repeats, float* times_ms);
void pdg_op_destroy(pdg_op* op);

/* Per-phase device timing (CUDA events on the library stream). Phases:
 * 0 space-time SpMV, 1 displacement solve, 2 flow solve, 3 other preconditioner
 * kernels, 4 Krylov vector kernels, 5 slab transforms / rhs. alg_bytes is the
 * algorithmic traffic summed over the calls. */
/* ---- Multi-GPU: one process per GPU, strips of cell rows ----
 * A communicator per rank: NCCL (rank 0 creates the id with pdg_nccl_unique_id and the
 * caller distributes it, e.g. by torch.distributed or MPI), or host-staged collectives
 * through caller callbacks (blocking; tests with several ranks on one GPU). The
 * distributed block is the transformed slab block of pdg_block_create (slab.hpp:154-171,
 * :220-234) with its rows owned by strips: every rank passes the whole operators (ops)
 * and its rows of the right-hand side; pdg_dblock_owned_rows gives their global indices. */
typedef struct pdg_comm pdg_comm;
typedef struct pdg_dblock pdg_dblock;
/* recv[r * count + j] = (send of rank r)[j]; return 0 on success */
typedef int (*pdg_host_allgather_fn)(void* user, const double* send, double* recv, long long count);
/* to peers[i]: send[i] (scount[i] doubles); from peers[i]: recv[i] (rcount[i]); 0 on success */
typedef int (*pdg_host_exchange_fn)(void* user, int npeers, const int* peers, const double* const* send,
                                    const long long* scount, double* const* recv, const long long* rcount);
int pdg_nccl_unique_id(unsigned char id[128]);
int pdg_comm_create_nccl(pdg_ctx* ctx, int nranks, int rank, const unsigned char id[128], pdg_comm** out);
int pdg_comm_create_host(pdg_ctx* ctx, int nranks, int rank, pdg_host_allgather_fn allgather,
                         pdg_host_exchange_fn exchange, void* user, pdg_comm** out);
void pdg_comm_destroy(pdg_comm* comm);
int pdg_dblock_create(pdg_ops* ops, pdg_comm* comm, int m, const double* theta_mxm, double tau, double lambda_pre,
                      const pdg_gmres_opts* opts, pdg_dblock** out);
/* rows owned here and rows of the whole block (m * n_total) */
int pdg_dblock_rows(const pdg_dblock* blk, long long* n_owned, long long* n_global);
int pdg_dblock_owned_rows(const pdg_dblock* blk, long long* rows);
/* GMRES across the ranks (collective: every rank calls it), owned rows, device pointers */
int pdg_dblock_solve_device(pdg_dblock* blk, const double* rhs_owned, double* x_owned, pdg_report* rep);
/* the operator rows and the preconditioner (collective), owned rows, device pointers */
int pdg_dblock_apply_device(pdg_dblock* blk, const double* x_owned, double* y_owned);
int pdg_dblock_precondition_device(pdg_dblock* blk, const double* r_owned, double* z_owned);
void pdg_dblock_destroy(pdg_dblock* blk);

/* Setup stage timers, cumulative seconds since pdg_setup_reset: [0] device assembly,
 * [1..3] displacement nested-dissection analysis / numeric factorization / solve schedule,
 * [4..6] the same for the flow Schur complement, [7] space-time operator build,
 * [8] whole block/slab solver construction (includes 1..7 when built there).
 * Writes min(n, 9) values and returns 9. */
void pdg_setup_reset(void);
int pdg_setup_read(double* seconds, int n);
void pdg_profile_enable(int on);
void pdg_profile_reset(void);
int pdg_profile_read(int phase, double* ms, long long* calls, double* alg_bytes);

/* Diagnostics: run one preconditioner application of `blk` with per-step
 * %globaltimer stamps in the last recurrence of solver `which` (0 displacement,
 * 1 flow); out[(cta * nsteps + step) * 4 + phase] (ns), phases: step start,
 * sources gathered, rows stored, streamed rows ready (0 when not recorded).
 * *ctas / *nsteps receive the shape. */
int pdg_debug_recurrence_timing(pdg_block* blk, int which, unsigned long long* out, long long cap, int* ctas,
                                int* nsteps);

/* Slab solver for dG(r), 0 <= r <= 5 (SlabSolver, slab.hpp:133-274): one block solver per
 * diagonal block of the ordered real Schur form (1x1: a real eigenvalue, 2x2: a standardized
 * complex pair), sharing the displacement factorisation (slab.hpp:155); solve() transforms,
 * back-substitutes through the T_ij D y_j couplings in descending block order
 * (slab.hpp:194-203), solves each block by preconditioned GMRES and transforms back. The
 * report handed back is that of the block with the most iterations (final_rel_res the maximum
 * over the blocks, device time and launches summed); pdg_slab_block_reports gives every
 * block's iterations and final relative residual of the last solve (BlockReport, slab.hpp:113-119).
 * Non-convergence: PDG_NOT_CONVERGED with "slab block g: GMRES did not converge (rel res ...)". */
int pdg_slab_create(pdg_ops* ops, int r, double tau, const pdg_gmres_opts* opts, pdg_slab** out);
int pdg_slab_block_reports(const pdg_slab* slab, int* n_blocks, int* block_sizes, int* iterations,
                           double* final_rel_res);
/* rhs: (r+1) * n_total stacked per Radau node (SlabSystem::rhs); out: (r+1) * n_total solution comps. */
int pdg_slab_solve(pdg_slab* slab, const double* rhs, double* out, pdg_report* rep);
int pdg_slab_solve_device(pdg_slab* slab, const double* rhs_dev, double* out_dev, pdg_report* rep);
/* Slab right-hand side (build_slab_system, slab.hpp:58-87) on the device: jump data u_prev/p_prev
 * (device), slab start t0 and length tau (the slab's own length, march.hpp:63-64; it may differ in
 * the last bits from the tau the solver was built with, as in the reference) -> rhs_dev
 * ((r+1) * n_total). */
int pdg_slab_rhs_device(pdg_slab* slab, double t0, double tau, const double* u_prev_dev, const double* p_prev_dev,
                        double* rhs_dev);
/* One step of the march's slab loop on the device (march.hpp:62-79 for the monolithic-spectral
 * branch): build_slab_system for [t0, t0 + tau] from the previous end trace prev_state_dev
 * ([u q p], n_total doubles; NULL = zero initial data) and solve it into out_dev ((r+1) n_total),
 * with ONE synchronization at the end. prev_state_dev must not alias out_dev (use two output
 * buffers alternately and pass the last component of the previous one). Constant boundary data. */
int pdg_slab_step_device(pdg_slab* slab, double t0, double tau, const double* prev_state_dev, double* out_dev,
                         pdg_report* rep);
/* The same with sampled data: samples[i] holds the fields at the slab's Radau node i,
 * t = t0 + nodes[i] * tau (r + 1 entries; pdg_time_constants gives the nodes). */
int pdg_slab_rhs_sampled_device(pdg_slab* slab, double tau, const pdg_rhs_samples* samples, const double* u_prev_dev,
                                const double* p_prev_dev, double* rhs_dev);
void pdg_slab_destroy(pdg_slab* slab);

/* Order-fixed CSR SpMV (SparseMatrix::apply) on device buffers. */
int pdg_spmv_csr_device(int rows, const long long* row_offsets_dev, const int* col_indices_dev,
                        const double* values_dev, const double* x_dev, double* y_dev);

/* dG(r) time constants, 0 <= r <= 5 (time_matrices + real_schur, time_basis.hpp:135-182,
 * schur.hpp:101-173): nodes, weights, phi(0) [r+1], T and Q [(r+1)^2 row-major]; blocks of T
 * ordered by ascending (Re, |Im|) of their eigenvalues, 2x2 blocks standardized. */
/* Fixed-stress solver of the fixed-stress march (FixedStressSolver::solve,
 * fixed_stress.hpp:144-172, as built at march.hpp:83-84: Theta = G_hat, kappa =
 * the Radau weights): sweeps on the untransformed slab block from x0 (null =
 * zero) until ||rhs - A x|| <= tol ||rhs||; rep->iterations = sweeps
 * (BlockReport::fs_sweeps). Fails with PDG_NOT_CONVERGED and the reference's
 * text "fixed-stress did not converge (rel res ...)". Device path: dG(0). */
typedef struct pdg_fs pdg_fs;
typedef struct {
    double tol;     /* FixedStressConfig::tol (default 1e-10) */
    int max_sweeps; /* FixedStressConfig::max_sweeps (default 200) */
    double stab;    /* < 0: b^2 / K_dr */
} pdg_fs_opts;
int pdg_fs_create(pdg_ops* ops, int r, double tau, const pdg_fs_opts* opts, pdg_fs** out);
/* rhs, x0, x: (r+1) * n_total stacked per Radau node (host buffers / device pointers) */
int pdg_fs_solve(pdg_fs* fs, const double* rhs, const double* x0, double* x, pdg_report* rep);
int pdg_fs_solve_device(pdg_fs* fs, const double* rhs_dev, const double* x0_dev, double* x_dev, pdg_report* rep);
void pdg_fs_destroy(pdg_fs* fs);

/* Exact SPD block-tridiagonal solver (the inner solves of the fixed-stress
 * preconditioner, fixed_stress.hpp:109-139) for a host CSR that is block
 * tridiagonal under the symmetric permutation perm (new -> old; NULL =
 * identity) with the given block sizes. allow_local (flags): bit 0 = use the
 * chunk-local sweep when the couplings are 8x8 cell-local; bit 1 = the matrix is
 * NOT symmetric (twisted block LU with in-block partial pivoting instead of
 * Cholesky; no pivoting across blocks). solve: nrhs <= 2 columns of n doubles
 * (device pointers, contiguous). Used for the strip interiors of the multi-GPU
 * substructured solve. */
typedef struct pdg_tri pdg_tri;
int pdg_tri_create(pdg_ctx* ctx, const pdg_csr* A, const int* perm, const int* block_sizes, int nblocks,
                   int allow_local, pdg_tri** out);
int pdg_tri_solve_device(pdg_tri* t, const double* b_dev, double* x_dev, int nrhs);
void pdg_tri_destroy(pdg_tri* t);

/* local_mass_residual (slab.hpp:292-318): the discrete per-cell mass balance of
 * one slab. rhs and state are (r+1)*n_total doubles stacked per Radau node
 * (the slab system right-hand side and its solution, [u q p] per node);
 * residual receives |residual| per cell (n_p), *scale the maximum over cells of
 * the summed constituent magnitudes. Bit-identical to the reference's arithmetic.
 * pdg_mass_residual takes host buffers, the _device variant device pointers
 * (*scale is always a host pointer). */
int pdg_mass_residual(pdg_ops* ops, int r, double tau, const double* rhs, const double* state, double* residual,
                      double* scale);
int pdg_mass_residual_device(pdg_ops* ops, int r, double tau, const double* rhs_dev, const double* state_dev,
                             double* residual_dev, double* scale);

int pdg_time_constants(int r, double* nodes, double* weights, double* phi0, double* T, double* Q);
/* The diagonal blocks of T (sizes 1 | 2, first rows; up to r + 1 entries) and G_hat [(r+1)^2]
 * (any output may be NULL except n_blocks). */
int pdg_time_schur_blocks(int r, int* n_blocks, int* block_sizes, int* block_starts, double* G_hat);

/* Seeded workload generators (Inputs). */
void pdg_util_uniform(unsigned long long seed, long long n, double* out);
void pdg_util_lognormal(unsigned long long seed, long long n, double sigma, double* out);
/* Number of library kernel launches issued on the calling thread so far. */
long long pdg_util_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif
