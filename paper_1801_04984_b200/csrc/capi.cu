// C ABI of porodg_b200 (include/porodg_b200.h).
#include <cstdio>
#include <cstring>
#include <random>

#include "block.cuh"
#include "dist.cuh"
#include "timebasis.hpp"

namespace pdg {
thread_local long long g_launches = 0;
static thread_local std::string g_err;
}  // namespace pdg

using namespace pdg;

struct pdg_ctx {
    Ctx c;
};
struct pdg_ops {
    SpatialOps s;
    std::shared_ptr<ASolver> a;  // shared displacement factorisation (slab.hpp:155)
    std::shared_ptr<ASolver> a_fast;  // the same with the fp32-stored factor (pdg_gmres_opts.mode 1)
};
struct pdg_block {
    Block b;
    DBuf<double> io_a, io_b;
};
struct pdg_op {
    Ctx* ctx = nullptr;
    SpaceTimeOp op;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
};
struct pdg_tri {
    Ctx* ctx = nullptr;
    DCsr A;
    BlockTriChol chol;
};
struct pdg_fs {
    pdg_ops* ops = nullptr;
    FsSolver fs;
    pdg_fs_opts opts{};
    DBuf<double> io_a, io_b, io_c;
};
struct pdg_comm {
    std::unique_ptr<Comm> c;
};
struct pdg_dblock {
    DistBlock b;
};
struct pdg_slab {
    pdg_ops* ops = nullptr;
    TimeConsts tc;
    double tau = 0;
    // one solver per diagonal Schur block (slab.hpp:154-171), solved in descending order with the
    // T_ij D y_j couplings of the blocks above (slab.hpp:194-203); r <= 1: a single block
    std::vector<std::unique_ptr<pdg_block>> blks;
    std::vector<int> blk_iterations;        // per block, last solve (BlockReport::gmres_iterations)
    std::vector<double> blk_final_rel_res;  // per block, last solve
    DBuf<double> d_Q, d_w, d_phi0, shat, ysol, io_a, io_b, rhs_u, rhs_q, rhs_p, djump, et_u;
    DBuf<double> dpt;  // D y_j (p rows) of the solved components, n x n_p
    DBuf<double> d_T;  // the Schur form's T on the device (back-substitution couplings)
    DBuf<double> zero_state;  // n_total zeros: the initial data of pdg_slab_step_device(prev = NULL)
    bool rhs_const = false;   // rhs_u / rhs_q / rhs_p hold b(t) of the problem's constant boundary data (time-independent)
};

#define API_BEGIN try {
#define API_END                                 \
    }                                           \
    catch (const pdg::Error& e) {               \
        g_err = e.what();                       \
        return e.status;                        \
    }                                           \
    catch (const std::bad_alloc& e) {           \
        g_err = e.what();                       \
        return PDG_OUT_OF_MEMORY;               \
    }                                           \
    catch (const std::exception& e) {           \
        g_err = e.what();                       \
        return PDG_INVALID_ARGUMENT;            \
    }                                           \
    return PDG_OK;

namespace {

inline double bits_to_double(unsigned long long b) {
    double d;
    std::memcpy(&d, &b, sizeof d);
    return d;
}


__global__ void k_schur_fwd(int nn, long long nt, const double* Q, const double* w, const double* R, double* shat) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nn * nt; t += (long long)gridDim.x * blockDim.x) {
        const int i = static_cast<int>(t / nt);
        const long long k = t % nt;
        double s = 0.0;
        for (int j = 0; j < nn; ++j) s += Q[j * nn + i] * (R[j * nt + k] / w[j]);
        shat[t] = s;
    }
}
__global__ void k_schur_bwd(int nn, long long nt, const double* Q, const double* y, double* X) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nn * nt; t += (long long)gridDim.x * blockDim.x) {
        const int i = static_cast<int>(t / nt);
        const long long k = t % nt;
        double s = 0.0;
        for (int j = 0; j < nn; ++j) s += Q[i * nn + j] * y[j * nt + k];
        X[t] = s;
    }
}
// djump = (-b) E^T u - (1/M) (m_p p)   (assembly.hpp:409-413)
// D(u,p)_c = (-b) (E^T u)_c - (1/M) (m_p,c p_c)   (assembly.hpp:409-413); E^T u summed
// in ascending row order of E from 0.0 like SparseMatrix::apply_transpose
// (sparse.hpp:43-50), no FMA: bit-identical to the reference's arithmetic.
__device__ __forceinline__ double time_derivative_p(int c, double mb, double im, const int* et_off, const int* et_idx,
                                                    const double* et_val, const double* m_p, const double* u,
                                                    const double* p) {
    double s = 0.0;
    for (int k = et_off[c]; k < et_off[c + 1]; ++k) s = __dadd_rn(s, __dmul_rn(et_val[k], u[et_idx[k]]));
    return __dsub_rn(__dmul_rn(mb, s), __dmul_rn(im, __dmul_rn(m_p[c], p[c])));
}
// 8 lanes per cell: the lanes load the products e_k u_k of the cell's E^T row in parallel, lane 0
// adds them in ascending k (the sequential sum of apply_transpose, same bits as one thread)
__global__ void k_time_derivative(int np, double mb, double im, const int* et_off, const int* et_idx, const double* et_val,
                                  const double* m_p, const double* u, const double* p, double* out) {
    const int sub = threadIdx.x & 7;
    const unsigned gmask = 0xffu << (threadIdx.x & 24);
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < 8LL * ((np + 3) / 4 * 4);
         t += (long long)gridDim.x * blockDim.x) {
        const int c = static_cast<int>(t >> 3);
        const bool live = c < np;
        const int b = live ? et_off[c] : 0, e = live ? et_off[c + 1] : 0;
        double s = 0.0;
        for (int k0 = b; __any_sync(gmask, k0 < e); k0 += 8) {
            const int k = k0 + sub;
            const double prod = k < e ? __dmul_rn(et_val[k], u[et_idx[k]]) : 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const double v = __shfl_sync(gmask, prod, (threadIdx.x & 24) + q);
                if (k0 + q < e) s = __dadd_rn(s, v);
            }
        }
        if (live && sub == 0) out[c] = __dsub_rn(__dmul_rn(mb, s), __dmul_rn(im, __dmul_rn(m_p[c], p[c])));
    }
}
// R_i = (tau w_i) [u;q;p]_i + phi0_i djump (p rows)   (slab.hpp:76-84)
__global__ void k_slab_rhs(int nn, int nu, int nq, int np, double tau, const double* w, const double* phi0,
                           const double* ru, const double* rq, const double* rp, const double* djump, double* R) {
    const long long nt = (long long)nu + nq + np;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nn * nt; t += (long long)gridDim.x * blockDim.x) {
        const int i = static_cast<int>(t / nt);
        const long long k = t % nt;
        const double s = __dmul_rn(tau, w[i]);
        double v;
        if (k < nu)
            v = __dmul_rn(s, ru[(long long)i * nu + k]);
        else if (k < nu + nq)
            v = __dmul_rn(s, rq[(long long)i * nq + (k - nu)]);
        else
            v = __dadd_rn(__dmul_rn(s, rp[(long long)i * np + (k - nu - nq)]), __dmul_rn(phi0[i], djump[k - nu - nq]));
        R[t] = v;
    }
}

// local_mass_residual (slab.hpp:292-318), one thread per cell: for each time
// test function i, storage = sum_j G(i,j) D(u_j,p_j) (j ascending, zero entries
// skipped), flux = (tau w_i) (B^T q_i), src = p-rows of rhs_i;
// res += (storage + flux) - src, scale += (|storage| + |flux|) + |src|.
// Writes |res| per cell; the scale maximum is an order-free atomic max on the
// (non-negative) double bits. Same operation order as the reference, no FMA.
constexpr int kMaxNodes = kMaxTimeDegree + 1;
__global__ void k_mass_residual(int np, int nu, int nq, int n, const double* __restrict__ G, const double* __restrict__ w,
                                double tau, double mb, double im, const double* __restrict__ m_p, const int* et_off,
                                const int* et_idx, const double* et_val, const int* bt_off, const int* bt_idx,
                                const double* bt_val, const double* __restrict__ rhs, const double* __restrict__ state,
                                double* __restrict__ residual, unsigned long long* scale_bits) {
    const long long nt = (long long)nu + nq + np;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < np; c += gridDim.x * blockDim.x) {
        double dp[kMaxNodes], kp[kMaxNodes];
        for (int j = 0; j < n; ++j) {
            const double* x = state + j * nt;
            dp[j] = time_derivative_p(c, mb, im, et_off, et_idx, et_val, m_p, x, x + nu + nq);
            double s = 0.0;
            for (int k = bt_off[c]; k < bt_off[c + 1]; ++k) s = __dadd_rn(s, __dmul_rn(bt_val[k], x[nu + bt_idx[k]]));
            kp[j] = s;
        }
        double res = 0.0, sc = 0.0;
        for (int i = 0; i < n; ++i) {
            double storage = 0.0;
            for (int j = 0; j < n; ++j) {
                const double g = G[i * n + j];
                if (g != 0.0) storage = __dadd_rn(storage, __dmul_rn(g, dp[j]));
            }
            const double flux = __dmul_rn(__dmul_rn(tau, w[i]), kp[i]);
            const double src = rhs[i * nt + nu + nq + c];
            res = __dadd_rn(res, __dsub_rn(__dadd_rn(storage, flux), src));
            sc = __dadd_rn(sc, __dadd_rn(__dadd_rn(fabs(storage), fabs(flux)), fabs(src)));
        }
        residual[c] = fabs(res);
        atomicMax(scale_bits, static_cast<unsigned long long>(__double_as_longlong(sc)));
    }
}

// rhs_i (p rows) -= sum_{j >= j0} T(i, j) D y_j for the rows i of one Schur block (slab.hpp:197-200)
__global__ void k_schur_backsub(int np, int n, int i0, int m, int j0, const double* __restrict__ T,
                                const double* __restrict__ dp, long long nt, long long poff, double* shat) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * np;
         t += (long long)gridDim.x * blockDim.x) {
        const int bi = static_cast<int>(t / np), c = static_cast<int>(t % np);
        double r = shat[(i0 + bi) * nt + poff + c];
        for (int j = j0; j < n; ++j) {
            const double tij = T[(i0 + bi) * n + j];
            if (tij != 0.0) r = __dsub_rn(r, __dmul_rn(tij, dp[(long long)j * np + c]));
        }
        shat[(i0 + bi) * nt + poff + c] = r;
    }
}

void finish_ops(SpatialOps& s, cudaStream_t st) {
    csr_transpose(s.E, s.Et, st);
    csr_transpose(s.B, s.Bt, st);
}

}  // namespace

extern "C" {

const char* pdg_last_error(void) { return g_err.c_str(); }
const char* pdg_version(void) { return "porodg_b200 0.1 (sm_100a)"; }

int pdg_ctx_create(int device, pdg_ctx** out) {
    API_BEGIN
    require(out != nullptr, "pdg_ctx_create: null out");
    int n = 0;
    PDG_CUDA(cudaGetDeviceCount(&n));
    require(device >= 0 && device < n, "pdg_ctx_create: bad device index");
    PDG_CUDA(cudaSetDevice(device));
    auto c = std::make_unique<pdg_ctx>();
    c->c.device = device;
    PDG_CUDA(cudaStreamCreateWithFlags(&c->c.stream, cudaStreamNonBlocking));
    *out = c.release();
    API_END
}

void pdg_ctx_destroy(pdg_ctx* ctx) {
    if (!ctx) return;
    if (ctx->c.stream) cudaStreamDestroy(ctx->c.stream);
    delete ctx;
}

int pdg_nccl_unique_id(unsigned char id[128]) {
    API_BEGIN
    require(id != nullptr, "pdg_nccl_unique_id: null argument");
    nccl_unique_id(id);
    API_END
}

int pdg_comm_create_nccl(pdg_ctx* ctx, int nranks, int rank, const unsigned char id[128], pdg_comm** out) {
    API_BEGIN
    require(ctx && id && out, "pdg_comm_create_nccl: null argument");
    auto c = std::make_unique<pdg_comm>();
    c->c = make_nccl_comm(nranks, rank, id, ctx->c.device);
    *out = c.release();
    API_END
}

int pdg_comm_create_host(pdg_ctx* ctx, int nranks, int rank, pdg_host_allgather_fn allgather,
                         pdg_host_exchange_fn exchange, void* user, pdg_comm** out) {
    API_BEGIN
    require(ctx && out, "pdg_comm_create_host: null argument");
    auto c = std::make_unique<pdg_comm>();
    c->c = make_host_comm(nranks, rank, allgather, exchange, user);
    *out = c.release();
    API_END
}

void pdg_comm_destroy(pdg_comm* comm) { delete comm; }

int pdg_dblock_create(pdg_ops* ops, pdg_comm* comm, int m, const double* theta, double tau, double lambda_pre,
                      const pdg_gmres_opts* opts, pdg_dblock** out) {
    API_BEGIN
    require(ops && comm && theta && opts && out, "pdg_dblock_create: null argument");
    PDG_CUDA(cudaSetDevice(ops->s.ctx->device));
    auto b = std::make_unique<pdg_dblock>();
    b->b.create(ops->s, comm->c.get(), m, theta, tau, lambda_pre, *opts, ops->s.ctx->stream);
    *out = b.release();
    API_END
}

int pdg_dblock_rows(const pdg_dblock* blk, long long* n_owned, long long* n_global) {
    API_BEGIN
    require(blk && n_owned && n_global, "pdg_dblock_rows: null argument");
    *n_owned = blk->b.nown;
    *n_global = blk->b.nglob;
    API_END
}

int pdg_dblock_owned_rows(const pdg_dblock* blk, long long* rows) {
    API_BEGIN
    require(blk && rows, "pdg_dblock_owned_rows: null argument");
    std::copy(blk->b.own_rows_h.begin(), blk->b.own_rows_h.end(), rows);
    API_END
}

int pdg_dblock_solve_device(pdg_dblock* blk, const double* rhs, double* x, pdg_report* rep) {
    API_BEGIN
    require(blk && rhs && x, "pdg_dblock_solve_device: null argument");
    blk->b.solve(rhs, x, rep);
    PDG_CUDA(cudaStreamSynchronize(blk->b.ctx->stream));
    API_END
}

int pdg_dblock_apply_device(pdg_dblock* blk, const double* x, double* y) {
    API_BEGIN
    require(blk && x && y, "pdg_dblock_apply_device: null argument");
    blk->b.apply(x, y, blk->b.ctx->stream);
    PDG_CUDA(cudaStreamSynchronize(blk->b.ctx->stream));
    API_END
}

int pdg_dblock_precondition_device(pdg_dblock* blk, const double* r, double* z) {
    API_BEGIN
    require(blk && r && z, "pdg_dblock_precondition_device: null argument");
    blk->b.precondition(r, z, blk->b.ctx->stream);
    PDG_CUDA(cudaStreamSynchronize(blk->b.ctx->stream));
    API_END
}

void pdg_dblock_destroy(pdg_dblock* blk) { delete blk; }

int pdg_mesh_dims_from_operators(const pdg_csr* B, int n_q, int dims[2]) {
    API_BEGIN
    require(B && dims, "pdg_mesh_dims_from_operators: null argument");
    require(B->rows == n_q && B->cols > 0, "pdg_mesh_dims_from_operators: B must be n_q x n_p");
    // n_p = nx ny and n_q = nx (ny + 1) + ny (nx + 1), so nx + ny = n_q - 2 n_p and nx, ny are
    // the roots of t^2 - (nx + ny) t + nx ny
    const long long np = B->cols, s = (long long)n_q - 2 * np;
    require(s >= 2 && s * s >= 4 * np, "pdg_mesh_dims_from_operators: sizes do not fit a structured mesh");
    long long d = (long long)std::llround(std::sqrt((double)(s * s - 4 * np)));
    while (d * d > s * s - 4 * np) --d;
    while ((d + 1) * (d + 1) <= s * s - 4 * np) ++d;
    require(d * d == s * s - 4 * np && (s + d) % 2 == 0, "pdg_mesh_dims_from_operators: sizes do not fit a structured mesh");
    const int a = (int)((s + d) / 2), b = (int)((s - d) / 2);
    require(a >= 1 && b >= 1 && (long long)a * b == np, "pdg_mesh_dims_from_operators: sizes do not fit a structured mesh");
    // interior face rows of B hold exactly the two adjacent cells (no-flux rows only sit on the
    // boundary): the first interior horizontal face (j = 1, i = 0) is face nx with cells {0, nx};
    // with ny = 1 the first interior vertical face (i = 1, j = 0) is face 2 nx + 1 with cells {0, 1}
    auto fits = [&](int nx, int ny) {
        int face, c1;
        if (ny >= 2) {
            face = nx;
            c1 = nx;
        } else if (nx >= 2) {
            face = nx * (ny + 1) + ny;
            c1 = 1;
        } else {
            return true;  // 1 x 1
        }
        if (face >= B->rows) return false;
        const long long o0 = B->row_offsets[face], o1 = B->row_offsets[face + 1];
        return o1 - o0 == 2 && B->col_indices[o0] == 0 && B->col_indices[o0 + 1] == c1;
    };
    const bool fa = fits(a, b), fb = fits(b, a);
    require(fa || fb, "pdg_mesh_dims_from_operators: B does not match a structured mesh numbering");
    dims[0] = fa ? a : b;
    dims[1] = fa ? b : a;
    API_END
}

int pdg_ctx_create_devices(const int* devices, int n, pdg_ctx** out) {
    API_BEGIN
    require(devices && out && n >= 1, "pdg_ctx_create_devices: bad arguments");
    for (int i = 0; i < n; ++i) out[i] = nullptr;
    for (int i = 0; i < n; ++i) {
        const int rc = pdg_ctx_create(devices[i], &out[i]);
        if (rc != PDG_OK) {
            for (int j = 0; j < i; ++j) {
                pdg_ctx_destroy(out[j]);
                out[j] = nullptr;
            }
            return rc;
        }
    }
    API_END
}

int pdg_ops_upload(pdg_ctx* ctx, int nx, int ny, const pdg_csr* A, const pdg_csr* M_q, const pdg_csr* B, const pdg_csr* E,
                   const double* m_p_diag, const signed char* q_constrained, double biot_b, double inv_m, double k_dr,
                   pdg_ops** out) {
    API_BEGIN
    require(ctx && A && M_q && B && E && m_p_diag && out, "pdg_ops_upload: null argument");
    if (nx <= 0 && ny <= 0) {  // infer the structured mesh from the operators (mesh.hpp:42-60)
        int dims[2];
        const int rc = pdg_mesh_dims_from_operators(B, M_q->rows, dims);
        if (rc != PDG_OK) return rc;
        nx = dims[0];
        ny = dims[1];
    }
    require(nx > 0 && ny > 0, "pdg_ops_upload: mesh dimensions must be positive");
    PDG_CUDA(cudaSetDevice(ctx->c.device));
    cudaStream_t st = ctx->c.stream;
    auto o = std::make_unique<pdg_ops>();
    SpatialOps& s = o->s;
    s.ctx = &ctx->c;
    s.nx = nx;
    s.ny = ny;
    s.n_u = A->rows;
    s.n_q = M_q->rows;
    s.n_p = B->cols;
    require(A->cols == s.n_u && E->rows == s.n_u && E->cols == s.n_p && B->rows == s.n_q && M_q->cols == s.n_q,
            "pdg_ops_upload: block dimensions are inconsistent");
    require(s.n_u == 8 * nx * ny && s.n_p == nx * ny, "pdg_ops_upload: sizes do not match an nx x ny mesh");
    s.biot_b = biot_b;
    s.inv_m = inv_m;
    s.k_dr = k_dr;
    csr_upload(s.A, *A, st);
    csr_upload(s.M_q, *M_q, st);
    csr_upload(s.B, *B, st);
    csr_upload(s.E, *E, st);
    s.m_p.upload(m_p_diag, s.n_p, st);
    s.q_constrained.alloc(s.n_q);
    if (q_constrained) s.q_constrained.upload(q_constrained, s.n_q, st);
    finish_ops(s, st);
    *out = o.release();
    API_END
}

int pdg_ops_assemble(pdg_ctx* ctx, const pdg_problem* problem, pdg_ops** out) {
    API_BEGIN
    require(ctx && problem && out, "pdg_ops_assemble: null argument");
    PDG_CUDA(cudaSetDevice(ctx->c.device));
    cudaStream_t st = ctx->c.stream;
    auto o = std::make_unique<pdg_ops>();
    o->s.ctx = &ctx->c;
    SetupTimer timer(SETUP_ASSEMBLE, st);
    assemble_ops_device(o->s, *problem, st);
    finish_ops(o->s, st);
    *out = o.release();
    API_END
}

int pdg_ops_assemble3(pdg_ctx* ctx, const pdg_problem3* problem, pdg_ops** out) {
    API_BEGIN
    require(ctx && problem && out, "pdg_ops_assemble3: null argument");
    PDG_CUDA(cudaSetDevice(ctx->c.device));
    cudaStream_t st = ctx->c.stream;
    auto o = std::make_unique<pdg_ops>();
    o->s.ctx = &ctx->c;
    SetupTimer timer(SETUP_ASSEMBLE, st);
    assemble_ops_device3(o->s, *problem, st);
    finish_ops(o->s, st);
    *out = o.release();
    API_END
}

int pdg_ops_upload3(pdg_ctx* ctx, int nx, int ny, int nz, const pdg_csr* A, const pdg_csr* M_q, const pdg_csr* B,
                    const pdg_csr* E, const double* m_p_diag, const signed char* q_constrained, double biot_b,
                    double inv_m, double k_dr, pdg_ops** out) {
    API_BEGIN
    require(ctx && A && M_q && B && E && m_p_diag && out, "pdg_ops_upload3: null argument");
    require(nx > 0 && ny > 0 && nz > 0, "pdg_ops_upload3: mesh dimensions must be positive");
    PDG_CUDA(cudaSetDevice(ctx->c.device));
    cudaStream_t st = ctx->c.stream;
    auto o = std::make_unique<pdg_ops>();
    SpatialOps& s = o->s;
    s.ctx = &ctx->c;
    s.nx = nx;
    s.ny = ny;
    s.nz = nz;
    s.n_u = A->rows;
    s.n_q = M_q->rows;
    s.n_p = B->cols;
    require(A->cols == s.n_u && E->rows == s.n_u && E->cols == s.n_p && B->rows == s.n_q && M_q->cols == s.n_q,
            "pdg_ops_upload3: block dimensions are inconsistent");
    const long long nc = (long long)nx * ny * nz;
    require(s.n_u == 24 * nc && s.n_p == nc &&
                s.n_q == (long long)nx * ny * (nz + 1) + (long long)nx * (ny + 1) * nz + (long long)(nx + 1) * ny * nz,
            "pdg_ops_upload3: sizes do not match an nx x ny x nz mesh");
    s.biot_b = biot_b;
    s.inv_m = inv_m;
    s.k_dr = k_dr;
    csr_upload(s.A, *A, st);
    csr_upload(s.M_q, *M_q, st);
    csr_upload(s.B, *B, st);
    csr_upload(s.E, *E, st);
    s.m_p.upload(m_p_diag, s.n_p, st);
    s.q_constrained.alloc(s.n_q);
    if (q_constrained) s.q_constrained.upload(q_constrained, s.n_q, st);
    finish_ops(s, st);
    *out = o.release();
    API_END
}

int pdg_ops_sizes(const pdg_ops* ops, long long sizes[7]) {
    API_BEGIN
    require(ops && sizes, "pdg_ops_sizes: null argument");
    const SpatialOps& s = ops->s;
    sizes[0] = s.n_u;
    sizes[1] = s.n_q;
    sizes[2] = s.n_p;
    sizes[3] = s.A.nnz;
    sizes[4] = s.M_q.nnz;
    sizes[5] = s.B.nnz;
    sizes[6] = s.E.nnz;
    API_END
}

int pdg_ops_download(const pdg_ops* ops, int which, int* row_offsets, int* col_indices, double* values) {
    API_BEGIN
    require(ops != nullptr, "pdg_ops_download: null ops");
    const SpatialOps& s = ops->s;
    const DCsr* m = which == 0 ? &s.A : which == 1 ? &s.M_q : which == 2 ? &s.B : which == 3 ? &s.E : nullptr;
    require(m != nullptr, "pdg_ops_download: bad block id");
    cudaStream_t st = s.ctx->stream;
    PDG_CUDA(cudaMemcpyAsync(row_offsets, m->off.p, sizeof(int) * (m->rows + 1), cudaMemcpyDeviceToHost, st));
    if (m->nnz) {
        PDG_CUDA(cudaMemcpyAsync(col_indices, m->idx.p, sizeof(int) * m->nnz, cudaMemcpyDeviceToHost, st));
        PDG_CUDA(cudaMemcpyAsync(values, m->val.p, sizeof(double) * m->nnz, cudaMemcpyDeviceToHost, st));
    }
    PDG_CUDA(cudaStreamSynchronize(st));
    API_END
}

int pdg_ops_rhs(const pdg_ops* ops, double t, double* u, double* q, double* p) {
    API_BEGIN
    require(ops && u && q && p, "pdg_ops_rhs: null argument");
    const SpatialOps& s = ops->s;
    require(s.has_problem, "pdg_ops_rhs: operators were uploaded without a problem description");
    cudaStream_t st = s.ctx->stream;
    DBuf<double> du(s.n_u), dq(s.n_q), dp(s.n_p);
    assemble_rhs_device(s, t, du.p, dq.p, dp.p, st);
    PDG_CUDA(cudaMemcpyAsync(u, du.p, sizeof(double) * s.n_u, cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaMemcpyAsync(q, dq.p, sizeof(double) * s.n_q, cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaMemcpyAsync(p, dp.p, sizeof(double) * s.n_p, cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    API_END
}

int pdg_rhs_sample_points(const pdg_ops* ops, double* cell_xy, int* bface_ids, double* bface_xy) {
    API_BEGIN
    require(ops != nullptr, "pdg_rhs_sample_points: null ops");
    const SpatialOps& s = ops->s;
    require(s.has_problem, "pdg_rhs_sample_points: needs a problem description (pdg_ops_assemble / pdg_ops_assemble3)");
    if (s.nz > 0) {  // 3D: [cell][216][3], boundary faces ascending, [bface][36][3]
        const int nx = s.nx, ny = s.ny, nz = s.nz;
        const double h[3] = {s.prob3.lx / nx, s.prob3.ly / ny, s.prob3.lz / nz};
        std::vector<double> pts, wts;
        tc_gauss(6, pts, wts);
        if (cell_xy)
            for (int c = 0; c < nx * ny * nz; ++c) {
                const double o[3] = {(c % nx) * h[0], ((c / nx) % ny) * h[1], (c / (nx * ny)) * h[2]};
                for (int i = 0; i < 6; ++i)
                    for (int j = 0; j < 6; ++j)
                        for (int k = 0; k < 6; ++k) {
                            double* d = cell_xy + ((size_t)c * 216 + (i * 6 + j) * 6 + k) * 3;
                            d[0] = o[0] + pts[i] * h[0];
                            d[1] = o[1] + pts[j] * h[1];
                            d[2] = o[2] + pts[k] * h[2];
                        }
            }
        const int nzf = nx * ny * (nz + 1), nyf = nx * (ny + 1) * nz;
        size_t b = 0;
        // axis: normal axis; (ci, cj, ck): the adjacent cell; fixed: reference coordinate of the face in it
        auto face = [&](int f, int axis, int ci, int cj, int ck, double fixed) {
            if (bface_ids) bface_ids[b] = f;
            if (bface_xy)
                for (int qa = 0; qa < 6; ++qa)
                    for (int qb = 0; qb < 6; ++qb) {
                        double rp[3];
                        if (axis == 0) { rp[0] = fixed; rp[1] = pts[qa]; rp[2] = pts[qb]; }
                        else if (axis == 1) { rp[0] = pts[qa]; rp[1] = fixed; rp[2] = pts[qb]; }
                        else { rp[0] = pts[qa]; rp[1] = pts[qb]; rp[2] = fixed; }
                        double* d = bface_xy + (b * 36 + qa * 6 + qb) * 3;
                        d[0] = ci * h[0] + rp[0] * h[0];
                        d[1] = cj * h[1] + rp[1] * h[1];
                        d[2] = ck * h[2] + rp[2] * h[2];
                    }
            ++b;
        };
        for (int j = 0; j < ny; ++j) for (int i = 0; i < nx; ++i) face((0 * ny + j) * nx + i, 2, i, j, 0, 0.0);
        for (int j = 0; j < ny; ++j) for (int i = 0; i < nx; ++i) face((nz * ny + j) * nx + i, 2, i, j, nz - 1, 1.0);
        for (int k = 0; k < nz; ++k) for (int i = 0; i < nx; ++i) face(nzf + (0 * nz + k) * nx + i, 1, i, 0, k, 0.0);
        for (int k = 0; k < nz; ++k) for (int i = 0; i < nx; ++i) face(nzf + (ny * nz + k) * nx + i, 1, i, ny - 1, k, 1.0);
        for (int k = 0; k < nz; ++k) for (int j = 0; j < ny; ++j) face(nzf + nyf + (0 * nz + k) * ny + j, 0, 0, j, k, 0.0);
        for (int k = 0; k < nz; ++k) for (int j = 0; j < ny; ++j) face(nzf + nyf + (nx * nz + k) * ny + j, 0, nx - 1, j, k, 1.0);
        return PDG_OK;
    }
    const int nx = s.nx, ny = s.ny;
    const double hx = s.prob.lx / nx, hy = s.prob.ly / ny;
    std::vector<double> pts, wts;
    tc_gauss(6, pts, wts);
    if (cell_xy)
        for (int c = 0; c < nx * ny; ++c) {
            const double x0 = (c % nx) * hx, y0 = (c / nx) * hy;
            for (int i = 0; i < 6; ++i)
                for (int j = 0; j < 6; ++j) {
                    cell_xy[((size_t)c * 36 + i * 6 + j) * 2] = x0 + pts[i] * hx;
                    cell_xy[((size_t)c * 36 + i * 6 + j) * 2 + 1] = y0 + pts[j] * hy;
                }
        }
    const int nh = nx * (ny + 1);
    int k = 0;
    auto face = [&](int f, double x0, double y0, double x1, double y1) {
        if (bface_ids) bface_ids[k] = f;
        if (bface_xy)
            for (int q = 0; q < 6; ++q) {
                bface_xy[((size_t)k * 6 + q) * 2] = x0 + pts[q] * (x1 - x0);
                bface_xy[((size_t)k * 6 + q) * 2 + 1] = y0 + pts[q] * (y1 - y0);
            }
        ++k;
    };
    for (int i = 0; i < nx; ++i) face(i, i * hx, 0 * hy, (i + 1) * hx, 0 * hy);
    for (int i = 0; i < nx; ++i) face(ny * nx + i, i * hx, ny * hy, (i + 1) * hx, ny * hy);
    for (int j = 0; j < ny; ++j) face(nh + j, 0 * hx, j * hy, 0 * hx, (j + 1) * hy);
    for (int j = 0; j < ny; ++j) face(nh + nx * ny + j, nx * hx, j * hy, nx * hx, (j + 1) * hy);
    API_END
}

int pdg_ops_rhs_sampled(const pdg_ops* ops, const pdg_rhs_samples* samples, double* u, double* q, double* p) {
    API_BEGIN
    require(ops && samples && u && q && p, "pdg_ops_rhs_sampled: null argument");
    const SpatialOps& s = ops->s;
    require(s.has_problem, "pdg_ops_rhs_sampled: operators were uploaded without a problem description");
    cudaStream_t st = s.ctx->stream;
    DBuf<double> du(s.n_u), dq(s.n_q), dp(s.n_p);
    assemble_rhs_sampled_device(s, *samples, du.p, dq.p, dp.p, st);
    PDG_CUDA(cudaMemcpyAsync(u, du.p, sizeof(double) * s.n_u, cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaMemcpyAsync(q, dq.p, sizeof(double) * s.n_q, cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaMemcpyAsync(p, dp.p, sizeof(double) * s.n_p, cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    API_END
}

void pdg_ops_destroy(pdg_ops* ops) { delete ops; }

int pdg_block_create(pdg_ops* ops, int m, const double* theta, double tau, double lambda_pre,
                     const pdg_gmres_opts* opts, pdg_block** out) {
    API_BEGIN
    require(ops && theta && opts && out, "pdg_block_create: null argument");
    PDG_CUDA(cudaSetDevice(ops->s.ctx->device));
    require(opts->mode == 0 || opts->mode == 1, "pdg_block_create: mode must be 0 (parity) or 1 (fast)");
    auto& aslot = opts->mode == 1 ? ops->a_fast : ops->a;
    if (!aslot) aslot = make_a_solver(ops->s, 2, ops->s.ctx->stream, opts->mode == 1);
    auto b = std::make_unique<pdg_block>();
    b->b.create(ops->s, m, theta, tau, lambda_pre, *opts, aslot);
    const long long n = b->b.rows();
    b->io_a.alloc(n);
    b->io_b.alloc(n);
    *out = b.release();
    API_END
}

int pdg_block_rows(const pdg_block* blk, long long* rows, long long* nnz) {
    API_BEGIN
    require(blk && rows && nnz, "pdg_block_rows: null argument");
    *rows = blk->b.op.rows;
    *nnz = blk->b.op.nnz;
    API_END
}

int pdg_block_solve(pdg_block* blk, const double* rhs, double* x, pdg_report* rep) {
    API_BEGIN
    require(blk && rhs && x, "pdg_block_solve: null argument");
    cudaStream_t st = blk->b.ctx->stream;
    const long long n = blk->b.rows();
    PDG_CUDA(cudaMemcpyAsync(blk->io_a.p, rhs, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    blk->b.solve(blk->io_a.p, blk->io_b.p, rep);
    PDG_CUDA(cudaMemcpyAsync(x, blk->io_b.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    API_END
}

int pdg_block_solve_device(pdg_block* blk, const double* rhs_dev, double* x_dev, pdg_report* rep) {
    API_BEGIN
    require(blk && rhs_dev && x_dev, "pdg_block_solve_device: null argument");
    blk->b.solve(rhs_dev, x_dev, rep);
    PDG_CUDA(cudaStreamSynchronize(blk->b.ctx->stream));
    API_END
}

int pdg_block_apply(pdg_block* blk, int mode, const double* x, double* y) {
    API_BEGIN
    require(blk && x && y, "pdg_block_apply: null argument");
    require(mode == 0, "pdg_block_apply: unknown mode");
    cudaStream_t st = blk->b.ctx->stream;
    const long long n = blk->b.rows();
    PDG_CUDA(cudaMemcpyAsync(blk->io_a.p, x, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    blk->b.op.apply(blk->io_a.p, blk->io_b.p, st);
    PDG_CUDA(cudaMemcpyAsync(y, blk->io_b.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    API_END
}

int pdg_block_apply_device(pdg_block* blk, int mode, const double* x_dev, double* y_dev, int repeats, float* ms) {
    API_BEGIN
    require(blk && x_dev && y_dev, "pdg_block_apply_device: null argument");
    require(mode == 0, "pdg_block_apply_device: unknown mode");
    cudaStream_t st = blk->b.ctx->stream;
    if (repeats < 1) repeats = 1;
    PDG_CUDA(cudaEventRecord(blk->b.ev0, st));
    for (int i = 0; i < repeats; ++i) blk->b.op.apply(x_dev, y_dev, st);
    PDG_CUDA(cudaEventRecord(blk->b.ev1, st));
    PDG_CUDA(cudaEventSynchronize(blk->b.ev1));
    float t = 0.f;
    PDG_CUDA(cudaEventElapsedTime(&t, blk->b.ev0, blk->b.ev1));
    if (ms) *ms = t;
    API_END
}

int pdg_block_precondition(pdg_block* blk, const double* r, double* z) {
    API_BEGIN
    require(blk && r && z, "pdg_block_precondition: null argument");
    cudaStream_t st = blk->b.ctx->stream;
    const long long n = blk->b.rows();
    PDG_CUDA(cudaMemcpyAsync(blk->io_a.p, r, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    blk->b.pre.apply(blk->io_a.p, blk->io_b.p, st);
    PDG_CUDA(cudaMemcpyAsync(z, blk->io_b.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    API_END
}

int pdg_block_download_csr(const pdg_block* blk, long long* row_offsets, int* col_indices, double* values) {
    API_BEGIN
    require(blk && row_offsets && col_indices && values, "pdg_block_download_csr: null argument");
    std::vector<long long> off;
    std::vector<int> idx;
    std::vector<double> val;
    blk->b.op.to_csr(off, idx, val, blk->b.ctx->stream);
    std::memcpy(row_offsets, off.data(), sizeof(long long) * off.size());
    std::memcpy(col_indices, idx.data(), sizeof(int) * idx.size());
    std::memcpy(values, val.data(), sizeof(double) * val.size());
    API_END
}

void pdg_block_destroy(pdg_block* blk) { delete blk; }

int pdg_debug_recurrence_timing(pdg_block* blk, int which, unsigned long long* out, long long cap, int* ctas,
                                int* nsteps) {
    API_BEGIN
    require(blk && out && ctas && nsteps, "pdg_debug_recurrence_timing: null argument");
    BlockTriChol& c = which == 0 ? blk->b.pre.a->chol : blk->b.pre.flow;
    cudaStream_t st = blk->b.ctx->stream;
    c.debug_timing = true;
    PDG_CUDA(cudaMemsetAsync(blk->io_a.p, 0, sizeof(double) * blk->b.rows(), st));
    blk->b.pre.apply(blk->io_a.p, blk->io_b.p, st);
    PDG_CUDA(cudaStreamSynchronize(st));
    c.debug_timing = false;
    std::vector<unsigned long long> h = c.dbg.download(st);
    *ctas = c.local ? 2 * c.sw_g : c.nchains * c.d_g;
    *nsteps = c.dbg_steps;
    std::memcpy(out, h.data(), sizeof(unsigned long long) * std::min<long long>(cap, (long long)h.size()));
    API_END
}

int pdg_op_create(pdg_ops* ops, int m, const double* theta, double tau, pdg_op** out) {
    API_BEGIN
    require(ops && theta && out, "pdg_op_create: null argument");
    require(tau > 0.0, "pdg_op_create: tau must be positive");
    PDG_CUDA(cudaSetDevice(ops->s.ctx->device));
    auto o = std::make_unique<pdg_op>();
    o->ctx = ops->s.ctx;
    o->op.build(ops->s, m, theta, tau, o->ctx->stream);
    PDG_CUDA(cudaEventCreate(&o->e0));
    PDG_CUDA(cudaEventCreate(&o->e1));
    PDG_CUDA(cudaStreamSynchronize(o->ctx->stream));
    *out = o.release();
    API_END
}

int pdg_op_rows(const pdg_op* op, long long* rows, long long* nnz) {
    API_BEGIN
    require(op && rows && nnz, "pdg_op_rows: null argument");
    *rows = op->op.rows;
    *nnz = op->op.nnz;
    API_END
}

int pdg_op_apply_device(pdg_op* op, const double* x_dev, double* y_dev, int repeats, float* times_ms) {
    API_BEGIN
    require(op && x_dev && y_dev, "pdg_op_apply_device: null argument");
    cudaStream_t st = op->ctx->stream;
    for (int i = 0; i < std::max(repeats, 1); ++i) {
        PDG_CUDA(cudaEventRecord(op->e0, st));
        op->op.apply(x_dev, y_dev, st);
        PDG_CUDA(cudaEventRecord(op->e1, st));
        if (times_ms) {
            PDG_CUDA(cudaEventSynchronize(op->e1));
            PDG_CUDA(cudaEventElapsedTime(&times_ms[i], op->e0, op->e1));
        }
    }
    PDG_CUDA(cudaStreamSynchronize(st));
    API_END
}

int pdg_op_set_strip(pdg_op* op, int nx, int ny, int r0, int r1) {
    API_BEGIN
    require(op, "pdg_op_set_strip: null argument");
    op->op.set_strip(nx, ny, r0, r1, op->ctx->stream);
    API_END
}

int pdg_op_apply_strip_device(pdg_op* op, const double* x_dev, double* y_dev, int repeats, float* times_ms) {
    API_BEGIN
    require(op && x_dev && y_dev, "pdg_op_apply_strip_device: null argument");
    cudaStream_t st = op->ctx->stream;
    for (int i = 0; i < std::max(repeats, 1); ++i) {
        PDG_CUDA(cudaEventRecord(op->e0, st));
        op->op.apply_strip(x_dev, y_dev, st);
        PDG_CUDA(cudaEventRecord(op->e1, st));
        if (times_ms) {
            PDG_CUDA(cudaEventSynchronize(op->e1));
            PDG_CUDA(cudaEventElapsedTime(&times_ms[i], op->e0, op->e1));
        }
    }
    PDG_CUDA(cudaStreamSynchronize(st));
    API_END
}

int pdg_op_download_csr(const pdg_op* op, long long* row_offsets, int* col_indices, double* values) {
    API_BEGIN
    require(op && row_offsets && col_indices && values, "pdg_op_download_csr: null argument");
    std::vector<long long> off;
    std::vector<int> idx;
    std::vector<double> val;
    op->op.to_csr(off, idx, val, op->ctx->stream);
    std::memcpy(row_offsets, off.data(), sizeof(long long) * off.size());
    std::memcpy(col_indices, idx.data(), sizeof(int) * idx.size());
    std::memcpy(values, val.data(), sizeof(double) * val.size());
    API_END
}

void pdg_op_destroy(pdg_op* op) {
    if (!op) return;
    if (op->e0) cudaEventDestroy(op->e0);
    if (op->e1) cudaEventDestroy(op->e1);
    delete op;
}

int pdg_slab_create(pdg_ops* ops, int r, double tau, const pdg_gmres_opts* opts, pdg_slab** out) {
    API_BEGIN
    require(ops && opts && out, "pdg_slab_create: null argument");
    require(r >= 0 && r <= kMaxTimeDegree, "pdg_slab_create: r must be in [0, 5]");
    require(tau > 0.0, "build_slab_system: tau must be positive");
    auto s = std::make_unique<pdg_slab>();
    s->ops = ops;
    s->tc = time_consts(r);
    s->tau = tau;
    const int nn = r + 1;
    for (int g = 0; g < s->tc.n_blocks(); ++g) {
        const int m = s->tc.block_sizes[g], i0 = s->tc.block_starts[g];
        double theta[4];
        for (int a = 0; a < m; ++a)
            for (int c = 0; c < m; ++c) theta[a * m + c] = s->tc.T[(i0 + a) * nn + i0 + c];
        pdg_block* b = nullptr;
        // per-time-component preconditioner lambda = T_gg(0,0) (2x2 blocks are standardized, slab.hpp:166-169)
        const int rc = pdg_block_create(ops, m, theta, tau, theta[0], opts, &b);
        if (rc != PDG_OK) return rc;
        s->blks.emplace_back(b);
    }
    s->blk_iterations.assign(s->tc.n_blocks(), 0);
    s->blk_final_rel_res.assign(s->tc.n_blocks(), 0.0);
    cudaStream_t st = ops->s.ctx->stream;
    if (s->tc.n_blocks() > 1) {
        s->dpt.alloc((size_t)nn * ops->s.n_p);
        s->d_T.upload(s->tc.T, st);
    }
    s->d_Q.upload(s->tc.Q, st);
    s->d_w.upload(s->tc.weights, st);
    s->d_phi0.upload(s->tc.phi0, st);
    const long long nt = ops->s.n_total();
    s->shat.alloc(nn * nt);
    s->ysol.alloc(nn * nt);
    s->io_a.alloc(nn * nt);
    s->io_b.alloc(nn * nt);
    *out = s.release();
    API_END
}

int pdg_slab_solve_device(pdg_slab* s, const double* rhs_dev, double* out_dev, pdg_report* rep) {
    API_BEGIN
    require(s && rhs_dev && out_dev, "pdg_slab_solve: null argument");
    cudaStream_t st = s->ops->s.ctx->stream;
    const int nn = s->tc.n;
    const long long nt = s->ops->s.n_total();
    { ProfScope prof(PROF_SLAB, st, 8.0 * 3 * nn * nt);
    k_schur_fwd<<<grid_for(nn * nt, 256), 256, 0, st>>>(nn, nt, s->d_Q.p, s->d_w.p, rhs_dev, s->shat.p); }
    count_launch();
    PDG_CHECK_LAUNCH();
    const int nb = s->tc.n_blocks();
    if (nb == 1) {
        s->blks[0]->b.solve(s->shat.p, s->ysol.p, rep, 0);
        if (rep) {
            s->blk_iterations[0] = rep->iterations;
            s->blk_final_rel_res[0] = rep->final_rel_res;
        }
    } else {
        // blocks in descending order (slab.hpp:194-235); the report handed back is the block
        // with the most iterations (march.hpp logs the maximum), device time and launches summed
        const SpatialOps& o = s->ops->s;
        DBuf<double>& dT = s->d_T;
        pdg_report best{};
        double ms = 0.0;
        int launches = 0;
        bool have = false;
        for (int g = nb - 1; g >= 0; --g) {
            const int m = s->tc.block_sizes[g], i0 = s->tc.block_starts[g];
            if (i0 + m < nn) {
                k_schur_backsub<<<grid_for((long long)m * o.n_p, 256), 256, 0, st>>>(o.n_p, nn, i0, m, i0 + m, dT.p, s->dpt.p,
                                                                                     nt, (long long)o.n_u + o.n_q, s->shat.p);
                count_launch();
                PDG_CHECK_LAUNCH();
            }
            pdg_report br{};
            if (rep) {
                br.history = rep->history;  // the last solved block's history ends up in the caller's buffer
                br.history_cap = rep->history_cap;
            }
            s->blks[g]->b.solve(s->shat.p + (long long)i0 * nt, s->ysol.p + (long long)i0 * nt, &br, g);
            s->blk_iterations[g] = br.iterations;
            s->blk_final_rel_res[g] = br.final_rel_res;
            ms += br.device_ms;
            launches += br.kernel_launches;
            if (!have || br.iterations > best.iterations) best = br;
            have = true;
            if (g > 0)
                for (int bi = 0; bi < m; ++bi) {
                    const double* yj = s->ysol.p + (long long)(i0 + bi) * nt;
                    k_time_derivative<<<grid_for(8LL * o.n_p, 256), 256, 0, st>>>(o.n_p, -o.biot_b, o.inv_m, o.Et.off.p, o.Et.idx.p,
                                                                             o.Et.val.p, o.m_p.p, yj, yj + o.n_u + o.n_q,
                                                                             s->dpt.p + (size_t)(i0 + bi) * o.n_p);
                    count_launch();
                    PDG_CHECK_LAUNCH();
                }
        }
        if (rep) {
            double worst = 0.0;
            for (double v : s->blk_final_rel_res) worst = std::max(worst, v);
            double* hist = rep->history;
            const int cap = rep->history_cap;
            *rep = best;
            rep->history = hist;
            rep->history_cap = cap;
            rep->final_rel_res = worst;
            rep->device_ms = ms;
            rep->kernel_launches = launches;
        }
    }
    { ProfScope prof(PROF_SLAB, st, 8.0 * 2 * nn * nt);
    k_schur_bwd<<<grid_for(nn * nt, 256), 256, 0, st>>>(nn, nt, s->d_Q.p, s->ysol.p, out_dev); }
    count_launch();
    PDG_CHECK_LAUNCH();
    PDG_CUDA(cudaStreamSynchronize(st));
    API_END
}

int pdg_slab_solve(pdg_slab* s, const double* rhs, double* out, pdg_report* rep) {
    API_BEGIN
    require(s && rhs && out, "pdg_slab_solve: null argument");
    cudaStream_t st = s->ops->s.ctx->stream;
    const long long n = s->tc.n * (long long)s->ops->s.n_total();
    PDG_CUDA(cudaMemcpyAsync(s->io_a.p, rhs, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    const int rc = pdg_slab_solve_device(s, s->io_a.p, s->io_b.p, rep);
    if (rc != PDG_OK) return rc;
    PDG_CUDA(cudaMemcpyAsync(out, s->io_b.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    API_END
}

namespace {
// build_slab_system (slab.hpp:58-87) on the slab's stream, constant boundary data; no synchronize
void slab_rhs_enqueue(pdg_slab* s, double t0, double tau, const double* u_prev_dev, const double* p_prev_dev,
                      double* rhs_dev) {
    const SpatialOps& o = s->ops->s;
    cudaStream_t st = o.ctx->stream;
    const int nn = s->tc.n;
    if (!s->rhs_u.n) {
        s->rhs_u.alloc((size_t)nn * o.n_u);
        s->rhs_q.alloc((size_t)nn * o.n_q);
        s->rhs_p.alloc((size_t)nn * o.n_p);
        s->djump.alloc(o.n_p);
    }
    ProfScope prof(PROF_SLAB, st, 8.0 * 2 * nn * o.n_total());
    // b(t_i) of the problem description: constant boundary data, so the same vector at every node and
    // slab (assemble_rhs_device ignores t); assembled once per handle, as long as nothing else
    // (the sampled variant) overwrites the buffers
    if (!s->rhs_const) {
        for (int i = 0; i < nn; ++i)
            assemble_rhs_device(o, t0 + s->tc.nodes[i] * tau, s->rhs_u.p + (size_t)i * o.n_u, s->rhs_q.p + (size_t)i * o.n_q,
                                s->rhs_p.p + (size_t)i * o.n_p, st);
        s->rhs_const = true;
    }
    k_time_derivative<<<grid_for(8LL * o.n_p, 256), 256, 0, st>>>(o.n_p, -o.biot_b, o.inv_m, o.Et.off.p, o.Et.idx.p, o.Et.val.p,
                                                             o.m_p.p, u_prev_dev, p_prev_dev, s->djump.p);
    k_slab_rhs<<<grid_for((long long)nn * o.n_total(), 256), 256, 0, st>>>(nn, o.n_u, o.n_q, o.n_p, tau, s->d_w.p,
                                                                           s->d_phi0.p, s->rhs_u.p, s->rhs_q.p,
                                                                           s->rhs_p.p, s->djump.p, rhs_dev);
    count_launch(2);
    PDG_CHECK_LAUNCH();
}
}  // namespace

int pdg_slab_rhs_device(pdg_slab* s, double t0, double tau, const double* u_prev_dev, const double* p_prev_dev,
                        double* rhs_dev) {
    API_BEGIN
    require(s && u_prev_dev && p_prev_dev && rhs_dev, "pdg_slab_rhs_device: null argument");
    require(tau > 0.0, "build_slab_system: tau must be positive");
    require(s->ops->s.has_problem, "pdg_slab_rhs_device: operators were uploaded without a problem description");
    slab_rhs_enqueue(s, t0, tau, u_prev_dev, p_prev_dev, rhs_dev);
    // like every other *_device entry point: rhs_dev is complete when the call returns, so a
    // caller on another stream (torch's) may read it without a library-stream dependency
    PDG_CUDA(cudaStreamSynchronize(s->ops->s.ctx->stream));
    API_END
}

int pdg_slab_step_device(pdg_slab* s, double t0, double tau, const double* prev_state_dev, double* out_dev,
                         pdg_report* rep) {
    API_BEGIN
    require(s && out_dev, "pdg_slab_step_device: null argument");
    require(tau > 0.0, "build_slab_system: tau must be positive");
    const SpatialOps& o = s->ops->s;
    require(o.has_problem, "pdg_slab_step_device: operators were uploaded without a problem description");
    cudaStream_t st = o.ctx->stream;
    const long long nt = o.n_total();
    if (!s->zero_state.n) {
        s->zero_state.alloc(nt);
        s->zero_state.zero(st);
    }
    const double* prev = prev_state_dev ? prev_state_dev : s->zero_state.p;
    // the right-hand side is consumed (Schur transform) before the solve writes out_dev, all in
    // stream order: prev_state_dev may be the last component of the previous call's out_dev only
    // if that is a different buffer than this call's out_dev
    slab_rhs_enqueue(s, t0, tau, prev, prev + o.n_u + o.n_q, s->io_a.p);
    return pdg_slab_solve_device(s, s->io_a.p, out_dev, rep);
    API_END
}

int pdg_slab_block_reports(const pdg_slab* s, int* n_blocks, int* block_sizes, int* iterations, double* final_rel_res) {
    API_BEGIN
    require(s && n_blocks, "pdg_slab_block_reports: null argument");
    *n_blocks = s->tc.n_blocks();
    for (int g = 0; g < s->tc.n_blocks(); ++g) {
        if (block_sizes) block_sizes[g] = s->tc.block_sizes[g];
        if (iterations) iterations[g] = s->blk_iterations[g];
        if (final_rel_res) final_rel_res[g] = s->blk_final_rel_res[g];
    }
    API_END
}

int pdg_slab_rhs_sampled_device(pdg_slab* s, double tau, const pdg_rhs_samples* samples, const double* u_prev_dev,
                                const double* p_prev_dev, double* rhs_dev) {
    API_BEGIN
    require(s && samples && u_prev_dev && p_prev_dev && rhs_dev, "pdg_slab_rhs_sampled_device: null argument");
    require(tau > 0.0, "build_slab_system: tau must be positive");
    const SpatialOps& o = s->ops->s;
    require(o.has_problem, "pdg_slab_rhs_sampled_device: operators were uploaded without a problem description");
    cudaStream_t st = o.ctx->stream;
    const int nn = s->tc.n;
    if (!s->rhs_u.n) {
        s->rhs_u.alloc((size_t)nn * o.n_u);
        s->rhs_q.alloc((size_t)nn * o.n_q);
        s->rhs_p.alloc((size_t)nn * o.n_p);
        s->djump.alloc(o.n_p);
    }
    s->rhs_const = false;  // the buffers no longer hold the constant-data vectors
    for (int i = 0; i < nn; ++i)
        assemble_rhs_sampled_device(o, samples[i], s->rhs_u.p + (size_t)i * o.n_u, s->rhs_q.p + (size_t)i * o.n_q,
                                    s->rhs_p.p + (size_t)i * o.n_p, st);
    k_time_derivative<<<grid_for(8LL * o.n_p, 256), 256, 0, st>>>(o.n_p, -o.biot_b, o.inv_m, o.Et.off.p, o.Et.idx.p, o.Et.val.p,
                                                             o.m_p.p, u_prev_dev, p_prev_dev, s->djump.p);
    k_slab_rhs<<<grid_for((long long)nn * o.n_total(), 256), 256, 0, st>>>(nn, o.n_u, o.n_q, o.n_p, tau, s->d_w.p,
                                                                           s->d_phi0.p, s->rhs_u.p, s->rhs_q.p,
                                                                           s->rhs_p.p, s->djump.p, rhs_dev);
    count_launch(2);
    PDG_CHECK_LAUNCH();
    PDG_CUDA(cudaStreamSynchronize(st));
    API_END
}

void pdg_slab_destroy(pdg_slab* s) { delete s; }

int pdg_spmv_csr_device(int rows, const long long* off, const int* idx, const double* val, const double* x, double* y) {
    API_BEGIN
    spmv_csr_device(rows, off, idx, val, x, y, 0);
    PDG_CUDA(cudaStreamSynchronize(0));
    API_END
}

int pdg_mass_residual_device(pdg_ops* ops, int r, double tau, const double* rhs_dev, const double* state_dev,
                             double* residual_dev, double* scale) {
    API_BEGIN
    require(ops && rhs_dev && state_dev && residual_dev && scale, "pdg_mass_residual: null argument");
    require(r >= 0 && r + 1 <= kMaxNodes, "pdg_mass_residual: unsupported dG degree");
    require(tau > 0.0, "build_slab_system: tau must be positive");
    const SpatialOps& o = ops->s;
    cudaStream_t st = o.ctx->stream;
    const TimeConsts tc = time_consts(r);
    DBuf<double> g, w;
    g.upload(tc.G, st);
    w.upload(tc.weights, st);
    DBuf<unsigned long long> sb(1);
    sb.zero(st);
    ProfScope prof(PROF_SLAB, st, 8.0 * 2 * tc.n * o.n_total());
    k_mass_residual<<<grid_for(o.n_p, 256), 256, 0, st>>>(o.n_p, o.n_u, o.n_q, tc.n, g.p, w.p, tau, -o.biot_b, o.inv_m,
                                                           o.m_p.p, o.Et.off.p, o.Et.idx.p, o.Et.val.p, o.Bt.off.p,
                                                           o.Bt.idx.p, o.Bt.val.p, rhs_dev, state_dev, residual_dev, sb.p);
    count_launch();
    PDG_CHECK_LAUNCH();
    unsigned long long bits = 0;
    PDG_CUDA(cudaMemcpyAsync(&bits, sb.p, sizeof(bits), cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    *scale = bits_to_double(bits);
    API_END
}

int pdg_mass_residual(pdg_ops* ops, int r, double tau, const double* rhs, const double* state, double* residual,
                      double* scale) {
    API_BEGIN
    require(ops && rhs && state && residual && scale, "pdg_mass_residual: null argument");
    require(r >= 0 && r + 1 <= kMaxNodes, "pdg_mass_residual: unsupported dG degree");
    const SpatialOps& o = ops->s;
    cudaStream_t st = o.ctx->stream;
    const size_t len = (size_t)(r + 1) * o.n_total();
    DBuf<double> drhs, dstate, dres(o.n_p);
    drhs.upload(rhs, len, st);
    dstate.upload(state, len, st);
    const int rc = pdg_mass_residual_device(ops, r, tau, drhs.p, dstate.p, dres.p, scale);
    if (rc != PDG_OK) return rc;
    PDG_CUDA(cudaMemcpyAsync(residual, dres.p, sizeof(double) * o.n_p, cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    API_END
}

int pdg_fs_create(pdg_ops* ops, int r, double tau, const pdg_fs_opts* opts, pdg_fs** out) {
    API_BEGIN
    require(ops && opts && out, "pdg_fs_create: null argument");
    require(opts->tol > 0.0 && opts->tol < 1.0, "fixed-stress: tol must be in (0,1)");
    require(opts->max_sweeps >= 1, "fixed-stress: sweep counts must be >= 1");
    PDG_CUDA(cudaSetDevice(ops->s.ctx->device));
    auto f = std::make_unique<pdg_fs>();
    f->ops = ops;
    f->opts = *opts;
    if (!ops->a) ops->a = make_a_solver(ops->s, 2, ops->s.ctx->stream);
    f->fs.create(ops->s, r, tau, opts->stab, ops->a);
    *out = f.release();
    API_END
}

int pdg_fs_solve_device(pdg_fs* f, const double* rhs_dev, const double* x0_dev, double* x_dev, pdg_report* rep) {
    API_BEGIN
    require(f && rhs_dev && x_dev, "pdg_fs_solve: null argument");
    f->fs.solve(rhs_dev, x0_dev, x_dev, f->opts.tol, f->opts.max_sweeps, rep);
    API_END
}

int pdg_fs_solve(pdg_fs* f, const double* rhs, const double* x0, double* x, pdg_report* rep) {
    API_BEGIN
    require(f && rhs && x, "pdg_fs_solve: null argument");
    cudaStream_t st = f->ops->s.ctx->stream;
    const size_t n = (size_t)f->fs.m * f->ops->s.n_total();
    if (!f->io_a.n) {
        f->io_a.alloc(n);
        f->io_b.alloc(n);
        f->io_c.alloc(n);
    }
    PDG_CUDA(cudaMemcpyAsync(f->io_a.p, rhs, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    if (x0) PDG_CUDA(cudaMemcpyAsync(f->io_c.p, x0, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    f->fs.solve(f->io_a.p, x0 ? f->io_c.p : nullptr, f->io_b.p, f->opts.tol, f->opts.max_sweeps, rep);
    PDG_CUDA(cudaMemcpyAsync(x, f->io_b.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    API_END
}

void pdg_fs_destroy(pdg_fs* f) { delete f; }

int pdg_tri_create(pdg_ctx* ctx, const pdg_csr* A, const int* perm, const int* block_sizes, int nblocks,
                   int allow_local, pdg_tri** out) {
    API_BEGIN
    require(ctx && A && block_sizes && out && nblocks >= 1, "pdg_tri_create: null argument");
    require(A->rows == A->cols, "pdg_tri_create: matrix must be square");
    PDG_CUDA(cudaSetDevice(ctx->c.device));
    auto t = std::make_unique<pdg_tri>();
    t->ctx = &ctx->c;
    cudaStream_t st = ctx->c.stream;
    csr_upload(t->A, *A, st);
    std::vector<int> p;
    if (perm) p.assign(perm, perm + A->rows);
    t->chol.allow_local = (allow_local & 1) != 0;
    t->chol.symmetric = (allow_local & 2) == 0;
    t->chol.factor(A->rows, t->A.off.p, t->A.idx.p, t->A.val.p, p, std::vector<int>(block_sizes, block_sizes + nblocks), 2,
                   st);
    *out = t.release();
    API_END
}

int pdg_tri_solve_device(pdg_tri* t, const double* b_dev, double* x_dev, int nrhs) {
    API_BEGIN
    require(t && b_dev && x_dev, "pdg_tri_solve: null argument");
    t->chol.solve(b_dev, t->chol.n, x_dev, t->chol.n, nrhs, t->ctx->stream);
    PDG_CUDA(cudaStreamSynchronize(t->ctx->stream));
    API_END
}

void pdg_tri_destroy(pdg_tri* t) { delete t; }

int pdg_time_constants(int r, double* nodes, double* weights, double* phi0, double* T, double* Q) {
    API_BEGIN
    require(nodes && weights && phi0 && T && Q, "pdg_time_constants: null argument");
    const TimeConsts tc = time_consts(r);
    for (int i = 0; i < tc.n; ++i) {
        nodes[i] = tc.nodes[i];
        weights[i] = tc.weights[i];
        phi0[i] = tc.phi0[i];
    }
    for (int i = 0; i < tc.n * tc.n; ++i) {
        T[i] = tc.T[i];
        Q[i] = tc.Q[i];
    }
    API_END
}

int pdg_time_schur_blocks(int r, int* n_blocks, int* block_sizes, int* block_starts, double* G_hat) {
    API_BEGIN
    require(n_blocks != nullptr, "pdg_time_schur_blocks: null argument");
    const TimeConsts tc = time_consts(r);
    *n_blocks = tc.n_blocks();
    for (int g = 0; g < tc.n_blocks(); ++g) {
        if (block_sizes) block_sizes[g] = tc.block_sizes[g];
        if (block_starts) block_starts[g] = tc.block_starts[g];
    }
    if (G_hat)
        for (int i = 0; i < tc.n * tc.n; ++i) G_hat[i] = tc.G[i];
    API_END
}

void pdg_util_uniform(unsigned long long seed, long long n, double* out) {
    std::mt19937_64 g(seed);
    for (long long i = 0; i < n; ++i) out[i] = -1.0 + 2.0 * (static_cast<double>(g() >> 11) * 0x1.0p-53);
}

void pdg_util_lognormal(unsigned long long seed, long long n, double sigma, double* out) {
    std::mt19937_64 g(seed);
    for (long long i = 0; i < n; ++i) {
        const double u1 = (static_cast<double>(g() >> 11) + 1.0) * 0x1.0p-53;
        const double u2 = static_cast<double>(g() >> 11) * 0x1.0p-53;
        out[i] = std::exp(sigma * (std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2)));
    }
}

long long pdg_util_launch_count(void) { return g_launches; }

}  // extern "C"
