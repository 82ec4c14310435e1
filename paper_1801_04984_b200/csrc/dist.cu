// Multi-GPU slab block solve (see dist.cuh).
#include <cublas_v2.h>
#include <cusolverDn.h>
#include <nccl.h>

#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>

#include "blocktri.cuh"
#include "dist.cuh"
#include "gmres_ls.cuh"

namespace pdg {

// NCCL is resolved at run time, not linked: inside a PyTorch process the NCCL that torch
// loaded is used (RTLD_NOLOAD), elsewhere PDG_NCCL_LIB or the system libnccl.so.2. (Linking
// libnccl.so.2 would bind whichever copy the loader meets first, possibly older than torch's.)
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
const NcclApi& nccl() {
    static NcclApi api;
    static bool loaded = false;
    if (loaded) return api;
    void* h = nullptr;
    if (const char* p = std::getenv("PDG_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw Error(PDG_NCCL_ERROR, "NCCL library not found (libnccl.so.2; set PDG_NCCL_LIB)");
    auto sym = [&](const char* n) {
        void* f = dlsym(h, n);
        if (!f) throw Error(PDG_NCCL_ERROR, std::string("NCCL symbol missing: ") + n);
        return f;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    loaded = true;
    return api;
}

#define PDG_NCCL(call)                                                                                      \
    do {                                                                                                    \
        ncclResult_t r_ = (call);                                                                           \
        if (r_ != ncclSuccess)                                                                              \
            throw ::pdg::Error(PDG_NCCL_ERROR, std::string(#call) + ": " + nccl().GetErrorString(r_));     \
    } while (0)
#define PDG_DBLAS(call)                                                                                     \
    do {                                                                                                    \
        cublasStatus_t s_ = (call);                                                                         \
        if (s_ != CUBLAS_STATUS_SUCCESS)                                                                    \
            throw ::pdg::Error(PDG_CUDA_ERROR, std::string(#call) + ": cublas status " + std::to_string((int)s_)); \
    } while (0)
#define PDG_DSOLVER(call)                                                                                     \
    do {                                                                                                      \
        cusolverStatus_t s_ = (call);                                                                         \
        if (s_ != CUSOLVER_STATUS_SUCCESS)                                                                    \
            throw ::pdg::Error(PDG_CUDA_ERROR, std::string(#call) + ": cusolver status " + std::to_string((int)s_)); \
    } while (0)

namespace {

// ---- communicators ----------------------------------------------------------
struct NcclComm : Comm {
    ncclComm_t c = nullptr;
    ~NcclComm() override {
        if (c) nccl().CommDestroy(c);
    }
    void allgather(const double* send, double* recv, size_t count, cudaStream_t st) override {
        PDG_NCCL(nccl().AllGather(send, recv, count, ncclDouble, c, st));
    }
    void exchange(const std::vector<int>& peers, const std::vector<const double*>& sbuf, const std::vector<size_t>& scount,
                  const std::vector<double*>& rbuf, const std::vector<size_t>& rcount, cudaStream_t st) override {
        PDG_NCCL(nccl().GroupStart());
        for (size_t i = 0; i < peers.size(); ++i) {
            if (scount[i]) PDG_NCCL(nccl().Send(sbuf[i], scount[i], ncclDouble, peers[i], c, st));
            if (rcount[i]) PDG_NCCL(nccl().Recv(rbuf[i], rcount[i], ncclDouble, peers[i], c, st));
        }
        PDG_NCCL(nccl().GroupEnd());
    }
};

// Host-staged collectives through caller callbacks (blocking): the device data goes
// to the host, the callback moves it between the processes, the result comes back.
struct HostComm : Comm {
    pdg_host_allgather_fn ag = nullptr;
    pdg_host_exchange_fn ex = nullptr;
    void* user = nullptr;
    std::vector<double> hs, hr;
    void allgather(const double* send, double* recv, size_t count, cudaStream_t st) override {
        hs.resize(std::max<size_t>(count, 1));
        hr.resize(std::max<size_t>(count * nranks, 1));
        if (count) PDG_CUDA(cudaMemcpyAsync(hs.data(), send, sizeof(double) * count, cudaMemcpyDeviceToHost, st));
        PDG_CUDA(cudaStreamSynchronize(st));
        if (ag(user, hs.data(), hr.data(), static_cast<long long>(count)) != 0)
            throw Error(PDG_NCCL_ERROR, "host communicator: all-gather callback failed");
        if (count) PDG_CUDA(cudaMemcpyAsync(recv, hr.data(), sizeof(double) * count * nranks, cudaMemcpyHostToDevice, st));
        PDG_CUDA(cudaStreamSynchronize(st));
    }
    void exchange(const std::vector<int>& peers, const std::vector<const double*>& sbuf, const std::vector<size_t>& scount,
                  const std::vector<double*>& rbuf, const std::vector<size_t>& rcount, cudaStream_t st) override {
        const size_t np = peers.size();
        std::vector<std::vector<double>> s(np), r(np);
        for (size_t i = 0; i < np; ++i) {
            s[i].resize(std::max<size_t>(scount[i], 1));
            r[i].resize(std::max<size_t>(rcount[i], 1));
            if (scount[i])
                PDG_CUDA(cudaMemcpyAsync(s[i].data(), sbuf[i], sizeof(double) * scount[i], cudaMemcpyDeviceToHost, st));
        }
        PDG_CUDA(cudaStreamSynchronize(st));
        std::vector<const double*> sp(np);
        std::vector<double*> rp(np);
        std::vector<long long> sc(np), rc(np);
        for (size_t i = 0; i < np; ++i) {
            sp[i] = s[i].data();
            rp[i] = r[i].data();
            sc[i] = static_cast<long long>(scount[i]);
            rc[i] = static_cast<long long>(rcount[i]);
        }
        if (ex(user, static_cast<int>(np), peers.data(), sp.data(), sc.data(), rp.data(), rc.data()) != 0)
            throw Error(PDG_NCCL_ERROR, "host communicator: exchange callback failed");
        for (size_t i = 0; i < np; ++i)
            if (rcount[i])
                PDG_CUDA(cudaMemcpyAsync(rbuf[i], r[i].data(), sizeof(double) * rcount[i], cudaMemcpyHostToDevice, st));
        PDG_CUDA(cudaStreamSynchronize(st));
    }
};

// ---- small kernels -------------------------------------------------------------
__global__ void k_rank_sum(int P, long long count, const double* __restrict__ in, double* __restrict__ out) {
    // out[j] = ((in_0 + in_1) + in_2) + ... in rank order: identical bits on every rank
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < count; j += (long long)gridDim.x * blockDim.x) {
        double s = in[j];
        for (int r = 1; r < P; ++r) s += in[(long long)r * count + j];
        out[j] = s;
    }
}
__global__ void k_pack(long long n, int ncomp, long long stride, const long long* __restrict__ idx,
                       const double* __restrict__ x, double* __restrict__ buf) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n * ncomp; t += (long long)gridDim.x * blockDim.x) {
        const long long k = t % n, c = t / n;
        buf[t] = x[c * stride + idx[k]];
    }
}
__global__ void k_unpack(long long n, int ncomp, long long stride, const long long* __restrict__ idx,
                         const double* __restrict__ buf, double* __restrict__ x) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n * ncomp; t += (long long)gridDim.x * blockDim.x) {
        const long long k = t % n, c = t / n;
        x[c * stride + idx[k]] = buf[t];
    }
}
// dst[idx[k] + c * sstride] <- src[k + c * lstride] (scatter) and the gather
__global__ void k_scatter(long long n, int ncomp, const long long* __restrict__ idx, const double* __restrict__ src,
                          long long lstride, double* __restrict__ dst, long long gstride) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n * ncomp; t += (long long)gridDim.x * blockDim.x) {
        const long long k = t % n, c = t / n;
        dst[c * gstride + idx[k]] = src[c * lstride + k];
    }
}
__global__ void k_gather(long long n, int ncomp, const long long* __restrict__ idx, const double* __restrict__ src,
                         long long gstride, double* __restrict__ dst, long long lstride) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n * ncomp; t += (long long)gridDim.x * blockDim.x) {
        const long long k = t % n, c = t / n;
        dst[c * lstride + k] = src[c * gstride + idx[k]];
    }
}
// y_r = sum_k val * x[local col] over CSR rows, for nrhs right-hand sides (x: ld, y: ldy); y = sign * (.) + (base ? base : 0)
__global__ void k_csr_rows(int rows, int nrhs, const int* __restrict__ off, const int* __restrict__ idx,
                           const double* __restrict__ val, const double* __restrict__ x, long long ldx, double* __restrict__ y,
                           long long ldy) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)rows * nrhs; t += (long long)gridDim.x * blockDim.x) {
        const int r = static_cast<int>(t % rows), k = static_cast<int>(t / rows);
        double s = 0.0;
        for (int q = off[r]; q < off[r + 1]; ++q) s += val[q] * x[(long long)k * ldx + idx[q]];
        y[(long long)k * ldy + r] = s;
    }
}
// g[so + i] (+)= (b[sep[i]] if b) - a[i], per rhs (g: ld ns, a: ld s)
__global__ void k_sep_rhs(int s, int nrhs, const long long* __restrict__ sep, const double* __restrict__ b, long long ldb,
                          const double* __restrict__ a, double* __restrict__ g, long long so, int ns) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)s * nrhs; t += (long long)gridDim.x * blockDim.x) {
        const int i = static_cast<int>(t % s), k = static_cast<int>(t / s);
        const double bv = b ? b[(long long)k * ldb + sep[i]] : 0.0;
        g[(long long)k * ns + so + i] = bv - a[(long long)k * s + i];
    }
}
__global__ void k_dense_scatter(long long nt, const long long* __restrict__ pos, const double* __restrict__ val, double* __restrict__ D) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nt; t += (long long)gridDim.x * blockDim.x)
        D[pos[t]] = val[t];
}
// fixed-stress sweep pieces on owned entries (fixed_stress.hpp:109-139; as k_flow_rq / k_flow_p / k_mech_rhs)
__global__ void k_d_fp(int m, int no, const int* __restrict__ oc, int np, int nt, int nuq, const double* __restrict__ r,
                       double* __restrict__ fp) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * no; t += (long long)gridDim.x * blockDim.x) {
        const int i = static_cast<int>(t / no), c = oc[t % no];
        fp[(long long)i * np + c] = r[(long long)i * nt + nuq + c];
    }
}
__global__ void k_d_rq(int m, int no, const int* __restrict__ of, int nq, int np, int nt, int nu, double w,
                       const double* __restrict__ r, const double* __restrict__ fp, const int* b_off, const int* b_idx,
                       const double* b_val, const double* __restrict__ dinv, double* __restrict__ rq) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * no; t += (long long)gridDim.x * blockDim.x) {
        const int i = static_cast<int>(t / no), f = of[t % no];
        double v = r[(long long)i * nt + nu + f];
        for (int k = b_off[f]; k < b_off[f + 1]; ++k) {
            const int c = b_idx[k];
            v -= w * b_val[k] * (dinv[c] * fp[(long long)i * np + c]);
        }
        rq[(long long)i * nq + f] = v;
    }
}
__global__ void k_d_p(int m, int no, const int* __restrict__ oc, int np, int nq, double w, const double* __restrict__ fp,
                      const int* bt_off, const int* bt_idx, const double* bt_val, const double* __restrict__ dinv,
                      const double* __restrict__ q, double* __restrict__ p) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * no; t += (long long)gridDim.x * blockDim.x) {
        const int i = static_cast<int>(t / no), c = oc[t % no];
        double btq = 0.0;
        for (int k = bt_off[c]; k < bt_off[c + 1]; ++k) btq += bt_val[k] * q[(long long)i * nq + bt_idx[k]];
        p[(long long)i * np + c] = dinv[c] * (fp[(long long)i * np + c] - w * btq);
    }
}
__global__ void k_d_mech(int m, int no, const int* __restrict__ ou, int nu, int nt, int np, double w, double b,
                         const double* __restrict__ r, const double* __restrict__ p, const int* e_off, const int* e_idx,
                         const double* e_val, double* __restrict__ mech) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * no; t += (long long)gridDim.x * blockDim.x) {
        const int i = static_cast<int>(t / no), d = ou[t % no];
        double ep = 0.0;
        for (int k = e_off[d]; k < e_off[d + 1]; ++k) ep += e_val[k] * p[(long long)i * np + e_idx[k]];
        mech[(long long)i * nu + d] = r[(long long)i * nt + d] / w + b * ep;
    }
}
// z_own[k] from the per-component result buffers at the owned global row rows[k]
__global__ void k_d_collect(long long nown, const long long* __restrict__ rows, int nt, int nu, int nq, int np,
                            const double* __restrict__ u, const double* __restrict__ q, const double* __restrict__ p,
                            double* __restrict__ z) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nown; k += (long long)gridDim.x * blockDim.x) {
        const long long g = rows[k];
        const int i = static_cast<int>(g / nt), l = static_cast<int>(g % nt);
        z[k] = l < nu ? u[(long long)i * nu + l] : l < nu + nq ? q[(long long)i * nq + l - nu] : p[(long long)i * np + l - nu - nq];
    }
}
constexpr int kDotThreads = 256;
// deterministic multi-block dots: partials[blk][j] of V_j . w over a fixed grid-stride row
// set, then out[j] = the partials summed in block order (one thread per column)
constexpr int kDotBlocks = 148;
__global__ void __launch_bounds__(kDotThreads) k_dot_partials(long long n, int ncols, const double* __restrict__ V,
                                                              const double* __restrict__ w, double* __restrict__ part) {
    __shared__ double sh[8][kDotThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int j0 = 0; j0 < ncols; j0 += 8) {
        double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
            const double wr = w[r];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (j0 + q < ncols) a[q] += V[(long long)(j0 + q) * n + r] * wr;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
            for (int o = 16; o; o >>= 1) a[q] += __shfl_xor_sync(0xffffffffu, a[q], o);
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < 8; ++q) sh[q][warp] = a[q];
        __syncthreads();
        if (threadIdx.x < 8 && j0 + threadIdx.x < ncols) {
            double t = 0.0;
            for (int i = 0; i < kDotThreads / 32; ++i) t += sh[threadIdx.x][i];
            part[(long long)blockIdx.x * ncols + j0 + threadIdx.x] = t;
        }
        __syncthreads();
    }
}
__global__ void k_dot_final(int nblk, int ncols, const double* __restrict__ part, double* __restrict__ out) {
    for (int j = threadIdx.x; j < ncols; j += blockDim.x) {
        double t = 0.0;
        for (int b = 0; b < nblk; ++b) t += part[(long long)b * ncols + j];
        out[j] = t;
    }
}
__global__ void k_sqrt_scale(long long n, const double* __restrict__ nrm2, const double* __restrict__ w, double* __restrict__ v,
                             double* __restrict__ nrm_out) {
    const double d = sqrt(nrm2[0]);
    if (blockIdx.x == 0 && threadIdx.x == 0) nrm_out[0] = d;
    if (!v) return;
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x)
        v[r] = w[r] / d;
}

// w -= V h (h on the device), out = base + V y
__global__ void k_sub_vh(long long n, int ncols, const double* __restrict__ V, const double* __restrict__ h, double* __restrict__ w) {
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
        double v = w[r];
        for (int j = 0; j < ncols; ++j) v -= h[j] * V[(long long)j * n + r];
        w[r] = v;
    }
}
__global__ void k_vy(long long n, int ncols, const double* __restrict__ V, const double* __restrict__ y,
                     const double* __restrict__ base, double* __restrict__ out) {
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int j = 0; j < ncols; ++j) s += V[(long long)j * n + r] * y[j];
        out[r] = base ? base[r] + s : s;
    }
}
__global__ void k_axpby(long long n, double a, const double* __restrict__ x, double b, const double* __restrict__ y,
                        double* __restrict__ out) {
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x)
        out[r] = a * x[r] + (b == 0.0 ? 0.0 : b * y[r]);
}

void ordered_allreduce(Comm& c, const double* in, double* out, size_t count, DBuf<double>& gall, cudaStream_t st) {
    if (gall.n < count * c.nranks) gall.alloc(count * c.nranks);
    c.allgather(in, gall.p, count, st);
    k_rank_sum<<<grid_for((long long)count, 256), 256, 0, st>>>(c.nranks, (long long)count, gall.p, out);
    count_launch();
    PDG_CHECK_LAUNCH();
}

std::vector<std::pair<int, int>> balanced_strips(int ny, int P) {
    require(P >= 1 && ny >= 2 * P, "distributed block: need at least two cell rows per rank");
    std::vector<std::pair<int, int>> out;
    const int base = ny / P, extra = ny % P;
    int r = 0;
    for (int k = 0; k < P; ++k) {
        const int h = base + (k < extra ? 1 : 0);
        out.push_back({r, r + h});
        r += h;
    }
    return out;
}

// halo lists for a CSR whose rows / columns have owners: recv[p] = columns owned by p that
// the rows owned by `me` read; send[p] = my columns that rows owned by p read
void halo_lists(const std::vector<long long>& off, const std::vector<int>& idx, const std::vector<int>& row_owner,
                const std::vector<int>& col_owner, int me, int P, std::vector<int>& peers,
                std::vector<std::vector<long long>>& send, std::vector<std::vector<long long>>& recv) {
    const long long rows = static_cast<long long>(row_owner.size());
    std::vector<std::vector<long long>> need(P);  // need[p]: columns not owned by p read by p's rows
    std::vector<int> mark(col_owner.size(), -1);
    std::vector<std::vector<char>> seen(P, std::vector<char>(col_owner.size(), 0));
    for (long long r = 0; r < rows; ++r) {
        const int o = row_owner[r];
        for (long long k = off[r]; k < off[r + 1]; ++k) {
            const int c = idx[k];
            if (col_owner[c] != o && !seen[o][c]) {
                seen[o][c] = 1;
                need[o].push_back(c);
            }
        }
    }
    (void)mark;
    peers.clear();
    send.clear();
    recv.clear();
    for (int p = 0; p < P; ++p) {
        if (p == me) continue;
        std::vector<long long> s, r;
        for (long long c : need[p])
            if (col_owner[c] == me) s.push_back(c);
        for (long long c : need[me])
            if (col_owner[c] == p) r.push_back(c);
        if (s.empty() && r.empty()) continue;
        std::sort(s.begin(), s.end());
        std::sort(r.begin(), r.end());
        peers.push_back(p);
        send.push_back(std::move(s));
        recv.push_back(std::move(r));
    }
}

}  // namespace

void nccl_unique_id(unsigned char* id) {
    ncclUniqueId u;
    PDG_NCCL(nccl().GetUniqueId(&u));
    std::memcpy(id, &u, sizeof(u));
}

std::unique_ptr<Comm> make_nccl_comm(int nranks, int rank, const unsigned char* id, int device) {
    require(nranks >= 1 && rank >= 0 && rank < nranks, "communicator: bad rank");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    auto c = std::make_unique<NcclComm>();
    c->rank = rank;
    c->nranks = nranks;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    PDG_CUDA(cudaSetDevice(device));
    PDG_NCCL(nccl().CommInitRank(&c->c, nranks, u, rank));
    return c;
}

std::unique_ptr<Comm> make_host_comm(int nranks, int rank, pdg_host_allgather_fn ag, pdg_host_exchange_fn ex, void* user) {
    require(nranks >= 1 && rank >= 0 && rank < nranks, "communicator: bad rank");
    require(ag && ex, "communicator: null callback");
    auto c = std::make_unique<HostComm>();
    c->rank = rank;
    c->nranks = nranks;
    c->ag = ag;
    c->ex = ex;
    c->user = user;
    return c;
}

// ---- Halo ---------------------------------------------------------------------
void Halo::build(const std::vector<int>& peers_, const std::vector<std::vector<long long>>& send,
                 const std::vector<std::vector<long long>>& recv, int ncomp_, long long stride_, cudaStream_t st) {
    peers = peers_;
    ncomp = ncomp_;
    stride = stride_;
    const size_t np = peers.size();
    sidx.clear();
    ridx.clear();
    sbuf.clear();
    rbuf.clear();
    sidx.resize(np);
    ridx.resize(np);
    sbuf.resize(np);
    rbuf.resize(np);
    for (size_t i = 0; i < np; ++i) {
        sidx[i].upload(send[i], st);
        ridx[i].upload(recv[i], st);
        sidx[i].n = send[i].size();
        ridx[i].n = recv[i].size();
        sbuf[i].alloc(std::max<size_t>(1, send[i].size() * ncomp));
        rbuf[i].alloc(std::max<size_t>(1, recv[i].size() * ncomp));
    }
}

void Halo::run(Comm& c, double* x, cudaStream_t st) {
    if (peers.empty()) return;
    std::vector<const double*> sp;
    std::vector<double*> rp;
    std::vector<size_t> sc, rc;
    for (size_t i = 0; i < peers.size(); ++i) {
        const long long ns = static_cast<long long>(sidx[i].n), nr = static_cast<long long>(ridx[i].n);
        if (ns) k_pack<<<grid_for(ns * ncomp, 256), 256, 0, st>>>(ns, ncomp, stride, sidx[i].p, x, sbuf[i].p);
        sp.push_back(sbuf[i].p);
        rp.push_back(rbuf[i].p);
        sc.push_back(static_cast<size_t>(ns) * ncomp);
        rc.push_back(static_cast<size_t>(nr) * ncomp);
    }
    count_launch(static_cast<int>(peers.size()));
    PDG_CHECK_LAUNCH();
    c.exchange(peers, sp, sc, rp, rc, st);
    for (size_t i = 0; i < peers.size(); ++i) {
        const long long nr = static_cast<long long>(ridx[i].n);
        if (nr) k_unpack<<<grid_for(nr * ncomp, 256), 256, 0, st>>>(nr, ncomp, stride, ridx[i].p, rbuf[i].p, x);
    }
    count_launch(static_cast<int>(peers.size()));
    PDG_CHECK_LAUNCH();
}

// ---- DistSub --------------------------------------------------------------------
void DistSub::setup(Comm& c, const HCsr& K, const std::vector<int>& block_of, const std::vector<std::pair<int, int>>& parts,
                    const std::vector<int>& node_of, const std::vector<double>& cx, const std::vector<double>& cy, int prof,
                    cudaStream_t st) {
    P = c.nranks;
    rank = c.rank;
    n = K.rows;
    require(static_cast<int>(parts.size()) == P, "distributed solve: one block range per rank");
    // separators: the first block of every rank but the first
    std::vector<std::vector<long long>> sep(std::max(P - 1, 0));
    std::vector<int> sep_of_block(static_cast<size_t>(parts.back().second) + 1, -1);
    for (int t = 0; t + 1 < P; ++t) sep_of_block[parts[t + 1].first] = t;
    std::vector<long long> I;
    const int b0 = parts[rank].first + (rank > 0 ? 1 : 0), b1 = parts[rank].second;
    for (int d = 0; d < n; ++d) {
        const int bl = block_of[d];
        if (sep_of_block[bl] >= 0) sep[sep_of_block[bl]].push_back(d);
        if (bl >= b0 && bl < b1 && sep_of_block[bl] < 0) I.push_back(d);
    }
    so.assign(P, 0);
    for (int t = 0; t + 1 < P; ++t) so[t + 1] = so[t] + static_cast<long long>(sep[t].size());
    ns = static_cast<int>(so[P - 1]);
    ni = static_cast<int>(I.size());
    require(ni > 0, "distributed solve: empty strip interior");
    t_top = rank > 0 ? rank - 1 : -1;
    t_bot = rank < P - 1 ? rank : -1;
    s_top = t_top >= 0 ? static_cast<int>(sep[t_top].size()) : 0;
    s_bot = t_bot >= 0 ? static_cast<int>(sep[t_bot].size()) : 0;
    std::vector<int> loc(n, -1);
    for (int i = 0; i < ni; ++i) loc[I[i]] = i;
    // interior matrix and its nested-dissection factor (compact node numbering)
    {
        std::vector<int> off(ni + 1, 0), idx;
        std::vector<double> val;
        std::vector<int> node_map(cx.size(), -1), nodes;
        std::vector<double> ncx, ncy;
        std::vector<int> nloc(ni);
        for (int i = 0; i < ni; ++i) {
            const long long d = I[i];
            for (int k = K.off[d]; k < K.off[d + 1]; ++k)
                if (loc[K.idx[k]] >= 0) {
                    idx.push_back(loc[K.idx[k]]);
                    val.push_back(K.val[k]);
                }
            off[i + 1] = static_cast<int>(idx.size());
            const int nd_ = node_of[d];
            if (node_map[nd_] < 0) {
                node_map[nd_] = static_cast<int>(ncx.size());
                ncx.push_back(cx[nd_]);
                ncy.push_back(cy[nd_]);
            }
            nloc[i] = node_map[nd_];
        }
        nd.prof_phase = prof;
        nd.factor(ni, off, idx, val, nloc, ncx, ncy, nd_leaf_dofs(128), 2, st);
    }
    la = std::make_unique<LaHandles>(st);
    // K_IS of the two separators: dense on the device for the spikes and the Schur products
    auto dense_is = [&](int t, DBuf<double>& D) {
        const int s = static_cast<int>(sep[t].size());
        D.alloc((size_t)ni * s);
        D.zero(st);
        std::vector<long long> pos;
        std::vector<double> val;
        for (int j = 0; j < s; ++j) {
            const long long d = sep[t][j];  // K symmetric: column d of K_IS = row d restricted to I
            for (int k = K.off[d]; k < K.off[d + 1]; ++k)
                if (loc[K.idx[k]] >= 0) {
                    pos.push_back((long long)j * ni + loc[K.idx[k]]);
                    val.push_back(K.val[k]);
                }
        }
        DBuf<long long> dp;
        DBuf<double> dv;
        dp.upload(pos, st);
        dv.upload(val, st);
        if (!pos.empty())
            k_dense_scatter<<<grid_for((long long)pos.size(), 256), 256, 0, st>>>((long long)pos.size(), dp.p, dv.p, D.p);
        PDG_CHECK_LAUNCH();
        PDG_CUDA(cudaStreamSynchronize(st));
    };
    auto sparse_si = [&](int t, DCsr& A) {  // K_SI rows of separator t, local interior columns
        std::vector<int> off(1, 0), idx;
        std::vector<double> val;
        for (long long d : sep[t]) {
            for (int k = K.off[d]; k < K.off[d + 1]; ++k)
                if (loc[K.idx[k]] >= 0) {
                    idx.push_back(loc[K.idx[k]]);
                    val.push_back(K.val[k]);
                }
            off.push_back(static_cast<int>(idx.size()));
        }
        pdg_csr h{static_cast<int>(sep[t].size()), ni, static_cast<int>(val.size()), off.data(), idx.data(), val.data()};
        csr_upload(A, h, st);
        PDG_CUDA(cudaStreamSynchronize(st));
    };
    auto spikes = [&](const DBuf<double>& D, int s, DBuf<double>& W) {
        W.alloc((size_t)ni * s);
        for (int c0 = 0; c0 < s; c0 += 2)
            nd.solve(D.p + (size_t)c0 * ni, ni, W.p + (size_t)c0 * ni, ni, std::min(2, s - c0), st);
        PDG_CUDA(cudaStreamSynchronize(st));
    };
    const int smax = std::max(1, static_cast<int>(std::max(s_top, s_bot)));
    int sall = 1;
    for (auto& v : sep) sall = std::max(sall, static_cast<int>(v.size()));
    // this rank's contributions: [D_top | D_bot | C_top,bot], each sall x sall (column-major, ld sall)
    const size_t bs = (size_t)sall * sall;
    DBuf<double> contrib(3 * bs);
    contrib.zero(st);
    const double one = 1.0, mone = -1.0;
    DBuf<double> Dt, Db;
    if (t_top >= 0) {
        dense_is(t_top, Dt);
        spikes(Dt, s_top, Wt);
        sparse_si(t_top, Ast);
        // K_SS of the own separator, then - K_IS^T W_top
        std::vector<long long> pos;
        std::vector<double> val;
        std::vector<int> sl(n, -1);
        for (int j = 0; j < s_top; ++j) sl[sep[t_top][j]] = j;
        for (int i = 0; i < s_top; ++i) {
            const long long d = sep[t_top][i];
            for (int k = K.off[d]; k < K.off[d + 1]; ++k)
                if (sl[K.idx[k]] >= 0) {
                    pos.push_back(i + (long long)sl[K.idx[k]] * sall);
                    val.push_back(K.val[k]);
                }
        }
        DBuf<long long> dp;
        DBuf<double> dv;
        dp.upload(pos, st);
        dv.upload(val, st);
        if (!pos.empty())
            k_dense_scatter<<<grid_for((long long)pos.size(), 256), 256, 0, st>>>((long long)pos.size(), dp.p, dv.p, contrib.p);
        PDG_CHECK_LAUNCH();
        PDG_DBLAS(cublasDgemm(la->blas, CUBLAS_OP_T, CUBLAS_OP_N, s_top, s_top, ni, &mone, Dt.p, ni, Wt.p, ni, &one, contrib.p, sall));
        PDG_CUDA(cudaStreamSynchronize(st));
    }
    if (t_bot >= 0) {
        dense_is(t_bot, Db);
        spikes(Db, s_bot, Wb);
        sparse_si(t_bot, Asb);
        PDG_DBLAS(cublasDgemm(la->blas, CUBLAS_OP_T, CUBLAS_OP_N, s_bot, s_bot, ni, &mone, Db.p, ni, Wb.p, ni, &one,
                              contrib.p + bs, sall));
        if (t_top >= 0)
            PDG_DBLAS(cublasDgemm(la->blas, CUBLAS_OP_T, CUBLAS_OP_N, s_top, s_bot, ni, &mone, Dt.p, ni, Wb.p, ni, &one,
                                  contrib.p + 2 * bs, sall));
        PDG_CUDA(cudaStreamSynchronize(st));
    }
    (void)smax;
    // separator Schur complement: the ranks' contributions in rank order, factored redundantly
    if (ns > 0) {
        DBuf<double> all;
        all.alloc(3 * bs * P);
        c.allgather(contrib.p, all.p, 3 * bs, st);
        const std::vector<double> h = all.download(st);
        std::vector<double> S((size_t)ns * ns, 0.0);
        auto add = [&](int ti, int tj, const double* blk, bool trans) {
            const int si = static_cast<int>(so[ti + 1] - so[ti]), sj = static_cast<int>(so[tj + 1] - so[tj]);
            for (int j = 0; j < sj; ++j)
                for (int i = 0; i < si; ++i) {
                    const double v = trans ? blk[j + (size_t)i * sall] : blk[i + (size_t)j * sall];
                    S[(size_t)(so[ti] + i) + (size_t)(so[tj] + j) * ns] += v;
                }
        };
        for (int r = 0; r < P; ++r) {
            const double* p = h.data() + 3 * bs * r;
            if (r > 0) add(r - 1, r - 1, p, false);
            if (r < P - 1) add(r, r, p + bs, false);
            if (r > 0 && r < P - 1) {
                add(r - 1, r, p + 2 * bs, false);
                add(r, r - 1, p + 2 * bs, true);
            }
        }
        Sfac.upload(S, st);
        PDG_DSOLVER(cusolverDnDpotrf_bufferSize(la->solver, CUBLAS_FILL_MODE_LOWER, ns, Sfac.p, ns, &lwork));
        work.alloc(std::max(lwork, 1));
        info.alloc(1);
        PDG_DSOLVER(cusolverDnDpotrf(la->solver, CUBLAS_FILL_MODE_LOWER, ns, Sfac.p, ns, work.p, lwork, info.p));
        int hinfo = 0;
        PDG_CUDA(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        PDG_CUDA(cudaStreamSynchronize(st));
        require(hinfo == 0, "distributed solve: separator Schur complement not positive definite");
    }
    I_d.upload(I, st);
    I_d.n = I.size();
    if (t_top >= 0) {
        Stop_d.upload(sep[t_top], st);
        Stop_d.n = sep[t_top].size();
    }
    bI.alloc((size_t)2 * ni);
    yI.alloc((size_t)2 * ni);
    g.alloc((size_t)2 * std::max(ns, 1));
    PDG_CUDA(cudaStreamSynchronize(st));
}

void DistSub::solve(Comm& c, const double* b, double* x, long long ld, int nrhs, cudaStream_t st) {
    require(nrhs >= 1 && nrhs <= 2, "distributed solve: at most 2 right-hand sides");
    k_gather<<<grid_for((long long)ni * nrhs, 256), 256, 0, st>>>(ni, nrhs, I_d.p, b, ld, bI.p, ni);
    count_launch();
    nd.solve(bI.p, ni, yI.p, ni, nrhs, st);
    if (ns > 0) {
        PDG_CUDA(cudaMemsetAsync(g.p, 0, sizeof(double) * 2 * ns, st));
        DBuf<double>& tmp = work;  // K_SI y (s x nrhs), reuses the factor workspace size check below
        const int smax = std::max(s_top, s_bot);
        if (tmp.n < (size_t)2 * smax) tmp.alloc((size_t)2 * smax);
        if (t_top >= 0) {
            k_csr_rows<<<grid_for((long long)s_top * nrhs, 256), 256, 0, st>>>(s_top, nrhs, Ast.off.p, Ast.idx.p, Ast.val.p, yI.p,
                                                                             ni, tmp.p, s_top);
            k_sep_rhs<<<grid_for((long long)s_top * nrhs, 256), 256, 0, st>>>(s_top, nrhs, Stop_d.p, b, ld, tmp.p, g.p, so[t_top], ns);
        }
        if (t_bot >= 0) {
            k_csr_rows<<<grid_for((long long)s_bot * nrhs, 256), 256, 0, st>>>(s_bot, nrhs, Asb.off.p, Asb.idx.p, Asb.val.p, yI.p,
                                                                             ni, tmp.p, s_bot);
            k_sep_rhs<<<grid_for((long long)s_bot * nrhs, 256), 256, 0, st>>>(s_bot, nrhs, nullptr, nullptr, 0, tmp.p, g.p,
                                                                            so[t_bot], ns);
        }
        count_launch(4);
        PDG_CHECK_LAUNCH();
        // one all-gather of the separator right-hand sides, summed in rank order
        DBuf<double>& gs = gsum;
        if (gs.n < (size_t)2 * ns) gs.alloc((size_t)2 * ns);
        ordered_allreduce(c, g.p, gs.p, (size_t)2 * ns, gall, st);
        PDG_DSOLVER(cusolverDnDpotrs(la->solver, CUBLAS_FILL_MODE_LOWER, ns, nrhs, Sfac.p, ns, gs.p, ns, info.p));
        const double mone = -1.0, one = 1.0;
        if (t_top >= 0)
            PDG_DBLAS(cublasDgemm(la->blas, CUBLAS_OP_N, CUBLAS_OP_N, ni, nrhs, s_top, &mone, Wt.p, ni, gs.p + so[t_top], ns,
                                  &one, yI.p, ni));
        if (t_bot >= 0)
            PDG_DBLAS(cublasDgemm(la->blas, CUBLAS_OP_N, CUBLAS_OP_N, ni, nrhs, s_bot, &mone, Wb.p, ni, gs.p + so[t_bot], ns,
                                  &one, yI.p, ni));
        if (t_top >= 0) {
            k_scatter<<<grid_for((long long)s_top * nrhs, 256), 256, 0, st>>>(s_top, nrhs, Stop_d.p, gs.p + so[t_top], ns, x, ld);
            count_launch();
        }
    }
    k_scatter<<<grid_for((long long)ni * nrhs, 256), 256, 0, st>>>(ni, nrhs, I_d.p, yI.p, ni, x, ld);
    count_launch();
    PDG_CHECK_LAUNCH();
}

// ---- DistBlock --------------------------------------------------------------------
void DistBlock::create(const SpatialOps& o, Comm* c, int m_, const double* theta, double tau_, double lambda_,
                       const pdg_gmres_opts& op_, cudaStream_t st) {
    ops = &o;
    ctx = o.ctx;
    comm = c;
    m = m_;
    tau = tau_;
    lambda = lambda_;
    opts = op_;
    require(m == 1 || m == 2, "distributed block: m must be 1 or 2");
    require(opts.tol > 0.0 && opts.tol < 1.0, "gmres: tol must be in (0,1)");
    require(opts.restart >= 1 && opts.max_iter >= 1, "gmres: bad iteration limits");
    require(tau > 0.0, "FixedStressSolver: tau must be positive");
    require(opts.sweeps == 1, "distributed block: one fixed-stress sweep per preconditioner application");
    P = c->nranks;
    rank = c->rank;
    const int nx = o.nx, ny = o.ny, nt = o.n_total(), nu = o.n_u, nq = o.n_q, np = o.n_p;
    strips = balanced_strips(ny, P);
    r0 = strips[rank].first;
    r1 = strips[rank].second;
    w = tau * 1.0;
    stab = opts.stab < 0.0 ? o.biot_b * o.biot_b / o.k_dr : opts.stab;
    require(lambda * (o.inv_m + stab) > 0.0, "fixed-stress: flow storage block must be negative definite");
    // ownership: cells by cell row, faces by face row (mesh.hpp:59-60), displacement dofs by cell
    std::vector<int> row_rank(ny);
    for (int k = 0; k < P; ++k)
        for (int j = strips[k].first; j < strips[k].second; ++j) row_rank[j] = k;
    std::vector<int> cell_own(np), face_own(nq), u_own(nu);
    std::vector<int> face_row(nq);
    const int nh = nx * (ny + 1);
    for (int cc = 0; cc < np; ++cc) cell_own[cc] = row_rank[cc / nx];
    for (int f = 0; f < nq; ++f) {
        face_row[f] = f < nh ? std::min(f / nx, ny - 1) : (f - nh) % ny;
        face_own[f] = row_rank[face_row[f]];
    }
    for (int d = 0; d < nu; ++d) u_own[d] = cell_own[d / 8];
    std::vector<int> comp_own(nt);
    for (int l = 0; l < nt; ++l) comp_own[l] = l < nu ? u_own[l] : l < nu + nq ? face_own[l - nu] : cell_own[l - nu - nq];
    nglob = (long long)m * nt;
    std::vector<int> glob_own(nglob);
    for (long long g = 0; g < nglob; ++g) glob_own[g] = comp_own[g % nt];
    own_rows_h.clear();
    for (long long g = 0; g < nglob; ++g)
        if (glob_own[g] == rank) own_rows_h.push_back(g);
    nown = static_cast<long long>(own_rows_h.size());
    own_rows.upload(own_rows_h, st);
    // operator: the strip's rows, halo of the x entries they read
    {
        SetupTimer t(SETUP_OPERATOR, st);
        op.build(o, m, theta, tau, st);
        op.set_strip(nx, ny, r0, r1, st);
    }
    {
        std::vector<long long> off;
        std::vector<int> idx;
        std::vector<double> val;
        op.to_csr(off, idx, val, st);
        std::vector<int> peers;
        std::vector<std::vector<long long>> send, recv;
        halo_lists(off, idx, glob_own, glob_own, rank, P, peers, send, recv);
        xhalo.build(peers, send, recv, 1, nglob, st);
    }
    xf.alloc(nglob);
    yf.alloc(nglob);
    xf.zero(st);
    // preconditioner: owned index lists, halos, D^{-1}, the two distributed inner solves
    std::vector<int> hoc, hof, hou;
    for (int cc = 0; cc < np; ++cc)
        if (cell_own[cc] == rank) hoc.push_back(cc);
    for (int f = 0; f < nq; ++f)
        if (face_own[f] == rank) hof.push_back(f);
    for (int d = 0; d < nu; ++d)
        if (u_own[d] == rank) hou.push_back(d);
    noc = static_cast<int>(hoc.size());
    nof = static_cast<int>(hof.size());
    nou = static_cast<int>(hou.size());
    oc.upload(hoc, st);
    of.upload(hof, st);
    ou.upload(hou, st);
    const HCsr hB = csr_download(o.B, st), hBt = csr_download(o.Bt, st), hE = csr_download(o.E, st);
    auto halo_of = [&](const HCsr& M, const std::vector<int>& rown, const std::vector<int>& cown, long long stride, Halo& H) {
        std::vector<long long> off(M.off.begin(), M.off.end());
        std::vector<int> peers;
        std::vector<std::vector<long long>> send, recv;
        halo_lists(off, M.idx, rown, cown, rank, P, peers, send, recv);
        H.build(peers, send, recv, m, stride, st);
    };
    halo_of(hB, face_own, cell_own, np, hfp);   // B rows (owned faces) read fp of cells
    halo_of(hBt, cell_own, face_own, nq, hq);   // B^T rows (owned cells) read q of faces
    halo_of(hE, u_own, cell_own, np, hp);       // E rows (owned u dofs) read p of cells
    std::vector<double> mp = o.m_p.download(st), di(np);
    for (int cc = 0; cc < np; ++cc) di[cc] = 1.0 / (-(lambda * (o.inv_m + stab)) * mp[cc]);
    dinv.upload(di, st);
    fp.alloc((size_t)m * np);
    pf.alloc((size_t)m * np);
    rq.alloc((size_t)m * nq);
    qf.alloc((size_t)m * nq);
    mech.alloc((size_t)m * nu);
    uf.alloc((size_t)m * nu);
    rfull.alloc((size_t)m * nt);
    for (auto* b : {&fp, &pf, &rq, &qf, &mech, &uf, &rfull}) b->zero(st);
    {
        // flux Schur complement in face-row blocks; displacement block in cell-row blocks
        const HCsr S = flow_schur_host(o, w, di, st);
        std::vector<int> node_f(nq);
        std::iota(node_f.begin(), node_f.end(), 0);
        std::vector<double> fcx, fcy;
        face_coords(nx, ny, fcx, fcy);
        flow.setup(*c, S, face_row, strips, node_f, fcx, fcy, PROF_FLOW_SOLVE, st);
        const HCsr A = csr_download(o.A, st);
        std::vector<int> blk_u(nu), node_u(nu);
        for (int d = 0; d < nu; ++d) {
            node_u[d] = d / 8;
            blk_u[d] = (d / 8) / nx;
        }
        std::vector<double> ccx(np), ccy(np);
        for (int cc = 0; cc < np; ++cc) {
            ccx[cc] = cc % nx + 0.5;
            ccy[cc] = cc / nx + 0.5;
        }
        mech_solver.setup(*c, A, blk_u, strips, node_u, ccx, ccy, PROF_A_SOLVE, st);
    }
    // GMRES buffers (owned rows)
    const int rs = opts.restart;
    V.alloc((size_t)nown * (rs + 1));
    Z.alloc((size_t)nown * rs);
    for (auto* b : {&wv, &x, &r, &cand, &t}) b->alloc(nown);
    ydev.alloc(rs + 2);
    dots.alloc(rs + 2);
    dsum.alloc(2 * rs + 4);
    if (!hhost) PDG_CUDA(cudaMallocHost(&hhost, sizeof(double) * (2 * rs + 4)));
    PDG_CUDA(cudaStreamSynchronize(st));
}

DistBlock::~DistBlock() {
    if (hhost) cudaFreeHost(hhost);
}

void DistBlock::apply(const double* x_own, double* y_own, cudaStream_t st) {
    k_scatter<<<grid_for(nown, 256), 256, 0, st>>>(nown, 1, own_rows.p, x_own, nown, xf.p, nglob);
    count_launch();
    xhalo.run(*comm, xf.p, st);
    op.apply_strip(xf.p, yf.p, st);
    k_gather<<<grid_for(nown, 256), 256, 0, st>>>(nown, 1, own_rows.p, yf.p, nglob, y_own, nown);
    count_launch();
    PDG_CHECK_LAUNCH();
}

void DistBlock::precondition(const double* r_own, double* z_own, cudaStream_t st) {
    const SpatialOps& o = *ops;
    const int nt = o.n_total(), nu = o.n_u, nq = o.n_q, np = o.n_p;
    k_scatter<<<grid_for(nown, 256), 256, 0, st>>>(nown, 1, own_rows.p, r_own, nown, rfull.p, nglob);
    k_d_fp<<<grid_for((long long)m * noc, 256), 256, 0, st>>>(m, noc, oc.p, np, nt, nu + nq, rfull.p, fp.p);
    count_launch(2);
    PDG_CHECK_LAUNCH();
    hfp.run(*comm, fp.p, st);
    k_d_rq<<<grid_for((long long)m * nof, 256), 256, 0, st>>>(m, nof, of.p, nq, np, nt, nu, w, rfull.p, fp.p, o.B.off.p,
                                                             o.B.idx.p, o.B.val.p, dinv.p, rq.p);
    count_launch();
    PDG_CHECK_LAUNCH();
    flow.solve(*comm, rq.p, qf.p, nq, m, st);
    hq.run(*comm, qf.p, st);
    k_d_p<<<grid_for((long long)m * noc, 256), 256, 0, st>>>(m, noc, oc.p, np, nq, w, fp.p, o.Bt.off.p, o.Bt.idx.p, o.Bt.val.p,
                                                            dinv.p, qf.p, pf.p);
    count_launch();
    PDG_CHECK_LAUNCH();
    hp.run(*comm, pf.p, st);
    k_d_mech<<<grid_for((long long)m * nou, 256), 256, 0, st>>>(m, nou, ou.p, nu, nt, np, w, o.biot_b, rfull.p, pf.p,
                                                               o.E.off.p, o.E.idx.p, o.E.val.p, mech.p);
    count_launch();
    PDG_CHECK_LAUNCH();
    mech_solver.solve(*comm, mech.p, uf.p, nu, m, st);
    k_d_collect<<<grid_for(nown, 256), 256, 0, st>>>(nown, own_rows.p, nt, nu, nq, np, uf.p, qf.p, pf.p, z_own);
    count_launch();
    PDG_CHECK_LAUNCH();
}

// ordered sums over the ranks of the local dots V_j . w, j < ncols, into out (device): no
// host round trip (NCCL runs on the stream; the host backend synchronizes inside)
void DistBlock::multidot_dev(const double* Vb, int ncols, const double* wv_, double* out, cudaStream_t st) {
    if (part.n < (size_t)kDotBlocks * ncols) part.alloc((size_t)kDotBlocks * ncols);
    k_dot_partials<<<kDotBlocks, kDotThreads, 0, st>>>(nown, ncols, Vb, wv_, part.p);
    k_dot_final<<<1, 64, 0, st>>>(kDotBlocks, ncols, part.p, dots.p);
    count_launch(2);
    PDG_CHECK_LAUNCH();
    ordered_allreduce(*comm, dots.p, out, ncols, gbuf, st);
}

double DistBlock::dot_sum(const double* a, const double* b, cudaStream_t st) {
    multidot_dev(a, 1, b, dsum.p, st);
    PDG_CUDA(cudaMemcpyAsync(hhost, dsum.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    return hhost[0];
}

// GMRES (gmres.hpp:40-139) on the owned rows; every reduction is a rank-ordered sum, so all
// ranks hold the same Hessenberg columns and make the same decisions. Candidate x + Z y
// (flexible) or x + P(V y) (reference), judged by the recomputed true residual.
void DistBlock::solve(const double* b, double* x_out, pdg_report* rep) {
    cudaStream_t st = ctx->stream;
    const long long n = nown;
    const unsigned gr = grid_for(n, 256);
    const long long launches0 = g_launches;
    cudaEvent_t e0, e1;
    PDG_CUDA(cudaEventCreate(&e0));
    PDG_CUDA(cudaEventCreate(&e1));
    PDG_CUDA(cudaEventRecord(e0, st));
    std::vector<double> hist;
    auto nrm = [&](const double* v) { return std::sqrt(dot_sum(v, v, st)); };
    const double bnorm = nrm(b);
    bool converged = false;
    int total = 0;
    double true_res = bnorm;
    const bool flexible = opts.candidate == 1;
    if (bnorm <= 1e-14) {  // gmres.hpp:56-62
        PDG_CUDA(cudaMemsetAsync(x_out, 0, sizeof(double) * n, st));
        converged = true;
        hist.push_back(bnorm);
        true_res = 0.0;
    } else {
        PDG_CUDA(cudaMemsetAsync(x.p, 0, sizeof(double) * n, st));
        hist.push_back(true_res);
        bool x_zero = true;
        const int restart = opts.restart, max_iter = opts.max_iter;
        while (total < max_iter) {
            if (x_zero) {
                PDG_CUDA(cudaMemcpyAsync(r.p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
            } else {
                apply(x.p, t.p, st);
                k_axpby<<<gr, 256, 0, st>>>(n, 1.0, b, -1.0, t.p, r.p);
                count_launch();
            }
            const double beta = nrm(r.p);
            if (beta / bnorm <= opts.tol) break;
            const int mm = std::min(restart, max_iter - total);
            std::vector<double> H((size_t)(mm + 1) * mm, 0.0);
            auto h = [&](int i, int j) -> double& { return H[(size_t)j * (mm + 1) + i]; };
            k_axpby<<<gr, 256, 0, st>>>(n, 1.0 / beta, r.p, 0.0, nullptr, V.p);
            count_launch();
            bool done = false;
            double* hd = dsum.p;  // [h pass 1 (k+1) | h pass 2 (k+1) | ||w||^2, ||w||]
            std::vector<double> cs(mm), sn(mm), gq(mm + 1, 0.0);
            gq[0] = beta;
            for (int k = 0; k < mm && !done; ++k) {
                double* vk = V.p + (size_t)k * n;
                double* zk = flexible ? Z.p + (size_t)k * n : cand.p;
                precondition(vk, zk, st);
                apply(zk, wv.p, st);
                // classical Gram-Schmidt, two passes, and the norm: rank-ordered sums on the stream,
                // the Hessenberg column comes back in one transfer
                for (int pass = 0; pass < 2; ++pass) {
                    multidot_dev(V.p, k + 1, wv.p, hd + (size_t)pass * (k + 1), st);
                    k_sub_vh<<<gr, 256, 0, st>>>(n, k + 1, V.p, hd + (size_t)pass * (k + 1), wv.p);
                    count_launch();
                }
                multidot_dev(wv.p, 1, wv.p, hd + 2 * (k + 1), st);
                k_sqrt_scale<<<gr, 256, 0, st>>>(n, hd + 2 * (k + 1), wv.p, V.p + (size_t)(k + 1) * n, hd + 2 * (k + 1) + 1);
                count_launch();
                PDG_CUDA(cudaMemcpyAsync(hhost, hd, sizeof(double) * (2 * (k + 1) + 2), cudaMemcpyDeviceToHost, st));
                PDG_CUDA(cudaStreamSynchronize(st));
                for (int pass = 0; pass < 2; ++pass)
                    for (int i = 0; i <= k; ++i) h(i, k) += hhost[(size_t)pass * (k + 1) + i];
                h(k + 1, k) = hhost[2 * (k + 1) + 1];
                double cn = 0.0;
                for (int i = 0; i <= mm; ++i) cn += h(i, k) * h(i, k);
                const bool breakdown = h(k + 1, k) <= 1e-14 * std::sqrt(cn);
                ++total;
                // residual estimate || beta e1 - H y || by Givens rotations (flexible candidate)
                double hk_ = h(0, k);
                for (int i = 0; i < k; ++i) hk_ = -sn[i] * hk_ + cs[i] * h(i + 1, k);
                const double rr = std::hypot(hk_, h(k + 1, k));
                cs[k] = rr == 0.0 ? 1.0 : hk_ / rr;
                sn[k] = rr == 0.0 ? 0.0 : h(k + 1, k) / rr;
                gq[k + 1] = -sn[k] * gq[k];
                gq[k] = cs[k] * gq[k];
                const bool cycle_end = breakdown || k == mm - 1 || total >= max_iter;
                if (flexible && std::fabs(gq[k + 1]) > opts.tol * bnorm && !cycle_end) {
                    hist.push_back(std::fabs(gq[k + 1]));  // estimate; the stop is confirmed explicitly
                    continue;
                }
                std::vector<double> hk((size_t)(k + 2) * (k + 1));
                for (int j = 0; j <= k; ++j)
                    for (int i = 0; i < k + 2; ++i) hk[(size_t)j * (k + 2) + i] = h(i, j);
                std::vector<double> e1v(k + 2, 0.0), tau_(k + 1), nrm_(k + 1), yv(k + 1);
                std::vector<int> piv(k + 1);
                e1v[0] = beta;
                ls_colpiv_raw(hk.data(), k + 2, k + 1, e1v.data(), tau_.data(), nrm_.data(), piv.data(), yv.data());
                PDG_CUDA(cudaMemcpyAsync(ydev.p, yv.data(), sizeof(double) * (k + 1), cudaMemcpyHostToDevice, st));
                if (flexible) {
                    k_vy<<<gr, 256, 0, st>>>(n, k + 1, Z.p, ydev.p, x.p, cand.p);
                    count_launch();
                } else {  // x + P(V y)
                    k_vy<<<gr, 256, 0, st>>>(n, k + 1, V.p, ydev.p, nullptr, t.p);
                    count_launch();
                    precondition(t.p, r.p, st);
                    k_axpby<<<gr, 256, 0, st>>>(n, 1.0, x.p, 1.0, r.p, cand.p);
                    count_launch();
                }
                // the true residual (gmres.hpp:68-72)
                apply(cand.p, t.p, st);
                k_axpby<<<gr, 256, 0, st>>>(n, 1.0, b, -1.0, t.p, r.p);
                count_launch();
                true_res = nrm(r.p);
                hist.push_back(true_res);
                const bool ok = true_res / bnorm <= opts.tol;
                if (ok || cycle_end) {  // else the cycle goes on (gmres.hpp:118-131)
                    PDG_CUDA(cudaMemcpyAsync(x.p, cand.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
                    x_zero = false;
                    done = true;
                    converged = ok;
                }
            }
            if (converged) break;
        }
        PDG_CUDA(cudaMemcpyAsync(x_out, x.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    }
    const double final_rel = bnorm > 0.0 ? true_res / bnorm : 0.0;
    if (!converged) converged = final_rel <= opts.tol;
    PDG_CUDA(cudaEventRecord(e1, st));
    PDG_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    PDG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (rep) {
        rep->converged = converged;
        rep->iterations = total;
        rep->final_rel_res = final_rel;
        rep->history_len = static_cast<int>(hist.size());
        if (rep->history)
            for (int i = 0; i < std::min<int>(rep->history_cap, (int)hist.size()); ++i) rep->history[i] = hist[i];
        rep->device_ms = ms;
        rep->kernel_launches = static_cast<int>(g_launches - launches0);
    }
    if (!converged) {
        char buf[64];
        std::snprintf(buf, sizeof(buf), "%f", final_rel);
        throw Error(PDG_NOT_CONVERGED, "slab block 0: GMRES did not converge (rel res " + std::string(buf) + ")");
    }
}

}  // namespace pdg
