// Shared device/host helpers of the porodg_b200 library (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "porodg_b200.h"

namespace pdg {

// Error carrying a pdg_status; converted to a return code at the C ABI.
struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#define PDG_CUDA(call)                                                                                    \
    do {                                                                                                  \
        cudaError_t e_ = (call);                                                                          \
        if (e_ != cudaSuccess)                                                                            \
            throw ::pdg::Error(e_ == cudaErrorMemoryAllocation ? PDG_OUT_OF_MEMORY : PDG_CUDA_ERROR,      \
                               std::string(#call) + ": " + cudaGetErrorString(e_));                       \
    } while (0)

#define PDG_CHECK_LAUNCH() PDG_CUDA(cudaGetLastError())

inline void require(bool ok, const std::string& msg) {
    if (!ok) throw Error(PDG_INVALID_ARGUMENT, msg);
}

// RAII device buffer.
template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) {
        o.p = nullptr;
        o.n = 0;
    }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) PDG_CUDA(cudaMalloc(&p, count * sizeof(T)));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void upload(const T* h, size_t count, cudaStream_t s = 0) {
        if (count > n) alloc(count);
        if (count) PDG_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void upload(const std::vector<T>& h, cudaStream_t s = 0) { upload(h.data(), h.size(), s); }
    std::vector<T> download(cudaStream_t s = 0) const {
        std::vector<T> h(n);
        if (n) {
            PDG_CUDA(cudaMemcpyAsync(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, s));
            PDG_CUDA(cudaStreamSynchronize(s));
        }
        return h;
    }
    void zero(cudaStream_t s = 0) {
        if (n) PDG_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
    }
};

// Device CSR (int32 offsets/indices, fp64 values).
struct DCsr {
    int rows = 0, cols = 0, nnz = 0;
    DBuf<int> off, idx;
    DBuf<double> val;
};

// Host CSR mirror used during setup.
struct HCsr {
    int rows = 0, cols = 0;
    std::vector<int> off, idx;
    std::vector<double> val;
    int nnz() const { return static_cast<int>(val.size()); }
};

inline int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

inline unsigned grid_for(long long n, int block, int max_blocks_per_sm = 8) {
    long long g = (n + block - 1) / block;
    const long long cap = static_cast<long long>(num_sms()) * max_blocks_per_sm;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return static_cast<unsigned>(g);
}

// Kernel launch counter (reported as gpu_launches by bench.py).
extern thread_local long long g_launches;
inline void count_launch(int n = 1) { g_launches += n; }

// Per-phase device timing with CUDA events on the launching stream
// (pdg_profile_*). A ProfScope records an event pair around a phase when
// profiling is enabled; the pairs are resolved at read time.
enum ProfPhase { PROF_SPMV = 0, PROF_A_SOLVE = 1, PROF_FLOW_SOLVE = 2, PROF_PRE_OTHER = 3, PROF_KRYLOV = 4,
                 PROF_SLAB = 5, PROF_NPHASES = 6 };
bool prof_enabled();
void prof_push(int phase, cudaEvent_t a, cudaEvent_t b, double bytes);
cudaEvent_t prof_event();
struct ProfScope {
    int phase;
    cudaStream_t st;
    double bytes;
    cudaEvent_t a = nullptr;
    ProfScope(int ph, cudaStream_t s, double b) : phase(ph), st(s), bytes(b) {
        if (prof_enabled()) {
            a = prof_event();
            cudaEventRecord(a, st);
        }
    }
    ~ProfScope() {
        if (a) {
            cudaEvent_t b = prof_event();
            cudaEventRecord(b, st);
            prof_push(phase, a, b, bytes);
        }
    }
};

// Setup stage timers (host wall clock, the stream synchronized at the end of each
// stage) behind pdg_setup_read: assembly, and per nested-dissection factor (A and the
// flow Schur complement) the analysis (graph + dissection + dense-front maps, host),
// the numeric factorization (cuSOLVER/cuBLAS on the fronts, device) and the solve
// schedule (task lists, host + upload); the space-time operator build; the whole
// block / slab solver construction.
enum SetupStage { SETUP_ASSEMBLE = 0, SETUP_A_ANALYSIS = 1, SETUP_A_FACTOR = 2, SETUP_A_SCHEDULE = 3,
                  SETUP_F_ANALYSIS = 4, SETUP_F_FACTOR = 5, SETUP_F_SCHEDULE = 6, SETUP_OPERATOR = 7,
                  SETUP_SOLVER_TOTAL = 8, SETUP_NSTAGES = 9 };
void setup_add(int stage, double seconds);
double setup_clock();  // seconds, monotonic
struct SetupTimer {
    int stage;
    cudaStream_t st;
    double t0;
    SetupTimer(int s, cudaStream_t stream) : stage(s), st(stream), t0(setup_clock()) {}
    void next(int s) {  // close the current stage, open stage s
        cudaStreamSynchronize(st);
        const double t = setup_clock();
        setup_add(stage, t - t0);
        stage = s;
        t0 = t;
    }
    ~SetupTimer() {
        cudaStreamSynchronize(st);
        setup_add(stage, setup_clock() - t0);
    }
};

}  // namespace pdg
