// Per-phase CUDA-event profiler behind pdg_profile_* (see common.cuh).
#include <chrono>
#include <mutex>

#include "common.cuh"

namespace pdg {

namespace {
struct Pending {
    int phase;
    cudaEvent_t a, b;
    double bytes;
};
struct State {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    std::vector<Pending> pending;
    double ms[PROF_NPHASES] = {};
    long long calls[PROF_NPHASES] = {};
    double bytes[PROF_NPHASES] = {};
};
State& st() {
    static State s;
    return s;
}
void resolve() {
    State& s = st();
    for (const Pending& p : s.pending) {
        float t = 0.f;
        cudaEventSynchronize(p.b);
        cudaEventElapsedTime(&t, p.a, p.b);
        s.ms[p.phase] += t;
        s.calls[p.phase] += 1;
        s.bytes[p.phase] += p.bytes;
        s.pool.push_back(p.a);
        s.pool.push_back(p.b);
    }
    s.pending.clear();
}
}  // namespace

bool prof_enabled() { return st().on; }

cudaEvent_t prof_event() {
    State& s = st();
    if (s.pool.empty()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
    cudaEvent_t e = s.pool.back();
    s.pool.pop_back();
    return e;
}

namespace {
double g_setup[SETUP_NSTAGES] = {};
}
void setup_add(int stage, double seconds) {
    if (stage >= 0 && stage < SETUP_NSTAGES) g_setup[stage] += seconds;
}
double setup_clock() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void prof_push(int phase, cudaEvent_t a, cudaEvent_t b, double bytes) {
    State& s = st();
    s.pending.push_back({phase, a, b, bytes});
    if (s.pending.size() > 8192) resolve();
}

}  // namespace pdg

extern "C" {
void pdg_profile_enable(int on) { pdg::st().on = on != 0; }
void pdg_profile_reset(void) {
    pdg::resolve();
    pdg::State& s = pdg::st();
    for (int i = 0; i < pdg::PROF_NPHASES; ++i) {
        s.ms[i] = 0.0;
        s.calls[i] = 0;
        s.bytes[i] = 0.0;
    }
}
void pdg_setup_reset(void) {
    for (int i = 0; i < pdg::SETUP_NSTAGES; ++i) pdg::g_setup[i] = 0.0;
}
int pdg_setup_read(double* seconds, int n) {
    if (!seconds || n < 0) return PDG_INVALID_ARGUMENT;
    for (int i = 0; i < n && i < pdg::SETUP_NSTAGES; ++i) seconds[i] = pdg::g_setup[i];
    return pdg::SETUP_NSTAGES;
}
int pdg_profile_read(int phase, double* ms, long long* calls, double* alg_bytes) {
    if (phase < 0 || phase >= pdg::PROF_NPHASES) return PDG_INVALID_ARGUMENT;
    pdg::resolve();
    pdg::State& s = pdg::st();
    if (ms) *ms = s.ms[phase];
    if (calls) *calls = s.calls[phase];
    if (alg_bytes) *alg_bytes = s.bytes[phase];
    return PDG_OK;
}
}
