// Host C++ over the C ABI: BASELINE config 0 (16^2, dG(0)), first slab,
// assembled on the device, solved by SlabSolver. Build:
//   g++ -std=c++17 -O2 -I include examples/slab_solve.cpp
//       -L paper_1801_04984_b200/_lib -lporodg_b200 -Wl,-rpath,$PWD/paper_1801_04984_b200/_lib
#include <cmath>
#include <cstdio>
#include <vector>

#include "porodg_b200.hpp"

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
    const int disp[4] = {1, 1, 0, 1};  // left, right traction-free; bottom fixed; top traction
    const int flow[4] = {1, 1, 1, 0};  // no flux except top pressure
    for (int s = 0; s < 4; ++s) {
        p.disp_kind[s] = disp[s];
        p.flow_kind[s] = flow[s];
    }
    p.disp_data[3][1] = -1.0;
    try {
        Context ctx(0);
        SpatialOperators ops(ctx, p);
        const long long nt = ops.n_total();
        long long sz[7];
        check(pdg_ops_sizes(ops.get(), sz));
        std::vector<double> u(sz[0]), q(sz[1]), pr(sz[2]);
        check(pdg_ops_rhs(ops.get(), 0.1, u.data(), q.data(), pr.data()));
        const double tau = 0.1;
        std::vector<double> rhs;  // R_0 = tau * w_0 * b(t_1) (zero initial jump), w_0 = 1 for dG(0)
        for (double v : u) rhs.push_back(tau * v);
        for (double v : q) rhs.push_back(tau * v);
        for (double v : pr) rhs.push_back(tau * v);
        SolveOptions opt;
        opt.gmres.restart = 50;
        SlabSolver slab(ops, 0, tau, opt);
        auto [x, rep] = slab.solve(rhs);
        double nrm = 0.0;
        for (double v : x) nrm += v * v;
        std::printf("config0 slab 0: converged=%d iterations=%d rel_res=%.3e |x|=%.6e n_total=%lld\n", rep.converged,
                    rep.iterations, rep.final_relative_residual, std::sqrt(nrm), nt);
        // local mass balance of the solved slab (slab.hpp:292-318)
        auto [res, scale] = mass_residual(ops, 0, tau, rhs, x);
        double worst = 0.0;
        for (double v : res) worst = std::fmax(worst, v);
        std::printf("mass balance: max|res|/scale=%.3e\n", scale > 0.0 ? worst / scale : 0.0);
        // the same slab by the fixed-stress method (march.hpp:80-108)
        FixedStressSolver fs(ops, 0, tau);
        auto [xf, rf] = fs.solve(rhs);
        double d = 0.0;
        for (size_t i = 0; i < x.size(); ++i) d += (x[i] - xf[i]) * (x[i] - xf[i]);
        std::printf("fixed-stress: converged=%d sweeps=%d |x_fs - x|/|x|=%.3e\n", rf.converged, rf.iterations,
                    std::sqrt(d / nrm));
        return rep.converged && rf.converged ? 0 : 1;
    } catch (const std::exception& e) {
        std::printf("error: %s\n", e.what());
        return 2;
    }
}
