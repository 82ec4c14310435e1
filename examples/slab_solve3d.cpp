// Host C++ over the C ABI, 3D extension: a BASELINE config-2-type problem (n^3 hexahedra,
// dG(0), fixed bottom, loaded drained top, 8 permeability layers) assembled on the device
// and solved for its first slab; a second argument "fast" selects SolveOptions::fast (the
// fp32-stored streaming factor; it only differs from parity mode where the displacement solve
// streams, i.e. from about 14^3). Build:
//   g++ -std=c++17 -O2 -I include examples/slab_solve3d.cpp
//       -L paper_1801_04984_b200/_lib -lporodg_b200 -Wl,-rpath,$PWD/paper_1801_04984_b200/_lib
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "porodg_b200.hpp"

int main(int argc, char** argv) {
    using namespace porodg_b200;
    const int n = argc > 1 ? std::atoi(argv[1]) : 8;
    const bool fast = argc > 2 && std::string(argv[2]) == "fast";
    pdg_problem3 p{};
    p.nx = p.ny = p.nz = n;
    p.lx = p.ly = p.lz = 1.0;
    p.lambda = 1e4 * 0.3 / ((1.3) * (1.0 - 0.6));
    p.mu = 1e4 / 2.6;
    p.k_perm = 1.0;
    p.eta = 1.0;
    p.biot_m = 1e3;
    p.biot_b = 0.9;
    p.penalty = 10.0;
    std::vector<double> k(static_cast<size_t>(n) * n * n);
    for (int c = 0; c < n * n * n; ++c) k[c] = std::pow(10.0, -3.0 + 3.0 * ((c / (n * n)) * 8 / n) / 8.0);  // 8 layers
    p.k_perm_cells = k.data();
    for (int s = 0; s < 6; ++s) {
        p.disp_kind[s] = s == 4 ? 0 : 1;  // zlo fixed, everything else traction
        p.flow_kind[s] = s == 5 ? 0 : 1;  // zhi drained, no flux elsewhere
    }
    p.disp_data[5][2] = -1.0;  // unit load on the top
    try {
        Context ctx(0);
        SpatialOperators ops(ctx, p);
        long long sz[7];
        check(pdg_ops_sizes(ops.get(), sz));
        const long long nt = sz[0] + sz[1] + sz[2];
        std::vector<double> u(sz[0]), q(sz[1]), pr(sz[2]);
        check(pdg_ops_rhs(ops.get(), 0.0, u.data(), q.data(), pr.data()));
        const double tau = 0.1;
        SolveOptions opt;
        opt.gmres.restart = 50;
        opt.fast = fast;
        SlabSolver slab(ops, 0, tau, opt);
        // first slab from rest: R = tau b(t_1) (slab.hpp:76-84 with zero jump data)
        std::vector<double> rhs(nt);
        for (long long i = 0; i < sz[0]; ++i) rhs[i] = tau * u[i];
        for (long long i = 0; i < sz[1]; ++i) rhs[sz[0] + i] = tau * q[i];
        for (long long i = 0; i < sz[2]; ++i) rhs[sz[0] + sz[1] + i] = tau * pr[i];
        auto [x, rep] = slab.solve(rhs);
        if (!rep.converged) return 1;
        auto [res, scale] = mass_residual(ops, 0, tau, rhs, x);
        double worst_mass = 0.0;
        for (double v : res) worst_mass = std::fmax(worst_mass, v);
        worst_mass = scale > 0.0 ? worst_mass / scale : 0.0;
        const int worst_it = rep.iterations;
        double uz_min = 0.0;
        for (long long i = 2; i < sz[0]; i += 3) uz_min = std::fmin(uz_min, x[i]);
        std::printf("config2-type %d^3 (%s mode): n_total=%lld iterations=%d mass max|res|/scale=%.3e min u_z=%.6e\n", n, fast ? "fast" : "parity", nt, worst_it,
                    worst_mass, uz_min);
        return 0;
    } catch (const std::exception& e) {
        std::printf("error: %s\n", e.what());
        return 2;
    }
}
