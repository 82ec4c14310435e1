// Device-resident spatial operators (SpatialOperators, assembly.hpp:38-52).
#pragma once

#include <memory>

#include "common.cuh"

namespace pdg {

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
};

struct SpatialOps {
    Ctx* ctx = nullptr;
    int nx = 0, ny = 0;
    int nz = 0;  // > 0: 3D mesh (assembly3d.cu), 24 displacement dofs per cell
    int n_u = 0, n_q = 0, n_p = 0;
    double biot_b = 0.8, inv_m = 0.1, k_dr = 2.0;
    DCsr A, M_q, B, E;  // as assembled (ascending columns per row)
    DCsr Et, Bt;        // transposes, entries in ascending source row
    DBuf<double> m_p;   // n_p
    DBuf<signed char> q_constrained;
    // problem description kept for rhs assembly (pdg_ops_assemble path or upload + problem)
    bool has_problem = false;
    pdg_problem prob{};
    pdg_problem3 prob3{};
    int dofs_per_cell() const { return nz > 0 ? 24 : 8; }
    std::vector<double> k_cells;
    int n_total() const { return n_u + n_q + n_p; }
};

void csr_upload(DCsr& d, const pdg_csr& h, cudaStream_t st);
void csr_transpose(const DCsr& a, DCsr& t, cudaStream_t st);
void csr_spmv(const DCsr& a, const double* x, double* y, cudaStream_t st);  // order-fixed, thread per row
void assemble_ops_device(SpatialOps& ops, const pdg_problem& p, cudaStream_t st);
void assemble_ops_device3(SpatialOps& ops, const pdg_problem3& p, cudaStream_t st);
void assemble_rhs_device3(const SpatialOps& ops, double t, double* u, double* q, double* p, cudaStream_t st);
void assemble_rhs_sampled_device3(const SpatialOps& ops, const pdg_rhs_samples& samples, double* u, double* q, double* p,
                                  cudaStream_t st);
void assemble_rhs_sampled_device(const SpatialOps& ops, const pdg_rhs_samples& samples, double* u, double* q, double* p,
                                 cudaStream_t st);
void assemble_rhs_device(const SpatialOps& ops, double t, double* u, double* q, double* p, cudaStream_t st);

}  // namespace pdg
