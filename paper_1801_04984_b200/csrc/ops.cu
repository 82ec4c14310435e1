// Device CSR utilities: upload, deterministic transpose, order-fixed SpMV.
#include <cub/cub.cuh>

#include "ops.cuh"

namespace pdg {

void csr_upload(DCsr& d, const pdg_csr& h, cudaStream_t st) {
    require(h.rows >= 0 && h.cols >= 0 && h.nnz >= 0, "pdg_ops_upload: negative CSR dimensions");
    require(h.row_offsets != nullptr, "pdg_ops_upload: null row_offsets");
    require(h.row_offsets[0] == 0 && h.row_offsets[h.rows] == h.nnz, "pdg_ops_upload: CSR offsets inconsistent with nnz");
    d.rows = h.rows;
    d.cols = h.cols;
    d.nnz = h.nnz;
    d.off.upload(h.row_offsets, h.rows + 1, st);
    d.idx.alloc(h.nnz);
    d.val.alloc(h.nnz);
    if (h.nnz) {
        PDG_CUDA(cudaMemcpyAsync(d.idx.p, h.col_indices, sizeof(int) * h.nnz, cudaMemcpyHostToDevice, st));
        PDG_CUDA(cudaMemcpyAsync(d.val.p, h.values, sizeof(double) * h.nnz, cudaMemcpyHostToDevice, st));
    }
}

__global__ void k_count_cols(int rows, const int* off, const int* idx, int* cnt) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x)
        for (int k = off[r]; k < off[r + 1]; ++k) atomicAdd(&cnt[idx[k]], 1);
}

__global__ void k_fill_t(int rows, const int* off, const int* idx, const double* val, int* fill, int* tidx,
                         double* tval) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x)
        for (int k = off[r]; k < off[r + 1]; ++k) {
            const int pos = atomicAdd(&fill[idx[k]], 1);
            tidx[pos] = r;
            tval[pos] = val[k];
        }
}

// Restore ascending source-row order inside each transposed row (the atomic
// fill order is arbitrary); insertion sort, rows are short.
__global__ void k_sort_rows(int rows, const int* off, int* idx, double* val) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
        const int b = off[r], e = off[r + 1];
        for (int i = b + 1; i < e; ++i) {
            const int ki = idx[i];
            const double vi = val[i];
            int j = i - 1;
            while (j >= b && idx[j] > ki) {
                idx[j + 1] = idx[j];
                val[j + 1] = val[j];
                --j;
            }
            idx[j + 1] = ki;
            val[j + 1] = vi;
        }
    }
}

void csr_transpose(const DCsr& a, DCsr& t, cudaStream_t st) {
    t.rows = a.cols;
    t.cols = a.rows;
    t.nnz = a.nnz;
    DBuf<int> cnt(static_cast<size_t>(a.cols) + 1);
    cnt.zero(st);
    t.off.alloc(static_cast<size_t>(a.cols) + 1);
    t.idx.alloc(a.nnz);
    t.val.alloc(a.nnz);
    if (a.rows) {
        k_count_cols<<<grid_for(a.rows, 256), 256, 0, st>>>(a.rows, a.off.p, a.idx.p, cnt.p);
        PDG_CHECK_LAUNCH();
    }
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt.p, t.off.p, a.cols + 1, st);
    DBuf<unsigned char> tmp(tmp_bytes + 1);
    cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, cnt.p, t.off.p, a.cols + 1, st);
    DBuf<int> fill(static_cast<size_t>(a.cols) + 1);
    PDG_CUDA(cudaMemcpyAsync(fill.p, t.off.p, sizeof(int) * (a.cols + 1), cudaMemcpyDeviceToDevice, st));
    if (a.rows) {
        k_fill_t<<<grid_for(a.rows, 256), 256, 0, st>>>(a.rows, a.off.p, a.idx.p, a.val.p, fill.p, t.idx.p, t.val.p);
        PDG_CHECK_LAUNCH();
    }
    if (t.rows) {
        k_sort_rows<<<grid_for(t.rows, 256), 256, 0, st>>>(t.rows, t.off.p, t.idx.p, t.val.p);
        PDG_CHECK_LAUNCH();
    }
    PDG_CUDA(cudaStreamSynchronize(st));
}

// y_i = sum_k v_k x_{c_k}, s from 0.0, stored order, no FMA (sparse.hpp:30-40).
template <typename OffT>
__global__ void k_csr_spmv(int rows, const OffT* __restrict__ off, const int* __restrict__ idx,
                           const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (OffT k = off[r]; k < off[r + 1]; ++k) s = __dadd_rn(s, __dmul_rn(__ldg(&val[k]), __ldg(&x[__ldg(&idx[k])])));
        y[r] = s;
    }
}

void csr_spmv(const DCsr& a, const double* x, double* y, cudaStream_t st) {
    if (!a.rows) return;
    k_csr_spmv<int><<<grid_for(a.rows, 256), 256, 0, st>>>(a.rows, a.off.p, a.idx.p, a.val.p, x, y);
    count_launch();
    PDG_CHECK_LAUNCH();
}

void spmv_csr_device(int rows, const long long* off, const int* idx, const double* val, const double* x, double* y,
                     cudaStream_t st) {
    if (!rows) return;
    k_csr_spmv<long long><<<grid_for(rows, 256), 256, 0, st>>>(rows, off, idx, val, x, y);
    count_launch();
    PDG_CHECK_LAUNCH();
}

}  // namespace pdg
