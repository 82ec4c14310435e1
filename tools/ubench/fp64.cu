// Micro-benchmark: FP64 FMA latency / throughput and shuffle+add latency on this GPU.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
template <int CH>
__global__ void k_fma(int iters, double* out, long long* cyc) {
    double a[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * 1e-3 + i;
    const double m = 1.0000001, c = 1e-9;
    const long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) a[i] = fma(a[i], m, c);
    }
    const long long c1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
}
__global__ void k_shfl(int iters, double* out, long long* cyc) {
    double a = threadIdx.x * 1e-3;
    const long long c0 = clock64();
    for (int it = 0; it < iters; ++it) a += __shfl_xor_sync(0xffffffffu, a, 1 + (it & 15));
    const long long c1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
}
template <int CH>
void run(int threads) {
    double* out; long long* cyc; long long h;
    cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&cyc, 148 * 8);
    const int iters = 4096;
    k_fma<CH><<<148, threads>>>(iters, out, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double per = (double)h / iters;
    printf("DFMA chains=%2d threads/SM=%4d: %.2f clk per iteration -> %.1f DFMA/clk/SM (%s)\n", CH, threads, per,
           CH * threads / per, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out); cudaFree(cyc);
}
int main() {
    run<1>(32); run<4>(32); run<8>(32); run<8>(256); run<8>(1024); run<16>(256); run<16>(512);
    double* out; long long* cyc; long long h;
    cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&cyc, 148 * 8);
    k_shfl<<<148, 32>>>(4096, out, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("shfl.f64 + dadd chain latency: %.1f clk (%s)\n", (double)h / 4096, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
