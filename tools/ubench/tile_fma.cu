// Micro-benchmark: cycles for one warp to multiply an 8-row smem tile (w columns) by a
// 2-column input (the nested-dissection solve's inner loop), 8 warps per CTA.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
template <int N>
__device__ __forceinline__ double rs(double (&v)[N], int lane) {
#pragma unroll
    for (int o = 16; o >= N; o >>= 1)
#pragma unroll
        for (int i = 0; i < N; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
#pragma unroll
    for (int o = N / 2; o >= 1; o >>= 1) {
        const bool up = lane & o;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const double send = up ? v[i] : v[i + o];
            const double keep = up ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0];
}
__global__ void k(int iters, int w2, double* out, long long* cyc) {
    extern __shared__ double2 sm[];
    double2* v = sm;                 // 2 x 768
    double2* tiles = sm + 1536;      // 8 warps x 8 x w2
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 1536 + 8 * 8 * w2; i += blockDim.x) sm[i] = make_double2(1e-3 * i, 2e-3);
    __syncthreads();
    const double2* tile = tiles + warp * 8 * w2;
    const long long c0 = clock64();
    double keep = 0;
    for (int it = 0; it < iters; ++it) {
        double acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = 0.0;
        const int vo = (it & 3) * 96;
        for (int c2 = lane; c2 < w2; c2 += 32) {
            const double2 a0 = v[vo + c2], a1 = v[768 + vo + c2];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const double2 m = tile[r * w2 + c2];
                acc[2 * r] = fma(m.y, a0.y, fma(m.x, a0.x, acc[2 * r]));
                acc[2 * r + 1] = fma(m.y, a1.y, fma(m.x, a1.x, acc[2 * r + 1]));
            }
        }
        keep += rs<16>(acc, lane);
    }
    const long long c1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = keep;
    if (lane == 0) cyc[blockIdx.x * 8 + warp] = c1 - c0;
}
int main(int argc, char** argv) {
    int w2 = argc > 1 ? atoi(argv[1]) : 96, iters = 1000;
    size_t smem = (1536 + 8 * 8 * w2) * sizeof(double2);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    double* out; long long* cyc;
    cudaMalloc(&out, 148 * 256 * 8); cudaMalloc(&cyc, 148 * 8 * 8);
    k<<<148, 256, smem>>>(iters, w2, out, cyc);
    cudaDeviceSynchronize();
    long long h[8];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("err=%s  cycles per 8x%d tile per warp (8 warps/SM): %.1f  -> %.1f B/clk/SM\n", cudaGetErrorString(cudaGetLastError()),
           2 * w2, (double)h[0] / iters, 8.0 * 8 * 2 * w2 * 8 / ((double)h[0] / iters));
    return 0;
}
