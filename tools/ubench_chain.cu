// Microbenchmark: per-step latency of a grid-wide dataflow chain on one GPU.
// G CTAs; at step s every CTA needs all M values produced at step s-1 (8 per
// CTA), as in the block-tridiagonal recurrence. Variants:
//   0: LL lines (value+flag, relaxed.gpu v4), all threads poll their lines
//   1: per-CTA flag (release/acquire) + plain data, one thread polls flags
//   2: atomic step counter barrier (acq_rel) + plain data
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_chain ubench_chain.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void st_ll(uint4* p, double v, unsigned f) {
    unsigned long long b = (unsigned long long)__double_as_longlong(v);
    asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"((unsigned)b), "r"(f), "r"((unsigned)(b >> 32)), "r"(f) : "memory");
}
__device__ __forceinline__ uint4 ld_ll(const uint4* p) {
    uint4 v;
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void chain(int variant, int steps, int M, uint4* ll, double* data, unsigned* flags, unsigned* counter,
                      unsigned flag0, double* sink) {
    extern __shared__ double ysh[];
    const int row0 = blockIdx.x * 8;
    double acc = 0.0;
    for (int s = 1; s <= steps; ++s) {
        const unsigned want = flag0 + s - 1;
        if (variant == 0) {
            constexpr int PER = 8;
            uint4 v[PER];
#pragma unroll
            for (int q = 0; q < PER; ++q) {
                const int t = threadIdx.x + q * blockDim.x;
                if (t < M) v[q] = ld_ll(&ll[(size_t)(s - 1) % 2 * M + t]);
            }
#pragma unroll
            for (int q = 0; q < PER; ++q) {
                const int t = threadIdx.x + q * blockDim.x;
                if (t < M) {
                    while (v[q].y != want || v[q].w != want) v[q] = ld_ll(&ll[(size_t)(s - 1) % 2 * M + t]);
                    ysh[t] = __longlong_as_double(((long long)v[q].z << 32) | v[q].x);
                }
            }
        } else if (variant == 1) {
            if (threadIdx.x < gridDim.x)
                while (ld_acq(&flags[((s - 1) % 2) * gridDim.x + threadIdx.x]) != want) {
                }
            __syncthreads();
            for (int t = threadIdx.x; t < M; t += blockDim.x) ysh[t] = __ldcg(&data[(size_t)(s - 1) % 2 * M + t]);
        } else {
            if (threadIdx.x == 0)
                while (ld_acq(counter) < gridDim.x * (unsigned)(s - 1)) {
                }
            __syncthreads();
            for (int t = threadIdx.x; t < M; t += blockDim.x) ysh[t] = __ldcg(&data[(size_t)(s - 1) % 2 * M + t]);
        }
        __syncthreads();
        // "compute": warp w produces row row0+w from ysh
        const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
        double a = 0.0;
        for (int c = lane; c < M; c += 32) a += ysh[c] * 1e-3;
        for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        acc += a;
        const int r = row0 + w;
        if (lane == 0 && r < M) {
            if (variant == 0)
                st_ll(&ll[(size_t)s % 2 * M + r], a, flag0 + s);
            else
                data[(size_t)s % 2 * M + r] = a;
        }
        __syncthreads();
        if (variant == 1 && threadIdx.x == 0) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(&flags[(s % 2) * gridDim.x + blockIdx.x]), "r"(flag0 + s) : "memory");
        }
        if (variant == 2 && threadIdx.x == 0) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            atomicAdd(counter, 1u);
        }
    }
    if (threadIdx.x == 0) sink[blockIdx.x] = acc;
}

__global__ void init(int M, uint4* ll, double* data, unsigned* flags, unsigned flag0, int G) {
    for (int t = threadIdx.x + blockIdx.x * blockDim.x; t < M; t += gridDim.x * blockDim.x) {
        unsigned long long b = (unsigned long long)__double_as_longlong(1.0);
        ll[t] = make_uint4((unsigned)b, flag0, (unsigned)(b >> 32), flag0);
        data[t] = 1.0;
    }
    for (int t = threadIdx.x + blockIdx.x * blockDim.x; t < G; t += gridDim.x * blockDim.x) flags[t] = flag0;
}

int main() {
    const int steps = 1000;
    for (int M : {257, 1032}) {
        const int G = (M + 7) / 8;
        uint4* ll;
        double *data, *sink;
        unsigned *flags, *counter;
        cudaMalloc(&ll, sizeof(uint4) * 2 * M);
        cudaMalloc(&data, sizeof(double) * 2 * M);
        cudaMalloc(&flags, sizeof(unsigned) * 2 * G);
        cudaMalloc(&counter, sizeof(unsigned));
        cudaMalloc(&sink, sizeof(double) * G);
        cudaMemset(ll, 0, sizeof(uint4) * 2 * M);
        cudaMemset(flags, 0, sizeof(unsigned) * 2 * G);
        for (int variant = 0; variant < 3; ++variant) {
            unsigned flag0 = 100 + variant * 5000;
            cudaMemset(ll, 0, sizeof(uint4) * 2 * M);
            cudaMemset(flags, 0, sizeof(unsigned) * 2 * G);
            init<<<8, 256>>>(M, ll, data, flags, flag0, G);
            cudaMemset(counter, 0, 4);
            int s_ = steps, M_ = M, v_ = variant;
            void* args[] = {&v_, &s_, &M_, &ll, &data, &flags, &counter, &flag0, &sink};
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            if (variant == 2) {  // counter semantics: step s waits for G*(s-1) arrivals
                cudaMemset(counter, 0, 4);
            }
            cudaEventRecord(a);
            cudaError_t e = cudaLaunchCooperativeKernel((void*)chain, G, 256, args, sizeof(double) * M, 0);
            cudaEventRecord(b);
            cudaError_t e2 = cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            printf("M=%d G=%d variant=%d: %.3f us/step (%s %s)\n", M, G, variant, ms * 1e3 / steps, cudaGetErrorString(e),
                   cudaGetErrorString(e2));
        }
        cudaFree(ll);
        cudaFree(data);
        cudaFree(flags);
        cudaFree(counter);
        cudaFree(sink);
    }
    return 0;
}
