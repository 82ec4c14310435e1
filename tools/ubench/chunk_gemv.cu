// Micro-benchmark: cycles for one warp to multiply a [nrow x ld2] double2 chunk in shared
// memory by a 2-column input (the nested-dissection solve's inner loop), 8 warps per SM,
// for three inner-loop designs: the 8-row tile with a warp reduce-scatter (old), groups
// of G lanes per row with an unrolled column loop, and one lane per row (odd ld2).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ double rs16(double (&v)[16], int lane) {
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) {
        const bool up = lane & o;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const double send = up ? v[i] : v[i + o];
            const double keep = up ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}

// variant 0: old 8-row tile
__device__ double chunk_tile(const double2* rows2, int nrow, int ld2, const double2* va, const double2* vb, int lane, double* out) {
    double keep = 0;
    for (int rb = 0; rb < nrow; rb += 8) {
        const int rn = min(8, nrow - rb);
        double acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = 0.0;
        for (int c2 = lane; c2 < ld2; c2 += 32) {
            const double2 p = va[c2], q = vb[c2];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const double2 m = r < rn ? rows2[(rb + r) * ld2 + c2] : make_double2(0.0, 0.0);
                acc[2 * r] = fma(m.y, p.y, fma(m.x, p.x, acc[2 * r]));
                acc[2 * r + 1] = fma(m.y, q.y, fma(m.x, q.x, acc[2 * r + 1]));
            }
        }
        keep += rs16(acc, lane);
    }
    return keep;
}
// variant 1: groups of G lanes per row, column loop unrolled by U
template <int G, int U>
__device__ double chunk_group(const double2* rows2, int nrow, int ld2, const double2* va, const double2* vb, int lane) {
    const int lg = lane & (G - 1), grp = lane / G;
    double keep = 0;
    for (int rb = 0; rb < nrow; rb += 32 / G) {
        const int row = rb + grp;
        double ax[U], ay[U], bx[U], by[U];
#pragma unroll
        for (int u = 0; u < U; ++u) ax[u] = ay[u] = bx[u] = by[u] = 0.0;
        if (row < nrow) {
            const double2* rp = rows2 + row * ld2;
            int c2 = lg;
            for (; c2 + (U - 1) * G < ld2; c2 += U * G) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const double2 m = rp[c2 + u * G], p = va[c2 + u * G], q = vb[c2 + u * G];
                    ax[u] = fma(m.x, p.x, ax[u]);
                    ay[u] = fma(m.y, p.y, ay[u]);
                    bx[u] = fma(m.x, q.x, bx[u]);
                    by[u] = fma(m.y, q.y, by[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (c2 + u * G < ld2) {
                    const double2 m = rp[c2 + u * G], p = va[c2 + u * G], q = vb[c2 + u * G];
                    ax[u] = fma(m.x, p.x, ax[u]);
                    ay[u] = fma(m.y, p.y, ay[u]);
                    bx[u] = fma(m.x, q.x, bx[u]);
                    by[u] = fma(m.y, q.y, by[u]);
                }
        }
        double s0 = 0, s1 = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            s0 += ax[u] + ay[u];
            s1 += bx[u] + by[u];
        }
#pragma unroll
        for (int o = G / 2; o >= 1; o >>= 1) {
            s0 += __shfl_xor_sync(0xffffffffu, s0, o);
            s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        }
        keep += s0 + s1;
    }
    return keep;
}

// variant 2: groups of G lanes, R rows per group sharing each v load
template <int G, int R>
__device__ double chunk_rows(const double2* rows2, int nrow, int ld2, const double2* va, const double2* vb, int lane) {
    const int lg = lane & (G - 1), grp = lane / G;
    double keep = 0;
    for (int rb = 0; rb < nrow; rb += (32 / G) * R) {
        const int row0 = rb + grp * R;
        double acc[R][4];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r][0] = acc[r][1] = acc[r][2] = acc[r][3] = 0.0;
        for (int c2 = lg; c2 < ld2; c2 += G) {
            const double2 p = va[c2], q = vb[c2];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double2 m = row0 + r < nrow ? rows2[(row0 + r) * ld2 + c2] : make_double2(0.0, 0.0);
                acc[r][0] = fma(m.x, p.x, acc[r][0]);
                acc[r][1] = fma(m.y, p.y, acc[r][1]);
                acc[r][2] = fma(m.x, q.x, acc[r][2]);
                acc[r][3] = fma(m.y, q.y, acc[r][3]);
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            double s0 = acc[r][0] + acc[r][1], s1 = acc[r][2] + acc[r][3];
#pragma unroll
            for (int o = G / 2; o >= 1; o >>= 1) {
                s0 += __shfl_xor_sync(0xffffffffu, s0, o);
                s1 += __shfl_xor_sync(0xffffffffu, s1, o);
            }
            keep += s0 + s1;
        }
    }
    return keep;
}

template <int V, int G, int U>
__global__ void k(int iters, int nrow, int ld2, double* out, long long* cyc) {
    extern __shared__ double2 sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double2* va = sm;
    double2* vb = sm + 1400;
    double2* chunks = sm + 2800;
    const int csz = nrow * ld2;
    for (int i = threadIdx.x; i < 2800 + 4 * csz; i += blockDim.x) sm[i] = make_double2(1e-3 * (i % 97), 2e-3);
    __syncthreads();
    const double2* rows2 = chunks + (warp & 3) * csz;
    const long long c0 = clock64();
    double keep = 0;
    for (int it = 0; it < iters; ++it) {
        if (V == 0) keep += chunk_tile(rows2, nrow, ld2, va + (it & 1), vb, lane, nullptr);
        else if (V == 1) keep += chunk_group<G, U>(rows2, nrow, ld2, va + (it & 1), vb, lane);
        else keep += chunk_rows<G, U>(rows2, nrow, ld2, va + (it & 1), vb, lane);
    }
    const long long c1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = keep;
    if (lane == 0) cyc[blockIdx.x * 8 + warp] = c1 - c0;
}

template <int V, int G, int U>
void run(const char* name, int nrow, int ld2) {
    const int iters = 200;
    const size_t smem = (2800 + 4 * (size_t)nrow * ld2) * sizeof(double2);
    if (smem > 227 * 1024) { printf("%-14s %3d x %4d: too big\n", name, nrow, ld2); return; }
    cudaFuncSetAttribute(k<V, G, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    double* out; long long* cyc;
    cudaMalloc(&out, 148 * 256 * 8); cudaMalloc(&cyc, 148 * 8 * 8);
    k<V, G, U><<<148, 256, smem>>>(iters, nrow, ld2, out, cyc);
    cudaDeviceSynchronize();
    long long h[8];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double c = (double)h[0] / iters;
    printf("%-14s %3d x %4d: %7.0f clk/chunk/warp -> %5.1f B/clk/SM (%s)\n", name, nrow, ld2, c, 8.0 * nrow * ld2 * 16 / c,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(out); cudaFree(cyc);
}
int main() {
    const int shapes[][2] = {{37, 36}, {32, 37}, {24, 86}, {24, 87}, {10, 256}, {2, 1024}, {1, 1300}};
    for (auto& sh : shapes) {
        const int nr = sh[0], l2 = sh[1];
        run<0, 32, 1>("tile8", nr, l2);
        run<1, 4, 4>("G4 U4", nr, l2);
        run<1, 32, 4>("G32 U4", nr, l2);
        run<1, 1, 4>("G1 U4", nr, l2);
        run<1, 1, 8>("G1 U8", nr, l2);
        run<2, 1, 2>("G1 R2", nr, l2);
        run<2, 4, 2>("G4 R2", nr, l2);
        run<2, 4, 4>("G4 R4", nr, l2);
        run<2, 8, 4>("G8 R4", nr, l2);
        run<2, 16, 2>("G16 R2", nr, l2);
        run<2, 32, 2>("G32 R2", nr, l2);
        run<2, 32, 4>("G32 R4", nr, l2);
    }
    return 0;
}
