// Device primitives of the persistent recurrence kernels: mbarriers, 1D TMA
// bulk copies into shared memory, and LL lines (value + flag in one 16-byte
// store) for barrier-free dataflow between CTAs.
#pragma once

#include <cuda_runtime.h>

namespace pdg {
namespace dev {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1D bulk copy global -> shared (TMA engine), completion counted on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// LL line (the NCCL "LL" idea): a double travels as two 32-bit halves, each
// paired with a 32-bit flag in one 8-byte-atomic unit, 16 bytes per value: one
// store publishes value + flag, a reader accepts the line when both flags
// match -- no fences on the critical path.
__device__ __forceinline__ void ll_store(uint4* p, double v, unsigned flag) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(static_cast<unsigned>(b)),
                 "r"(flag), "r"(static_cast<unsigned>(b >> 32)), "r"(flag)
                 : "memory");
}
__device__ __forceinline__ uint4 ll_peek(const uint4* p) {
    uint4 v;
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
__device__ __forceinline__ double ll_value(const uint4& v) {
    return __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(v.z) << 32) | v.x));
}
__device__ __forceinline__ bool ll_ready(const uint4& v, unsigned flag) { return v.y == flag && v.w == flag; }
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

}  // namespace dev
}  // namespace pdg
