// Small PTX helpers shared by the shared-memory-pipeline kernels
// (mbarrier, TMA bulk copies).  Internal header.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace poset {
namespace ptx {
typedef unsigned long long u64;
}

template <typename T>
__device__ __forceinline__ T bits_to(unsigned long long x);
template <>
__device__ __forceinline__ unsigned long long bits_to<unsigned long long>(unsigned long long x) { return x; }
template <>
__device__ __forceinline__ double bits_to<double>(unsigned long long x) {
    return __longlong_as_double((long long)x);
}

// ------------------------------------------------------ PTX helpers -------
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}


}  // namespace poset
