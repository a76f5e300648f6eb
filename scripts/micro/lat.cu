// Latency microbenchmarks (tuning aid, not part of the library): dependent
// chains of LDS.64, DADD, IADD.64, SHFL, __syncthreads, mbarrier try_wait on a
// completed phase, clock64 itself.  One CTA, results in cycles per op.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__global__ void k(long long *out, int iters, double seed) {
    __shared__ u64 sm[1024];
    __shared__ __align__(8) u64 bar;
    const int tid = threadIdx.x;
    for (int i = tid; i < 1024; i += blockDim.x) sm[i] = (u64)((i * 37 + 11) & 1023);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
    }
    __syncthreads();
    long long t0, t1;
    // LDS chain
    u64 p = tid & 1023;
    t0 = clock64();
    for (int i = 0; i < iters; i++) p = sm[p];
    t1 = clock64();
    if (tid == 0) out[0] = (t1 - t0) / iters;
    // DADD chain
    double d = seed + tid;
    t0 = clock64();
    for (int i = 0; i < iters; i++) d = d + 1.0000001;
    t1 = clock64();
    if (tid == 0) out[1] = (t1 - t0) / iters;
    // IADD64 chain
    u64 q = p + tid;
    t0 = clock64();
    for (int i = 0; i < iters; i++) q = q + 0x100000001ull;
    t1 = clock64();
    if (tid == 0) out[2] = (t1 - t0) / iters;
    // SHFL chain
    int s = tid;
    t0 = clock64();
    for (int i = 0; i < iters; i++) s = __shfl_xor_sync(0xffffffffu, s, 1) + 1;
    t1 = clock64();
    if (tid == 0) out[3] = (t1 - t0) / iters;
    // syncthreads
    t0 = clock64();
    for (int i = 0; i < iters; i++) __syncthreads();
    t1 = clock64();
    if (tid == 0) out[4] = (t1 - t0) / iters;
    // clock64 back to back
    t0 = clock64();
    long long acc = 0;
    for (int i = 0; i < iters; i++) acc += clock64();
    t1 = clock64();
    if (tid == 0) out[5] = (t1 - t0) / iters;
    // mbarrier try_wait on completed phase (parity 0)
    t0 = clock64();
    for (int i = 0; i < iters; i++) {
        asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W%=;\n}\n" ::"r"(
            (unsigned)__cvta_generic_to_shared(&bar)));
    }
    t1 = clock64();
    if (tid == 0) out[6] = (t1 - t0) / iters;
    // DFMA chain
    double e = seed;
    t0 = clock64();
    for (int i = 0; i < iters; i++) e = fma(e, 1.0000001, 0.5);
    t1 = clock64();
    if (tid == 0) out[7] = (t1 - t0) / iters;
    if (tid == 0) out[15] = (long long)d + (long long)q + s + acc + (long long)e;
}
int main() {
    long long *d, h[16];
    cudaMalloc(&d, 16 * sizeof(long long));
    for (int nt : {32, 128, 224, 512}) {
        k<<<1, nt>>>(d, 4096, 1.5);
        k<<<1, nt>>>(d, 4096, 1.5);
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        printf("threads=%d  LDS %lld  DADD %lld  IADD64 %lld  SHFL %lld  BAR %lld  CLOCK64 %lld  MBAR_TRYWAIT %lld  DFMA %lld (cycles per dependent op)\n",
               nt, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
    }
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
