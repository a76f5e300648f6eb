// RINGDF skeleton (tuning aid): 8 warps own levels round-robin; the owner of
// level L waits (mbarrier) for L-1, does the per-level tail, arrives on L.
// Components toggled by MODE bits:
//   1: try_wait on two older phases first (far L-7, mid L-3)
//   2: Fprev LDS + DADDs + ring STS (the element tail)
//   4: global store of f after the arrive
//   8: all 32 lanes active instead of 25
//  16: level bounds via shfl from a register cache + staged-counter poll (LDS)
// Prints cycles per level.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ unsigned sa(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_ph(u64 *bar, int L) {
    if (L < 0) return;
    asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(
                     sa(&bar[L & 15])),
                 "r"((L >> 4) & 1)
                 : "memory");
}
template <int MODE>
__global__ void k(long long *out, int levels, double *gout, const int *lvl) {
    __shared__ __align__(8) u64 bars[16];
    __shared__ __align__(8) double ring[4097];
    __shared__ int ctrl;
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 4097; i += blockDim.x) ring[i] = 0.0;
    if (tid == 0) {
        for (int i = 0; i < 16; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[i])));
        ctrl = 1 << 30;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int cache = lvl[lane];
    long long t0 = clock64();
    double fo = 0;
    for (int L = w; L < levels; L += 8) {
        int lo = L * 25, hi = lo + 25;
        if (MODE & 16) {
            lo = __shfl_sync(0xffffffffu, cache, (L >> 3) & 31) + L * 25;
            hi = lo + 25;
            int st;
            do { asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(st) : "r"(sa(&ctrl)) : "memory"); } while (st < hi);
        }
        const bool act = (MODE & 8) ? true : (lane < 25);
        if (MODE & 1) { wait_ph(bars, L - 7); wait_ph(bars, L - 3); }
        wait_ph(bars, L - 1);
        if (MODE & 2) {
            const int e = lo + lane;
            const double Fp = ring[(e - 64) & 4095];
            const double Fx = 1.0 - (0.5 + Fp * 0.0);
            if (act) ring[e & 4095] = Fx;
            fo = Fx - Fp;
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(sa(&bars[L & 15])) : "memory");
        if ((MODE & 4) && act) gout[(size_t)(lo + lane) * 32] = fo;
    }
    long long t1 = clock64();
    if (tid == 0) out[0] = (t1 - t0) / levels;
}
int main() {
    long long *d, h;
    double *g;
    int *lvl;
    cudaMalloc(&d, 8);
    cudaMalloc(&g, (size_t)40000 * 25 * 32 * 8 + 64);
    cudaMalloc(&lvl, 32 * 4);
    cudaMemset(lvl, 0, 128);
    const int L = 40000;
#define RUN(M)                                                        \
    k<M><<<1, 256>>>(d, L, g, lvl);                                   \
    cudaDeviceSynchronize();                                          \
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);                     \
    printf("mode %2d: %lld cycles/level\n", M, h);
    RUN(0) RUN(1) RUN(2) RUN(3) RUN(6) RUN(7) RUN(15) RUN(23) RUN(31)
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
