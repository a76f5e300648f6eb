// Cross-warp hand-off latency (tuning aid): warps 0 and 1 of one CTA pass a
// token back and forth N times; cycles per hand-off for
//  0: mbarrier arrive.release (1 arrival) / try_wait.parity (acquire)
//  1: st.release.cta / ld.acquire.cta spin on a shared counter
//  2: st.relaxed (volatile) / ld.volatile spin
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ unsigned sa(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int MODE>
__global__ void k(long long *out, int N) {
    __shared__ __align__(8) u64 bars[64];
    __shared__ int flag;
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int i = 0; i < 64; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[i])));
        flag = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < N; i++) {
        const int me = i & 1;   // warp that acts at step i
        if (w == me) {
            // wait for step i-1 to be done
            if (i > 0) {
                if (MODE == 0) {
                    const int j = i - 1;
                    asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(
                                     sa(&bars[j & 63])),
                                 "r"((j >> 6) & 1));
                } else if (MODE == 1) {
                    int v;
                    do { asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"(sa(&flag)) : "memory"); } while (v < i);
                } else {
                    int v;
                    do { asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(sa(&flag)) : "memory"); } while (v < i);
                }
            }
            __syncwarp();
            if (lane == 0) {
                if (MODE == 0)
                    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(sa(&bars[i & 63])) : "memory");
                else if (MODE == 1)
                    asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"(sa(&flag)), "r"(i + 1) : "memory");
                else
                    asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(sa(&flag)), "r"(i + 1) : "memory");
            }
        }
    }
    long long t1 = clock64();
    if (tid == 0) out[MODE] = (t1 - t0) / N;
}
int main() {
    long long *d, h[4] = {0};
    cudaMalloc(&d, sizeof h);
    k<0><<<1, 64>>>(d, 20000);
    k<1><<<1, 64>>>(d, 20000);
    k<2><<<1, 64>>>(d, 20000);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("cycles per hand-off: mbarrier %lld | release/acquire flag %lld | volatile flag %lld\n", h[0], h[1], h[2]);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
