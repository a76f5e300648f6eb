// DSMEM hand-off latency between the two CTAs of a cluster (tuning aid for
// RINGCL): round trips of (a) st.async + remote complete_tx, waited with
// try_wait / test_wait, and (b) st.shared::cluster + remote
// mbarrier.arrive.release.cluster, waited with try_wait.acquire.cluster.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ unsigned sa(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned rank_() { unsigned r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ unsigned mapa(unsigned a, unsigned r) { unsigned o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) k(long long *out, int iters) {
    __shared__ __align__(8) u64 bar[2];
    __shared__ __align__(8) u64 data[32];
    const unsigned me = rank_(), peer = me ^ 1;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[0])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
    const unsigned rbar = mapa(sa(&bar[0]), peer), rdat = mapa(sa(&data[threadIdx.x]), peer);
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        // rank 0 sends on even turns, rank 1 answers
        if ((int)me == 1 || i > 0) {
            // wait for phase i - (me == 0) ... each side waits its own phases in order
            const unsigned ph = (unsigned)((me == 0 ? i - 1 : i) & 1);
            if (MODE == 0 || MODE == 2) {
                if (threadIdx.x == 0 && MODE == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 256;" ::"r"(sa(&bar[0])));
                if (MODE == 0)
                    asm volatile("{\n.reg .pred p;\nW0:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W0;\n}" ::"r"(sa(&bar[0])), "r"(ph) : "memory");
                else
                    asm volatile("{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}" ::"r"(sa(&bar[0])), "r"(ph) : "memory");
            } else {
                if (threadIdx.x == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 256;" ::"r"(sa(&bar[0])));
                asm volatile("{\n.reg .pred p;\nW1:\nmbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W1;\n}" ::"r"(sa(&bar[0])), "r"(ph) : "memory");
            }
        }
        if (MODE == 2) {
            asm volatile("st.shared::cluster.b64 [%0], %1;" ::"r"(rdat), "l"((u64)i) : "memory");
            __syncwarp();
            if (threadIdx.x == 0) asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
        } else {
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(rdat), "l"((u64)i), "r"(rbar) : "memory");
        }
        if (me == 0 && i == iters - 1) {
            // wait for the final answer
            if (MODE != 2 && threadIdx.x == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 256;" ::"r"(sa(&bar[0])));
            asm volatile("{\n.reg .pred p;\nW3:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W3;\n}" ::"r"(sa(&bar[0])), "r"((unsigned)(i & 1)) : "memory");
        }
    }
    long long t1 = clock64();
    if (me == 0 && threadIdx.x == 0) out[MODE] = (t1 - t0) / iters;
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
}
int main() {
    long long *d, h[3] = {0, 0, 0};
    cudaMalloc(&d, 24);
    cudaMemset(d, 0, 24);
    k<0><<<2, 32>>>(d, 10000);
    cudaDeviceSynchronize();
    printf("st.async + try_wait: %s\n", cudaGetErrorString(cudaGetLastError()));
    k<1><<<2, 32>>>(d, 10000);
    cudaDeviceSynchronize();
    printf("st.async + test_wait: %s\n", cudaGetErrorString(cudaGetLastError()));
    k<2><<<2, 32>>>(d, 10000);
    cudaDeviceSynchronize();
    printf("st.cluster + arrive.release.cluster: %s\n", cudaGetErrorString(cudaGetLastError()));
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("round trip cycles: st.async/try_wait %lld | st.async/test_wait %lld | st+arrive.release %lld\n", h[0], h[1], h[2]);
    return 0;
}
