// Grid barrier cost in isolation (tuning aid, not part of the library):
// 148 persistent 1024-thread CTAs, N barriers.  Variants: the CSR kernel's
// barrier (every CTA: red.release.gpu + ld.acquire.gpu spin on one counter)
// and a two-level one over clusters of 2 (cluster barrier, then one CTA per
// cluster on the global counter, then the cluster barrier again).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void gsync(unsigned *bar, unsigned nb, unsigned t) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        const unsigned target = (t + 1) * nb;
        unsigned v;
        do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory"); } while ((int)(v - target) < 0);
    }
    __syncthreads();
}
__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned crank() { unsigned r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(unsigned *bar, int N, long long *out) {
    long long t0 = clock64();
    for (int t = 0; t < N; t++) {
        if (MODE == 0) gsync(bar, gridDim.x, t);
        else {
            csync();
            if (crank() == 0) {
                if (threadIdx.x == 0) {
                    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
                    const unsigned target = (t + 1) * (gridDim.x / 2);
                    unsigned v;
                    do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory"); } while ((int)(v - target) < 0);
                }
                __syncthreads();
            }
            csync();
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[MODE] = clock64() - t0;
}
int main() {
    unsigned *bar; long long *out, h[2];
    cudaMalloc(&bar, 8); cudaMalloc(&out, 16);
    const int N = 20000;
    cudaMemset(bar, 0, 8);
    k<0><<<148, 1024>>>(bar, N, out);
    cudaDeviceSynchronize();
    cudaMemset(bar, 0, 8);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148); cfg.blockDim = dim3(1024);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k<1>, bar, N, out);
    cudaDeviceSynchronize();
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("flat grid barrier: %.0f cycles (%.2f us)\\n", (double)h[0] / N, (double)h[0] / N / 1965.0);
    printf("cluster-2 + global: %.0f cycles (%.2f us) (%s)\\n", (double)h[1] / N, (double)h[1] / N / 1965.0, cudaGetErrorString(cudaGetLastError()));
}
