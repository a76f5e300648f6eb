// Critical-warp level loop in isolation (tuning aid, not part of the library):
// warp 0 per level: read a 16-byte record (near offsets + value), 4 ring loads,
// adds, ring store, __syncwarp, lane-0 mbarrier arrive.  Other warps (NW-1)
// optionally wait on the level barriers like the RINGCW level warps.
// Prints cycles per level for each MODE.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ unsigned su(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int MODE>
__global__ void k(long long *out, int levels) {
    __shared__ __align__(16) u64 ring[4096 + 16];
    __shared__ __align__(16) uint4 hb[16][32];
    __shared__ __align__(8) u64 bar[16];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < 4096 + 16; i += blockDim.x) ring[i] = i;
    for (int i = tid; i < 16 * 32; i += blockDim.x) {
        const int l = i & 31;
        const unsigned o = ((l * 37 + 5) & 4095) * 8, o2 = ((l * 11 + 900) & 4095) * 8;
        hb[i >> 5][l] = make_uint4(1, 0, o | (o2 << 16), o2 | (o << 16));
    }
    if (tid < 16) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[tid])));
    __syncthreads();
    if (warp == 0) {
        long long t0 = clock64();
        int lo = 0;
        u64 acc = 0;
        for (int L = 0; L < levels; L++) {
            uint4 r;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(su(&hb[L & 15][lane])));
            u64 v[4];
            const unsigned base = su(ring);
            if (MODE & 1) {
                asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v[0]) : "r"(base + (r.z & 0xfff8u)));
                asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v[1]) : "r"(base + ((r.z >> 16) & 0xfff8u)));
                asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v[2]) : "r"(base + (r.w & 0xfff8u)));
                asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v[3]) : "r"(base + ((r.w >> 16) & 0xfff8u)));
            } else {
                v[0] = r.x; v[1] = r.y; v[2] = r.z; v[3] = r.w;
            }
            const u64 F = (((u64)r.y << 32) | r.x) - ((v[0] + v[1]) + (v[2] + v[3]));
            asm volatile("st.shared.b64 [%0], %1;" ::"r"(base + ((lo + lane) & 4095) * 8), "l"(F) : "memory");
            __syncwarp();
            if ((MODE & 2) && lane == 0)
                asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su(&bar[L & 15])) : "memory");
            lo += 25;
            acc += F;
        }
        long long t1 = clock64();
        if (lane == 0) out[0] = (t1 - t0);
        if (acc == 12345) out[1] = acc;
    } else if (MODE & 4) {
        // waiters: warp w waits for levels L = w (mod NW-1)
        for (int L = warp - 1; L < levels; L += blockDim.x / 32 - 1) {
            asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(su(&bar[L & 15])), "r"((L / 16) & 1) : "memory");
        }
    }
}
template <int MODE>
void run(int nw, const char *name) {
    long long *d;
    cudaMalloc(&d, 16);
    const int levels = 100000;
    k<MODE><<<1, 32 * nw>>>(d, levels);
    k<MODE><<<1, 32 * nw>>>(d, levels);
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-40s warps %2d: %.1f cycles/level (%s)\n", name, nw, (double)h[0] / levels, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}
int main() {
    run<0>(1, "rec only + STS + syncwarp");
    run<1>(1, "rec + 4 near LDS + STS");
    run<3>(1, "rec + near + arrive");
    run<7>(9, "rec + near + arrive, 8 waiters");
    run<7>(17, "rec + near + arrive, 16 waiters");
    return 0;
}
