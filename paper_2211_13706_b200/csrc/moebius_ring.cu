// Kernel (v), schedule RING: the Möbius U-solve of Alg. 4 (first loop,
// P:L655-661) fused with its second loop (chain difference) for
// posets whose dependencies reach back a bounded distance in rank order
// (chain-local posets).
//
//   F(x) = g(x) - Σ_{j ≠ id(x)} F(niv_j(x))           (U-solve, y' of Alg. 4)
//   f(x) = F(x) - F(next(x))                            (V^{-1})
//
// One CTA per column of the batch sweeps the antichain levels bottom-up
// (Alg. 5, with a CTA barrier instead of a grid barrier).  The
// last RING values of F live in a shared-memory ring indexed by rank mod
// RING; every dependency of rank r is a lower rank r - d with 1 <= d <= R,
// and RING >= R + max level width, so a ring entry is never overwritten
// while it can still be read.  Nothing but the result leaves the SM:
//
//   D   [npad][kp] uint16, rank-major ring-slot table: D[r][0] = ring slot
//       of next(r), D[r][1+j] = ring slot of niv_j(r) for j ≠ id(r); ring
//       slot of rank p = p mod RING; RING (the zero entry) where there is no
//       dependency.  Built once per poset (k_build_dist).
//
// Per element the kernel sums S = Σ_row F[slot] over the whole row (the
// predecessor included), so f(x) = g(x) - S directly and F(x) = f(x) +
// F(next(x)) goes into the ring.  LPE lanes share one element's row.
//   gP  [B][npad] the input g permuted to rank order (k_to_rank_major).
//
// D, gP and rank->user rows are streamed into a NSTAGE-deep shared-memory
// pipeline by cp.async.bulk (TMA bulk copies, one mbarrier per stage); the
// level boundaries are read 31 levels ahead through a per-warp register
// cache, so the only latency on the critical path of a level is shared
// memory + one barrier.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "kernels.cuh"

namespace poset {

typedef unsigned long long u64;

// ------------------------------------------------ setup: reach + table ----
// max over (r, j) of r - rank(dep), dep = niv_j(r) (j ≠ id(r)) or next(r)
__global__ void k_reach_max(const int32_t *__restrict__ M, int32_t n, int32_t k,
                            const int32_t *__restrict__ chain, const int32_t *__restrict__ slot,
                            const int32_t *__restrict__ slot_rank, unsigned *out) {
    unsigned best = 0;
    const int64_t total = (int64_t)n * (k + 1);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t j = (int32_t)(i / n), r = (int32_t)(i % n);
        int32_t dep = -1;
        if (j < k) {
            const int32_t s = __ldcs(M + i);
            if (s != n && chain[r] != j) dep = slot_rank[s];
        } else {
            const int32_t s = slot[r];
            if (s > 0 && slot_rank[s - 1] < r && chain[slot_rank[s - 1]] == chain[r]) dep = slot_rank[s - 1];
        }
        if (dep >= 0) best = max(best, (unsigned)(r - dep));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0 && best) atomicMax(out, best);
}

// D[r][*] (see header).  CTA = 32 ranks; the chain-major table is read in
// coalesced 32-rank rows, transposed through shared memory, written as
// contiguous rank rows.
__global__ void __launch_bounds__(256) k_build_dist(const int32_t *__restrict__ M, int32_t n,
                                                    int32_t k, int32_t kp, int32_t ring,
                                                    const int32_t *__restrict__ chain,
                                                    const int32_t *__restrict__ slot,
                                                    const int32_t *__restrict__ slot_rank,
                                                    uint16_t *__restrict__ D) {
    extern __shared__ uint16_t tile[];   // [32][kp + 2]
    const int stride = kp + 2;
    const int r0 = blockIdx.x * 32;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int r = r0 + lane;
    const int mask = ring - 1;
    for (int j = w; j < kp; j += nw) {
        int dep = -1;
        if (r < n) {
            if (j == 0) {
                const int32_t s = slot[r];
                if (s > 0) {
                    const int32_t p = slot_rank[s - 1];
                    if (chain[p] == chain[r]) dep = p;
                }
            } else if (j <= k) {
                const int32_t s = M[(size_t)(j - 1) * n + r];
                if (s != n && chain[r] != j - 1) dep = slot_rank[s];
            }
        }
        tile[lane * stride + j] = (uint16_t)(dep >= 0 ? (dep & mask) : ring);
    }
    __syncthreads();
    // rows r0..r0+31 are contiguous in D: write 16-bit words coalesced
    const int64_t base = (int64_t)r0 * kp;
    for (int t = threadIdx.x; t < 32 * kp; t += blockDim.x) {
        const int rr = t / kp, j = t % kp;
        D[base + t] = tile[rr * stride + j];
    }
}

cudaError_t launch_reach_max(const DevPoset &P, const int32_t *slot_rank, unsigned *out,
                             cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned), s);
    if (e != cudaSuccess || P.n == 0) return e;
    const int64_t total = (int64_t)P.n * (P.k + 1);
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    k_reach_max<<<blocks, 256, 0, s>>>(P.M, P.n, P.k, P.chain, P.slot, slot_rank, out);
    launches_add(1);
    return cudaGetLastError();
}

cudaError_t launch_build_dist(const DevPoset &P, const int32_t *slot_rank, int32_t kp, int32_t ring,
                              int64_t npad, uint16_t *D, cudaStream_t s) {
    // padding rows/columns point at the zero entry (RING)
    cudaError_t e = cudaMemsetAsync(D, 0, (size_t)npad * kp * 2, s);
    if (e != cudaSuccess || P.n == 0) return e;
    const size_t smem = (size_t)32 * (kp + 2) * 2;
    e = cudaFuncSetAttribute(k_build_dist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_build_dist<<<(unsigned)(npad / 32), 256, smem, s>>>(P.M, P.n, P.k, kp, ring, P.chain, P.slot,
                                                          slot_rank, D);
    launches_add(1);
    return cudaGetLastError();
}

// --------------------------------------------- g -> rank-major columns ----
// gP[b][r] = g[user(r)][b]   (tile transpose through shared memory)
template <typename T>
__global__ void __launch_bounds__(256) k_to_rank_major(const T *__restrict__ g,
                                                       const int32_t *__restrict__ rank_user,
                                                       int32_t n, int32_t B, int64_t npad,
                                                       T *__restrict__ gP) {
    __shared__ T t[32][33];
    const int r0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
    const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;   // 8 rows of 32
    for (int i = ly; i < 32; i += 8) {
        const int r = r0 + i, b = b0 + lx;
        if (r < n && b < B) t[i][lx] = g[(size_t)rank_user[r] * B + b];
    }
    __syncthreads();
    for (int i = ly; i < 32; i += 8) {
        const int b = b0 + i, r = r0 + lx;
        if (r < n && b < B) gP[(size_t)b * npad + r] = t[lx][i];
    }
}

cudaError_t launch_to_rank_major(const DevPoset &P, int dtype, const void *g, int64_t B,
                                 int64_t npad, void *gP, cudaStream_t s) {
    dim3 grid((unsigned)((P.n + 31) / 32), (unsigned)((B + 31) / 32));
    launches_add(1);
    if (dtype == 0)
        k_to_rank_major<u64><<<grid, 256, 0, s>>>((const u64 *)g, P.rank_user, P.n, (int32_t)B, npad,
                                                  (u64 *)gP);
    else
        k_to_rank_major<double><<<grid, 256, 0, s>>>((const double *)g, P.rank_user, P.n, (int32_t)B,
                                                     npad, (double *)gP);
    return cudaGetLastError();
}

// ------------------------------------------------------ PTX helpers -------
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(u64 *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u64 *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(u64 *bar, unsigned parity) {
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
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, u64 *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// ------------------------------------------------------- the kernel -------
struct RingArgs {
    const uint16_t *D;          // [npad][kp] ring-slot rows
    const void *gP;             // [B][npad]
    const int32_t *ru;          // [npad] rank -> user (padded)
    const int32_t *lvl_ptr;     // [ell + 1]
    void *f;                    // [n][B] output, user order
    int64_t npad;
    int32_t n, kp, ell, B;
    int32_t ring_mask;          // RING - 1 (power of two)
    int32_t lg_ch, nstage;      // log2 ranks per staged chunk, pipeline depth (power of two)
};

template <typename T, int LPE>
__global__ void __launch_bounds__(512) k_moeb_ring(RingArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int RING = a.ring_mask + 1;
    const int ch = 1 << a.lg_ch;
    T *ring = reinterpret_cast<T *>(smem);                               // RING + 1 entries
    u64 *bars = reinterpret_cast<u64 *>(smem + (size_t)(RING + 2) * 8);  // nstage
    unsigned char *stage0 = smem + (size_t)(RING + 2) * 8 + 8 * ((a.nstage + 1) & ~1);
    const unsigned dbytes = (unsigned)ch * a.kp * 2, gbytes = (unsigned)ch * 8, ubytes = (unsigned)ch * 4;
    const unsigned sbytes = dbytes + gbytes + ubytes;
    const int b = blockIdx.x;
    const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31;
    const int sub = tid & (LPE - 1), grp = tid / LPE, NG = NT / LPE;
    const unsigned gmask = LPE == 32 ? 0xffffffffu : (((1u << LPE) - 1u) << (lane & ~(LPE - 1)));
    const int Q = a.kp / LPE;   // row entries per lane (even)
    const T *gcol = reinterpret_cast<const T *>(a.gP) + (size_t)b * a.npad;
    T *f = reinterpret_cast<T *>(a.f);
    const int32_t nchunks = (int32_t)(a.npad >> a.lg_ch);

    if (tid == 0) ring[RING] = T(0);   // target of "no dependency"
    if (tid == 0) {
        for (int s = 0; s < a.nstage; s++) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int32_t issued = 0;   // chunks issued (meaningful in thread 0)
    auto issue = [&](int32_t c) {
        const int s = c & (a.nstage - 1);
        unsigned char *st = stage0 + (size_t)s * sbytes;
        mbar_expect_tx(&bars[s], sbytes);
        bulk_g2s(st, a.D + ((size_t)c << a.lg_ch) * a.kp, dbytes, &bars[s]);
        bulk_g2s(st + dbytes, gcol + ((size_t)c << a.lg_ch), gbytes, &bars[s]);
        bulk_g2s(st + dbytes + gbytes, a.ru + ((size_t)c << a.lg_ch), ubytes, &bars[s]);
    };
    if (tid == 0)
        for (; issued < nchunks && issued < a.nstage; issued++) issue(issued);

    int32_t ready = 0;                // chunks [0, ready) observed complete
    int32_t cache_base = 0;           // lv = lvl_ptr[cache_base + lane]
    int32_t lv = a.lvl_ptr[min(lane, a.ell)];
    int32_t lv_next = a.lvl_ptr[min(31 + lane, a.ell)];
    for (int32_t L = 0; L < a.ell; L++) {
        if (L - cache_base == 31) {
            cache_base += 31;
            lv = lv_next;
            lv_next = a.lvl_ptr[min(cache_base + 31 + lane, a.ell)];
        }
        const int32_t lo = __shfl_sync(0xffffffffu, lv, L - cache_base);
        const int32_t hi = __shfl_sync(0xffffffffu, lv, L - cache_base + 1);
        const int32_t need = ((hi - 1) >> a.lg_ch) + 1;
        for (; ready < need; ready++)
            mbar_wait(&bars[ready & (a.nstage - 1)], (unsigned)((ready / a.nstage) & 1));
        for (int32_t e = lo + grp; e < hi; e += NG) {   // uniform within an LPE group
            const int off = e & (ch - 1);
            const unsigned char *st = stage0 + (size_t)((e >> a.lg_ch) & (a.nstage - 1)) * sbytes;
            const uint16_t *row = reinterpret_cast<const uint16_t *>(st) + (size_t)off * a.kp + sub * Q;
            const unsigned dpred = row[0];   // meaningful in sub 0 (entry 0 of the row)
            T s = T(0);
            for (int q = 0; q < Q; q += 8) {
                unsigned w[4];
#pragma unroll
                for (int h = 0; h < 4; h++)
                    w[h] = (q + 2 * h < Q) ? *reinterpret_cast<const unsigned *>(row + q + 2 * h)
                                           : (unsigned)RING * 0x10001u;
                T v[8];
#pragma unroll
                for (int h = 0; h < 4; h++) {
                    v[2 * h] = ring[w[h] & 0xffffu];
                    v[2 * h + 1] = ring[w[h] >> 16];
                }
                s += ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
            }
#pragma unroll
            for (int o = LPE / 2; o; o >>= 1) s += __shfl_xor_sync(gmask, s, o);
            if (sub == 0) {
                const T fx = reinterpret_cast<const T *>(st + dbytes)[off] - s;
                const int32_t u = reinterpret_cast<const int32_t *>(st + dbytes + gbytes)[off];
                f[(size_t)u * a.B + b] = fx;
                ring[e & a.ring_mask] = fx + ring[dpred];
            }
        }
        if (NT == 32) __syncwarp();
        else __syncthreads();
        // chunks entirely below hi are finished: refill their stages
        if (tid == 0) {
            while (issued < nchunks && ((int64_t)(issued - a.nstage + 1) << a.lg_ch) <= hi) {
                issue(issued);
                issued++;
            }
        }
    }
}

static constexpr size_t kSmemCap = 227 * 1024;

void ring_plan(int32_t n, int32_t k, int32_t ell, int32_t max_level_width, unsigned reach,
               RingPlan &R) {
    R.ok = false;
    R.reach = reach;
    if (n <= 0 || k + 1 > 2048) return;
    int64_t ring = 32;
    while (ring < (int64_t)reach + max_level_width + 1) ring <<= 1;
    if (ring > (1 << 15)) return;   // ring slots are uint16, RING itself included
    const double avg_w = (double)n / std::max(ell, 1);
    int lpe = 4;
    while (lpe > 1 && avg_w * lpe > 512) lpe >>= 1;
    // row = [pred, chain 0 .. k-1], padded to 8*lpe entries
    const int32_t unit = 8 * lpe;
    const int32_t kp = (k + 1 + unit - 1) / unit * unit;
    int threads = (int)std::min<int64_t>(512, ((int64_t)std::ceil(avg_w * lpe) + 31) / 32 * 32);
    threads = std::max(threads, 32);
    for (int nstage : {4, 2}) {
        for (int ch : {256, 128, 64, 32, 16, 8, 4}) {
            if ((int64_t)max_level_width > (int64_t)(nstage - 1) * ch) break;
            if (ring_smem_bytes((int)ring, kp, ch, nstage) <= kSmemCap) {
                R.ok = true;
                R.kp = kp;
                R.ring = (int32_t)ring;
                R.ch = ch;
                R.nstage = nstage;
                R.lpe = lpe;
                R.threads = threads;
                R.npad = ((int64_t)n + ch - 1) / ch * ch;
                return;
            }
        }
    }
}

size_t ring_smem_bytes(int ring, int kp, int ch, int nstage) {
    return (size_t)(ring + 2) * 8 + 8 * ((nstage + 1) & ~1) +
           (size_t)nstage * ch * ((size_t)kp * 2 + 8 + 4);
}

cudaError_t launch_moebius_ring(const DevPoset &P, const RingPlan &R, int dtype, const void *gP,
                                void *f, int64_t B, cudaStream_t s) {
    if (P.n == 0) return cudaSuccess;
    RingArgs a;
    a.D = R.D;
    a.gP = gP;
    a.ru = R.ru_pad;
    a.lvl_ptr = P.lvl_ptr;
    a.f = f;
    a.npad = R.npad;
    a.n = P.n;
    a.kp = R.kp;
    a.ell = P.ell;
    a.B = (int32_t)B;
    a.ring_mask = R.ring - 1;
    a.lg_ch = 0;
    while ((1 << a.lg_ch) < R.ch) a.lg_ch++;
    a.nstage = R.nstage;
    const size_t smem = ring_smem_bytes(R.ring, R.kp, R.ch, R.nstage);
    void *fn;
#define RING_FN(LPE) (dtype == 0 ? (void *)k_moeb_ring<u64, LPE> : (void *)k_moeb_ring<double, LPE>)
    fn = R.lpe == 4 ? RING_FN(4) : R.lpe == 2 ? RING_FN(2) : RING_FN(1);
#undef RING_FN
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    void *args[] = {&a};
    launches_add(1);
    return cudaLaunchKernel(fn, dim3((unsigned)B), dim3(R.threads), args, smem, s);
}

}  // namespace poset
