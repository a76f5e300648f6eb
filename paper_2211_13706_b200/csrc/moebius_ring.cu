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
//   D   [npad][kp] uint16, rank-major ring-slot rows: the ring slots
//       (rank mod RING) of niv_j(r) for j ≠ id(r), sorted by bank key,
//       padded with RING (the zero entry); 64 entries per lane, LPE lanes
//       per element.  Pn [npad]: ring slot of next(r) (RING at a chain
//       bottom).  Built once per poset (k_build_dist).
//
// Per element: F(x) = g(x) - Σ_row F[slot] goes into the ring and
// f(x) = F(x) - F(next(x)) to global memory.
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
#include "ptx.cuh"

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

// D rows and next slots (see header).  CTA = 32 ranks: the chain-major
// table is read in coalesced 32-rank rows into shared memory, each row is
// counting-sorted by its bank key, and the rows are written out contiguous.
// Bank key of a dependency slot s of rank r: ((s - r) mod 16) -- the ring
// holds 8-byte entries, so slot s lives in bank pair s mod 16; after the sort,
// the lanes of a warp (consecutive ranks) reading their q-th entries hit
// different bank pairs instead of colliding at random.
__global__ void __launch_bounds__(256) k_build_dist(const int32_t *__restrict__ M, int32_t n,
                                                    int32_t k, int32_t kp, int32_t ring,
                                                    const int32_t *__restrict__ chain,
                                                    const int32_t *__restrict__ slot,
                                                    const int32_t *__restrict__ slot_rank,
                                                    uint16_t *__restrict__ D, uint16_t *__restrict__ Pn) {
    extern __shared__ uint16_t tile[];   // [2][32][kp + 2]
    const int stride = kp + 2;
    uint16_t *raw = tile, *srt = tile + 32 * stride;
    const int r0 = blockIdx.x * 32;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int r = r0 + lane;
    const int mask = ring - 1;
    for (int j = w; j < k; j += nw) {
        int dep = -1;
        if (r < n) {
            const int32_t s = M[(size_t)j * n + r];
            if (s != n && chain[r] != j) dep = slot_rank[s];
        }
        raw[lane * stride + j] = (uint16_t)(dep >= 0 ? (dep & mask) : ring);
    }
    if (w == 0) {
        int dep = -1;
        if (r < n) {
            const int32_t s = slot[r];
            if (s > 0) {
                const int32_t p = slot_rank[s - 1];
                if (chain[p] == chain[r]) dep = p;
            }
        }
        Pn[r] = (uint16_t)(dep >= 0 ? (dep & mask) : ring);
    }
    __syncthreads();
    if (w == 0) {   // counting sort of row `lane` by bank key; "none" entries last
        int cnt[17];
#pragma unroll
        for (int c = 0; c < 17; c++) cnt[c] = 0;
        const uint16_t *in = raw + lane * stride;
        for (int j = 0; j < k; j++) {
            const int s = in[j];
            cnt[s == ring ? 16 : ((s - r) & 15)]++;
        }
        int pos[17], acc = 0;
#pragma unroll
        for (int c = 0; c < 17; c++) { pos[c] = acc; acc += cnt[c]; }
        uint16_t *out = srt + lane * stride;
        for (int j = 0; j < k; j++) {
            const int s = in[j];
            const int c = s == ring ? 16 : ((s - r) & 15);
#pragma unroll
            for (int cc = 0; cc < 17; cc++)
                if (cc == c) out[pos[cc]++] = (uint16_t)s;
        }
        for (int j = k; j < kp; j++) out[j] = (uint16_t)ring;
    }
    __syncthreads();
    // rows r0..r0+31 are contiguous in D: write 16-bit words coalesced
    const int64_t base = (int64_t)r0 * kp;
    for (int t = threadIdx.x; t < 32 * kp; t += blockDim.x) {
        const int rr = t / kp, j = t % kp;
        D[base + t] = srt[rr * stride + j];
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
                              int64_t npad, uint16_t *D, uint16_t *Pn, cudaStream_t s) {
    if (P.n == 0) return cudaSuccess;
    const size_t smem = (size_t)2 * 32 * (kp + 2) * 2;
    cudaError_t e;
    e = cudaFuncSetAttribute(k_build_dist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_build_dist<<<(unsigned)(npad / 32), 256, smem, s>>>(P.M, P.n, P.k, kp, ring, P.chain, P.slot,
                                                          slot_rank, D, Pn);
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

// ------------------------------------------------------- the kernel -------
struct RingArgs {
    const uint16_t *D;          // [npad][kp] sorted ring-slot rows
    const uint16_t *Pn;         // [npad] ring slot of next(r)
    const void *gP;             // [B][npad]
    const int32_t *ru;          // [npad] rank -> user (padded)
    const int32_t *lvl_ptr;     // [ell + 1]
    void *f;                    // [n][B] output, user order
    int64_t npad;
    int32_t n, kp, ell, B;
    int32_t ring_mask;          // RING - 1 (power of two)
    int32_t lg_ch, nstage;      // log2 ranks per staged chunk, pipeline depth (power of two)
    int32_t debug;              // tuning experiments only: bit 0 = skip the global store of f,
                                // (the per-phase clock64 instrumentation of round 1 is retired;
                                // DESIGN.md §5.4 records what it measured)
    unsigned long long *dbg;
};

// 8 shared-memory loads in one asm block: issued back to back, so all 32
// loads of a row chunk are in flight before the first add (the compiler's own
// schedule interleaves them 4 at a time with the additions).
__device__ __forceinline__ void lds64x8(unsigned base, const unsigned (&w)[4], u64 (&v)[8]) {
    asm volatile(
        "{\n\t.reg .u32 a<8>;\n\t"
        "and.b32 a0, %8, 65535;\n\tshr.u32 a1, %8, 16;\n\t"
        "and.b32 a2, %9, 65535;\n\tshr.u32 a3, %9, 16;\n\t"
        "and.b32 a4, %10, 65535;\n\tshr.u32 a5, %10, 16;\n\t"
        "and.b32 a6, %11, 65535;\n\tshr.u32 a7, %11, 16;\n\t"
        "mad.lo.u32 a0, a0, 8, %12;\n\tmad.lo.u32 a1, a1, 8, %12;\n\t"
        "mad.lo.u32 a2, a2, 8, %12;\n\tmad.lo.u32 a3, a3, 8, %12;\n\t"
        "mad.lo.u32 a4, a4, 8, %12;\n\tmad.lo.u32 a5, a5, 8, %12;\n\t"
        "mad.lo.u32 a6, a6, 8, %12;\n\tmad.lo.u32 a7, a7, 8, %12;\n\t"
        "ld.shared.b64 %0, [a0];\n\tld.shared.b64 %1, [a1];\n\t"
        "ld.shared.b64 %2, [a2];\n\tld.shared.b64 %3, [a3];\n\t"
        "ld.shared.b64 %4, [a4];\n\tld.shared.b64 %5, [a5];\n\t"
        "ld.shared.b64 %6, [a6];\n\tld.shared.b64 %7, [a7];\n\t}"
        : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]), "=l"(v[4]), "=l"(v[5]), "=l"(v[6]),
          "=l"(v[7])
        : "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(base));
}

// Σ of the ring entries named by E consecutive row words (E/8 x LDS.128 of
// slots, E independent LDS.64, balanced tree).
template <typename T, int E>
__device__ __forceinline__ T ring_sum(const T *ring, const uint16_t *row) {
    T v[E];
    if constexpr (E >= 8) {
        uint4 w[E / 8];
#pragma unroll
        for (int i = 0; i < E / 8; i++) w[i] = reinterpret_cast<const uint4 *>(row)[i];
#pragma unroll
        for (int i = 0; i < E / 8; i++) {
            const unsigned ws[4] = {w[i].x, w[i].y, w[i].z, w[i].w};
#pragma unroll
            for (int h = 0; h < 4; h++) {
                v[8 * i + 2 * h] = ring[ws[h] & 0xffffu];
                v[8 * i + 2 * h + 1] = ring[ws[h] >> 16];
            }
        }
    } else {
        const uint2 w = *reinterpret_cast<const uint2 *>(row);
        v[0] = ring[w.x & 0xffffu];
        v[1] = ring[w.x >> 16];
        v[2] = ring[w.y & 0xffffu];
        v[3] = ring[w.y >> 16];
    }
#pragma unroll
    for (int st = 1; st < E; st <<= 1)
#pragma unroll
        for (int i = 0; i < E; i += 2 * st) v[i] += v[i + st];
    return v[0];
}

// shared-memory accessors on 32-bit shared addresses (the generic-to-shared
// window base is computed once, not per access)
__device__ __forceinline__ uint4 lds128(unsigned addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ u64 lds64(unsigned addr) {
    u64 v;
    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ unsigned lds32(unsigned addr) {
    unsigned v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ unsigned lds16(unsigned addr) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts64(unsigned addr, u64 v) {
    asm volatile("st.shared.b64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
template <typename T>
__device__ __forceinline__ u64 tobits(T x);
template <>
__device__ __forceinline__ u64 tobits<u64>(u64 x) { return x; }
template <>
__device__ __forceinline__ u64 tobits<double>(double x) { return (u64)__double_as_longlong(x); }

// Σ_{i < E} ring[slot_i] for the E slots packed in w (two per 32-bit word)
template <typename T, int E>
__device__ __forceinline__ T ring_sum_w(unsigned ring_base, const uint4 (&w)[E / 8]) {
    T v[E];
#pragma unroll
    for (int i = 0; i < E / 8; i++) {
        const unsigned ws[4] = {w[i].x, w[i].y, w[i].z, w[i].w};
#pragma unroll
        for (int h = 0; h < 4; h++) {
            v[8 * i + 2 * h] = bits_to<T>(lds64(ring_base + ((ws[h] & 0xffffu) << 3)));
            v[8 * i + 2 * h + 1] = bits_to<T>(lds64(ring_base + ((ws[h] >> 16) << 3)));
        }
    }
#pragma unroll
    for (int st = 1; st < E; st <<= 1)
#pragma unroll
        for (int i = 0; i < E; i += 2 * st) v[i] += v[i + st];
    return v[0];
}

__device__ __forceinline__ int ld_acq(unsigned addr) {
    int v;
    asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel(unsigned addr, int v) {
    asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void bar_consumers(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// Warp roles: warps 0 .. NW-2 are consumers (one level at a time, named
// barrier 1 between levels); the last warp is the producer: it issues the TMA
// bulk copies of the staged chunks, waits for their mbarriers and publishes
// ready_rank (ranks < ready_rank are staged); consumers publish done_rank
// (ranks < done_rank are finished) so the producer can recycle stages.  Per
// consumer level (uniform trip counts so every shuffle is a full-warp one):
// pass p handles ranks lo + grp + p*NG; the first pass of the next level has
// its row words, g, rank->user and next-slot loaded into registers before the
// barrier, and level bounds are read two levels ahead, so after the barrier
// only the ring reads, the lane reduction and the tail are on the critical path.
template <typename T, int LPE, int E>
__global__ void __launch_bounds__(544) k_moeb_ring(RingArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int RING = a.ring_mask + 1;
    const int ch = 1 << a.lg_ch;
    const unsigned sbase = smem_u32(smem);
    const unsigned ring_base = sbase;                                    // RING + 1 entries
    u64 *bars = reinterpret_cast<u64 *>(smem + (size_t)(RING + 2) * 8);  // nstage
    const unsigned ctrl = smem_u32(bars + ((a.nstage + 1) & ~1));        // [0] ready_rank [1] done_rank
    unsigned char *stage0 = smem + (size_t)(RING + 2) * 8 + 8 * ((a.nstage + 1) & ~1) + 16;
    const unsigned stage_base = smem_u32(stage0);
    const unsigned dbytes = (unsigned)ch * a.kp * 2, gbytes = (unsigned)ch * 8;
    const unsigned ubytes = (unsigned)ch * 4, pbytes = (unsigned)ch * 2;
    const unsigned sbytes = dbytes + gbytes + ubytes + pbytes;
    const int b = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31;
    const int NTC = blockDim.x - 32;   // consumer threads
    const T *gcol = reinterpret_cast<const T *>(a.gP) + (size_t)b * a.npad;
    const int32_t nchunks = (int32_t)(a.npad >> a.lg_ch);

    if (tid == 0) {
        sts64(ring_base + (unsigned)RING * 8, 0ull);   // target of "no dependency"
        for (int s = 0; s < a.nstage; s++) mbar_init(&bars[s], 1);
        asm volatile("st.shared.s32 [%0], 0;\n\tst.shared.s32 [%0+4], 0;" ::"r"(ctrl) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (tid >= NTC) {
        // ------------------------------------------------------ producer --
        if (lane == 0) {
            auto issue = [&](int32_t c) {
                const int s = c & (a.nstage - 1);
                unsigned char *st = stage0 + (size_t)s * sbytes;
                const size_t r0 = (size_t)c << a.lg_ch;
                mbar_expect_tx(&bars[s], sbytes);
                bulk_g2s(st, a.D + r0 * a.kp, dbytes, &bars[s]);
                bulk_g2s(st + dbytes, gcol + r0, gbytes, &bars[s]);
                bulk_g2s(st + dbytes + gbytes, a.ru + r0, ubytes, &bars[s]);
                bulk_g2s(st + dbytes + gbytes + ubytes, a.Pn + r0, pbytes, &bars[s]);
            };
            int32_t issued = 0, arrived = 0;
            for (; issued < nchunks && issued < a.nstage; issued++) issue(issued);
            while (arrived < nchunks) {
                mbar_wait(&bars[arrived & (a.nstage - 1)], (unsigned)((arrived / a.nstage) & 1));
                arrived++;
                st_rel(ctrl, arrived << a.lg_ch);
                // refill every stage whose previous chunk the consumers have finished
                while (issued < nchunks) {
                    const int32_t done = ld_acq(ctrl + 4);
                    if (((int64_t)(issued - a.nstage + 1) << a.lg_ch) > done) {
                        if (arrived < issued) break;   // go wait for the next arrival
                        __nanosleep(64);
                        continue;
                    }
                    issue(issued);
                    issued++;
                }
            }
        }
        return;
    }

    // ---------------------------------------------------------- consumers --
    const int sub = tid & (LPE - 1), grp = tid / LPE, NG = NTC / LPE;
    T *f = reinterpret_cast<T *>(a.f);
    const unsigned zero_words = (unsigned)RING * 0x10001u;   // two "no dependency" slots
    auto stage_addr = [&](int32_t e) {
        return stage_base + (unsigned)((e >> a.lg_ch) & (a.nstage - 1)) * sbytes;
    };
    auto load_elem = [&](int32_t e, bool act, uint4 (&w)[E / 8], T &gx, int32_t &u, unsigned &pn) {
        if (act) {
            const unsigned st = stage_addr(e), off = (unsigned)(e & (ch - 1));
            const unsigned row = st + (off * (unsigned)a.kp + (unsigned)(sub * E)) * 2;
#pragma unroll
            for (int i = 0; i < E / 8; i++) w[i] = lds128(row + 16 * i);
            gx = bits_to<T>(lds64(st + dbytes + off * 8));
            u = (int32_t)lds32(st + dbytes + gbytes + off * 4);
            pn = lds16(st + dbytes + gbytes + ubytes + off * 2);
        } else {
#pragma unroll
            for (int i = 0; i < E / 8; i++) w[i] = make_uint4(zero_words, zero_words, zero_words, zero_words);
            gx = T(0);
            u = 0;
            pn = (unsigned)RING;
        }
    };
    int32_t staged = 0;   // ranks < staged are known to be in shared memory
    auto wait_staged = [&](int32_t rank_hi) {
        while (staged < rank_hi) staged = ld_acq(ctrl);
    };
    int32_t cache_base = 0;           // lv = lvl_ptr[cache_base + lane]
    int32_t lv = a.lvl_ptr[min(lane, a.ell)];
    int32_t lv_next = a.lvl_ptr[min(31 + lane, a.ell)];
    auto level_bounds = [&](int32_t L, int32_t &lo, int32_t &hi) {   // L non-decreasing
        if (L >= a.ell) { lo = hi = a.n; return; }
        if (L - cache_base >= 31) {
            cache_base += 31;
            lv = lv_next;
            lv_next = a.lvl_ptr[min(cache_base + 31 + lane, a.ell)];
        }
        lo = __shfl_sync(0xffffffffu, lv, L - cache_base);
        hi = __shfl_sync(0xffffffffu, lv, L - cache_base + 1);
    };

    int32_t lo, hi, nlo, nhi;
    level_bounds(0, lo, hi);
    level_bounds(1, nlo, nhi);
    wait_staged(hi);
    uint4 pw[E / 8];
    T pg;
    int32_t pu;
    unsigned ppn;
    load_elem(lo + grp, lo + grp < hi, pw, pg, pu, ppn);
    for (int32_t L = 0; L < a.ell; L++) {
        int32_t nnlo, nnhi;
        level_bounds(L + 2, nnlo, nnhi);   // two levels ahead, off the critical path
        for (int32_t base = lo; base < hi; base += NG) {
            const int32_t e = base + grp;
            const bool act = e < hi;
            uint4 w[E / 8];
            T gx;
            int32_t u;
            unsigned pn;
            if (base == lo) {
#pragma unroll
                for (int i = 0; i < E / 8; i++) w[i] = pw[i];
                gx = pg;
                u = pu;
                pn = ppn;
            } else {
                load_elem(e, act, w, gx, u, pn);
            }
            const T Fprev = bits_to<T>(lds64(ring_base + pn * 8));
            T s = ring_sum_w<T, E>(ring_base, w);
#pragma unroll
            for (int o = LPE / 2; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (sub == 0 && act) {
                const T Fx = gx - s;
                if (!(a.debug & 1)) f[(size_t)u * a.B + b] = Fx - Fprev;
                sts64(ring_base + (unsigned)(e & a.ring_mask) * 8, tobits<T>(Fx));
            }
        }
        // the next level's first pass: staged data into registers before the barrier
        if (L + 1 < a.ell) {
            wait_staged(nhi);
            load_elem(nlo + grp, nlo + grp < nhi, pw, pg, pu, ppn);
        }
        bar_consumers(NTC);
        if (tid == 0) st_rel(ctrl + 4, hi);   // ranks < hi are done: their stages may be recycled
        lo = nlo;
        hi = nhi;
        nlo = nnlo;
        nhi = nnhi;
    }
}

static constexpr size_t kSmemCap = 227 * 1024;

void ring_plan(int32_t n, int32_t k, int32_t ell, int32_t max_level_width, unsigned reach,
               RingPlan &R) {
    R.ok = false;
    R.reach = reach;
    if (n <= 0 || k > 256) return;
    int64_t ring = 32;
    while (ring < (int64_t)reach + max_level_width + 1) ring <<= 1;
    if (ring > (1 << 15)) return;   // ring slots are uint16, RING itself included
    const int entries = k <= 64 ? 64 : k <= 128 ? 128 : 256;
    // row stride = 16 B x odd: consecutive rows start in different bank quads
    const int32_t kp = entries + 8;
    const int lpe = std::min(32, entries / 8);   // 8 entries per lane (measured best)
    const double avg_w = (double)n / std::max(ell, 1);
    (void)avg_w;
    for (int nstage : {4, 2}) {
        for (int ch : {256, 128, 64, 32, 16, 8}) {
            // the current and the next level must be staged at once (prefetch)
            if (2 * (int64_t)max_level_width > (int64_t)(nstage - 1) * ch) break;
            if (ring_smem_bytes((int)ring, kp, ch, nstage) <= kSmemCap) {
                R.ok = true;
                R.kp = kp;
                R.ring = (int32_t)ring;
                R.ch = ch;
                R.nstage = nstage;
                R.lpe = lpe;
                R.entries = entries;
                R.npad = ((int64_t)n + ch - 1) / ch * ch;
                return;
            }
        }
    }
}

size_t ring_smem_bytes(int ring, int kp, int ch, int nstage) {
    return (size_t)(ring + 2) * 8 + 8 * ((nstage + 1) & ~1) + 16 +
           (size_t)nstage * ch * ((size_t)kp * 2 + 8 + 4 + 2);
}

cudaError_t launch_moebius_ring(const DevPoset &P, const RingPlan &R, int dtype, const void *gP,
                                void *f, int64_t B, cudaStream_t s) {
    if (P.n == 0) return cudaSuccess;
    RingArgs a;
    a.D = R.D;
    a.Pn = R.Pn;
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
    a.debug = R.debug;
    a.dbg = R.dbg;
    const size_t smem = ring_smem_bytes(R.ring, R.kp, R.ch, R.nstage);
    const int lpe = R.lpe, E = R.entries / R.lpe;
    void *fn = nullptr;
#define RING_FN(L, EE)                                                                          \
    if (lpe == L && E == EE)                                                                    \
        fn = dtype == 0 ? (void *)k_moeb_ring<u64, L, EE> : (void *)k_moeb_ring<double, L, EE>;
    RING_FN(1, 64) RING_FN(2, 32) RING_FN(4, 16) RING_FN(8, 8)
    RING_FN(2, 64) RING_FN(4, 32) RING_FN(8, 16) RING_FN(16, 8)
    RING_FN(4, 64) RING_FN(8, 32) RING_FN(16, 16) RING_FN(32, 8)
#undef RING_FN
    if (!fn) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const double avg_w = (double)P.n / std::max(P.ell, 1);
    int threads = (int)std::min<int64_t>(512, ((int64_t)std::ceil(avg_w * lpe) + 31) / 32 * 32);
    threads = std::max(threads, 32) + 32;   // + the producer warp
    void *args[] = {&a};
    launches_add(1);
    return cudaLaunchKernel(fn, dim3((unsigned)B), dim3(threads), args, smem, s);
}

}  // namespace poset
