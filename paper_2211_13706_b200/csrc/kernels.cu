// sm_100a kernels of the chain-decomposition zeta / Moebius transforms
// (arXiv 2211.13706; PAPER.md cited as P:Lnnn).  DESIGN.md §5 describes each
// kernel, its roofline and its algorithmic bytes.
//
//   (ii)  k_mtable       Thm. 4: m(x,j) = max_{z child of x} m(z,j),
//                        own chain -> pos(x).  One warp per chain j sweeps the
//                        antichain levels bottom-up (chains are independent).
//   (iii) k_scan_*       Eq. zeta_cache: per-chain prefix sums
//                        F = V f, a three-phase segmented scan in slot order.
//   (iv)  k_gather       Eq. zeta-fast: g(x) = Σ_j F[M[j][x]],
//                        chain-major index stream, near-broadcast F gathers,
//                        one thread = one element x, CB columns, 8..32-byte
//                        vector loads.
//   (v)   k_moeb_*       Alg. 4 first loop: back-substitution
//                        F(x) = g(x) - Σ_{j≠id(x)} F[M[j][x]] level by level.
//         k_chain_diff   Alg. 4 second loop: f = V^{-1} F.
//
// Arithmetic: T = unsigned long long (int64 in Z/2^64) or double.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <vector>

#include "kernels.cuh"

namespace poset {

typedef unsigned long long u64;

static std::atomic<int64_t> g_launches{0};
int64_t launches_take() { return g_launches.exchange(0); }
void launches_add(int64_t c) { g_launches += c; }
#define COUNT_LAUNCH(c) launches_add(c)

// ------------------------------------------------------------------ loads --
enum { LD_CA = 0, LD_NC = 1, LD_CG = 2 };

template <int V, int C>
__device__ __forceinline__ void ldv(const u64 *p, u64 *o);

#define POSET_LDV(V, C, OP, REGS, ...)                                               \
    template <>                                                                      \
    __device__ __forceinline__ void ldv<V, C>(const u64 *p, u64 *o) {                \
        asm volatile(OP REGS ", [%" #V "];" : __VA_ARGS__ : "l"(p));                 \
    }
POSET_LDV(1, LD_CA, "ld.global.b64 ", "%0", "=l"(o[0]))
POSET_LDV(1, LD_NC, "ld.global.nc.b64 ", "%0", "=l"(o[0]))
POSET_LDV(1, LD_CG, "ld.global.cg.b64 ", "%0", "=l"(o[0]))
POSET_LDV(2, LD_CA, "ld.global.v2.b64 ", "{%0,%1}", "=l"(o[0]), "=l"(o[1]))
POSET_LDV(2, LD_NC, "ld.global.nc.v2.b64 ", "{%0,%1}", "=l"(o[0]), "=l"(o[1]))
POSET_LDV(2, LD_CG, "ld.global.cg.v2.b64 ", "{%0,%1}", "=l"(o[0]), "=l"(o[1]))
POSET_LDV(4, LD_CA, "ld.global.v4.b64 ", "{%0,%1,%2,%3}", "=l"(o[0]), "=l"(o[1]), "=l"(o[2]), "=l"(o[3]))
POSET_LDV(4, LD_NC, "ld.global.nc.v4.b64 ", "{%0,%1,%2,%3}", "=l"(o[0]), "=l"(o[1]), "=l"(o[2]), "=l"(o[3]))
POSET_LDV(4, LD_CG, "ld.global.cg.v4.b64 ", "{%0,%1,%2,%3}", "=l"(o[0]), "=l"(o[1]), "=l"(o[2]), "=l"(o[3]))
#undef POSET_LDV

template <int V>
__device__ __forceinline__ void stv(u64 *p, const u64 *o);
template <>
__device__ __forceinline__ void stv<1>(u64 *p, const u64 *o) {
    asm volatile("st.global.b64 [%0], %1;" ::"l"(p), "l"(o[0]) : "memory");
}
template <>
__device__ __forceinline__ void stv<2>(u64 *p, const u64 *o) {
    asm volatile("st.global.v2.b64 [%0], {%1,%2};" ::"l"(p), "l"(o[0]), "l"(o[1]) : "memory");
}
template <>
__device__ __forceinline__ void stv<4>(u64 *p, const u64 *o) {
    asm volatile("st.global.v4.b64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(o[0]), "l"(o[1]), "l"(o[2]),
                 "l"(o[3])
                 : "memory");
}

template <typename T>
__device__ __forceinline__ T from_bits(u64 x);
template <>
__device__ __forceinline__ u64 from_bits<u64>(u64 x) { return x; }
template <>
__device__ __forceinline__ double from_bits<double>(u64 x) { return __longlong_as_double((long long)x); }
template <typename T>
__device__ __forceinline__ u64 to_bits(T x);
template <>
__device__ __forceinline__ u64 to_bits<u64>(u64 x) { return x; }
template <>
__device__ __forceinline__ u64 to_bits<double>(double x) { return (u64)__double_as_longlong(x); }

// CB consecutive columns of one row, VEC elements (8 B each) per instruction
template <typename T, int CB, int VEC, int C>
__device__ __forceinline__ void load_row(const T *p, T (&o)[CB]) {
#pragma unroll
    for (int v = 0; v < CB; v += VEC) {
        u64 t[VEC];
        ldv<VEC, C>(reinterpret_cast<const u64 *>(p + v), t);
#pragma unroll
        for (int i = 0; i < VEC; i++) o[v + i] = from_bits<T>(t[i]);
    }
}
template <typename T, int CB, int VEC>
__device__ __forceinline__ void store_row(T *p, const T (&o)[CB]) {
#pragma unroll
    for (int v = 0; v < CB; v += VEC) {
        u64 t[VEC];
#pragma unroll
        for (int i = 0; i < VEC; i++) t[i] = to_bits<T>(o[v + i]);
        stv<VEC>(reinterpret_cast<u64 *>(p + v), t);
    }
}

__device__ __forceinline__ int32_t ld_stream_i32(const int32_t *p) { return __ldcs(p); }

// ---------------------------------------------------- (ii) m-table build --
// One warp per chain j.  For every level L (bottom-up) and every rank r of L:
//   M[j][r] = slot(r)                               if chain(r) == j
//           = max_{c child of r} M[j][c]  (n = ∞ = smallest)   otherwise.
// Children lie in lower levels, already written by this warp; __syncwarp()
// orders those global stores before the next level's loads (plain ld.global,
// coherent within the SM).
__global__ void __launch_bounds__(128) k_mtable(DevPoset P, int32_t *M) {
    const int lane = threadIdx.x & 31;
    const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (j >= P.k) return;
    const int32_t n = P.n;
    int32_t *Mj = M + (size_t)j * n;
    for (int32_t L = 0; L < P.ell; L++) {
        const int32_t lo = P.lvl_ptr[L], hi = P.lvl_ptr[L + 1];
        for (int32_t base = lo; base < hi; base += 32) {
            const int32_t r = base + lane;
            if (r < hi) {
                int32_t v;
                if (P.chain[r] == j) {
                    v = P.slot[r];
                } else {
                    int32_t best = -1;
                    const int64_t a = P.child_ptr[r], b = P.child_ptr[r + 1];
                    for (int64_t t = a; t < b; t++) {
                        int32_t x = Mj[P.child[t]];
                        best = max(best, x == n ? -1 : x);
                    }
                    v = best < 0 ? n : best;
                }
                Mj[r] = v;
            }
        }
        __syncwarp();
    }
}

// The same propagation with chain j's recent values in a shared-memory ring
// (rank mod RING, RING >= the children's rank reach + the widest level) and
// the next level's child lists, chain ids and slots prefetched into
// registers one level ahead: the per-level chain of a warp is then ring
// loads -> max -> ring store -> __syncwarp instead of dependent global
// loads (~1 µs per level on C5w, 630k levels).  One warp (CTA) per chain.
constexpr int kMtCh = 4;   // children prefetched per element (more: loaded in place)
__global__ void __launch_bounds__(32) k_mtable_ring(DevPoset P, int32_t *M, int ring_mask) {
    extern __shared__ int32_t mring[];
    const int lane = threadIdx.x;
    const int j = blockIdx.x;
    const int32_t n = P.n;
    int32_t *Mj = M + (size_t)j * n;
    // prefetched first pass of the next level: element, chain, slot, children
    int32_t nr = -1, nchain = -1, nslot = 0, nc[kMtCh], nhi = 0;
    int64_t na = 0, nb = 0;
    auto fetch = [&](int32_t L) {
        nr = -1;
        if (L >= P.ell) return;
        const int32_t lo = P.lvl_ptr[L], hi = P.lvl_ptr[L + 1];
        nhi = hi;
        const int32_t r = lo + lane;
        if (r < hi) {
            nr = r;
            nchain = P.chain[r];
            nslot = P.slot[r];
            na = P.child_ptr[r];
            nb = P.child_ptr[r + 1];
#pragma unroll
            for (int t = 0; t < kMtCh; t++) nc[t] = na + t < nb ? P.child[na + t] : 0;
        }
    };
    auto value = [&](int32_t r, int32_t ch, int32_t sl, int64_t a, int64_t b, const int32_t *c4) {
        if (ch == j) return sl;
        int32_t best = -1;
        for (int64_t t = a; t < b; t++) {
            const int32_t c = (t - a < kMtCh && c4) ? c4[t - a] : P.child[t];
            const int32_t x = mring[c & ring_mask];
            best = max(best, x == n ? -1 : x);
        }
        return best < 0 ? n : best;
    };
    int32_t lo_next = P.lvl_ptr[0];
    fetch(0);
    for (int32_t L = 0; L < P.ell; L++) {
        const int32_t lo = lo_next, hi = nhi;   // prefetched with the level's first pass
        lo_next = hi;
        const int32_t r0 = nr, ch0 = nchain, sl0 = nslot;
        const int64_t a0 = na, b0 = nb;
        int32_t c0[kMtCh];
#pragma unroll
        for (int t = 0; t < kMtCh; t++) c0[t] = nc[t];
        fetch(L + 1);   // independent of this level's values: in flight meanwhile
        if (r0 >= 0) {
            const int32_t v = value(r0, ch0, sl0, a0, b0, c0);
            mring[r0 & ring_mask] = v;
            Mj[r0] = v;
        }
        for (int32_t base = lo + 32; base < hi; base += 32) {   // wide levels: further passes
            const int32_t r = base + lane;
            if (r < hi) {
                const int32_t v = value(r, P.chain[r], P.slot[r], P.child_ptr[r], P.child_ptr[r + 1], nullptr);
                mring[r & ring_mask] = v;
                Mj[r] = v;
            }
        }
        __syncwarp();
    }
}

cudaError_t launch_mtable(const DevPoset &P, int32_t *M, cudaStream_t s, int32_t child_reach,
                          int32_t max_level_width) {
    if (P.k == 0) return cudaSuccess;
    int ring = 32;
    while (ring < child_reach + max_level_width + 1) ring <<= 1;
    if (child_reach >= 0 && ring <= 16384) {   // ring of <= 64 KB per chain
        const size_t smem = (size_t)ring * 4;
        cudaError_t e = cudaFuncSetAttribute(k_mtable_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_mtable_ring<<<(unsigned)P.k, 32, smem, s>>>(P, M, ring - 1);
        COUNT_LAUNCH(1);
        return cudaGetLastError();
    }
    const int wpb = 4;
    k_mtable<<<(P.k + wpb - 1) / wpb, 32 * wpb, 0, s>>>(P, M);
    COUNT_LAUNCH(1);
    return cudaGetLastError();
}

__global__ void k_count_nnz(const int32_t *__restrict__ M, int64_t total, int32_t n,
                            unsigned long long *out) {
    unsigned long long c = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x)
        c += (__ldcs(M + i) < n);
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

cudaError_t launch_count_nnz(const int32_t *M, int64_t total, int32_t n,
                             unsigned long long *out, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    if (total == 0) return cudaSuccess;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    k_count_nnz<<<blocks, 256, 0, s>>>(M, total, n, out);
    COUNT_LAUNCH(1);
    return cudaGetLastError();
}

// ------------------------------------------- D_U: depth of the U-solve ----
// D(r) = 1 + max { D(y) : y = chain_j[m(r,j)], j ≠ chain(r), m(r,j) ≥ 0 }
// (1 with no cross-chain dependency); D_U = max_r D(r), the length of the
// longest dependency path of Alg. 4's first loop -- the PRAM depth of the
// triangular solve.  One CTA sweeps the levels in order (a
// level's dependencies lie in lower levels); warp per element, lanes over
// chains.  Diagnostic only (poset_set_option "compute_depth_u").
__global__ void __launch_bounds__(1024) k_depth_u(DevPoset P, const int32_t *__restrict__ slot_rank,
                                                  int32_t *D, unsigned *out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned best = 0;
    for (int32_t L = 0; L < P.ell; L++) {
        const int32_t lo = P.lvl_ptr[L], hi = P.lvl_ptr[L + 1];
        for (int32_t r = lo + warp; r < hi; r += 32) {
            const int32_t c = P.chain[r];
            int d = 0;
            for (int32_t j = lane; j < P.k; j += 32) {
                const int32_t sl = P.M[(size_t)j * P.n + r];
                if (j != c && sl != P.n) d = max(d, D[slot_rank[sl]]);
            }
            d = __reduce_max_sync(0xffffffffu, d) + 1;
            if (lane == 0) {
                D[r] = d;
                best = max(best, (unsigned)d);
            }
        }
        __syncthreads();
    }
    if (lane == 0) atomicMax(out, best);
}

cudaError_t launch_depth_u(const DevPoset &P, const int32_t *slot_rank, int32_t *D, unsigned *out,
                           cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned), s);
    if (e != cudaSuccess || P.n == 0) return e;
    k_depth_u<<<1, 1024, 0, s>>>(P, slot_rank, D, out);
    COUNT_LAUNCH(1);
    return cudaGetLastError();
}

// ------------------------------------------------ (iii) segmented scan ----
// Slot range [lo, lo+rows).  A CTA tile = RG row groups x CB columns; a
// thread scans R consecutive slots of one column serially, row-group
// aggregates are combined with a Hillis-Steele segmented scan in shared
// memory.  Segment operator on (flag, value) pairs describing a contiguous
// range (flag = the range contains a chain start, value = sum after the last
// start, or of everything):  (fa,va) ⊕ (fb,vb) = (fa|fb, fb ? vb : va+vb).
struct ScanGeom {
    int CB, RG, R;
    int64_t tile_rows, ntiles;
    int gy;
};
static ScanGeom scan_geom(int64_t rows, int64_t B) {
    ScanGeom g;
    g.CB = (int)std::min<int64_t>(B, 32);
    g.RG = 256 / g.CB;
    g.R = 16;
    g.tile_rows = (int64_t)g.RG * g.R;
    g.ntiles = (rows + g.tile_rows - 1) / g.tile_rows;
    g.gy = (int)((B + g.CB - 1) / g.CB);
    return g;
}

size_t scan_scratch_bytes(int64_t rows, int64_t B) {
    ScanGeom g = scan_geom(rows, B);
    // agg values, carry values (8 B each) + agg flags (4 B)
    return (size_t)std::max<int64_t>(g.ntiles, 1) * B * (8 + 8 + 4) + 256;
}

template <typename T>
__device__ __forceinline__ void seg_block_scan(T &v, int &fl, int rg, int bl, int RG, int CB,
                                               T *sv, int *sf) {
    // inclusive segmented scan of (fl, v) over rg for each column bl
    for (int d = 1; d < RG; d <<= 1) {
        __syncthreads();
        if (rg < RG) { sv[rg * CB + bl] = v; sf[rg * CB + bl] = fl; }
        __syncthreads();
        if (rg < RG && rg >= d) {
            T pv = sv[(rg - d) * CB + bl];
            int pf = sf[(rg - d) * CB + bl];
            if (!fl) v = pv + v;
            fl |= pf;
        }
    }
    __syncthreads();
    if (rg < RG) { sv[rg * CB + bl] = v; sf[rg * CB + bl] = fl; }
    __syncthreads();
}

// NVLS multicast store: one st through the multicast
// address reaches the same offset of every device's buffer bound to the
// multicast object (NVSwitch replicates it) -- the all-gather of F fused into
// the scan epilogue.
__device__ __forceinline__ void mc_st64(void *p, unsigned long long v) {
    asm volatile("multimem.st.weak.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <typename T>
__global__ void __launch_bounds__(256) k_scan_tiles(const T *__restrict__ f, T *__restrict__ F,
                                                    const int32_t *__restrict__ slot_user,
                                                    int64_t lo, int64_t rows, int32_t B, int CB,
                                                    int RG, int R, T *agg_v, int *agg_f,
                                                    const T *carry, int phase, T *Fmc = nullptr) {
    __shared__ T sv[256];
    __shared__ int sf[256];
    const int bl = threadIdx.x % CB, rg = threadIdx.x / CB;
    const int b = blockIdx.y * CB + bl;
    const bool act = rg < RG && b < B;
    const int64_t t = blockIdx.x;
    const int64_t s0 = lo + t * (int64_t)RG * R + (int64_t)rg * R;
    const int64_t end = lo + rows;
    T v = T(0);
    int fl = 0;
    if (act) {
        for (int i = 0; i < R; i++) {
            int64_t s = s0 + i;
            if (s >= end) break;
            int32_t u = slot_user[s];
            if (u < 0) { fl = 1; v = T(0); }
            v += f[(size_t)(u & 0x7fffffff) * B + b];
        }
    }
    seg_block_scan<T>(v, fl, rg, bl, RG, CB, sv, sf);
    if (phase == 1) {
        if (act && rg == RG - 1) {
            agg_v[t * B + b] = v;
            agg_f[t * B + b] = fl;
        }
        return;
    }
    if (!act) return;
    // exclusive prefix for this row group, seeded by the tile carry
    T run = carry[t * B + b];
    if (rg > 0) {
        T pv = sv[(rg - 1) * CB + bl];
        int pf = sf[(rg - 1) * CB + bl];
        run = pf ? pv : run + pv;
    }
    for (int i = 0; i < R; i++) {
        int64_t s = s0 + i;
        if (s >= end) break;
        int32_t u = slot_user[s];
        if (u < 0) run = T(0);
        run += f[(size_t)(u & 0x7fffffff) * B + b];
        if (Fmc) mc_st64(Fmc + (size_t)s * B + b, to_bits<T>(run));
        else F[(size_t)s * B + b] = run;
    }
    if (Fmc) __threadfence_system();   // the rows are visible to every peer at kernel end
}

// carry[t] = value of the exclusive segmented prefix over tiles < t (per column)
template <typename T>
__global__ void __launch_bounds__(1024) k_scan_carry_tiles(const T *agg_v, const int *agg_f,
                                                           T *carry, int64_t ntiles, int32_t B,
                                                           T *tail) {
    __shared__ T sv[1024];
    __shared__ int sf[1024];
    const int b = blockIdx.x;
    const int tid = threadIdx.x;
    const int64_t chunk = (ntiles + 1023) / 1024;
    const int64_t a = tid * chunk, e = (a + chunk < ntiles) ? a + chunk : ntiles;
    T v = T(0);
    int fl = 0;
    for (int64_t i = a; i < e; i++) {
        int af = agg_f[i * B + b];
        T av = agg_v[i * B + b];
        v = af ? av : v + av;
        fl |= af;
    }
    seg_block_scan<T>(v, fl, tid, 0, 1024, 1, sv, sf);
    T run = T(0);
    int rf = 0;
    if (tid > 0) { run = sv[tid - 1]; rf = sf[tid - 1]; }
    for (int64_t i = a; i < e; i++) {
        carry[i * B + b] = run;
        int af = agg_f[i * B + b];
        T av = agg_v[i * B + b];
        run = af ? av : run + av;
        rf |= af;
    }
    if (tail && tid == 1023) {
        reinterpret_cast<u64 *>(tail)[b] = (u64)(sf[1023] != 0);
        tail[B + b] = sv[1023];
    }
}

template <typename T>
static cudaError_t scan_t(const DevPoset &P, const void *f, void *F, int64_t lo, int64_t hi,
                          int64_t B, void *scratch, void *tail, cudaStream_t s, void *Fmc) {
    const int64_t rows = hi - lo;
    if (rows <= 0) {
        if (tail) return cudaMemsetAsync(tail, 0, sizeof(T) * 2 * B, s);
        return cudaSuccess;
    }
    ScanGeom g = scan_geom(rows, B);
    T *agg_v = reinterpret_cast<T *>(scratch);
    T *carry = agg_v + g.ntiles * B;
    int *agg_f = reinterpret_cast<int *>(carry + g.ntiles * B);
    dim3 grid((unsigned)g.ntiles, (unsigned)g.gy);
    k_scan_tiles<T><<<grid, 256, 0, s>>>((const T *)f, (T *)F, P.slot_user, lo, rows, (int32_t)B,
                                         g.CB, g.RG, g.R, agg_v, agg_f, nullptr, 1);
    k_scan_carry_tiles<T><<<(unsigned)B, 1024, 0, s>>>(agg_v, agg_f, carry, g.ntiles, (int32_t)B,
                                                       (T *)tail);
    k_scan_tiles<T><<<grid, 256, 0, s>>>((const T *)f, (T *)F, P.slot_user, lo, rows, (int32_t)B,
                                         g.CB, g.RG, g.R, agg_v, agg_f, carry, 3, (T *)Fmc);
    COUNT_LAUNCH(3);
    return cudaGetLastError();
}

cudaError_t launch_scan(const DevPoset &P, int dtype, const void *f, void *F, int64_t lo,
                        int64_t hi, int64_t B, void *scratch, void *tail, cudaStream_t s, void *Fmc) {
    return dtype == 0 ? scan_t<u64>(P, f, F, lo, hi, B, scratch, tail, s, Fmc)
                      : scan_t<double>(P, f, F, lo, hi, B, scratch, tail, s, Fmc);
}

// ---------------------------------------- (iii) single-pass scan (zeta) ----
// Decoupled look-back: one pass over f.  Tiles of RG row groups x CB columns
// (R = 16 slots per thread, kept in registers) are taken in slot order from
// an atomic ticket (so every predecessor is running or done); a tile
// publishes its aggregate (flag, value) per column, looks back over its
// predecessors' published aggregates / inclusive prefixes until it meets a
// prefix or a chain start (the segmented operator restarts there), publishes
// its own inclusive prefix, and writes F from the registers.  f is read once
// and F written once: 16nB bytes (the three-kernel scan above read f twice).
// status[(t * B + b)]: {value, flag | state << 1}, state 0 = empty,
// 1 = aggregate, 2 = inclusive prefix.
struct ScanStatus { unsigned long long v; unsigned long long fs; };

template <typename T>
__device__ __forceinline__ void st_status(ScanStatus *p, T v, unsigned fl, unsigned state) {
    const unsigned long long bits = to_bits<T>(v);
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(bits),
                 "l"((unsigned long long)(fl | (state << 1)))
                 : "memory");
}
template <typename T>
__device__ __forceinline__ unsigned ld_status(const ScanStatus *p, T &v, unsigned &fl) {
    unsigned long long a, b;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
    v = from_bits<T>(a);
    fl = (unsigned)(b & 1u);
    return (unsigned)(b >> 1);
}

template <typename T>
__global__ void __launch_bounds__(256) k_scan_1p(const T *__restrict__ f, T *__restrict__ F,
                                                 const int32_t *__restrict__ slot_user, int64_t rows,
                                                 int32_t B, int CB, int RG, ScanStatus *status,
                                                 unsigned *ticket, int64_t ntiles) {
    constexpr int R = 16;
    __shared__ T sv[256];
    __shared__ int sf[256];
    __shared__ T sexcl[32];
    __shared__ int sexf[32];
    __shared__ int64_t stile;
    const int bl = threadIdx.x % CB, rg = threadIdx.x / CB;
    const int b = blockIdx.y * CB + bl;
    const bool act = rg < RG && b < B;
    if (threadIdx.x == 0) stile = atomicAdd(ticket + blockIdx.y, 1u);
    __syncthreads();
    const int64_t t = stile;
    const int64_t s0 = t * (int64_t)RG * R + (int64_t)rg * R;
    T x[R];
    int st[R];
    T v = T(0);
    int fl = 0;
#pragma unroll
    for (int i = 0; i < R; i++) {
        const int64_t sl = s0 + i;
        x[i] = T(0);
        st[i] = 0;
        if (act && sl < rows) {
            const int32_t u = slot_user[sl];
            st[i] = u < 0;
            x[i] = f[(size_t)(u & 0x7fffffff) * B + b];
            if (st[i]) { fl = 1; v = T(0); }
            v += x[i];
        }
    }
    seg_block_scan<T>(v, fl, rg, bl, RG, CB, sv, sf);
    // tile aggregate per column = inclusive value of the last row group
    if (act && rg == RG - 1) {
        ScanStatus *my = status + (size_t)t * B + b;
        if (t == 0) {
            st_status<T>(my, v, (unsigned)fl, 2u);
            sexcl[bl] = T(0);
            sexf[bl] = 0;
        } else {
            st_status<T>(my, v, (unsigned)fl, 1u);
            // look back: running = (predecessors' aggregates) ⊕ ..., right to left
            T run = T(0);
            int rf = 0;
            for (int64_t p = t - 1;; p--) {
                T pv;
                unsigned pf, state;
                do { state = ld_status<T>(status + (size_t)p * B + b, pv, pf); } while (state == 0);
                run = rf ? run : pv + run;   // (pf, pv) ⊕ (rf, run)
                rf |= (int)pf;
                if (state == 2 || pf) break;
            }
            sexcl[bl] = run;
            sexf[bl] = rf;
            // this tile's inclusive prefix = exclusive ⊕ aggregate
            const T inc = fl ? v : run + v;
            st_status<T>(my, inc, (unsigned)(fl | rf), 2u);
        }
    }
    __syncthreads();
    if (!act) return;
    // this row group's exclusive prefix: tile exclusive ⊕ earlier row groups
    T run = sexcl[bl];
    if (rg > 0) {
        const T pv = sv[(rg - 1) * CB + bl];
        const int pf = sf[(rg - 1) * CB + bl];
        run = pf ? pv : run + pv;
    }
#pragma unroll
    for (int i = 0; i < R; i++) {
        const int64_t sl = s0 + i;
        if (sl < rows) {
            if (st[i]) run = T(0);
            run += x[i];
            F[(size_t)sl * B + b] = run;
        }
    }
}

size_t scan1p_scratch_bytes(int64_t rows, int64_t B) {
    ScanGeom g = scan_geom(rows, B);
    return (size_t)std::max<int64_t>(g.ntiles, 1) * B * sizeof(ScanStatus) + 64 * sizeof(unsigned) + 256;
}

template <typename T>
static cudaError_t scan1p_t(const DevPoset &P, const void *f, void *F, int64_t B, void *scratch,
                            cudaStream_t s) {
    const int64_t rows = P.n;
    if (rows <= 0) return cudaSuccess;
    ScanGeom g = scan_geom(rows, B);
    if (g.gy > 64) return cudaErrorInvalidValue;   // B > 2048: the caller uses the three-kernel scan
    ScanStatus *status = reinterpret_cast<ScanStatus *>(scratch);
    unsigned *ticket = reinterpret_cast<unsigned *>(status + (size_t)g.ntiles * B);
    cudaError_t e = cudaMemsetAsync(scratch, 0, scan1p_scratch_bytes(rows, B), s);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)g.ntiles, (unsigned)g.gy);
    k_scan_1p<T><<<grid, 256, 0, s>>>((const T *)f, (T *)F, P.slot_user, rows, (int32_t)B, g.CB, g.RG, status,
                                      ticket, g.ntiles);
    COUNT_LAUNCH(1);
    return cudaGetLastError();
}

cudaError_t launch_scan_1p(const DevPoset &P, int dtype, const void *f, void *F, int64_t B, void *scratch,
                           cudaStream_t s) {
    return dtype == 0 ? scan1p_t<u64>(P, f, F, B, scratch, s) : scan1p_t<double>(P, f, F, B, scratch, s);
}

template <typename T>
__global__ void k_add_carry(T *F, const T *carry, int64_t lo, int64_t end, int32_t B) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t tot = (end - lo) * B;
    if (i >= tot) return;
    F[(size_t)lo * B + i] += carry[i % B];
}

cudaError_t launch_scan_carry(const DevPoset &P, int dtype, void *F, const void *carry,
                              int64_t lo, int64_t end, int64_t B, cudaStream_t s) {
    int64_t tot = (end - lo) * B;
    if (tot <= 0) return cudaSuccess;
    unsigned blocks = (unsigned)((tot + 255) / 256);
    COUNT_LAUNCH(1);
    if (dtype == 0)
        k_add_carry<u64><<<blocks, 256, 0, s>>>((u64 *)F, (const u64 *)carry, lo, end, (int32_t)B);
    else
        k_add_carry<double><<<blocks, 256, 0, s>>>((double *)F, (const double *)carry, lo, end,
                                                   (int32_t)B);
    return cudaGetLastError();
}

// carry into rank `rank` = value of (tail_0 ⊕ ... ⊕ tail_{rank-1})
template <typename T>
__global__ void k_combine_tails(const T *tails, int64_t rank, T *carry, int32_t B) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    T run = T(0);
    for (int64_t p = 0; p < rank; p++) {
        const T *tp = tails + (size_t)p * 2 * B;
        u64 fl = reinterpret_cast<const u64 *>(tp)[b];
        T v = tp[B + b];
        run = fl ? v : run + v;
    }
    carry[b] = run;
}

cudaError_t launch_combine_tails(int dtype, const void *tails, int64_t world, int64_t rank,
                                void *carry, int64_t B, cudaStream_t s) {
    (void)world;
    unsigned blocks = (unsigned)((B + 127) / 128);
    COUNT_LAUNCH(1);
    if (dtype == 0)
        k_combine_tails<u64><<<blocks, 128, 0, s>>>((const u64 *)tails, rank, (u64 *)carry, (int32_t)B);
    else
        k_combine_tails<double><<<blocks, 128, 0, s>>>((const double *)tails, rank, (double *)carry,
                                                      (int32_t)B);
    return cudaGetLastError();
}

// ---------------------------------------------- (iv) zeta gather-reduce ---
// Lane = one rank r (a warp owns 32 consecutive ranks, so the chain-major
// index row M[j][r..r+31] is one coalesced 128-B load); CB <= 8 consecutive
// columns per thread.  The WG warps of a CTA that own the same 32 ranks take
// WG different column groups and share each index row through L1
// (ld.global.nc).  Index loads run U chains ahead of the F loads (register
// double buffer), which keeps ~U x 128 B of the HBM index stream in flight
// per warp.  F rows gathered by a warp are near-identical for chain-local
// posets (1.6-2.4 distinct sectors per warp-gather), so the F
// loads are L1 broadcasts.  Block id: column-group block fastest, then
// j-slice, then rank tile.
template <typename T, int CB, int VEC, int U>
__global__ void __launch_bounds__(256) k_gather(const int32_t *__restrict__ M, int32_t n, int32_t k, int64_t ldm,
                                                const T *__restrict__ F, T *__restrict__ out,
                                                const int32_t *__restrict__ rank_user,
                                                int64_t row_lo, int64_t row_hi, int32_t B, int GB,
                                                int WG, int S, int mode) {
    const int64_t bid = blockIdx.x;
    const int cgb = (int)(bid % GB);
    const int64_t rest = bid / GB;
    const int slice = (int)(rest % S);
    const int64_t tile = rest / S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wc = warp % WG, wr = warp / WG;
    const int ranks_per_cta = 32 * (8 / WG);
    const int64_t r = row_lo + tile * ranks_per_cta + wr * 32 + lane;
    if (r >= row_hi) return;
    const int j0 = (int)((int64_t)slice * k / S), j1 = (int)((int64_t)(slice + 1) * k / S);
    const int c0 = (cgb * WG + wc) * CB;
    T acc[CB];
#pragma unroll
    for (int c = 0; c < CB; c++) acc[c] = T(0);
    const int32_t *Mr = M + r;
    const T *Fc = F + c0;
    int32_t idx[U];
#pragma unroll
    for (int u = 0; u < U; u++) idx[u] = (j0 + u < j1) ? __ldg(Mr + (size_t)(j0 + u) * ldm) : n;
    for (int j = j0; j < j1; j += U) {
        int32_t nidx[U];
#pragma unroll
        for (int u = 0; u < U; u++)
            nidx[u] = (j + U + u < j1) ? __ldg(Mr + (size_t)(j + U + u) * ldm) : n;
#pragma unroll
        for (int u = 0; u < U; u++) {
            T v[CB];
            load_row<T, CB, VEC, LD_NC>(Fc + (size_t)idx[u] * B, v);
#pragma unroll
            for (int c = 0; c < CB; c++) acc[c] += v[c];
        }
#pragma unroll
        for (int u = 0; u < U; u++) idx[u] = nidx[u];
    }
    T *dst;
    if (mode == 0)
        dst = out + (size_t)rank_user[r] * B + c0;
    else if (mode == 1)
        dst = out + (size_t)(r - row_lo) * B + c0;
    else
        dst = out + ((size_t)slice * (row_hi - row_lo) + (r - row_lo)) * B + c0;
    store_row<T, CB, VEC>(dst, acc);
}

// Lanes over COLUMNS (B % 32 == 0): a warp owns TR = 8 consecutive ranks and
// 32 consecutive columns.  For chain j the 8 indices M[j][r..r+7] are
// warp-uniform; each DISTINCT row of F among them (a "run head") is fetched
// once as one coalesced 256-B load and forwarded in registers to the rest of
// its run (chain-local posets: 1-3 distinct rows per 8 ranks).  This removes
// the L1 data-pipe bound of the lanes-over-ranks kernel (8 B returned to every
// lane per rank, chain and column).  Index chunks (KCH chains x 8 ranks) are
// staged in shared memory by cp.async one chunk ahead; the row loads of chain
// j+1 are issued before chain j is resolved (software pipeline).
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// raw[t] = *(row of id[t]) if id[t] starts a run (t == 0 or id[t] != id[t-1]),
// undefined otherwise; one asm block so the 8 loads stay independent.
__device__ __forceinline__ void head_loads8(const char *Fb, unsigned rowbytes, const int32_t (&id)[8],
                                           u64 (&raw)[8]) {
    const char *p[8];
#pragma unroll
    for (int t = 0; t < 8; t++) p[t] = Fb + (size_t)(unsigned)id[t] * rowbytes;
    asm("{\n\t.reg .pred q<8>;\n\t"
        "setp.ne.s32 q1, %9, %8;\n\tsetp.ne.s32 q2, %10, %9;\n\tsetp.ne.s32 q3, %11, %10;\n\t"
        "setp.ne.s32 q4, %12, %11;\n\tsetp.ne.s32 q5, %13, %12;\n\tsetp.ne.s32 q6, %14, %13;\n\t"
        "setp.ne.s32 q7, %15, %14;\n\t"
        "ld.global.nc.b64 %0, [%16];\n\t"
        "@q1 ld.global.nc.b64 %1, [%17];\n\t@q2 ld.global.nc.b64 %2, [%18];\n\t"
        "@q3 ld.global.nc.b64 %3, [%19];\n\t@q4 ld.global.nc.b64 %4, [%20];\n\t"
        "@q5 ld.global.nc.b64 %5, [%21];\n\t@q6 ld.global.nc.b64 %6, [%22];\n\t"
        "@q7 ld.global.nc.b64 %7, [%23];\n\t}"
        : "=l"(raw[0]), "=l"(raw[1]), "=l"(raw[2]), "=l"(raw[3]), "=l"(raw[4]), "=l"(raw[5]),
          "=l"(raw[6]), "=l"(raw[7])
        : "r"(id[0]), "r"(id[1]), "r"(id[2]), "r"(id[3]), "r"(id[4]), "r"(id[5]), "r"(id[6]),
          "r"(id[7]), "l"(p[0]), "l"(p[1]), "l"(p[2]), "l"(p[3]), "l"(p[4]), "l"(p[5]), "l"(p[6]),
          "l"(p[7]));
}

template <typename T, int KCH>
__global__ void __launch_bounds__(256, 2) k_gather_cols(const int32_t *__restrict__ M, int32_t n,
                                                        int32_t k, int64_t ldm, const T *__restrict__ F,
                                                        T *__restrict__ out,
                                                        const int32_t *__restrict__ rank_user,
                                                        int64_t row_lo, int64_t row_hi, int32_t B,
                                                        int G32, int mode) {
    constexpr int TR = 8;
    __shared__ __align__(16) int32_t sidx[2][8][KCH][TR];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cg = (int)(blockIdx.x % G32);
    const int64_t tile = blockIdx.x / G32;
    const int64_t r0 = row_lo + (tile * 8 + warp) * TR;
    if (r0 >= row_hi) return;
    const int col = cg * 32 + lane;
    const char *Fb = reinterpret_cast<const char *>(F + col);
    const unsigned rowbytes = (unsigned)B * sizeof(T);
    const int nchunk = (k + KCH - 1) / KCH;
    // word w of a chunk (KCH*TR words, KCH*TR/32 per lane): chain w / TR, rank w % TR
    auto stage = [&](int c) {
        int32_t (*S)[TR] = sidx[c & 1][warp];
        const int j0 = c * KCH;
#pragma unroll 4
        for (int i = 0; i < KCH * TR / 32; i++) {
            const int w = i * 32 + lane, jj = w / TR, t = w % TR;
            const int64_t r = r0 + t;
            if (j0 + jj < k && r < row_hi)
                cp_async4(&S[jj][t], M + (size_t)(j0 + jj) * ldm + r);
            else
                S[jj][t] = n;   // the zero row of F
        }
    };
    T acc[TR];
#pragma unroll
    for (int t = 0; t < TR; t++) acc[t] = T(0);
    stage(0);
    for (int c = 0; c < nchunk; c++) {
        cp_async_wait_all();
        __syncwarp();
        if (c + 1 < nchunk) stage(c + 1);   // next chunk in flight during this one
        int32_t (*S)[TR] = sidx[c & 1][warp];
        const int jn = min(KCH, k - c * KCH);
        // ping-pong register sets A / B: the loads of one chain are in flight
        // while the other chain is resolved (no register moves between them)
        int32_t idA[TR], idB[TR];
        u64 rawA[TR], rawB[TR];
        auto fetch = [&](int jj, int32_t (&id)[TR], u64 (&raw)[TR]) {
            const int4 q0 = *reinterpret_cast<const int4 *>(&S[jj][0]);
            const int4 q1 = *reinterpret_cast<const int4 *>(&S[jj][4]);
            id[0] = q0.x; id[1] = q0.y; id[2] = q0.z; id[3] = q0.w;
            id[4] = q1.x; id[5] = q1.y; id[6] = q1.z; id[7] = q1.w;
            head_loads8(Fb, rowbytes, id, raw);
        };
        auto resolve = [&](const int32_t (&id)[TR], const u64 (&raw)[TR]) {
            u64 v = raw[0];
#pragma unroll
            for (int t = 0; t < TR; t++) {
                if (t > 0) v = id[t] != id[t - 1] ? raw[t] : v;
                acc[t] += from_bits<T>(v);
            }
        };
        fetch(0, idA, rawA);
#pragma unroll 1
        for (int jj = 0; jj < jn; jj += 2) {
            if (jj + 1 < jn) fetch(jj + 1, idB, rawB);
            resolve(idA, rawA);
            if (jj + 2 < jn) fetch(jj + 2, idA, rawA);
            if (jj + 1 < jn) resolve(idB, rawB);
        }
        __syncwarp();
    }
#pragma unroll
    for (int t = 0; t < TR; t++) {
        const int64_t r = r0 + t;
        if (r < row_hi) {
            T *dst = mode == 0 ? out + (size_t)rank_user[r] * B : out + (size_t)(r - row_lo) * B;
            dst[col] = acc[t];
        }
    }
}

// Lanes over (rank, 4 columns) -- B % 32 == 0, the batched configs.  A warp
// owns 16 consecutive ranks: lane group q = lane / 8 (4 groups) walks ranks
// 4q .. 4q+3 one after the other, lane l % 8 owns columns 4(l%8) .. 4(l%8)+3
// of a 32-column group.  For each chain j a lane keeps the F row it last
// used (4 values) in registers and reloads it -- one predicated 32-byte load
// straight into the held registers -- only when the chain's index changes
// from the previous rank (the "run" structure of chain-local posets).  Per
// (rank, chain, 32 columns) this costs 1/4 of a compare, address and load
// issue plus the 32 adds, against ~7 instructions of the lanes-over-columns
// form.  Index chunks (64 chains x 16 ranks per warp) are staged by cp.async.
__device__ __forceinline__ void ld4_if_ne(u64 (&v)[4], const void *p, int32_t a, int32_t b) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %4, %5;\n\t"
                 "@q ld.global.nc.v4.b64 {%0,%1,%2,%3}, [%6];\n\t}"
                 : "+l"(v[0]), "+l"(v[1]), "+l"(v[2]), "+l"(v[3])
                 : "r"(a), "r"(b), "l"(p));
}

template <typename T, int KCH, int KC = 4, int MINB = 2>
__global__ void __launch_bounds__(256, MINB) k_gather_r4(const int32_t *__restrict__ M, int32_t n,
                                                      int32_t k, int64_t ldm, const T *__restrict__ F,
                                                      T *__restrict__ out,
                                                      const int32_t *__restrict__ rank_user,
                                                      int64_t row_lo, int64_t row_hi, int32_t B,
                                                      int G32, int mode) {
    constexpr int TS = 4, TRW = 16;   // ranks per lane, ranks per warp; KC chains per step
    // rank-major id tile, row stride KCH + 2 words: the staging writes (lanes
    // over 16 ranks x 2 chains) and the 4 lane groups' 8-byte reads of rows
    // 4q + ts both fall on distinct banks (ncu: the unpadded 64-word stride
    // made shared-memory wavefronts the bulk of the L1 data-pipe load)
    constexpr int SW = KCH + 2;
    __shared__ __align__(16) int32_t sid[8][TRW][SW];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = lane >> 3, cq = lane & 7;
    const int cg = (int)(blockIdx.x % G32);
    const int64_t tile = blockIdx.x / G32;
    const int64_t r0 = row_lo + (tile * 8 + warp) * TRW;
    if (r0 >= row_hi) return;
    const int col0 = cg * 32 + cq * 4;
    const char *Fb = reinterpret_cast<const char *>(F + col0);
    const unsigned rowbytes = (unsigned)B * sizeof(T);
    int32_t (*S)[SW] = sid[warp];
    T acc[TS][4];
#pragma unroll
    for (int ts = 0; ts < TS; ts++)
#pragma unroll
        for (int c = 0; c < 4; c++) acc[ts][c] = T(0);
    for (int j0 = 0; j0 < k; j0 += KCH) {
        __syncwarp();
        // word w: chain w / TRW, rank w % TRW (16 consecutive ranks = 64 B)
#pragma unroll 4
        for (int i = 0; i < KCH * TRW / 32; i++) {
            const int w = i * 32 + lane, jj = w / TRW, t = w % TRW;
            const int64_t r = r0 + t;
            if (j0 + jj < k && r < row_hi)
                cp_async4(&S[t][jj], M + (size_t)(j0 + jj) * ldm + r);
            else
                S[t][jj] = n;   // the zero row of F
        }
        cp_async_wait_all();
        __syncwarp();
        const int jn = min(KCH, k - j0);
        for (int jj = 0; jj < jn; jj += KC) {
            u64 v[KC][4];
            int32_t prev[KC];
#pragma unroll
            for (int u = 0; u < KC; u++) prev[u] = -1;   // never an index: first rank loads
#pragma unroll
            for (int ts = 0; ts < TS; ts++) {
                int32_t id[KC];
#pragma unroll
                for (int u = 0; u < KC; u += 2) {
                    const int2 id2 = *reinterpret_cast<const int2 *>(&S[q * TS + ts][jj + u]);
                    id[u] = id2.x;
                    id[u + 1] = id2.y;
                }
#pragma unroll
                for (int u = 0; u < KC; u++) {
                    ld4_if_ne(v[u], Fb + (size_t)(unsigned)id[u] * rowbytes, id[u], prev[u]);
                    prev[u] = id[u];
                }
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    T t = from_bits<T>(v[0][c]);
#pragma unroll
                    for (int u = 1; u < KC; u++) t += from_bits<T>(v[u][c]);
                    acc[ts][c] += t;
                }
            }
        }
    }
#pragma unroll
    for (int ts = 0; ts < TS; ts++) {
        const int64_t r = r0 + q * TS + ts;
        if (r < row_hi) {
            T *dst = mode == 0 ? out + (size_t)rank_user[r] * B : out + (size_t)(r - row_lo) * B;
            u64 o[4];
#pragma unroll
            for (int c = 0; c < 4; c++) o[c] = to_bits<T>(acc[ts][c]);
            stv<4>(reinterpret_cast<u64 *>(dst + col0), o);
        }
    }
}

template <typename T>
__global__ void k_gather_reduce(const T *__restrict__ part, T *__restrict__ out,
                                const int32_t *__restrict__ rank_user, int64_t row_lo,
                                int64_t rows, int32_t B, int S, int mode) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows * B) return;
    int64_t rr = i / B;
    int b = (int)(i % B);
    T acc = T(0);
    for (int sl = 0; sl < S; sl++) acc += part[((size_t)sl * rows + rr) * B + b];
    if (mode == 0)
        out[(size_t)rank_user[row_lo + rr] * B + b] = acc;
    else
        out[(size_t)rr * B + b] = acc;
}

// Dense-gather variant for B % 32 == 0 (process-wide; poset_set_option
// "gather_variant"): 0 = gather order (gather_pi.cu; rank-order k_gather_r4
// for row ranges and when the order table does not fit), 1 = k_gather_cols,
// 2 = k_gather (lanes over ranks), 3 / 4 = k_gather_r4 with 4 / 2 chains per step.
static std::atomic<int> g_gather_variant{0};
void set_gather_variant(int v) { g_gather_variant = v; }
static int gather_variant() { return g_gather_variant.load(); }
int gather_variant_get() { return gather_variant(); }

static int gather_cb(int64_t B) {
    for (int cb : {8, 4, 2, 1})
        if (B % cb == 0) return cb;
    return 1;
}

static int pick_cb(int64_t B) {
    for (int cb : {32, 16, 8, 4, 2, 1})
        if (B % cb == 0) return cb;
    return 1;
}

static int gather_slices(const DevPoset &P, int64_t rows, int64_t B, int num_sms) {
    int CB = gather_cb(B);
    int64_t G = B / CB;
    int64_t warps = ((rows + 31) / 32) * G;
    int64_t target = (int64_t)num_sms * 48;
    if (warps >= target || P.k < 16) return 1;
    int64_t S = (target + warps - 1) / warps;
    S = std::min<int64_t>(S, P.k / 8);
    return (int)std::max<int64_t>(S, 1);
}

size_t gather_partial_bytes(const DevPoset &P, int64_t rows, int64_t B, int num_sms) {
    int S = gather_slices(P, rows, B, num_sms);
    return S > 1 ? (size_t)S * rows * B * 8 : 0;
}

template <typename T, int CB>
static cudaError_t gather_launch(const DevPoset &P, const void *F, void *g, int64_t lo, int64_t hi,
                                 int64_t B, int mode, void *partial, int S, cudaStream_t s) {
    constexpr int VEC = (CB % 4 == 0) ? 4 : (CB % 2 == 0 ? 2 : 1);
    constexpr int U = CB >= 8 ? 4 : (CB >= 4 ? 8 : 16);
    const int G = (int)(B / CB);
    const int WG = (G % 4 == 0) ? 4 : (G % 2 == 0 ? 2 : 1);
    const int GB = G / WG;
    const int64_t rows = hi - lo;
    const int64_t per_cta = 32 * (8 / WG);
    const int64_t tiles = (rows + per_cta - 1) / per_cta;
    const int64_t blocks = tiles * S * GB;
    void *dst = S > 1 ? partial : g;
    int m = S > 1 ? 2 : mode;
    k_gather<T, CB, VEC, U><<<(unsigned)blocks, 256, 0, s>>>(P.M, P.n, P.k, P.ldm, (const T *)F, (T *)dst,
                                                             P.rank_user, lo, hi, (int32_t)B, GB, WG,
                                                             S, m);
    COUNT_LAUNCH(S > 1 ? 2 : 1);
    if (S > 1) {
        int64_t tot = rows * B;
        k_gather_reduce<T><<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(
            (const T *)partial, (T *)g, P.rank_user, lo, rows, (int32_t)B, S, mode);
    }
    return cudaGetLastError();
}

template <typename T>
static cudaError_t gather_t(const DevPoset &P, const void *F, void *g, int64_t lo, int64_t hi,
                            int64_t B, int mode, void *partial, int num_sms, cudaStream_t s) {
    int S = gather_slices(P, hi - lo, B, num_sms);
    if (S > 1 && !partial) S = 1;
    if (B % 32 == 0 && S == 1 && (gather_variant() == 0 || gather_variant() == 3 || gather_variant() == 4)) {
        const int G32 = (int)(B / 32);
        const int64_t tiles = (hi - lo + 8 * 16 - 1) / (8 * 16);
        if (gather_variant() != 3)   // 2 chains per step: fewer registers, 3 CTAs per SM (measured best)
            k_gather_r4<T, 64, 2, 3><<<(unsigned)(tiles * G32), 256, 0, s>>>(
                P.M, P.n, P.k, P.ldm, (const T *)F, (T *)g, P.rank_user, lo, hi, (int32_t)B, G32, mode);
        else
            k_gather_r4<T, 64><<<(unsigned)(tiles * G32), 256, 0, s>>>(
                P.M, P.n, P.k, P.ldm, (const T *)F, (T *)g, P.rank_user, lo, hi, (int32_t)B, G32, mode);
        COUNT_LAUNCH(1);
        return cudaGetLastError();
    }
    if (B % 32 == 0 && S == 1 && gather_variant() == 1) {
        constexpr int TR = 8, KCH = 64;
        const int G32 = (int)(B / 32);
        const int64_t tiles = (hi - lo + 8 * TR - 1) / (8 * TR);
        k_gather_cols<T, KCH><<<(unsigned)(tiles * G32), 256, 0, s>>>(
            P.M, P.n, P.k, P.ldm, (const T *)F, (T *)g, P.rank_user, lo, hi, (int32_t)B, G32, mode);
        COUNT_LAUNCH(1);
        return cudaGetLastError();
    }
    switch (gather_cb(B)) {
        case 8: return gather_launch<T, 8>(P, F, g, lo, hi, B, mode, partial, S, s);
        case 4: return gather_launch<T, 4>(P, F, g, lo, hi, B, mode, partial, S, s);
        case 2: return gather_launch<T, 2>(P, F, g, lo, hi, B, mode, partial, S, s);
        default: return gather_launch<T, 1>(P, F, g, lo, hi, B, mode, partial, S, s);
    }
}

cudaError_t launch_gather(const DevPoset &P, int dtype, const void *F, void *g, int64_t lo,
                          int64_t hi, int64_t B, int out_rank, void *partial, int num_sms,
                          cudaStream_t s) {
    if (hi <= lo) return cudaSuccess;
    return dtype == 0 ? gather_t<u64>(P, F, g, lo, hi, B, out_rank, partial, num_sms, s)
                      : gather_t<double>(P, F, g, lo, hi, B, out_rank, partial, num_sms, s);
}

// ------------------------------------------------ (v) Moebius U-solve -----
// Body shared by the three schedules: one rank r, CB columns from c0.
//   F[slot(r)] = g[user(r)] - Σ_{j : M[j][r] ∉ {slot(r), n}} F[M[j][r]]
template <typename T, int CB, int VEC, int CF>
__device__ __forceinline__ void moeb_row(const DevPoset &P, const T *__restrict__ g, T *F,
                                         int32_t r, int32_t B, int c0) {
    const int32_t n = P.n;
    const int32_t my = P.slot[r];
    T acc[CB];
    load_row<T, CB, VEC, LD_NC>(g + (size_t)P.rank_user[r] * B + c0, acc);
    const int32_t *Mr = P.M + r;
    constexpr int U = 8;
    int j = 0;
    for (; j + U <= P.k; j += U) {
        int32_t idx[U];
#pragma unroll
        for (int u = 0; u < U; u++) idx[u] = ld_stream_i32(Mr + (size_t)(j + u) * n);
#pragma unroll
        for (int u = 0; u < U; u++) {
            if (idx[u] != my && idx[u] != n) {
                T v[CB];
                load_row<T, CB, VEC, CF>(F + (size_t)idx[u] * B + c0, v);
#pragma unroll
                for (int c = 0; c < CB; c++) acc[c] -= v[c];
            }
        }
    }
    for (; j < P.k; j++) {
        int32_t idx = ld_stream_i32(Mr + (size_t)j * n);
        if (idx != my && idx != n) {
            T v[CB];
            load_row<T, CB, VEC, CF>(F + (size_t)idx * B + c0, v);
#pragma unroll
            for (int c = 0; c < CB; c++) acc[c] -= v[c];
        }
    }
    store_row<T, CB, VEC>(F + (size_t)my * B + c0, acc);
}

// (a) one launch per level (Alg. 5 with the kernel boundary as the barrier)
template <typename T, int CB, int VEC>
__global__ void __launch_bounds__(256) k_moeb_level(DevPoset P, const T *__restrict__ g, T *F,
                                                    int32_t B, int G, int32_t lo, int32_t hi) {
    const int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int32_t w = hi - lo;
    if (item >= (int64_t)w * G) return;
    const int32_t r = lo + (int32_t)(item % w);
    const int cg = (int)(item / w);
    moeb_row<T, CB, VEC, LD_NC>(P, g, F, r, B, cg * CB);
}

// (b) persistent cooperative kernel: grid barrier between levels
__device__ __forceinline__ void grid_barrier(unsigned *bar, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *gen = bar + 1;
        unsigned g0 = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == nblocks - 1) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            unsigned rounds = 0;
            while (*gen == g0) {
                __nanosleep(32);
                if (++rounds == (1u << 26)) __trap();   // watchdog (see ptx.cuh)
            }
        }
        __threadfence();
    }
    __syncthreads();
}

template <typename T, int CB, int VEC>
__global__ void __launch_bounds__(512) k_moeb_grid(DevPoset P, const T *__restrict__ g, T *F,
                                                   int32_t B, int G, unsigned *bar) {
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int32_t L = 0; L < P.ell; L++) {
        const int32_t lo = P.lvl_ptr[L], hi = P.lvl_ptr[L + 1];
        const int32_t w = hi - lo;
        for (int64_t item = tid; item < (int64_t)w * G; item += nth) {
            const int32_t r = lo + (int32_t)(item % w);
            moeb_row<T, CB, VEC, LD_CG>(P, g, F, r, B, (int)(item / w) * CB);
        }
        if (L + 1 < P.ell) grid_barrier(bar, gridDim.x);
    }
}

// (c) one warp per column group sweeps every level; lanes over the level's
// ranks; __syncwarp() orders this warp's F stores before the next level's
// loads (only this warp writes its columns).
template <typename T, int CB, int VEC>
__global__ void __launch_bounds__(32) k_moeb_warp(DevPoset P, const T *__restrict__ g, T *F,
                                                  int32_t B, int G) {
    const int wid = blockIdx.x;
    if (wid >= G) return;
    const int lane = threadIdx.x & 31;
    const int c0 = wid * CB;
    for (int32_t L = 0; L < P.ell; L++) {
        const int32_t lo = P.lvl_ptr[L], hi = P.lvl_ptr[L + 1];
        for (int32_t base = lo; base < hi; base += 32) {
            const int32_t r = base + lane;
            if (r < hi) moeb_row<T, CB, VEC, LD_CA>(P, g, F, r, B, c0);
        }
        __syncwarp();
    }
}

static int warp_cb(int64_t B) {
    // columns per lane for the warp schedule: as many warps as columns up to 64
    for (int cb : {1, 2, 4, 8, 16, 32})
        if (B % cb == 0 && B / cb <= 64) return cb;
    return pick_cb(B);
}

int moebius_pick(const DevPoset &P, int64_t B, int max_level_width, int num_sms) {
    (void)max_level_width;
    if (P.ell <= 48) return MOEB_LEVEL;
    // work per level per warp in the warp schedule vs a grid barrier per level
    const double avg_w = (double)P.n / P.ell;
    const int64_t G = B / warp_cb(B);
    const double warp_cycles = P.ell * (std::ceil(avg_w / 32.0)) * (900.0 + 4.0 * P.k * warp_cb(B));
    const double grid_cycles = P.ell * 4000.0 +
                               (double)P.n * P.k * B * 2.0 / (num_sms * 512.0);
    if (G >= 1 && warp_cycles < grid_cycles) return MOEB_WARP;
    return MOEB_GRID;
}

template <typename T, int CB>
static cudaError_t moeb_cb(const DevPoset &P, const int32_t *h_lvl, const void *g, void *F,
                           int64_t B, int which, unsigned *bar, int num_sms, cudaStream_t s) {
    constexpr int VEC = (CB % 4 == 0) ? 4 : (CB % 2 == 0 ? 2 : 1);
    const int G = (int)(B / CB);
    if (which == MOEB_LEVEL) {
        for (int32_t L = 0; L < P.ell; L++) {
            int32_t lo = h_lvl[L], hi = h_lvl[L + 1];
            int64_t items = (int64_t)(hi - lo) * G;
            k_moeb_level<T, CB, VEC><<<(unsigned)((items + 255) / 256), 256, 0, s>>>(
                P, (const T *)g, (T *)F, (int32_t)B, G, lo, hi);
        }
        COUNT_LAUNCH(P.ell);
        return cudaGetLastError();
    }
    if (which == MOEB_WARP) {
        k_moeb_warp<T, CB, VEC><<<G, 32, 0, s>>>(P, (const T *)g, (T *)F, (int32_t)B, G);
        COUNT_LAUNCH(1);
        return cudaGetLastError();
    }
    // GRID: one 512-thread CTA per SM, co-resident by cooperative launch
    cudaError_t e = cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    DevPoset Pc = P;
    const T *gp = (const T *)g;
    T *Fp = (T *)F;
    int32_t Bi = (int32_t)B;
    int Gi = G;
    void *args[] = {&Pc, &gp, &Fp, &Bi, &Gi, &bar};
    COUNT_LAUNCH(1);
    return cudaLaunchCooperativeKernel((void *)k_moeb_grid<T, CB, VEC>, dim3(num_sms), dim3(512),
                                       args, 0, s);
}

template <typename T>
static cudaError_t moeb_t(const DevPoset &P, const int32_t *h_lvl, const void *g, void *F,
                          int64_t B, int which, unsigned *bar, int num_sms, cudaStream_t s) {
    int cb = which == MOEB_WARP ? warp_cb(B) : pick_cb(B);
    switch (cb) {
        case 32: return moeb_cb<T, 32>(P, h_lvl, g, F, B, which, bar, num_sms, s);
        case 16: return moeb_cb<T, 16>(P, h_lvl, g, F, B, which, bar, num_sms, s);
        case 8: return moeb_cb<T, 8>(P, h_lvl, g, F, B, which, bar, num_sms, s);
        case 4: return moeb_cb<T, 4>(P, h_lvl, g, F, B, which, bar, num_sms, s);
        case 2: return moeb_cb<T, 2>(P, h_lvl, g, F, B, which, bar, num_sms, s);
        default: return moeb_cb<T, 1>(P, h_lvl, g, F, B, which, bar, num_sms, s);
    }
}

cudaError_t launch_moebius_solve(const DevPoset &P, const int32_t *h_lvl, int dtype, const void *g,
                                 void *F, int64_t B, int which, unsigned *bar, int num_sms,
                                 cudaStream_t s) {
    if (P.n == 0) return cudaSuccess;
    return dtype == 0 ? moeb_t<u64>(P, h_lvl, g, F, B, which, bar, num_sms, s)
                      : moeb_t<double>(P, h_lvl, g, F, B, which, bar, num_sms, s);
}

// ----------------------------------------------------- chain difference ---
template <typename T, int CB, int VEC>
__global__ void __launch_bounds__(256) k_chain_diff(const int32_t *__restrict__ slot_user,
                                                    int32_t n, const T *__restrict__ F,
                                                    T *__restrict__ f, int32_t B, int G) {
    const int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (item >= (int64_t)n * G) return;
    const int64_t s = item / G;
    const int c0 = (int)(item % G) * CB;
    const int32_t u = slot_user[s];
    T a[CB];
    load_row<T, CB, VEC, LD_NC>(F + (size_t)s * B + c0, a);
    if (u >= 0) {   // not a chain start: subtract the element below
        T p[CB];
        load_row<T, CB, VEC, LD_NC>(F + (size_t)(s - 1) * B + c0, p);
#pragma unroll
        for (int c = 0; c < CB; c++) a[c] -= p[c];
    }
    store_row<T, CB, VEC>(f + (size_t)(u & 0x7fffffff) * B + c0, a);
}

template <typename T, int CB, int VEC>
__global__ void __launch_bounds__(256) k_rank_to_user(const int32_t *__restrict__ rank_user,
                                                      int32_t n, const T *__restrict__ src,
                                                      T *__restrict__ dst, int32_t B, int G) {
    const int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (item >= (int64_t)n * G) return;
    const int64_t r = item / G;
    const int c0 = (int)(item % G) * CB;
    T a[CB];
    load_row<T, CB, VEC, LD_NC>(src + (size_t)r * B + c0, a);
    store_row<T, CB, VEC>(dst + (size_t)rank_user[r] * B + c0, a);
}

template <typename T>
static cudaError_t elementwise_t(const DevPoset &P, const void *in, void *out, int64_t B,
                                 int what, cudaStream_t s) {
    int cb = std::min(pick_cb(B), 4);
    int G = (int)(B / cb);
    unsigned blocks = (unsigned)(((int64_t)P.n * G + 255) / 256);
    if (blocks == 0) return cudaSuccess;
    COUNT_LAUNCH(1);
#define POSET_EW(CBV, VECV)                                                                      \
    if (what == 0)                                                                               \
        k_chain_diff<T, CBV, VECV><<<blocks, 256, 0, s>>>(P.slot_user, P.n, (const T *)in,        \
                                                         (T *)out, (int32_t)B, G);               \
    else                                                                                         \
        k_rank_to_user<T, CBV, VECV><<<blocks, 256, 0, s>>>(P.rank_user, P.n, (const T *)in,     \
                                                           (T *)out, (int32_t)B, G);
    if (cb == 4) { POSET_EW(4, 4) }
    else if (cb == 2) { POSET_EW(2, 2) }
    else { POSET_EW(1, 1) }
#undef POSET_EW
    return cudaGetLastError();
}

cudaError_t launch_chain_diff(const DevPoset &P, int dtype, const void *F, void *f, int64_t B,
                              cudaStream_t s) {
    return dtype == 0 ? elementwise_t<u64>(P, F, f, B, 0, s) : elementwise_t<double>(P, F, f, B, 0, s);
}

cudaError_t launch_rank_to_user(const DevPoset &P, int dtype, const void *g_rank, void *g_user,
                                int64_t B, cudaStream_t s) {
    return dtype == 0 ? elementwise_t<u64>(P, g_rank, g_user, B, 1, s)
                      : elementwise_t<double>(P, g_rank, g_user, B, 1, s);
}

}  // namespace poset
