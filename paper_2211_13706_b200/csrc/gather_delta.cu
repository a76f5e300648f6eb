// Kernel (iv), batched form with a DELTA LIST: the zeta gather-reduce
// g(x) = Σ_j F[niv_j(x)] (Eq. zeta-fast, Alg. 3)
// evaluated position by position along the per-tile gather order of
// gather_pi.cu, carrying the sum from one position to the next:
//
//   g(x_p) = g(x_{p-1}) + Σ_{j : niv_j(x_p) ≠ niv_j(x_{p-1})} (F[niv_j(x_p)] − F[niv_j(x_{p-1})])
//
// which telescopes per chain to the paper's sum (F[∞] = the zero row n,
// reading G12).  The greedy nearest-neighbour order makes consecutive rows
// differ in few chains (C5w: 14.0 entries per position, 63 chains), so a
// position costs ~14 pairs of row loads and adds instead of 63 dependent
// loads and adds.  MEASURED SLOWER than the default gather-order kernel
// (C5w 10.7 vs 7.9 ms, C4w 12.6 vs 4.7 ms: each change loads two rows, the
// old one mostly from L2) -- kept as option gather_pi_cfg 4.
//
// Error control (fp64; int64 is exact in Z/2^64 in any order): a carried sum
// has rounding error relative to the magnitudes of the previous positions'
// rows, not of x's own.  Positions whose down-set is small (|↓x| < 2048) or
// more than 4x smaller than the largest earlier one in the tile are summed
// from scratch (RESET: the carried sum is dropped and every finite entry of
// the row is added), as is the first position of every tile.  Then every
// carried magnitude is within 4x of x's own and the error stays at
// γ_{2E}·4·ζ(|f|)(x) with E ≤ 2·256·k entries per tile (C5w: ≈ 4e-12 relative,
// DESIGN.md §2 tolerance 1e-9).
//
//   k_delta_count   CTA per 256-position tile: per position the number of
//                   changed chains, |↓x| (= Σ_j pos + 1), the reset rule
//   k_delta_fill    CTA per tile: writes the entries {new | LAST, old | RESET}
//   k_gather_delta  warp per (tile, column group): entries staged 32 at a time
//                   in shared memory, U entries' 2U row loads issued together
//                   (independent of the running sum), then the adds; the sum
//                   is stored at every LAST entry.
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <cstdint>
#include <vector>

#include "kernels.cuh"

namespace poset {

typedef unsigned long long u64;

namespace {
constexpr int GT = 256;                 // tile = positions (same tiles as gather_pi.cu)
constexpr int64_t RESET_MIN = 2048;     // down-sets below this are summed from scratch
constexpr int64_t RESET_RATIO = 4;      // ... and those this much smaller than an earlier one
constexpr uint32_t LAST = 0x80000000u;  // in .x: last entry of a position
constexpr uint32_t RESET = 0x80000000u; // in .y: drop the carried sum before this entry
}

// ------------------------------------------------------------ build -----
__device__ __forceinline__ int64_t block_excl_max(int64_t v, int64_t *sw) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int64_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc = max(inc, o);
    }
    if (lane == 31) sw[warp] = inc;
    __syncthreads();
    int64_t pre = 0;
    for (int w = 0; w < warp; w++) pre = max(pre, sw[w]);
    int64_t ex = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) ex = 0;
    __syncthreads();
    return max(pre, ex);
}

__device__ __forceinline__ int block_excl_sum(int v, int *sw, int *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
    }
    if (lane == 31) sw[warp] = inc;
    __syncthreads();
    int pre = 0, tot = 0;
    for (int w = 0; w < GT / 32; w++) {
        if (w < warp) pre += sw[w];
        tot += sw[w];
    }
    __syncthreads();
    *total = tot;
    return pre + inc - v;
}

__global__ void __launch_bounds__(GT) k_delta_count(const int32_t *__restrict__ Mg,
                                                    const int32_t *__restrict__ out_user,
                                                    const int32_t *__restrict__ off, int64_t npad, int32_t n,
                                                    int32_t k, int32_t *__restrict__ cnt,
                                                    int64_t *__restrict__ tot,
                                                    unsigned long long *__restrict__ nreset) {
    __shared__ int64_t swm[GT / 32];
    __shared__ int sws[GT / 32];
    const int64_t p = (int64_t)blockIdx.x * GT + threadIdx.x;
    const bool pad = out_user[p] < 0;
    const bool first = threadIdx.x == 0;
    int64_t dsz = 0;
    int ch = 0, fin = 0;
    for (int j = 0; j < k; j++) {
        const int32_t v = Mg[(size_t)j * npad + p];
        const int32_t o = first ? n : Mg[(size_t)j * npad + p - 1];
        if (v < n) {
            dsz += v - __ldg(off + j) + 1;
            fin++;
        }
        ch += v != o;
    }
    const int64_t pmax = block_excl_max(pad ? 0 : dsz, swm);
    const bool reset = !pad && (first || dsz < RESET_MIN || dsz * RESET_RATIO < pmax);
    const int c = pad ? 1 : reset ? max(fin, 1) : max(ch, 1);
    cnt[p] = reset ? -c : c;
    int t = 0;
    block_excl_sum(c, sws, &t);
    const unsigned rb = __syncthreads_count(reset);
    if (first) {
        tot[blockIdx.x] = t;
        atomicAdd(nreset, (unsigned long long)rb);
    }
}

__global__ void __launch_bounds__(GT) k_delta_fill(const int32_t *__restrict__ Mg,
                                                   const int32_t *__restrict__ out_user, int64_t npad,
                                                   int32_t n, int32_t k, const int32_t *__restrict__ cnt,
                                                   const int64_t *__restrict__ Dptr, int2 *__restrict__ D) {
    __shared__ int sws[GT / 32];
    const int64_t p = (int64_t)blockIdx.x * GT + threadIdx.x;
    const int c0 = cnt[p];
    const bool reset = c0 < 0;
    int t = 0;
    int64_t e = Dptr[blockIdx.x] + block_excl_sum(reset ? -c0 : c0, sws, &t);
    if (out_user[p] < 0) {   // padding: one zero entry (F[n] - F[n])
        D[e] = make_int2((int)((uint32_t)n | LAST), n);
        return;
    }
    const bool first = threadIdx.x == 0;
    int2 pend = make_int2(-1, 0);
    bool have = false, first_entry = true;
    for (int j = 0; j < k; j++) {
        const int32_t v = Mg[(size_t)j * npad + p];
        int2 en;
        bool emit;
        if (reset) {
            emit = v < n;
            en = make_int2(v, (int)((uint32_t)n | (first_entry ? RESET : 0u)));
        } else {
            const int32_t o = first ? n : Mg[(size_t)j * npad + p - 1];
            emit = v != o;
            en = make_int2(v, o);
        }
        if (emit) {
            if (have) D[e++] = pend;
            pend = en;
            have = true;
            first_entry = false;
        }
    }
    if (!have) pend = make_int2(n, (int)((uint32_t)n | (reset ? RESET : 0u)));   // unchanged row
    pend.x = (int)((uint32_t)pend.x | LAST);
    D[e] = pend;
}

cudaError_t build_gather_delta(const DevPoset &P, const int32_t *chain_off, GatherPi &G, cudaStream_t s) {
    const int64_t tiles = G.npad / GT;
    cudaError_t e = cudaSuccess;
    int32_t *cnt = nullptr;
    int64_t *tot = nullptr;
    unsigned long long *nres = nullptr;
    int2 *D = nullptr;
    int64_t *Dptr = nullptr;
    std::vector<int64_t> h_tot(tiles), h_ptr(tiles + 1);
    unsigned long long h_nres = 0;
    size_t fb = 0, tb = 0;
    auto fail = [&](cudaError_t x) {
        cudaFree(cnt); cudaFree(tot); cudaFree(nres); cudaFree(D); cudaFree(Dptr);
        return x;
    };
    if ((e = cudaMalloc((void **)&cnt, (size_t)G.npad * 4)) != cudaSuccess) return fail(e);
    if ((e = cudaMalloc((void **)&tot, (size_t)tiles * 8)) != cudaSuccess) return fail(e);
    if ((e = cudaMalloc((void **)&nres, 8)) != cudaSuccess) return fail(e);
    if ((e = cudaMemsetAsync(nres, 0, 8, s)) != cudaSuccess) return fail(e);
    k_delta_count<<<(unsigned)tiles, GT, 0, s>>>(G.Mg, G.out_user, chain_off, G.npad, P.n, P.k, cnt, tot, nres);
    launches_add(1);
    if ((e = cudaGetLastError()) != cudaSuccess) return fail(e);
    if ((e = cudaMemcpyAsync(h_tot.data(), tot, (size_t)tiles * 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        return fail(e);
    if ((e = cudaMemcpyAsync(&h_nres, nres, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return fail(e);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return fail(e);
    h_ptr[0] = 0;
    for (int64_t t = 0; t < tiles; t++) h_ptr[t + 1] = h_ptr[t] + h_tot[t];
    const int64_t ne = h_ptr[tiles];
    if ((e = cudaMemGetInfo(&fb, &tb)) != cudaSuccess) return fail(e);
    if ((size_t)ne * 8 + ((size_t)1 << 30) > fb) return fail(cudaErrorMemoryAllocation);
    if ((e = cudaMalloc((void **)&D, (size_t)ne * 8)) != cudaSuccess) return fail(e);
    if ((e = cudaMalloc((void **)&Dptr, (size_t)(tiles + 1) * 8)) != cudaSuccess) return fail(e);
    if ((e = cudaMemcpyAsync(Dptr, h_ptr.data(), (size_t)(tiles + 1) * 8, cudaMemcpyHostToDevice, s)) !=
        cudaSuccess)
        return fail(e);
    k_delta_fill<<<(unsigned)tiles, GT, 0, s>>>(G.Mg, G.out_user, G.npad, P.n, P.k, cnt, Dptr, D);
    launches_add(1);
    if ((e = cudaGetLastError()) != cudaSuccess) return fail(e);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return fail(e);
    cudaFree(cnt);
    cudaFree(tot);
    cudaFree(nres);
    G.D = D;
    G.Dptr = Dptr;
    G.nentries = ne;
    G.nreset = (int64_t)h_nres;
    G.delta_ok = true;
    return cudaSuccess;
}

// ------------------------------------------------------------ gather ----
template <int CPL>
__device__ __forceinline__ void ldrow(u64 (&v)[CPL], const char *p) {
    if constexpr (CPL == 1) {
        asm volatile("ld.global.nc.b64 %0, [%1];" : "=l"(v[0]) : "l"(p));
    } else if constexpr (CPL == 2) {
        asm volatile("ld.global.nc.v2.b64 {%0,%1}, [%2];" : "=l"(v[0]), "=l"(v[1]) : "l"(p));
    } else {
        asm volatile("ld.global.nc.v4.b64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3])
                     : "l"(p));
    }
}
template <int CPL>
__device__ __forceinline__ void strow(char *p, const u64 (&v)[CPL]) {
    if constexpr (CPL == 1) {
        asm volatile("st.global.b64 [%0], %1;" ::"l"(p), "l"(v[0]) : "memory");
    } else if constexpr (CPL == 2) {
        asm volatile("st.global.v2.b64 [%0], {%1,%2};" ::"l"(p), "l"(v[0]), "l"(v[1]) : "memory");
    } else {
        asm volatile("st.global.v4.b64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(v[0]), "l"(v[1]), "l"(v[2]),
                     "l"(v[3])
                     : "memory");
    }
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

// Warp per item (tile, group of 32·CPL columns); lane = CPL consecutive
// columns.  Items run in tile order, so the warps resident at one time work
// on neighbouring tiles and share their F rows in L2.
//
// fp64 certificate: every add's rounding error is at most u·|its result|
// (u = 2^-53), so err(x) ≤ u·Σ|results| since the last reset =: u·errb.
// |g(x)| ≤ ζ(|f|)(x), so a position with u·errb ≤ 0.5e-9·|g(x)| (computed)
// meets the tolerance |Δ| ≤ 1e-9·ζ(|f|)(x) for ANY f; the others (g ≈ 0 by
// cancellation, or a tile-mate of much larger magnitude) are appended to
// `redo` and summed directly by k_gather_redo.
template <typename T, int CPL, int U>
__global__ void __launch_bounds__(256) k_gather_delta(const int2 *__restrict__ D, const int64_t *__restrict__ Dptr,
                                                      const int32_t *__restrict__ out_user, int64_t items, int G,
                                                      const T *__restrict__ F, T *__restrict__ out, int32_t B,
                                                      int32_t nrow, int64_t *__restrict__ redo,
                                                      unsigned long long *__restrict__ nredo) {
    constexpr bool FP = std::is_same<T, double>::value;
    __shared__ __align__(16) int2 sb[8][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t item = (int64_t)blockIdx.x * 8 + warp;
    if (item >= items) return;
    const int64_t tile = item / G;
    const int cg = (int)(item - tile * G);
    const int64_t e0 = Dptr[tile], e1 = Dptr[tile + 1];
    const size_t rowbytes = (size_t)B * sizeof(T);
    const char *Fb = reinterpret_cast<const char *>(F + cg * 32 * CPL + lane * CPL);
    char *Ob = reinterpret_cast<char *>(out + cg * 32 * CPL + lane * CPL);
    const int32_t *ou = out_user + tile * GT;
    int2 *S = sb[warp];
    T acc[CPL];
    double errb[CPL];
#pragma unroll
    for (int i = 0; i < CPL; i++) {
        acc[i] = T(0);
        errb[i] = 0.0;
    }
    int pos = 0;
    for (int64_t e = e0; e < e1; e += 32) {
        const int2 en = e + lane < e1 ? D[e + lane] : make_int2(nrow, nrow);   // dummy: adds F[n] - F[n] = 0
        __syncwarp();
        S[lane] = en;
        __syncwarp();
        const int m = e1 - e < 32 ? (int)(e1 - e) : 32;
        for (int t = 0; t < m; t += U) {
            int32_t nw[U], od[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int2 x = S[t + u];
                nw[u] = x.x;
                od[u] = x.y;
            }
            u64 a[U][CPL], b[U][CPL];
#pragma unroll
            for (int u = 0; u < U; u++) {
                ldrow<CPL>(a[u], Fb + (size_t)((uint32_t)nw[u] & 0x7fffffffu) * rowbytes);
                ldrow<CPL>(b[u], Fb + (size_t)((uint32_t)od[u] & 0x7fffffffu) * rowbytes);
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                if (od[u] < 0) {
#pragma unroll
                    for (int i = 0; i < CPL; i++) {
                        acc[i] = T(0);
                        errb[i] = 0.0;
                    }
                }
#pragma unroll
                for (int i = 0; i < CPL; i++) {
                    const T d = from_bits<T>(a[u][i]) - from_bits<T>(b[u][i]);
                    acc[i] += d;
                    if constexpr (FP) errb[i] += fabs((double)d) + fabs((double)acc[i]);
                }
                if (nw[u] < 0) {
                    const int p = pos++;
                    const int32_t usr = ou[p];
                    if (usr >= 0) {
                        u64 o[CPL];
#pragma unroll
                        for (int i = 0; i < CPL; i++) o[i] = to_bits<T>(acc[i]);
                        strow<CPL>(Ob + (size_t)usr * rowbytes, o);
                        if constexpr (FP) {
                            bool bad = false;
#pragma unroll
                            for (int i = 0; i < CPL; i++)
                                bad |= errb[i] * 0x1p-53 > 0.5e-9 * fabs((double)acc[i]);
                            const unsigned bm = __ballot_sync(0xffffffffu, bad);
                            if (bm && lane == 0) {
                                const unsigned long long w = atomicAdd(nredo, 1ull);
                                redo[w] = (tile * GT + p) * (int64_t)G + cg;
                            }
                        }
                    }
                }
            }
        }
    }
}

// The positions the certificate rejected, summed directly from the
// gather-order table Mg (the paper's Σ_j F[niv_j(x)], k loads): warp per
// entry of `redo` (position · G + column group).
template <typename T, int CPL>
__global__ void __launch_bounds__(256) k_gather_redo(const int32_t *__restrict__ Mg, int64_t npad, int32_t k,
                                                     const int32_t *__restrict__ out_user, int G,
                                                     const T *__restrict__ F, T *__restrict__ out, int32_t B,
                                                     const int64_t *__restrict__ redo,
                                                     const unsigned long long *__restrict__ nredo) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t cnt = (int64_t)*nredo;
    const size_t rowbytes = (size_t)B * sizeof(T);
    for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < cnt; w += nw) {
        const int64_t r = redo[w];
        const int64_t p = r / G;
        const int cg = (int)(r - p * G);
        const char *Fb = reinterpret_cast<const char *>(F + cg * 32 * CPL + lane * CPL);
        T acc[CPL];
#pragma unroll
        for (int i = 0; i < CPL; i++) acc[i] = T(0);
        for (int j = 0; j < k; j++) {
            u64 v[CPL];
            ldrow<CPL>(v, Fb + (size_t)Mg[(size_t)j * npad + p] * rowbytes);
#pragma unroll
            for (int i = 0; i < CPL; i++) acc[i] += from_bits<T>(v[i]);
        }
        u64 o[CPL];
#pragma unroll
        for (int i = 0; i < CPL; i++) o[i] = to_bits<T>(acc[i]);
        strow<CPL>(reinterpret_cast<char *>(out + cg * 32 * CPL + lane * CPL) + (size_t)out_user[p] * rowbytes, o);
    }
}

template <typename T, int CPL, int U>
static cudaError_t gather_delta_t(const GatherPi &G, int32_t n, int32_t k, const void *F, void *g, int64_t B,
                                  int num_sms, cudaStream_t s) {
    const int groups = (int)(B / (32 * CPL));
    const int64_t items = (G.npad / GT) * groups;
    constexpr bool FP = std::is_same<T, double>::value;
    cudaError_t e = cudaSuccess;
    if (FP && (e = cudaMemsetAsync(G.nredo, 0, 8, s)) != cudaSuccess) return e;
    k_gather_delta<T, CPL, U><<<(unsigned)((items + 7) / 8), 256, 0, s>>>(
        (const int2 *)G.D, G.Dptr, G.out_user, items, groups, (const T *)F, (T *)g, (int32_t)B, n, G.redo,
        G.nredo);
    launches_add(1);
    if (FP) {
        k_gather_redo<T, CPL><<<(unsigned)num_sms, 256, 0, s>>>(G.Mg, G.npad, k, G.out_user, groups, (const T *)F,
                                                                (T *)g, (int32_t)B, G.redo, G.nredo);
        launches_add(1);
    }
    return cudaGetLastError();
}

template <typename T>
static cudaError_t gather_delta_dt(const GatherPi &G, int32_t n, int32_t k, const void *F, void *g, int64_t B,
                                   int num_sms, cudaStream_t s) {
    if (B % 128 == 0) return gather_delta_t<T, 4, 4>(G, n, k, F, g, B, num_sms, s);
    if (B % 64 == 0) return gather_delta_t<T, 2, 8>(G, n, k, F, g, B, num_sms, s);
    return gather_delta_t<T, 1, 8>(G, n, k, F, g, B, num_sms, s);
}

cudaError_t launch_gather_delta(GatherPi &G, int32_t n, int32_t k, int dtype, const void *F, void *g,
                                int64_t B, int num_sms, cudaStream_t s) {
    if (!G.delta_ok || B % 32) return cudaErrorInvalidValue;
    if (dtype == 0) return gather_delta_dt<u64>(G, n, k, F, g, B, num_sms, s);
    // the redo list holds at most one entry per (position, column group)
    const int64_t groups = B % 128 == 0 ? B / 128 : B % 64 == 0 ? B / 64 : B / 32;
    if (groups * G.npad > G.redo_cap) {
        cudaError_t e = cudaSuccess;
        if (G.redo) cudaFree(G.redo);
        G.redo = nullptr;
        G.redo_cap = 0;
        if (!G.nredo && (e = cudaMalloc((void **)&G.nredo, 8)) != cudaSuccess) return e;
        if ((e = cudaMalloc((void **)&G.redo, (size_t)(groups * G.npad) * 8)) != cudaSuccess) return e;
        G.redo_cap = groups * G.npad;
    }
    return gather_delta_dt<double>(G, n, k, F, g, B, num_sms, s);
}

}  // namespace poset
