// Sparse (CSR) niv rows -- SURVEY.md §8(f) N1 -- and the two kernels that use
// them:
//
//   U-rows   for rank r: the F slots of niv_j(r) for j ≠ id(r), ∞ omitted
//            (the paper stores N sparse with ∞ dropped, and drops the
//            self entries in practice, P:L582 / P:L670).  int32 slots,
//            int64 row pointers, rank order.  Built from the dense table M.
//
//   k_gather_csr   zeta, Eq. zeta-fast:
//                  g(x) = F[slot(x)] + Σ_{s ∈ U-row(x)} F[s]
//                  (the self entry is niv_{id(x)}(x) = x).
//   k_moeb_csr     Möbius, Alg. 4: persistent cooperative
//                  kernel, one grid barrier per antichain level (Alg. 5,
//                  P:L692-705); warp-granular items, so wide rows (large k)
//                  are summed by 32 lanes in parallel instead of one thread:
//                    F(x) = g(x) - Σ_{s ∈ U-row(x)} F[s];  f(x) = F(x) - F(next(x))
//
// Two lane mappings: lanes over the row's entries (B % 32 != 0, one column
// at a time, warp-shuffle reduction) or lanes over columns (B % 32 == 0; each
// row entry is read once by the warp and broadcast by a shuffle, the F row is
// one coalesced 256-B load).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "kernels.cuh"

namespace poset {

typedef unsigned long long u64;

// ------------------------------------------------------------ build ------
__global__ void k_csr_count(const int32_t *__restrict__ M, int32_t n, int32_t k,
                            const int32_t *__restrict__ chain, int32_t *__restrict__ cnt) {
    const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int32_t own = chain[r];
    int32_t c = 0;
    for (int32_t j = 0; j < k; j++) c += (j != own) & (__ldcs(M + (size_t)j * n + r) != n);
    cnt[r] = c;
}

__global__ void k_csr_fill(const int32_t *__restrict__ M, int32_t n, int32_t k,
                           const int32_t *__restrict__ chain, const int64_t *__restrict__ ptr,
                           int32_t *__restrict__ idx) {
    const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int32_t own = chain[r];
    int64_t o = ptr[r];
    for (int32_t j = 0; j < k; j++) {
        const int32_t s = __ldcs(M + (size_t)j * n + r);
        if (j != own && s != n) idx[o++] = s;
    }
}

cudaError_t build_csr(const DevPoset &P, CsrRows &C, size_t free_budget) {
    C.ok = false;
    const int32_t n = P.n;
    if (n == 0) return cudaSuccess;
    int32_t *d_cnt = nullptr;
    cudaError_t e = cudaMalloc((void **)&d_cnt, (size_t)n * 4);
    if (e != cudaSuccess) return e;
    k_csr_count<<<(n + 255) / 256, 256>>>(P.M, n, P.k, P.chain, d_cnt);
    launches_add(1);
    std::vector<int32_t> cnt((size_t)n);
    e = cudaMemcpy(cnt.data(), d_cnt, (size_t)n * 4, cudaMemcpyDeviceToHost);
    cudaFree(d_cnt);
    if (e != cudaSuccess) return e;
    std::vector<int64_t> ptr((size_t)n + 1, 0);
    for (int32_t r = 0; r < n; r++) ptr[r + 1] = ptr[r] + cnt[r];
    C.nnz = ptr[n];
    const size_t bytes = (size_t)std::max<int64_t>(C.nnz, 1) * 4 + ((size_t)n + 1) * 8;
    if (bytes > free_budget) return cudaSuccess;   // not enough room: no CSR rows
    e = cudaMalloc((void **)&C.ptr, ((size_t)n + 1) * 8);
    if (e == cudaSuccess) e = cudaMalloc((void **)&C.idx, (size_t)std::max<int64_t>(C.nnz, 1) * 4);
    if (e != cudaSuccess) {
        cudaGetLastError();
        if (C.ptr) cudaFree(C.ptr);
        C.ptr = nullptr;
        C.idx = nullptr;
        return cudaSuccess;
    }
    e = cudaMemcpy(C.ptr, ptr.data(), ((size_t)n + 1) * 8, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return e;
    k_csr_fill<<<(n + 255) / 256, 256>>>(P.M, n, P.k, P.chain, C.ptr, C.idx);
    launches_add(1);
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return e;
    C.ok = true;
    return cudaSuccess;
}

// ------------------------------------------------ build without M (N1) ---
// The U-rows straight from the DAG, level by level, without the dense n x k
// table (the paper's sparse N, built bottom-up as in
// Alg. 2): by Thm. 4 the full niv row of x is the
// per-chain maximum over its children c of (U-row(c) ∪ {slot(c)}) -- slots
// are sorted by chain, then position, so "per-chain maximum" is "the last
// entry of each chain run" of the merged, sorted slot lists.  Entries on x's
// own chain are dropped (its own entry is implicit: slot(x)).
// One warp per element: lane i owns the chains [i k / 32, (i+1) k / 32), i.e.
// a contiguous slot range (chains are laid out contiguously), finds its
// segment of every child's row by binary search and merges it (m-way merge,
// m = out-degree <= 64); lane counts -> a warp prefix sum -> the element's
// row.  A count pass, a prefix sum over the level and a fill pass per level.
constexpr int kDirectMaxChildren = 64;

__device__ __forceinline__ int64_t lower_bound_i32(const int32_t *a, int64_t lo, int64_t hi, int32_t v) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

template <bool FILL>
__global__ void __launch_bounds__(128) k_csr_direct(int32_t lo, int32_t hi, int32_t k,
                                                    const int64_t *__restrict__ child_ptr,
                                                    const int32_t *__restrict__ child,
                                                    const int32_t *__restrict__ slot,
                                                    const int32_t *__restrict__ chain,
                                                    const int32_t *__restrict__ slot_chain,
                                                    const int32_t *__restrict__ chain_off, int64_t *ptr,
                                                    int32_t *idx, int64_t *cnt, int32_t *too_many) {
    const int lane = threadIdx.x & 31;
    const int32_t r = lo + (int32_t)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (r >= hi) return;
    const int64_t c0 = child_ptr[r], c1 = child_ptr[r + 1];
    const int m = (int)(c1 - c0);
    if (m > kDirectMaxChildren) {
        if (lane == 0) *too_many = 1;
        return;
    }
    // this lane's slot range
    const int32_t s_lo = chain_off[(int64_t)lane * k / 32], s_hi = chain_off[(int64_t)(lane + 1) * k / 32];
    const int32_t own_lo = chain_off[chain[r]], own_hi = chain_off[chain[r] + 1];
    int64_t cur[kDirectMaxChildren], end[kDirectMaxChildren];
    int32_t cs[kDirectMaxChildren];   // slot(c) if in this lane's range and not yet taken, else INT32_MAX
    for (int i = 0; i < m; i++) {
        const int32_t c = child[c0 + i];
        const int64_t a = ptr[c], b = ptr[c + 1];
        cur[i] = s_lo > 0 ? lower_bound_i32(idx, a, b, s_lo) : a;
        end[i] = lower_bound_i32(idx, cur[i], b, s_hi);
        const int32_t sc = slot[c];
        cs[i] = (sc >= s_lo && sc < s_hi) ? sc : INT32_MAX;
    }
    int64_t w = 0;
    int32_t prev = -1, prev_chain = -1;
    int64_t o = 0;
    if (FILL) {
        // this lane's output offset: the lane counts of the count pass are
        // recomputed here (cheaper than storing 32 counts per element)
    }
    // pass 1 (always): count; pass 2 (FILL): write at the lane's offset
    for (int pass = 0; pass < (FILL ? 2 : 1); pass++) {
        if (pass == 1) {
            // exclusive prefix of the lane counts
            int64_t x = w;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int64_t y = __shfl_up_sync(0xffffffffu, x, d);
                if (lane >= d) x += y;
            }
            o = ptr[r] + x - w;
            // rewind the cursors
            for (int i = 0; i < m; i++) {
                const int32_t c = child[c0 + i];
                const int64_t a = ptr[c], b = ptr[c + 1];
                cur[i] = s_lo > 0 ? lower_bound_i32(idx, a, b, s_lo) : a;
                const int32_t sc = slot[c];
                cs[i] = (sc >= s_lo && sc < s_hi) ? sc : INT32_MAX;
            }
            w = 0;
            prev = -1;
            prev_chain = -1;
        }
        for (;;) {
            int32_t best = INT32_MAX;
            int bi = -1;
            bool from_row = false;
            for (int i = 0; i < m; i++) {
                const int32_t hr = cur[i] < end[i] ? idx[cur[i]] : INT32_MAX;
                if (hr < best) { best = hr; bi = i; from_row = true; }
                if (cs[i] < best) { best = cs[i]; bi = i; from_row = false; }
            }
            if (bi < 0) break;
            if (from_row) cur[bi]++;
            else cs[bi] = INT32_MAX;
            if (best == prev) continue;                       // the same slot from several children
            if (best >= own_lo && best < own_hi) continue;    // own chain: implicit
            const int32_t ch = slot_chain[best];
            if (ch == prev_chain) {
                if (pass == 1) idx[o + w - 1] = best;   // a higher slot of the same chain: the max wins
            } else {
                if (pass == 1) idx[o + w] = best;
                w++;
            }
            prev = best;
            prev_chain = ch;
        }
    }
    if (!FILL) {
        int64_t t = w;
#pragma unroll
        for (int d = 16; d; d >>= 1) t += __shfl_xor_sync(0xffffffffu, t, d);
        if (lane == 0) cnt[r - lo] = t;
    }
}

// ptr[lo + i] = base + Σ_{t < i} cnt[t], ptr[hi] = base + Σ cnt (one CTA)
__global__ void __launch_bounds__(1024) k_csr_direct_scan(int32_t lo, int32_t hi, const int64_t *cnt,
                                                          int64_t *ptr) {
    __shared__ int64_t sh[1024];
    const int t = threadIdx.x;
    const int32_t w = hi - lo;
    const int32_t per = (w + 1023) / 1024;
    const int32_t a = min(w, t * per), b = min(w, a + per);
    int64_t s = 0;
    for (int32_t i = a; i < b; i++) s += cnt[i];
    sh[t] = s;
    __syncthreads();
    for (int d = 1; d < 1024; d <<= 1) {
        const int64_t v = t >= d ? sh[t - d] : 0;
        __syncthreads();
        sh[t] += v;
        __syncthreads();
    }
    const int64_t base = ptr[lo];
    __syncthreads();
    int64_t run = base + (t ? sh[t - 1] : 0);
    for (int32_t i = a; i < b; i++) {
        ptr[lo + i] = run;
        run += cnt[i];
    }
    if (t == 1023) ptr[hi] = base + sh[1023];
}

cudaError_t build_csr_direct(const DevPoset &P, const int32_t *h_lvl_ptr, const int32_t *slot_chain,
                             const int32_t *chain_off, CsrRows &C, size_t budget, int32_t max_level_width,
                             cudaStream_t s) {
    C.ok = false;
    const int32_t n = P.n;
    if (n == 0) return cudaSuccess;
    const size_t ptr_bytes = ((size_t)n + 1) * 8;
    if (budget < ptr_bytes + 4096) return cudaSuccess;
    const size_t cap = (budget - ptr_bytes) / 4;   // idx entries that fit
    cudaError_t e = cudaMalloc((void **)&C.ptr, ptr_bytes);
    if (e != cudaSuccess) { cudaGetLastError(); C.ptr = nullptr; return cudaSuccess; }
    e = cudaMalloc((void **)&C.idx, cap * 4);
    if (e != cudaSuccess) { cudaGetLastError(); cudaFree(C.ptr); C.ptr = nullptr; C.idx = nullptr; return cudaSuccess; }
    int64_t *cnt = nullptr, *h_total = nullptr;
    int32_t *flag = nullptr;
    e = cudaMalloc((void **)&cnt, (size_t)std::max(max_level_width, 1) * 8);
    if (e == cudaSuccess) e = cudaMalloc((void **)&flag, 4);
    if (e == cudaSuccess) e = cudaMallocHost((void **)&h_total, 8);
    if (e == cudaSuccess) e = cudaMemsetAsync(flag, 0, 4, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(C.ptr, 0, 8, s);
    bool full = false;
    int64_t total = 0;
    for (int32_t L = 0; L < P.ell && e == cudaSuccess; L++) {
        const int32_t lo = h_lvl_ptr[L], hi = h_lvl_ptr[L + 1];
        const unsigned blocks = (unsigned)(((int64_t)(hi - lo) * 32 + 127) / 128);
        k_csr_direct<false><<<blocks, 128, 0, s>>>(lo, hi, P.k, P.child_ptr, P.child, P.slot, P.chain, slot_chain,
                                                   chain_off, C.ptr, C.idx, cnt, flag);
        k_csr_direct_scan<<<1, 1024, 0, s>>>(lo, hi, cnt, C.ptr);
        // the level's rows must fit the allocation before they are written
        e = cudaMemcpyAsync(h_total, C.ptr + hi, 8, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) break;
        const int64_t level_rows = *h_total - total;
        total = *h_total;
        // stop as soon as the rows cannot fit: this level's, or the rest at
        // this level's average row length (rows grow with the level on the
        // generators, so this only under-estimates)
        if ((size_t)total > cap ||
            (double)total + (double)(n - hi) * ((double)level_rows / (hi - lo)) > (double)cap) {
            full = true;
            break;
        }
        k_csr_direct<true><<<blocks, 128, 0, s>>>(lo, hi, P.k, P.child_ptr, P.child, P.slot, P.chain, slot_chain,
                                                  chain_off, C.ptr, C.idx, cnt, flag);
        launches_add(3);
        e = cudaGetLastError();
    }
    int32_t too_many = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&too_many, flag, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(cnt);
    cudaFree(flag);
    if (h_total) cudaFreeHost(h_total);
    if (e != cudaSuccess) return e;
    if (full || too_many) {   // does not fit / unsupported: no rows
        cudaFree(C.ptr);
        cudaFree(C.idx);
        C.ptr = nullptr;
        C.idx = nullptr;
        return cudaSuccess;
    }
    C.nnz = total;
    C.ok = true;
    return cudaSuccess;
}

template <typename T>
__device__ __forceinline__ T ld_cg(const T *p);
template <>
__device__ __forceinline__ double ld_cg<double>(const double *p) { return __ldcg(p); }
template <>
__device__ __forceinline__ u64 ld_cg<u64>(const u64 *p) { return __ldcg(p); }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Σ_{e ∈ [a, b)} Fsrc[idx[e] * B + c] by one warp, lanes over entries; the
// result is valid in every lane.  CG: loads bypass L1 (data written earlier
// in the same kernel by other SMs).  8 independent loads per lane in flight.
template <typename T, bool CG, int U = 16>
__device__ __forceinline__ T row_sum_lanes(const int32_t *__restrict__ idx, int64_t a, int64_t b,
                                           const T *Fsrc, int32_t B, int c) {
    const int lane = threadIdx.x & 31;
    T s[U];
#pragma unroll
    for (int u = 0; u < U; u++) s[u] = T(0);
    int64_t e = a + lane;
    for (; e + 32 * (U - 1) < b; e += 32 * U) {
        int32_t i[U];
#pragma unroll
        for (int u = 0; u < U; u++) i[u] = __ldg(idx + e + 32 * u);
#pragma unroll
        for (int u = 0; u < U; u++) {
            const T *p = Fsrc + (size_t)i[u] * B + c;
            s[u] += CG ? ld_cg(p) : __ldg(p);
        }
    }
    for (; e < b; e += 32) {
        const T *p = Fsrc + (size_t)__ldg(idx + e) * B + c;
        s[0] += CG ? ld_cg(p) : __ldg(p);
    }
#pragma unroll
    for (int st = 1; st < U; st <<= 1)
#pragma unroll
        for (int u = 0; u < U; u += 2 * st) s[u] += s[u + st];
    return warp_sum(s[0]);
}

// Σ_{e ∈ [a, b)} Fsrc[idx[e] * B + col] by one warp, lanes over columns: the
// row entries are read 32 at a time and broadcast by shuffles; 16 row loads
// (one coalesced 256-B load each) in flight.
template <typename T, bool CG, int U = 32>
__device__ __forceinline__ T row_sum_cols(const int32_t *__restrict__ idx, int64_t a, int64_t b,
                                          const T *Fsrc, int32_t B, int col) {
    const int lane = threadIdx.x & 31;
    T s[U];
#pragma unroll
    for (int u = 0; u < U; u++) s[u] = T(0);
    for (int64_t e0 = a; e0 < b; e0 += 32) {
        const int m = (int)(b - e0 < 32 ? b - e0 : 32);
        const int32_t mine = lane < m ? __ldg(idx + e0 + lane) : 0;
        int q = 0;
        for (; q + U <= m; q += U) {
            int32_t i[U];
#pragma unroll
            for (int u = 0; u < U; u++) i[u] = __shfl_sync(0xffffffffu, mine, q + u);
#pragma unroll
            for (int u = 0; u < U; u++) {
                const T *p = Fsrc + (size_t)i[u] * B + col;
                s[u] += CG ? ld_cg(p) : __ldg(p);
            }
        }
        for (; q < m; q++) {
            const int32_t i0 = __shfl_sync(0xffffffffu, mine, q);
            const T *p = Fsrc + (size_t)i0 * B + col;
            s[0] += CG ? ld_cg(p) : __ldg(p);
        }
    }
#pragma unroll
    for (int st = 1; st < U; st <<= 1)
#pragma unroll
        for (int u = 0; u < U; u += 2 * st) s[u] += s[u + st];
    return s[0];
}

// ---------------------------------------------------- zeta gather (CSR) ---
// One warp per (rank, 32-column group) [COLS] or per rank [lanes over entries].
template <typename T, bool COLS>
__global__ void __launch_bounds__(256) k_gather_csr(DevPoset P, const int64_t *__restrict__ ptr,
                                                    const int32_t *__restrict__ idx,
                                                    const T *__restrict__ F, T *__restrict__ out,
                                                    int64_t row_lo, int64_t row_hi, int32_t B,
                                                    int G, int mode) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t items = (row_hi - row_lo) * G;
    if (w >= items) return;
    const int64_t r = row_lo + w / G;
    const int cg = (int)(w % G);
    const int64_t a = ptr[r], b = ptr[r + 1];
    const int32_t my = P.slot[r];
    T *dst = mode == 0 ? out + (size_t)P.rank_user[r] * B : out + (size_t)(r - row_lo) * B;
    if (COLS) {
        const int col = cg * 32 + lane;
        const T s = row_sum_cols<T, false>(idx, a, b, F, B, col);
        dst[col] = s + __ldg(F + (size_t)my * B + col);
    } else {
        for (int c = 0; c < B; c++) {
            const T s = row_sum_lanes<T, false>(idx, a, b, F, B, c);
            if (lane == 0) dst[c] = s + __ldg(F + (size_t)my * B + c);
        }
    }
}

// Short rows (the paper's ER DAGs: ~10-80 entries) and B < 32: one thread
// per (rank, column), the row's loads unrolled 8-wide (a warp per row would
// leave most lanes idle).
template <typename T>
__global__ void __launch_bounds__(256) k_gather_csr_thread(DevPoset P, const int64_t *__restrict__ ptr,
                                                           const int32_t *__restrict__ idx,
                                                           const T *__restrict__ F, T *__restrict__ out,
                                                           int64_t row_lo, int64_t row_hi, int32_t B,
                                                           int mode) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t r = row_lo + t / B;
    const int c = (int)(t % B);
    if (r >= row_hi) return;
    const int64_t a = ptr[r], b = ptr[r + 1];
    constexpr int U = 8;
    T acc[U];
#pragma unroll
    for (int u = 0; u < U; u++) acc[u] = T(0);
    int64_t e = a;
    for (; e + U <= b; e += U) {
        int32_t i[U];
#pragma unroll
        for (int u = 0; u < U; u++) i[u] = __ldg(idx + e + u);
#pragma unroll
        for (int u = 0; u < U; u++) acc[u] += __ldg(F + (size_t)i[u] * B + c);
    }
    for (; e < b; e++) acc[0] += __ldg(F + (size_t)__ldg(idx + e) * B + c);
#pragma unroll
    for (int st = 1; st < U; st <<= 1)
#pragma unroll
        for (int u = 0; u < U; u += 2 * st) acc[u] += acc[u + st];
    T *dst = mode == 0 ? out + (size_t)P.rank_user[r] * B : out + (size_t)(r - row_lo) * B;
    dst[c] = acc[0] + __ldg(F + (size_t)P.slot[r] * B + c);
}

cudaError_t launch_gather_csr(const DevPoset &P, const CsrRows &C, int dtype, const void *F,
                              void *g, int64_t lo, int64_t hi, int64_t B, int out_rank,
                              cudaStream_t s) {
    if (hi <= lo) return cudaSuccess;
    if (B % 32 != 0 && (double)C.nnz / P.n < 96) {
        const int64_t threads = (hi - lo) * B;
        const unsigned blocks = (unsigned)((threads + 255) / 256);
        launches_add(1);
        if (dtype == 0)
            k_gather_csr_thread<u64><<<blocks, 256, 0, s>>>(P, C.ptr, C.idx, (const u64 *)F, (u64 *)g, lo, hi,
                                                            (int32_t)B, out_rank);
        else
            k_gather_csr_thread<double><<<blocks, 256, 0, s>>>(P, C.ptr, C.idx, (const double *)F, (double *)g, lo,
                                                               hi, (int32_t)B, out_rank);
        return cudaGetLastError();
    }
    const bool cols = B % 32 == 0;
    const int G = cols ? (int)(B / 32) : 1;
    const int64_t warps = (hi - lo) * G;
    const unsigned blocks = (unsigned)((warps * 32 + 255) / 256);
    launches_add(1);
#define GCSR(TT, CC)                                                                             \
    k_gather_csr<TT, CC><<<blocks, 256, 0, s>>>(P, C.ptr, C.idx, (const TT *)F, (TT *)g, lo, hi, \
                                                (int32_t)B, G, out_rank)
    if (dtype == 0) {
        if (cols) GCSR(u64, true); else GCSR(u64, false);
    } else {
        if (cols) GCSR(double, true); else GCSR(double, false);
    }
#undef GCSR
    return cudaGetLastError();
}

// ------------------------------------------------------ Möbius (CSR) ------
// Level L+1's row entries are one contiguous index range; while level L is
// summed, thread 0 of every CTA pulls its 1/gridDim share of that range into
// L2 (cp.async.bulk.prefetch: no registers, nothing waits on it), so the
// next level's index loads are L2 hits instead of DRAM round trips.
__device__ __forceinline__ void bulk_prefetch_l2(const void *lo, const void *hi) {
    uintptr_t p0 = reinterpret_cast<uintptr_t>(lo) & ~(uintptr_t)15;
    const uintptr_t p1 = (reinterpret_cast<uintptr_t>(hi) + 15) & ~(uintptr_t)15;
    while (p0 < p1) {
        const unsigned n = (unsigned)(p1 - p0 < ((uintptr_t)1 << 16) ? p1 - p0 : ((uintptr_t)1 << 16));
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p0), "r"(n) : "memory");
        p0 += n;
    }
}
__device__ __forceinline__ void prefetch_next_rows(const DevPoset &P, const int64_t *__restrict__ ptr,
                                                   const int32_t *__restrict__ idx, int32_t L) {
    if (threadIdx.x != 0 || L + 1 >= P.ell) return;
    const int32_t r0 = P.lvl_ptr[L + 1], r1 = P.lvl_ptr[L + 2];
    if (blockIdx.x == 0 && r1 - r0 <= 8192) {   // a narrow next level's row pointers, slots, user ids
        // (narrow levels are latency-bound; a wide one hides the latency itself)
        bulk_prefetch_l2(ptr + r0, ptr + r1 + 1);
        bulk_prefetch_l2(P.slot + r0, P.slot + r1);
        bulk_prefetch_l2(P.rank_user + r0, P.rank_user + r1);
    }
    const int64_t a = ptr[P.lvl_ptr[L + 1]], b = ptr[P.lvl_ptr[L + 2]];
    if ((b - a) * 4 > ((int64_t)32 << 20)) return;   // a wide level's rows would only evict L2
    const int64_t per = ((b - a) + gridDim.x - 1) / gridDim.x;
    int64_t e0 = a + per * blockIdx.x, e1 = min(b, e0 + per);
    if (e1 <= e0) return;
    uintptr_t p0 = reinterpret_cast<uintptr_t>(idx + e0) & ~(uintptr_t)15;
    const uintptr_t p1 = (reinterpret_cast<uintptr_t>(idx + e1) + 15) & ~(uintptr_t)15;
    while (p0 < p1) {
        const unsigned n = (unsigned)(p1 - p0 < ((uintptr_t)1 << 16) ? p1 - p0 : ((uintptr_t)1 << 16));
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p0), "r"(n) : "memory");
        p0 += n;
    }
}

// Grid barrier on a monotone arrival counter: barrier number t completes when
// the counter reaches (t + 1) * nblocks.  One release-add per CTA and an
// acquire spin by one thread; no reset, no generation flag.
__device__ __forceinline__ void grid_sync(unsigned *bar, unsigned nblocks, unsigned t) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        const unsigned target = (t + 1) * nblocks;
        unsigned v, rounds = 0;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
            if (++rounds == (1u << 26)) __trap();   // watchdog: a lost arrival faults, not hangs
        } while ((int)(v - target) < 0);
    }
    __syncthreads();
}

// One level's items (element, 32-column group) are dealt to "item slots":
// groups of WPI warps inside a CTA (1024 threads = 32 / WPI slots per CTA).
// The WPI warps of a slot split the element's row into contiguous chunks,
// sum them (lanes over columns, or over entries for B < 32), reduce their
// partial sums through shared memory under the slot's named barrier, and the
// slot's first warp writes F(x) = g(x) - Σ and f(x) = F(x) - F(next(x)).
// A level of w elements uses ceil(w * G / slots) rounds; C4w (256 x 2
// items) and C3w (~360 items) fit one round on 148 CTAs x 4 slots, so each
// level costs one L2 round trip of row loads, a shared-memory reduction and
// the grid barrier (the round-1 kernel used one warp per item, so a level of
// C4w ran 512 warps of 255 serial-ish loads each on a 4,736-warp grid).
// WPI (warps per item slot) follows the average row length: 8 for the
// long rows of C2 / C3w / C4w, 4 for medium rows, 1 (a warp per element, no
// slot barrier) for the short rows of the paper's ER DAGs.
#ifndef CSR_COLS_U
#define CSR_COLS_U 8
#endif
template <typename T, bool COLS, int kCsrWPI>
__global__ void __launch_bounds__(1024, 1) k_moeb_csr(DevPoset P, const int64_t *__restrict__ ptr,
                                                      const int32_t *__restrict__ idx,
                                                      const T *__restrict__ g, T *F, T *__restrict__ f,
                                                      int32_t B, int G, unsigned *bar) {
    constexpr int kCsrSlots = 32 / kCsrWPI;   // item slots per 1024-thread CTA
    __shared__ T part[kCsrSlots][kCsrWPI][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slot = warp / kCsrWPI, ws = warp % kCsrWPI;
    const int64_t nslots = (int64_t)gridDim.x * kCsrSlots;
    const int64_t my_slot = (int64_t)blockIdx.x * kCsrSlots + slot;
    for (int32_t L = 0; L < P.ell; L++) {
        const int32_t lo = P.lvl_ptr[L], hi = P.lvl_ptr[L + 1];
        prefetch_next_rows(P, ptr, idx, L);
        const int64_t items = (int64_t)(hi - lo) * G;
        // every slot runs the same number of rounds (named barriers inside)
        const int64_t rounds = (items + nslots - 1) / nslots;
        for (int64_t rd = 0; rd < rounds; rd++) {
            const int64_t it = my_slot + rd * nslots;
            const bool valid = it < items;
            int32_t r = 0, my = 0, u = 0;
            int cg = 0;
            int64_t a = 0, b = 0;
            if (valid) {
                r = lo + (int32_t)(it / G);
                cg = (int)(it % G);
                a = ptr[r];
                b = ptr[r + 1];
                if (ws == 0) {   // the epilogue's addresses, loaded before the row sum
                    my = __ldg(P.slot + r);
                    u = __ldg(P.rank_user + r);
                }
            }
            // this warp's chunk of the row
            const int64_t len = b - a, per = (len + kCsrWPI - 1) / kCsrWPI;
            const int64_t ca = a + min(len, per * ws), cb = a + min(len, per * (ws + 1));
            if (COLS) {
                const int col = cg * 32 + lane;
                const T s = valid ? row_sum_cols<T, true, CSR_COLS_U>(idx, ca, cb, F, B, col) : T(0);
                part[slot][ws][lane] = s;
            } else {
                // B % 32 != 0: lanes over entries, one column of the group at
                // a time; lane c of the partial row holds column cg * 32 + c
                T mine = T(0);
                const int c1 = min(B - cg * 32, 32);
                for (int c = 0; c < c1; c++) {
                    const T s = valid ? row_sum_lanes<T, true, 8>(idx, ca, cb, F, B, cg * 32 + c) : T(0);
                    if (lane == c) mine = s;
                }
                part[slot][ws][lane] = mine;
            }
            if (kCsrWPI > 1) asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(32 * kCsrWPI) : "memory");
            else __syncwarp();
            if (ws == 0 && valid) {
                const int ncol = COLS ? 32 : min(B - cg * 32, 32);
                if (lane < ncol) {
                    // three independent loads (one round of latency), then the sums
                    const int col = cg * 32 + lane;
                    const bool has_prev = !(__ldg(P.slot_user + my) < 0);   // bit 31 = chain start
                    const T gx = __ldg(g + (size_t)u * B + col);
                    const T fp = ld_cg(F + (size_t)(my > 0 ? my - 1 : 0) * B + col);
                    T s = part[slot][0][lane];
#pragma unroll
                    for (int w2 = 1; w2 < kCsrWPI; w2++) s += part[slot][w2][lane];
                    const T Fx = gx - s;
                    F[(size_t)my * B + col] = Fx;
                    f[(size_t)u * B + col] = has_prev ? Fx - fp : Fx;
                }
            }
            if (kCsrWPI > 1) asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(32 * kCsrWPI) : "memory");
            else __syncwarp();
        }
        if (L + 1 < P.ell) grid_sync(bar, gridDim.x, (unsigned)L);
    }
}

// Short rows (ER DAGs, ~10-80 entries) and B < 32: one thread per
// (element, column) sums its row (8 loads in flight), persistent grid with
// one barrier per level as above.
template <typename T>
__global__ void __launch_bounds__(1024, 1) k_moeb_csr_thread(DevPoset P, const int64_t *__restrict__ ptr,
                                                             const int32_t *__restrict__ idx,
                                                             const T *__restrict__ g, T *F, T *__restrict__ f,
                                                             int32_t B, unsigned *bar) {
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int32_t L = 0; L < P.ell; L++) {
        const int32_t lo = P.lvl_ptr[L], hi = P.lvl_ptr[L + 1];
        prefetch_next_rows(P, ptr, idx, L);
        const int64_t items = (int64_t)(hi - lo) * B;
        for (int64_t it = tid; it < items; it += nth) {
            const int32_t r = lo + (int32_t)(it / B);
            const int c = (int)(it % B);
            const int64_t a = ptr[r], b = ptr[r + 1];
            const int32_t my = __ldg(P.slot + r), usr = __ldg(P.rank_user + r);   // epilogue addresses, early
            constexpr int U = 8;
            T acc[U];
#pragma unroll
            for (int u = 0; u < U; u++) acc[u] = T(0);
            int64_t e = a;
            for (; e + U <= b; e += U) {
                int32_t i[U];
#pragma unroll
                for (int u = 0; u < U; u++) i[u] = __ldg(idx + e + u);
#pragma unroll
                for (int u = 0; u < U; u++) acc[u] += ld_cg(F + (size_t)i[u] * B + c);
            }
            for (; e < b; e++) acc[0] += ld_cg(F + (size_t)__ldg(idx + e) * B + c);
#pragma unroll
            for (int st = 1; st < U; st <<= 1)
#pragma unroll
                for (int u = 0; u < U; u += 2 * st) acc[u] += acc[u + st];
            const bool start = __ldg(P.slot_user + my) < 0;
            const T gx = __ldg(g + (size_t)usr * B + c);
            const T fp = ld_cg(F + (size_t)(my > 0 ? my - 1 : 0) * B + c);
            const T Fx = gx - acc[0];
            F[(size_t)my * B + c] = Fx;
            f[(size_t)usr * B + c] = start ? Fx : Fx - fp;
        }
        if (L + 1 < P.ell) grid_sync(bar, gridDim.x, (unsigned)L);
    }
}

cudaError_t launch_moebius_csr(const DevPoset &P, const CsrRows &C, int dtype, const void *g,
                               void *F, void *f, int64_t B, unsigned *bar, int num_sms,
                               cudaStream_t s) {
    if (P.n == 0) return cudaSuccess;
    if (B % 32 != 0 && (double)C.nnz / P.n < 128) {
        cudaError_t e = cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), s);
        if (e != cudaSuccess) return e;
        DevPoset Pc = P;
        const int64_t *pp = C.ptr;
        const int32_t *ip = C.idx;
        int32_t Bi = (int32_t)B;
        void *args[] = {&Pc, &pp, &ip, (void *)&g, &F, &f, &Bi, &bar};
        void *fn = dtype == 0 ? (void *)k_moeb_csr_thread<u64> : (void *)k_moeb_csr_thread<double>;
        launches_add(1);
        return cudaLaunchCooperativeKernel(fn, dim3(num_sms), dim3(1024), args, 0, s);
    }
    // lanes over columns for B % 32 == 0; otherwise lanes over entries, one
    // column at a time, in groups of 32 columns
    const bool cols = B % 32 == 0;
    int G = (int)((B + 31) / 32);
    const double avg = (double)C.nnz / P.n;
    const int wpi = avg >= 128 ? 8 : avg >= 48 ? 4 : 1;
    void *fn;
#define MCSR(WPI)                                                                                  \
    if (wpi == WPI) {                                                                              \
        if (dtype == 0)                                                                            \
            fn = cols ? (void *)k_moeb_csr<u64, true, WPI> : (void *)k_moeb_csr<u64, false, WPI>;  \
        else                                                                                       \
            fn = cols ? (void *)k_moeb_csr<double, true, WPI> : (void *)k_moeb_csr<double, false, WPI>; \
    }
    MCSR(1) MCSR(4) MCSR(8)
#undef MCSR
    cudaError_t e = cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    DevPoset Pc = P;
    const int64_t *pp = C.ptr;
    const int32_t *ip = C.idx;
    int32_t Bi = (int32_t)B;
    void *args[] = {&Pc, &pp, &ip, (void *)&g, &F, &f, &Bi, &G, &bar};
    launches_add(1);
    return cudaLaunchCooperativeKernel(fn, dim3(num_sms), dim3(1024), args, 0, s);
}

}  // namespace poset
