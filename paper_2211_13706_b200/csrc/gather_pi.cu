// Kernel (iv), batched form: zeta gather-reduce g(x) = Σ_j F[M[j][x]]
// (Eq. zeta-fast, Alg. 3) in a per-tile GATHER ORDER
// chosen so that consecutive elements share most of their niv rows.
//
// Why: with B = 32 columns every (x, j) pair delivers a
// 256-byte row of F to registers, so the gather is bound by the SM load
// data path (128 B/clk/SM), not by HBM.  A lane that walks R consecutive
// elements keeps the row it last used per chain and reloads only when the
// index changes; the fraction of (x, j) pairs that reload is the "miss
// rate".  The gather itself is order-free (each g(x) is independent), so
// the order of elements inside each 256-element tile is chosen at setup by a
// greedy nearest-neighbour walk over the niv rows (Hamming distance).
// Measured on C5w (n = 40k sample): miss 0.64 for rank order with 4 elements
// per lane (round-1 kernel) -> 0.315 for the greedy order with 8 per lane.
//
//   k_gather_order   one CTA per tile of 256 ranks: greedy walk -> pi_rank
//   k_build_gtable   Mg[j][p] = M[j][pi_rank[p]] (chain-major, gather order),
//                    out_user[p] = user id of position p (-1 = padding)
//   k_gather_pi      persistent CTAs over (tile, 32-column group) items; the
//                    tile's index rows are staged by cp.async.bulk (TMA) into
//                    a two-stage shared-memory ring one chunk ahead; lane
//                    (q, c4) of a warp walks 8 consecutive positions
//                    (q = lane / 8) for 4 columns (c4 = lane % 8), reloading
//                    a row (one predicated 32-byte load) only on a change.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels.cuh"
#include "ptx.cuh"

namespace poset {

typedef unsigned long long u64;

namespace {
constexpr int GT = 256;     // tile = positions per CTA item
constexpr int GD = 64;      // chains sampled for the order's distance
constexpr int KCH = 32;     // chains per staged index chunk (32 KB)
constexpr int RPL = 8;      // consecutive positions per lane
}

// ------------------------------------------------------------ order -----
// Greedy nearest neighbour over the tile's rows (first element first):
// each step picks the unused element whose sampled row differs from the
// current one in the fewest chains.  Distance over <= 64 evenly spaced
// chains (all of them when k <= 64).
__global__ void __launch_bounds__(GT) k_gather_order(const int32_t *__restrict__ M, int32_t n,
                                                     int32_t k, int32_t *__restrict__ pi_rank) {
    __shared__ int32_t cur[GD];
    __shared__ unsigned wmin[GT / 32];
    __shared__ int32_t pick;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * GT;
    const int64_t r = r0 + tid;
    const bool valid = r < n;
    const int D = k < GD ? k : GD;
    int32_t row[GD];
#pragma unroll
    for (int c = 0; c < GD; c++) {
        const int j = (int)((int64_t)c * k / D);
        row[c] = (valid && c < D) ? __ldg(M + (size_t)j * n + r) : 0;
    }
    bool used = !valid;
    if (tid == 0) {
#pragma unroll
        for (int c = 0; c < GD; c++) cur[c] = row[c];
        used = true;
        pi_rank[r0] = valid ? (int32_t)r : -1;
    }
    const int nv = n > r0 ? (int)(n - r0 < GT ? n - r0 : GT) : 0;
    __syncthreads();
    for (int step = 1; step < GT; step++) {
        unsigned key = 0xffffffffu;
        if (!used) {
            int d = 0;
#pragma unroll
            for (int c = 0; c < GD; c++) d += (c < D) & (row[c] != cur[c]);
            key = ((unsigned)d << 8) | (unsigned)tid;
        }
        key = __reduce_min_sync(0xffffffffu, key);
        if (lane == 0) wmin[warp] = key;
        __syncthreads();
        if (warp == 0) {
            unsigned v = lane < GT / 32 ? wmin[lane] : 0xffffffffu;
            v = __reduce_min_sync(0xffffffffu, v);
            if (lane == 0) pick = v == 0xffffffffu ? -1 : (int)(v & 0xff);
        }
        __syncthreads();
        const int p = pick;
        if (p == tid) {
#pragma unroll
            for (int c = 0; c < GD; c++) cur[c] = row[c];
            used = true;
        }
        if (tid == 0) pi_rank[r0 + step] = (step < nv && p >= 0) ? (int32_t)(r0 + p) : -1;
        __syncthreads();
    }
}

__global__ void k_build_gtable(const int32_t *__restrict__ M, const int32_t *__restrict__ rank_user,
                               const int32_t *__restrict__ pi_rank, int32_t n, int32_t k, int64_t npad,
                               int32_t *__restrict__ Mg, int32_t *__restrict__ out_user) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npad) return;
    const int32_t r = pi_rank[p];
    const int j = blockIdx.y;
    Mg[(size_t)j * npad + p] = r >= 0 ? M[(size_t)j * n + r] : n;
    if (j == 0) out_user[p] = r >= 0 ? rank_user[r] : -1;
}

// Fr[tile][j] = (lowest, highest) F slot of chain j referenced by the tile
// (∞ = n excluded; empty = (n, -1)): the L2 prefetch ranges of k_gather_pi.
__global__ void k_build_franges(const int32_t *__restrict__ Mg, int64_t npad, int32_t n, int32_t k,
                                int2 *__restrict__ Fr) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t tiles = npad / GT;
    if (w >= tiles * k) return;
    const int64_t tile = w / k;
    const int j = (int)(w % k);
    int lo = n, hi = -1;
    for (int p = lane; p < GT; p += 32) {
        const int32_t v = Mg[(size_t)j * npad + tile * GT + p];
        if (v < n) { lo = min(lo, v); hi = max(hi, v); }
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if (lane == 0) Fr[w] = make_int2(lo, hi);
}

cudaError_t build_gather_pi(const DevPoset &P, GatherPi &G, cudaStream_t s) {
    G.npad = ((int64_t)P.n + GT - 1) / GT * GT;
    const int64_t tiles = G.npad / GT;
    cudaError_t e = cudaSuccess;
    int32_t *pi = nullptr;
    if ((e = cudaMalloc((void **)&pi, (size_t)G.npad * 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc((void **)&G.Mg, (size_t)G.npad * P.k * 4)) != cudaSuccess) { cudaFree(pi); G.Mg = nullptr; return e; }
    if ((e = cudaMalloc((void **)&G.out_user, (size_t)G.npad * 4)) != cudaSuccess) {
        cudaFree(pi); cudaFree(G.Mg); G.Mg = nullptr; G.out_user = nullptr; return e;
    }
    k_gather_order<<<(unsigned)tiles, GT, 0, s>>>(P.M, P.n, P.k, pi);
    k_build_gtable<<<dim3((unsigned)((G.npad + 255) / 256), (unsigned)P.k), 256, 0, s>>>(
        P.M, P.rank_user, pi, P.n, P.k, G.npad, G.Mg, G.out_user);
    if ((e = cudaMalloc((void **)&G.Fr, (size_t)tiles * P.k * sizeof(int2))) != cudaSuccess) {
        cudaFree(pi); return e;
    }
    k_build_franges<<<(unsigned)((tiles * P.k * 32 + 255) / 256), 256, 0, s>>>(G.Mg, G.npad, P.n, P.k,
                                                                                 (int2 *)G.Fr);
    launches_add(3);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(pi);
    G.ok = e == cudaSuccess;
    return e;
}

void free_gather_pi(GatherPi &G) {
    if (G.Mg) cudaFree(G.Mg);
    if (G.out_user) cudaFree(G.out_user);
    if (G.Fr) cudaFree(G.Fr);
    if (G.D) cudaFree(G.D);
    if (G.Dptr) cudaFree(G.Dptr);
    if (G.redo) cudaFree(G.redo);
    if (G.nredo) cudaFree(G.nredo);
    G = GatherPi{};
}

// ------------------------------------------------------------ gather ----
__device__ __forceinline__ void ld4_if_ne_pi(u64 (&v)[4], const void *p, int32_t a, int32_t b) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %4, %5;\n\t"
                 "@q ld.global.nc.v4.b64 {%0,%1,%2,%3}, [%6];\n\t}"
                 : "+l"(v[0]), "+l"(v[1]), "+l"(v[2]), "+l"(v[3])
                 : "r"(a), "r"(b), "l"(p));
}

template <typename T>
__device__ __forceinline__ T as_t(u64 x);
template <>
__device__ __forceinline__ u64 as_t<u64>(u64 x) { return x; }
template <>
__device__ __forceinline__ double as_t<double>(u64 x) { return __longlong_as_double((long long)x); }
template <typename T>
__device__ __forceinline__ u64 as_bits(T x);
template <>
__device__ __forceinline__ u64 as_bits<u64>(u64 x) { return x; }
template <>
__device__ __forceinline__ u64 as_bits<double>(double x) { return (u64)__double_as_longlong(x); }

// Items (tile, column group) are dealt to CTAs in contiguous runs
// (contig = 1; consecutive tiles share most of their F rows, which then stay
// in L1) or round-robin (contig = 0).
// STEP_IDS: load each step's KC indices from shared memory (KC registers)
// instead of holding the lane's 8 x KC indices (frees registers for 4
// chains per step).  Fr != null: at the start of an item, warp 0 prefetches
// into L2 the F rows the CTA's NEXT item reads (cp.async.bulk.prefetch, one
// contiguous slot range per chain), so first touches of F rows do not stall
// the dependent reuse walk on DRAM latency.
template <typename T, int KC, int MINB, bool STEP_IDS, int PFD, int RP = RPL>
__global__ void __launch_bounds__(32 * GT / (4 * RP), MINB) k_gather_pi(const int32_t *__restrict__ Mg, int64_t npad,
                                                         int32_t k, const T *__restrict__ F,
                                                         T *__restrict__ out,
                                                         const int32_t *__restrict__ out_user, int32_t B,
                                                         int G32, int64_t items, int contig,
                                                         const int2 *__restrict__ Fr) {
    extern __shared__ __align__(128) int32_t sidx[];   // [2][KCH][GT]
    __shared__ __align__(8) unsigned long long full[2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = lane >> 3, c4 = lane & 7;
    const int nchunk = (k + KCH - 1) / KCH;
    const int64_t per = (items + gridDim.x - 1) / gridDim.x;
    const int64_t ilo = contig ? min(items, (int64_t)blockIdx.x * per) : blockIdx.x;
    const int64_t my_items = contig ? min(items, ilo + per) - ilo
                                    : (items > blockIdx.x ? (items - 1 - blockIdx.x) / gridDim.x + 1 : 0);
    const int64_t istep = contig ? 1 : gridDim.x;
    const int64_t nstages = my_items * nchunk;
    if (threadIdx.x == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // stage s = (item index i = s / nchunk, chunk c = s % nchunk) -> buffer s & 1
    auto issue = [&](int64_t s) {
        const int64_t it = ilo + (s / nchunk) * istep;
        const int64_t tile = it / G32;
        const int c = (int)(s % nchunk);
        const int j0 = c * KCH, jn = min(KCH, k - j0);
        int32_t *dst = sidx + (size_t)(s & 1) * KCH * GT;
        mbar_expect_tx(&full[s & 1], (unsigned)(jn * GT * 4));
        for (int u = 0; u < jn; u++)
            bulk_g2s(dst + u * GT, Mg + (size_t)(j0 + u) * npad + tile * GT, GT * 4, &full[s & 1]);
    };
    if (threadIdx.x == 0) {
        if (nstages > 0) issue(0);
        if (nstages > 1) issue(1);
    }
    const unsigned rowbytes = (unsigned)B * sizeof(T);
    const int pos0 = warp * (4 * RP) + q * RP;   // this lane's first position in the tile
    T acc[RP][4];
    for (int64_t s = 0; s < nstages; s++) {
        const int c = (int)(s % nchunk);
        const int64_t it = ilo + (s / nchunk) * istep;
        const int cg = (int)(it % G32);
        if (c == 0) {
#pragma unroll
            for (int t = 0; t < RP; t++)
#pragma unroll
                for (int i = 0; i < 4; i++) acc[t][i] = T(0);
        }
        mbar_wait(&full[s & 1], (unsigned)((s >> 1) & 1));
        const int32_t *S = sidx + (size_t)(s & 1) * KCH * GT + pos0;
        const char *Fb = reinterpret_cast<const char *>(F + cg * 32 + c4 * 4);
        const int jn = min(KCH, k - c * KCH);
        if (Fr && c == 0 && warp == 0) {
            const int64_t nit = it + istep;
            if (nit < ilo + my_items * istep && (nit % G32) == 0) {
                const int2 *fr = Fr + (nit / G32) * k;
                for (int j = lane; j < k; j += 32) {
                    const int2 r = fr[j];
                    if (r.y >= r.x) {
                        const char *a = reinterpret_cast<const char *>(F + (size_t)r.x * B);
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a),
                                     "r"((unsigned)(r.y - r.x + 1) * rowbytes)
                                     : "memory");
                    }
                }
            }
        }
        if constexpr (STEP_IDS) {
            for (int jj = 0; jj < jn; jj += KC) {
                int32_t prev[KC];
                u64 v[KC][4];
#pragma unroll
                for (int u = 0; u < KC; u++) {
                    prev[u] = -1;
#pragma unroll
                    for (int i = 0; i < 4; i++) v[u][i] = 0;
                }
#pragma unroll
                for (int t = 0; t < RP; t++) {
                    int32_t id[KC];
#pragma unroll
                    for (int u = 0; u < KC; u++) id[u] = jj + u < jn ? S[(jj + u) * GT + t] : -1;
#pragma unroll
                    for (int u = 0; u < KC; u++) {
                        ld4_if_ne_pi(v[u], Fb + (size_t)(unsigned)id[u] * rowbytes, id[u], prev[u]);
                        prev[u] = id[u];
                    }
#pragma unroll
                    for (int i = 0; i < 4; i++) {
                        T x = as_t<T>(v[0][i]);
#pragma unroll
                        for (int u = 1; u < KC; u++) x += as_t<T>(v[u][i]);
                        acc[t][i] += x;
                    }
                }
            }
        } else
        for (int jj = 0; jj < jn; jj += KC) {
            int32_t id[KC][RP];
#pragma unroll
            for (int u = 0; u < KC; u++) {
                if (jj + u < jn) {
#pragma unroll
                    for (int h = 0; h < RP / 4; h++) {
                        const int4 a = *reinterpret_cast<const int4 *>(S + (jj + u) * GT + 4 * h);
                        id[u][4 * h] = a.x; id[u][4 * h + 1] = a.y; id[u][4 * h + 2] = a.z; id[u][4 * h + 3] = a.w;
                    }
                } else {
#pragma unroll
                    for (int t = 0; t < RP; t++) id[u][t] = -1;   // no chain: never loads
                }
            }
            if (PFD > 0 && jj + PFD * KC < jn) {
                // L1 prefetch of the rows PFD chain groups ahead (only where
                // the index changes: the rows the reuse walk will load)
#pragma unroll
                for (int u = 0; u < KC; u++) {
                    const int32_t *Sp = S + (jj + PFD * KC + u) * GT;
                    if (jj + PFD * KC + u < jn) {
                        int32_t w[RP];
#pragma unroll
                        for (int h = 0; h < RP / 4; h++) {
                            const int4 a = *reinterpret_cast<const int4 *>(Sp + 4 * h);
                            w[4 * h] = a.x; w[4 * h + 1] = a.y; w[4 * h + 2] = a.z; w[4 * h + 3] = a.w;
                        }
#pragma unroll
                        for (int t = 0; t < RP; t++)
                            if (t == 0 || w[t] != w[t - 1])
                                asm volatile("prefetch.global.L1 [%0];" ::"l"(Fb + (size_t)(unsigned)w[t] * rowbytes));
                    }
                }
            }
            u64 v[KC][4];
#pragma unroll
            for (int u = 0; u < KC; u++)
#pragma unroll
                for (int i = 0; i < 4; i++) v[u][i] = 0;   // also the value of an absent chain
#pragma unroll
            for (int t = 0; t < RP; t++) {
#pragma unroll
                for (int u = 0; u < KC; u++)
                    ld4_if_ne_pi(v[u], Fb + (size_t)(unsigned)id[u][t] * rowbytes, id[u][t],
                                 t ? id[u][t - 1] : (id[u][0] < 0 ? id[u][0] : -1));
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    T x = as_t<T>(v[0][i]);
#pragma unroll
                    for (int u = 1; u < KC; u++) x += as_t<T>(v[u][i]);
                    acc[t][i] += x;
                }
            }
        }
        if (c == nchunk - 1) {
            const int64_t tile = it / G32;
#pragma unroll
            for (int t = 0; t < RP; t++) {
                const int32_t usr = out_user[tile * GT + pos0 + t];
                if (usr >= 0) {
                    u64 o[4];
#pragma unroll
                    for (int i = 0; i < 4; i++) o[i] = as_bits<T>(acc[t][i]);
                    u64 *dst = reinterpret_cast<u64 *>(out + (size_t)usr * B + cg * 32 + c4 * 4);
                    asm volatile("st.global.v4.b64 [%0], {%1,%2,%3,%4};" ::"l"(dst), "l"(o[0]), "l"(o[1]),
                                 "l"(o[2]), "l"(o[3])
                                 : "memory");
                }
            }
        }
        __syncthreads();   // every warp is done with buffer s & 1
        if (threadIdx.x == 0 && s + 2 < nstages) issue(s + 2);
    }
}

static int g_pi_cfg = 0;
void set_gather_pi_cfg(int c) { g_pi_cfg = c; }

template <typename T, int KC, int MINB, bool STEP_IDS, int PFD, int RP = RPL>
static cudaError_t gather_pi_t(const GatherPi &G, int32_t k, const void *F, void *g, int64_t B, int num_sms,
                               int contig, bool prefetch, cudaStream_t s) {
    const int G32 = (int)(B / 32);
    const int64_t items = (G.npad / GT) * G32;
    const size_t smem = (size_t)2 * KCH * GT * 4;
    const int64_t grid = std::min<int64_t>(items, (int64_t)num_sms * MINB);
    auto kern = k_gather_pi<T, KC, MINB, STEP_IDS, PFD, RP>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)grid, 32 * GT / (4 * RP), smem, s>>>(G.Mg, G.npad, k, (const T *)F, (T *)g, G.out_user, (int32_t)B,
                                           G32, items, contig, prefetch ? (const int2 *)G.Fr : nullptr);
    launches_add(1);
    return cudaGetLastError();
}

int gather_pi_cfg_get() { return g_pi_cfg; }

// cfg (option "gather_pi_cfg", tuning; DESIGN.md §5.2 has the measured
// table): 0 = 2 chains per step, held indices, round-robin items, L1
// prefetch of the rows 2 chain groups ahead (default); 4 = the delta-list
// kernel (gather_delta.cu; its list is built on first use); 1 = as 0, contiguous
// items + L2 prefetch of the next item's rows; 2 = 2 chains per step, held
// indices, round-robin, no prefetch (first version); 3 = 4 chains per step,
// per-step index loads, round-robin
template <typename T>
static cudaError_t gather_pi_cfg(const GatherPi &G, int32_t k, const void *F, void *g, int64_t B,
                                 int num_sms, cudaStream_t s) {
    switch (g_pi_cfg) {
        case 1: return gather_pi_t<T, 2, 2, false, 2>(G, k, F, g, B, num_sms, 1, true, s);
        case 2: return gather_pi_t<T, 2, 2, false, 0>(G, k, F, g, B, num_sms, 0, false, s);
        case 3: return gather_pi_t<T, 4, 2, true, 0>(G, k, F, g, B, num_sms, 0, false, s);
        case 5: return gather_pi_t<T, 2, 2, false, 2, 4>(G, k, F, g, B, num_sms, 0, false, s);   // 4 positions per lane
        case 6: return gather_pi_t<T, 2, 4, false, 2, 16>(G, k, F, g, B, num_sms, 0, false, s);  // 16 per lane
        case 7: return gather_pi_t<T, 2, 1, false, 2, 4>(G, k, F, g, B, num_sms, 0, false, s);   // 4 per lane, 128 regs
        default: return gather_pi_t<T, 2, 2, false, 2>(G, k, F, g, B, num_sms, 0, false, s);
    }
}

cudaError_t launch_gather_pi(const GatherPi &G, int32_t k, int dtype, const void *F, void *g, int64_t B,
                             int num_sms, cudaStream_t s) {
    return dtype == 0 ? gather_pi_cfg<u64>(G, k, F, g, B, num_sms, s)
                      : gather_pi_cfg<double>(G, k, F, g, B, num_sms, s);
}

}  // namespace poset
