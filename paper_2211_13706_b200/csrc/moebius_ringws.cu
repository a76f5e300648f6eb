// Kernel (v), schedule RINGWS: the RING Möbius solve (moebius_ring.cu) with
// warp specialisation, for bounded-reach posets with narrow levels (C5w).
//
// Alg. 4 needs, for each x in topological order,
//     F(x) = g(x) - Σ_{j ≠ id(x)} F(niv_j(x)),   f(x) = F(x) - F(next(x)).
// The dependencies of an element of level L (Alg. 6 levels) split
// by their own level:
//   near  level >= L - LD:  at most NN of them (~2 on average for C5w, LD=2)
//   far   level <  L - LD:  the rest (~60 for C5w)
// The far part S_old(x) can be summed as soon as level L - LD - 1 is done,
// i.e. up to LD levels before x itself is due.  So:
//   * warp 0 ("fresh") sweeps the levels: for each x of the level it sums
//     its <= NN near entries, takes S_old(x) from a shared buffer, writes
//     F(x) into the ring and f(x) to global memory, then publishes
//     R_done = hi(level) -- only this short chain is on the critical path;
//   * warps 1..NWO ("old") walk the ranks in order, LPEO lanes per element,
//     wait until R_done >= thr(x) = lo(L(x) - LD), sum the far entries
//     and post S_old(x) (value, then tag = x) in a shared buffer.
// All sizes (ring, S_old buffer, pipeline depth) are chosen by the plan so
// that no entry is overwritten while it may still be read.
//
//   rows [npad][kp] uint16 (ring slots = rank mod RING, RING = zero entry):
//     [0, NN)           near entries, padded with RING
//     [NN, NN + FE)     far entries, sorted by bank key (see k_build_dist)
//     NN + FE           slot of next(x)
//     NN + FE + 1, +2   thr(x) low / high 16 bits
// rows, g (rank order) and rank->user are streamed by TMA bulk copies into a
// shared-memory pipeline as in RING.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "kernels.cuh"
#include "ptx.cuh"

namespace poset {

typedef unsigned long long u64;

// ------------------------------------------------------------ setup -------
// max number of dependencies (j ≠ id(r), niv_j(r) ≠ ∞) at level distance
// <= 1, 2, 3 over all ranks r
__global__ void k_near_max(const int32_t *__restrict__ M, int32_t n, int32_t k,
                           const int32_t *__restrict__ chain, const int32_t *__restrict__ level,
                           const int32_t *__restrict__ slot_rank, unsigned *out3) {
    const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned c1 = 0, c2 = 0, c3 = 0;
    if (r < n) {
        const int32_t own = chain[r], lr = level[r];
        for (int32_t j = 0; j < k; j++) {
            const int32_t s = __ldcs(M + (size_t)j * n + r);
            if (j == own || s == n) continue;
            const int32_t ld = lr - level[slot_rank[s]];
            c1 += ld <= 1;
            c2 += ld <= 2;
            c3 += ld <= 3;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        c1 = max(c1, __shfl_xor_sync(0xffffffffu, c1, o));
        c2 = max(c2, __shfl_xor_sync(0xffffffffu, c2, o));
        c3 = max(c3, __shfl_xor_sync(0xffffffffu, c3, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(out3, c1);
        atomicMax(out3 + 1, c2);
        atomicMax(out3 + 2, c3);
    }
}

__global__ void __launch_bounds__(256) k_build_ringws(
    const int32_t *__restrict__ M, int32_t n, int32_t k, int32_t kp, int32_t nn, int32_t fe,
    int32_t ld, int32_t ring, const int32_t *__restrict__ chain, const int32_t *__restrict__ slot,
    const int32_t *__restrict__ slot_rank, const int32_t *__restrict__ level,
    const int32_t *__restrict__ lvl_ptr, uint16_t *__restrict__ D) {
    extern __shared__ uint16_t tile[];   // raw [32][k + 1] slots, near flags [32][k+1], out [32][kp]
    const int ks = k + 1;
    uint16_t *raw = tile, *isnear = tile + 32 * ks, *outr = tile + 64 * ks;
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
        raw[lane * ks + j] = (uint16_t)(dep >= 0 ? (dep & mask) : ring);
        isnear[lane * ks + j] = (uint16_t)(dep >= 0 && level[r] - level[dep] <= ld);
    }
    __syncthreads();
    if (w == 0) {
        const uint16_t *in = raw + lane * ks, *nf = isnear + lane * ks;
        uint16_t *out = outr + lane * kp;
        int cnt[17], pos[17], acc = 0, nnear = 0;
#pragma unroll
        for (int c = 0; c < 17; c++) cnt[c] = 0;
        for (int j = 0; j < k; j++) {
            const int s = in[j];
            if (nf[j]) {
                if (nnear < nn) out[nnear] = (uint16_t)s;   // plan guarantees nnear <= nn
                nnear++;
            } else {
                cnt[s == ring ? 16 : ((s - r) & 15)]++;
            }
        }
        for (int j = nnear; j < nn; j++) out[j] = (uint16_t)ring;
#pragma unroll
        for (int c = 0; c < 17; c++) { pos[c] = acc; acc += cnt[c]; }
        for (int j = 0; j < k; j++) {
            if (nf[j]) continue;
            const int s = in[j];
            const int c = s == ring ? 16 : ((s - r) & 15);
#pragma unroll
            for (int cc = 0; cc < 17; cc++)
                if (cc == c) out[nn + pos[cc]++] = (uint16_t)s;
        }
        for (int j = nn + acc; j < kp; j++) out[j] = (uint16_t)ring;
        // next(r), thr(r)
        int pn = -1;
        int32_t thr = 0;
        if (r < n) {
            const int32_t s = slot[r];
            if (s > 0) {
                const int32_t p = slot_rank[s - 1];
                if (chain[p] == chain[r]) pn = p;
            }
            const int32_t L = level[r];
            thr = L - ld >= 0 ? lvl_ptr[L - ld] : 0;
        }
        out[nn + fe] = (uint16_t)(pn >= 0 ? (pn & mask) : ring);
        out[nn + fe + 1] = (uint16_t)(thr & 0xffff);
        out[nn + fe + 2] = (uint16_t)((unsigned)thr >> 16);
    }
    __syncthreads();
    const int64_t base = (int64_t)r0 * kp;
    for (int t = threadIdx.x; t < 32 * kp; t += blockDim.x) D[base + t] = outr[t];
}

// ------------------------------------------------------------ kernel ------
struct RWArgs {
    const uint16_t *D;          // [npad][kp]
    const void *gP;             // [B][npad]
    const int32_t *ru;          // [npad]
    const int32_t *lvl_ptr;     // [ell + 1]
    void *f;                    // [n][B]
    int64_t npad;
    int32_t n, kp, ell, B;
    int32_t ring_mask, sbuf_mask;
    int32_t lg_ch, nstage;
};

__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
    asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

template <typename T, int E>
__device__ __forceinline__ T slot_sum(const T *ring, const uint16_t *row) {
    T v[E];
    if constexpr (E >= 8) {
#pragma unroll
        for (int i = 0; i < E / 8; i++) {
            const uint4 w = reinterpret_cast<const uint4 *>(row)[i];
            const unsigned ws[4] = {w.x, w.y, w.z, w.w};
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

template <typename T, int NN, int LPEO, int EO, int NWO>
__global__ void __launch_bounds__(32 * (1 + NWO)) k_moeb_ringws(RWArgs a) {
    constexpr int FE = LPEO * EO;
    extern __shared__ __align__(16) unsigned char smem[];
    const int RING = a.ring_mask + 1, SBUF = a.sbuf_mask + 1;
    const int ch = 1 << a.lg_ch;
    T *ring = reinterpret_cast<T *>(smem);                                  // RING + 2
    T *sbuf = ring + RING + 2;                                              // SBUF
    int *stag = reinterpret_cast<int *>(sbuf + SBUF);                       // SBUF
    int *ctrl = stag + SBUF;                                                // [0] R_done, [1] issued
    u64 *bars = reinterpret_cast<u64 *>(ctrl + 4);                          // nstage
    unsigned char *stage0 = reinterpret_cast<unsigned char *>(bars + ((a.nstage + 1) & ~1));
    const unsigned dbytes = (unsigned)ch * a.kp * 2, gbytes = (unsigned)ch * 8, ubytes = (unsigned)ch * 4;
    const unsigned sbytes = dbytes + gbytes + ubytes;
    const int b = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const T *gcol = reinterpret_cast<const T *>(a.gP) + (size_t)b * a.npad;
    const int32_t nchunks = (int32_t)(a.npad >> a.lg_ch);

    for (int i = tid; i < SBUF; i += blockDim.x) stag[i] = -1;
    if (tid == 0) {
        ring[RING] = T(0);
        ctrl[0] = 0;
        ctrl[1] = 0;
        for (int s = 0; s < a.nstage; s++) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto stage_of = [&](int32_t c) { return stage0 + (size_t)(c & (a.nstage - 1)) * sbytes; };
    if (warp == 0) {
        // ------------------------------------------------ fresh warp ------
        int32_t issued = 0;
        auto issue = [&](int32_t c) {
            const int s = c & (a.nstage - 1);
            unsigned char *st = stage_of(c);
            const size_t r0 = (size_t)c << a.lg_ch;
            mbar_expect_tx(&bars[s], sbytes);
            bulk_g2s(st, a.D + r0 * a.kp, dbytes, &bars[s]);
            bulk_g2s(st + dbytes, gcol + r0, gbytes, &bars[s]);
            bulk_g2s(st + dbytes + gbytes, a.ru + r0, ubytes, &bars[s]);
        };
        if (lane == 0) {
            for (; issued < nchunks && issued < a.nstage; issued++) issue(issued);
            st_release(&ctrl[1], issued);
        }
        T *f = reinterpret_cast<T *>(a.f);
        int32_t ready = 0, cache_base = 0;
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
            for (int32_t e = lo + lane; e < hi; e += 32) {
                const int off = e & (ch - 1);
                const unsigned char *st = stage_of(e >> a.lg_ch);
                const uint16_t *row = reinterpret_cast<const uint16_t *>(st) + (size_t)off * a.kp;
                const T sn = slot_sum<T, NN>(ring, row);
                const T gx = reinterpret_cast<const T *>(st + dbytes)[off];
                const int32_t u = reinterpret_cast<const int32_t *>(st + dbytes + gbytes)[off];
                const unsigned pn = row[NN + FE];
                const int si = e & a.sbuf_mask;
                while (ld_acquire(&stag[si]) != e) {
                }
                const T Fx = gx - sbuf[si] - sn;
                f[(size_t)u * a.B + b] = Fx - ring[pn];
                ring[e & a.ring_mask] = Fx;
            }
            __syncwarp();
            if (lane == 0) {
                st_release(&ctrl[0], hi);
                bool more = false;
                while (issued < nchunks && ((int64_t)(issued - a.nstage + 1) << a.lg_ch) <= hi) {
                    issue(issued);
                    issued++;
                    more = true;
                }
                if (more) st_release(&ctrl[1], issued);
            }
        }
    } else {
        // ------------------------------------------------- old warps ------
        const int ot = tid - 32;
        const int sub = ot & (LPEO - 1), og = ot / LPEO;
        constexpr int NGO = 32 * NWO / LPEO;
        const unsigned gmask = LPEO == 32 ? 0xffffffffu : (((1u << LPEO) - 1u) << (lane & ~(LPEO - 1)));
        int32_t ready = 0;
        for (int32_t e = og; e < a.n; e += NGO) {   // uniform within an LPEO group
            const int32_t c = e >> a.lg_ch;
            while (ld_acquire(&ctrl[1]) <= c) {
            }
            for (; ready <= c; ready++)
                mbar_wait(&bars[ready & (a.nstage - 1)], (unsigned)((ready / a.nstage) & 1));
            const int off = e & (ch - 1);
            const uint16_t *row = reinterpret_cast<const uint16_t *>(stage_of(c)) + (size_t)off * a.kp;
            const int32_t thr = (int32_t)((unsigned)row[NN + FE + 1] | ((unsigned)row[NN + FE + 2] << 16));
            const int32_t need = max(thr, e - SBUF + 1);
            while (ld_acquire(&ctrl[0]) < need) {
            }
            T s = slot_sum<T, EO>(ring, row + NN + sub * EO);
#pragma unroll
            for (int o = LPEO / 2; o; o >>= 1) s += __shfl_xor_sync(gmask, s, o);
            if (sub == 0) {
                const int si = e & a.sbuf_mask;
                sbuf[si] = s;
                st_release(&stag[si], e);
            }
        }
    }
}

// ------------------------------------------------------------- host -------
static constexpr size_t kSmemCapWS = 227 * 1024;

size_t ringws_smem_bytes(int ring, int sbuf, int kp, int ch, int nstage) {
    return (size_t)(ring + 2) * 8 + (size_t)sbuf * 12 + 16 + 8 * ((nstage + 1) & ~1) +
           (size_t)nstage * ch * ((size_t)kp * 2 + 8 + 4);
}

void ringws_plan(int32_t n, int32_t k, int32_t max_level_width, unsigned reach,
                 const unsigned near_max[3], RingWSPlan &R) {
    R.ok = false;
    if (n <= 0 || k > 256) return;
    // LD: the most levels of slack whose near entries still fit NN = 8 (or
    // 16 at LD = 1)
    int ld = 0, nn = 8;
    for (int t = 3; t >= 1 && !ld; t--)
        if (near_max[t - 1] <= 8) ld = t;
    if (!ld && near_max[0] <= 16) { ld = 1; nn = 16; }
    if (!ld) return;
    const int fe = k <= 64 ? 64 : k <= 128 ? 128 : 256;
    int32_t kp = nn + fe + 8;
    if ((kp / 8) % 2 == 0) kp += 8;
    const int64_t ahead = (int64_t)(ld + 3) * max_level_width;   // old warps' lead, in ranks
    int64_t ring = 32;
    while (ring < (int64_t)reach + ahead + 1) ring <<= 1;
    if (ring > (1 << 15)) return;
    int64_t sbuf = 64;
    while (sbuf < ahead + 32) sbuf <<= 1;
    for (int nstage : {4, 2}) {
        for (int ch : {256, 128, 64, 32}) {
            if ((int64_t)(nstage - 1) * ch < ahead + max_level_width) break;
            if (ringws_smem_bytes((int)ring, (int)sbuf, kp, ch, nstage) <= kSmemCapWS) {
                R.ok = true;
                R.ld = ld;
                R.nn = nn;
                R.fe = fe;
                R.kp = kp;
                R.ring = (int32_t)ring;
                R.sbuf = (int32_t)sbuf;
                R.ch = ch;
                R.nstage = nstage;
                R.npad = ((int64_t)n + ch - 1) / ch * ch;
                // 16 far entries per lane, 4 old warps: the best of the
                // (nwo, lpeo) sweep on C5w (profiles/r1_ring_notes.md)
                R.lpeo = std::min(32, std::max(4, fe / 16));
                R.nwo = 4;
                return;
            }
        }
    }
}

cudaError_t launch_near_max(const DevPoset &P, const int32_t *level, const int32_t *slot_rank,
                            unsigned *out3, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(out3, 0, 3 * sizeof(unsigned), s);
    if (e != cudaSuccess || P.n == 0) return e;
    k_near_max<<<(P.n + 255) / 256, 256, 0, s>>>(P.M, P.n, P.k, P.chain, level, slot_rank, out3);
    launches_add(1);
    return cudaGetLastError();
}

cudaError_t launch_build_ringws(const DevPoset &P, const RingWSPlan &R, const int32_t *level,
                                const int32_t *slot_rank, cudaStream_t s) {
    if (P.n == 0) return cudaSuccess;
    const size_t smem = (size_t)64 * (P.k + 1) * 2 + (size_t)32 * R.kp * 2;
    cudaError_t e = cudaFuncSetAttribute(k_build_ringws, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    k_build_ringws<<<(unsigned)(R.npad / 32), 256, smem, s>>>(P.M, P.n, P.k, R.kp, R.nn, R.fe, R.ld,
                                                              R.ring, P.chain, P.slot, slot_rank,
                                                              level, P.lvl_ptr, R.D);
    launches_add(1);
    return cudaGetLastError();
}

cudaError_t launch_moebius_ringws(const DevPoset &P, const RingWSPlan &R, const int32_t *ru_pad,
                                  int dtype, const void *gP, void *f, int64_t B, cudaStream_t s) {
    if (P.n == 0) return cudaSuccess;
    RWArgs a;
    a.D = R.D;
    a.gP = gP;
    a.ru = ru_pad;
    a.lvl_ptr = P.lvl_ptr;
    a.f = f;
    a.npad = R.npad;
    a.n = P.n;
    a.kp = R.kp;
    a.ell = P.ell;
    a.B = (int32_t)B;
    a.ring_mask = R.ring - 1;
    a.sbuf_mask = R.sbuf - 1;
    a.lg_ch = 0;
    while ((1 << a.lg_ch) < R.ch) a.lg_ch++;
    a.nstage = R.nstage;
    const size_t smem = ringws_smem_bytes(R.ring, R.sbuf, R.kp, R.ch, R.nstage);
    void *fn = nullptr;
    const int E = R.fe / R.lpeo;
#define RWS_FN(NN, L, EE, W)                                                                    \
    if (R.nn == NN && R.lpeo == L && E == EE && R.nwo == W)                                     \
        fn = dtype == 0 ? (void *)k_moeb_ringws<u64, NN, L, EE, W>                              \
                        : (void *)k_moeb_ringws<double, NN, L, EE, W>;
#define RWS_NN(NN, W) RWS_FN(NN, 8, 8, W) RWS_FN(NN, 4, 16, W) RWS_FN(NN, 16, 8, W) RWS_FN(NN, 8, 16, W) \
    RWS_FN(NN, 32, 8, W) RWS_FN(NN, 16, 16, W)
    RWS_NN(8, 4) RWS_NN(8, 8) RWS_NN(8, 12) RWS_NN(16, 4) RWS_NN(16, 8) RWS_NN(16, 12)
#undef RWS_NN
#undef RWS_FN
    if (!fn) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    void *args[] = {&a};
    launches_add(1);
    return cudaLaunchKernel(fn, dim3((unsigned)B), dim3(32 * (1 + R.nwo)), args, smem, s);
}

}  // namespace poset
