// Kernel (v), schedule RINGDF: barrier-free level pipeline for the Möbius
// solve of bounded-reach posets (C5w) -- NEXT row N2, DESIGN.md §5.4.
//
// Alg. 4: F(x) = g(x) - Σ_{j ≠ id(x)} F(niv_j(x)),
// f(x) = F(x) - F(next(x)), swept over the antichain levels (Alg. 6,
// P:L709-733; Alg. 5 P:L692-705 puts a barrier between levels).
//
// Here there is no barrier.  One CTA per column; consumer warp w owns the
// levels L ≡ w (mod NWC), one lane per element.  Level completion is
// published on a small ring of mbarriers (arrive.release by the owner warp's
// lanes, try_wait.parity by later owners; levels finish in order) instead of
// a CTA barrier.  The dependencies of an element of level L are
// split by their own level when the tables are built:
//   far   level <= L - 7   summed once levels_done >= L - 6
//   mid   level in [L-6, L-3]   summed once levels_done >= L - 2
//   near  level >= L - 2   (at most NN) summed once levels_done >= L
// so while the other warps finish levels L-6 .. L-1, warp w has already done
// almost all of its work for level L; what remains on the critical path of a
// level is one poll of levels_done, <= NN shared-memory loads, a few adds, the
// ring store and the release of levels_done.  The ring of F values, the
// TMA-staged rows (producer warp) and the sizes follow RING; the plan makes
// RING >= reach + 12 * max level width so no slot is overwritten while any
// warp may still read it.
//
//   rows [npad][kp] uint16 ring slots (RING = the zero entry):
//     [0, NN) near | [NN, NN+NM) mid | [NN+NM, NN+NM+FE) far (bank-sorted) | pn
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "kernels.cuh"
#include "ptx.cuh"

namespace poset {

typedef unsigned long long u64;

static constexpr int kNear = 2;    // level distance <= kNear: near
static constexpr int kMid = 6;     // kNear < distance <= kMid: mid; beyond: far
static constexpr int kLB = 16;     // level-completion mbarriers (ring), > kMid + 1
static constexpr int kNP = 3;      // passes of 32 elements kept in registers per level

// ------------------------------------------------------------ setup -------
// max over ranks of (#deps at level distance <= kNear, #deps in (kNear, kMid])
__global__ void k_df_counts(const int32_t *__restrict__ M, int32_t n, int32_t k,
                            const int32_t *__restrict__ chain, const int32_t *__restrict__ level,
                            const int32_t *__restrict__ slot_rank, unsigned *out2) {
    const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned cn = 0, cm = 0;
    if (r < n) {
        const int32_t own = chain[r], lr = level[r];
        for (int32_t j = 0; j < k; j++) {
            const int32_t s = __ldcs(M + (size_t)j * n + r);
            if (j == own || s == n) continue;
            const int32_t ld = lr - level[slot_rank[s]];
            cn += ld <= kNear;
            cm += ld > kNear && ld <= kMid;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        cn = max(cn, __shfl_xor_sync(0xffffffffu, cn, o));
        cm = max(cm, __shfl_xor_sync(0xffffffffu, cm, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(out2, cn);
        atomicMax(out2 + 1, cm);
    }
}

__global__ void __launch_bounds__(256) k_build_ringdf(
    const int32_t *__restrict__ M, int32_t n, int32_t k, int32_t kp, int32_t nn, int32_t nm,
    int32_t fe, int32_t ring, const int32_t *__restrict__ chain, const int32_t *__restrict__ slot,
    const int32_t *__restrict__ slot_rank, const int32_t *__restrict__ level,
    uint16_t *__restrict__ D) {
    extern __shared__ uint16_t tile[];   // raw [32][k+1] slots, class [32][k+1], out [32][kp]
    const int ks = k + 1;
    uint16_t *raw = tile, *cls = tile + 32 * ks, *outr = tile + 64 * ks;
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
        raw[lane * ks + j] = (uint16_t)(dep >= 0 ? (dep & mask) : ring);   // slot; bytes on output
        int c = 3;   // 0 near, 1 mid, 2 far, 3 none
        if (dep >= 0) {
            const int32_t ld = level[r] - level[dep];
            c = ld <= kNear ? 0 : ld <= kMid ? 1 : 2;
        }
        cls[lane * ks + j] = (uint16_t)c;
    }
    __syncthreads();
    if (w == 0) {
        const uint16_t *in = raw + lane * ks, *cl = cls + lane * ks;
        uint16_t *out = outr + lane * kp;
        int nnear = 0, nmid = 0, cnt[16], pos[16], acc = 0;
#pragma unroll
        for (int c = 0; c < 16; c++) cnt[c] = 0;
        for (int j = 0; j < k; j++) {
            const int s = in[j];
            if (cl[j] == 0) { if (nnear < nn) out[nnear] = (uint16_t)s; nnear++; }
            else if (cl[j] == 1) { if (nmid < nm) out[nn + nmid] = (uint16_t)s; nmid++; }
            else if (cl[j] == 2) cnt[(s - r) & 15]++;
        }
        for (int j = nnear; j < nn; j++) out[j] = (uint16_t)ring;
        for (int j = nmid; j < nm; j++) out[nn + j] = (uint16_t)ring;
#pragma unroll
        for (int c = 0; c < 16; c++) { pos[c] = acc; acc += cnt[c]; }
        for (int j = 0; j < k; j++) {
            if (cl[j] != 2) continue;
            const int s = in[j];
            const int c = (s - r) & 15;
#pragma unroll
            for (int cc = 0; cc < 16; cc++)
                if (cc == c) out[nn + nm + pos[cc]++] = (uint16_t)s;
        }
        for (int j = nn + nm + acc; j < kp; j++) out[j] = (uint16_t)ring;
        int pn = -1;
        if (r < n) {
            const int32_t s = slot[r];
            if (s > 0) {
                const int32_t p = slot_rank[s - 1];
                if (chain[p] == chain[r]) pn = p;
            }
        }
        out[nn + nm + fe] = (uint16_t)(pn >= 0 ? (pn & mask) : ring);
        out[nn + nm + fe + 1] = (uint16_t)(min(nnear, nn) | (min(nmid, nm) << 8));
    }
    __syncthreads();
    // ring slots -> byte offsets into the ring (slot * 8; RING * 8 < 65536 by
    // the plan), except the counts word
    const int64_t base = (int64_t)r0 * kp;
    for (int t = threadIdx.x; t < 32 * kp; t += blockDim.x) {
        const int j = t % kp;
        const uint16_t v = outr[t];
        D[base + t] = j == nn + nm + fe + 1 ? v : (uint16_t)(v * 8);
    }
}

// ------------------------------------------------------------ kernel ------
struct RDFArgs {
    const uint16_t *D;          // [npad][kp]
    const void *gP;             // [B][npad]
    const int32_t *ru;          // [npad]
    const int32_t *lvl_ptr;     // [ell + 1]
    void *f;                    // [n][B]
    int64_t npad;
    int32_t n, kp, ell, B;
    int32_t ring_mask;
    int32_t lg_ch, nstage;
    int32_t sbuf;               // RINGFR: S_old buffer entries (power of two)
    int32_t skip_far;           // timing experiment only (results invalid): bit 0 far, bit 1 mid,
                                // bit 2 near sums skipped
    unsigned long long *dbg;    // PROF instantiation only: [0] Σ ready->publish, [1] Σ publish->ready
                                // (owner already waiting), [2] Σ lateness, [3] late levels, [4] levels
};

__device__ __forceinline__ uint4 df_lds128(unsigned addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ u64 df_lds64(unsigned addr) {
    u64 v;
    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ unsigned lds32u(unsigned addr) {
    unsigned v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ int df_acq(unsigned addr) {
    int v;
    asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void df_rel(unsigned addr, int v) {
    asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// Σ ring[slot] over E consecutive row words at shared address `row`
template <typename T, int E>
__device__ __forceinline__ T df_sum(unsigned ring_base, unsigned row) {
    static_assert(E == 8 || E % 16 == 0, "row segments are 8 or a multiple of 16 entries");
    T acc = T(0);
    if constexpr (E == 8) {
        const uint4 w0 = df_lds128(row);
        const unsigned ws[4] = {w0.x, w0.y, w0.z, w0.w};
        T v[8];
#pragma unroll
        for (int h = 0; h < 4; h++) {
            v[2 * h] = bits_to<T>(df_lds64(ring_base + (ws[h] & 0xffffu)));
            v[2 * h + 1] = bits_to<T>(df_lds64(ring_base + (ws[h] >> 16)));
        }
        return ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
    }
#pragma unroll
    for (int c = 0; c < E; c += 16) {
        const uint4 w0 = df_lds128(row + 2 * c), w1 = df_lds128(row + 2 * c + 16);
        const unsigned ws[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
        T v[16];
#pragma unroll
        for (int h = 0; h < 8; h++) {
            v[2 * h] = bits_to<T>(df_lds64(ring_base + (ws[h] & 0xffffu)));
            v[2 * h + 1] = bits_to<T>(df_lds64(ring_base + (ws[h] >> 16)));
        }
#pragma unroll
        for (int st = 1; st < 16; st <<= 1)
#pragma unroll
            for (int i = 0; i < 16; i += 2 * st) v[i] += v[i + st];
        acc += v[0];
    }
    return acc;
}
// Σ ring[slot] for E slots already in registers (two per 32-bit word)
template <typename T, int E>
__device__ __forceinline__ T df_sum_w(unsigned ring_base, const uint4 (&w)[E / 8]) {
    T v[E];
#pragma unroll
    for (int i = 0; i < E / 8; i++) {
        const unsigned ws[4] = {w[i].x, w[i].y, w[i].z, w[i].w};
#pragma unroll
        for (int h = 0; h < 4; h++) {
            v[8 * i + 2 * h] = bits_to<T>(df_lds64(ring_base + (ws[h] & 0xffffu)));
            v[8 * i + 2 * h + 1] = bits_to<T>(df_lds64(ring_base + (ws[h] >> 16)));
        }
    }
#pragma unroll
    for (int st = 1; st < E; st <<= 1)
#pragma unroll
        for (int i = 0; i < E; i += 2 * st) v[i] += v[i + st];
    return v[0];
}
// Σ ring[slot] over the first `cnt` of E slots in registers (the rest are
// padding; their loads are predicated off so they cost no wavefronts)
template <typename T, int E>
__device__ __forceinline__ T df_sum_wc(unsigned ring_base, const uint4 (&w)[E / 8], int cnt) {
    T v[E];
#pragma unroll
    for (int i = 0; i < E / 8; i++) {
        const unsigned ws[4] = {w[i].x, w[i].y, w[i].z, w[i].w};
#pragma unroll
        for (int h = 0; h < 4; h++) {
            const int j0 = 8 * i + 2 * h;
            v[j0] = j0 < cnt ? bits_to<T>(df_lds64(ring_base + (ws[h] & 0xffffu))) : T(0);
            v[j0 + 1] = j0 + 1 < cnt ? bits_to<T>(df_lds64(ring_base + (ws[h] >> 16))) : T(0);
        }
    }
#pragma unroll
    for (int st = 1; st < E; st <<= 1)
#pragma unroll
        for (int i = 0; i < E; i += 2 * st) v[i] += v[i + st];
    return v[0];
}
template <typename T>
__device__ __forceinline__ u64 df_bits(T x);
template <>
__device__ __forceinline__ u64 df_bits<u64>(u64 x) { return x; }
template <>
__device__ __forceinline__ u64 df_bits<double>(double x) { return (u64)__double_as_longlong(x); }

template <typename T, int NN, int NM, int FE, int kNWC, bool PROF = false>
__global__ void __launch_bounds__(32 * (kNWC + 1)) k_moeb_ringdf(RDFArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int RING = a.ring_mask + 1;
    const int ch = 1 << a.lg_ch;
    const unsigned ring_base = smem_u32(smem);                            // RING + 2 entries
    u64 *bars = reinterpret_cast<u64 *>(smem + (size_t)(RING + 2) * 8);
    const unsigned ctrl = smem_u32(bars + ((a.nstage + kLB + 1) & ~1));   // ready, done_rank
    unsigned char *stage0 = smem + (size_t)(RING + 2) * 8 + 8 * ((a.nstage + kLB + 1) & ~1) + 16;
    const unsigned stage_base = smem_u32(stage0);
    const unsigned dbytes = (unsigned)ch * a.kp * 2, gbytes = (unsigned)ch * 8, ubytes = (unsigned)ch * 4;
    const unsigned sbytes = dbytes + gbytes + ubytes;
    const int b = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const T *gcol = reinterpret_cast<const T *>(a.gP) + (size_t)b * a.npad;
    const int32_t nchunks = (int32_t)(a.npad >> a.lg_ch);

    if (tid == 0) {
        asm volatile("st.shared.b64 [%0], %1;" ::"r"(ring_base + (unsigned)RING * 8), "l"(0ull) : "memory");
        for (int s = 0; s < a.nstage; s++) mbar_init(&bars[s], 1);
        for (int s = 0; s < kLB; s++) mbar_init(&bars[a.nstage + s], 1);
        asm volatile("st.shared.s32 [%0], 0;\n\tst.shared.s32 [%0+4], 0;\n\tst.shared.s32 [%0+8], 0;" ::"r"(ctrl)
                     : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const unsigned ns = (unsigned)a.nstage;   // any stage count 2..8 (not only powers of two)

    if (warp == kNWC) {
        // ------------------------------------------------------ producer --
        if (lane == 0) {
            auto issue = [&](int32_t c) {
                const int s = (int)((unsigned)c % ns);
                unsigned char *st = stage0 + (size_t)s * sbytes;
                const size_t r0 = (size_t)c << a.lg_ch;
                mbar_expect_tx(&bars[s], sbytes);
                bulk_g2s(st, a.D + r0 * a.kp, dbytes, &bars[s]);
                bulk_g2s(st + dbytes, gcol + r0, gbytes, &bars[s]);
                bulk_g2s(st + dbytes + gbytes, a.ru + r0, ubytes, &bars[s]);
            };
            int32_t issued = 0, arrived = 0;
            for (; issued < nchunks && issued < a.nstage; issued++) issue(issued);
            while (arrived < nchunks) {
                mbar_wait(&bars[(unsigned)arrived % ns], ((unsigned)arrived / ns) & 1u);
                arrived++;
                df_rel(ctrl, arrived << a.lg_ch);
                while (issued < nchunks) {
                    const int32_t done = df_acq(ctrl + 4);
                    if (((int64_t)(issued - a.nstage + 1) << a.lg_ch) > done) {
                        if (arrived < issued) break;
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

    // ------------------------------------------------------- consumers ----
    // Level completion is published on a ring of kLB mbarriers: the 32 lanes
    // of the warp that owns level L arrive (release) on lvlbar[L % kLB] once
    // their ring stores are issued; a waiter for "level L done" try_waits
    // (acquire) on the phase (L / kLB) & 1.  Levels finish in order, so "L
    // done" means every level <= L is done, and no waiter ever looks more
    // than kMid + 1 < kLB levels back, so parities cannot alias.
    T *f = reinterpret_cast<T *>(a.f);
    u64 *lvlbar = bars + a.nstage;   // kLB barriers after the stage barriers
    __shared__ unsigned long long prof[8];
    __shared__ volatile unsigned long long prof_last;
    long long t_ready = 0;
    if (PROF && tid == 0) { for (int i = 0; i < 8; i++) prof[i] = 0; prof_last = clock64(); }
    if (PROF) asm volatile("bar.sync 1, %0;" ::"r"(32 * kNWC));
    auto wait_level = [&](int32_t Ld) {   // level Ld (and all below) done
        if (Ld < 0) return;
        mbar_wait(&lvlbar[Ld & (kLB - 1)], (unsigned)((Ld / kLB) & 1));
    };
    int32_t cb = 0;
    auto ld_bounds = [&](int32_t i0, int32_t &vlo, int32_t &vhi) {
        const int32_t L = warp + (i0 + lane) * kNWC;
        vlo = a.lvl_ptr[min(L, a.ell)];
        vhi = a.lvl_ptr[min(L + 1, a.ell)];
    };
    int32_t clo, chi;
    ld_bounds(0, clo, chi);
    int32_t staged = 0;
    for (int32_t i = 0;; i++) {
        const int32_t L = warp + i * kNWC;
        if (L >= a.ell) break;
        if (i - cb == 32) {
            cb += 32;
            ld_bounds(cb, clo, chi);
        }
        const int32_t lo = __shfl_sync(0xffffffffu, clo, i - cb);
        const int32_t hi = __shfl_sync(0xffffffffu, chi, i - cb);
        const int32_t npass = (hi - lo + 31) >> 5;
        const int32_t np = min(npass, kNP);
        while (staged < hi) staged = df_acq(ctrl);
        // per pass: row-derived data in registers (passes beyond kNP: serial below)
        T gx[kNP], sp[kNP];
        int32_t u[kNP];
        unsigned rowa[kNP], pn[kNP], cnt[kNP];
        uint4 nw[kNP][NN / 8];
#pragma unroll
        for (int p = 0; p < kNP; p++) {
            if (p < np) {
                const int32_t e = lo + 32 * p + lane;
                const int32_t ee = e < hi ? e : lo + 32 * p;
                const unsigned st = stage_base + ((unsigned)(ee >> a.lg_ch) % ns) * sbytes;
                const unsigned off = (unsigned)(ee & (ch - 1));
                rowa[p] = st + off * (unsigned)a.kp * 2;
                gx[p] = bits_to<T>(df_lds64(st + dbytes + off * 8));
                asm volatile("ld.shared.b32 %0, [%1];" : "=r"(u[p]) : "r"(st + dbytes + gbytes + off * 4));
                unsigned pc;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(pc) : "r"(rowa[p] + 2 * (NN + NM + FE)));
                pn[p] = pc & 0xffffu;
                cnt[p] = pc >> 16;   // near count | mid count << 8
#pragma unroll
                for (int q = 0; q < NN / 8; q++) nw[p][q] = df_lds128(rowa[p] + 16 * q);
                u[p] = e < hi ? u[p] : -1;
            }
        }
        wait_level(L - kMid - 1);   // far: levels <= L-7
#pragma unroll
        for (int p = 0; p < kNP; p++)
            if (p < np) sp[p] = (a.skip_far & 1) ? T(0) : df_sum<T, FE>(ring_base, rowa[p] + 2 * (NN + NM));
        wait_level(L - kNear - 1);  // mid: levels <= L-3
#pragma unroll
        for (int p = 0; p < kNP; p++) {
            if (p < np) {
                uint4 mw[NM / 8];
#pragma unroll
                for (int q = 0; q < NM / 8; q++) mw[q] = df_lds128(rowa[p] + 2 * NN + 16 * q);
                if (!(a.skip_far & 2)) sp[p] += df_sum_wc<T, NM>(ring_base, mw, (int)(cnt[p] >> 8));
            }
        }
        long long t_wait = 0;
        if (PROF) t_wait = clock64();
        wait_level(L - 1);          // near: the critical path
        if (PROF) {
            t_ready = clock64();
            if (lane == 0 && b == 0 && L > 0) {
                const long long tp = (long long)prof_last;
                if (t_wait > tp) { prof[2] += t_wait - tp; prof[3] += 1; }
                else prof[1] += t_ready - tp;
            }
        }
        T fo[kNP];
#pragma unroll
        for (int p = 0; p < kNP; p++) {
            if (p < np) {
                const T sn = (a.skip_far & 4) ? T(0) : df_sum_wc<T, NN>(ring_base, nw[p], (int)(cnt[p] & 0xffu));
                if (PROF && p == 0 && lane == 0 && b == 0) {
                    // force the near sum to complete before the stamp
                    asm volatile("" ::"l"(df_bits<T>(sn)));
                    prof[7] += clock64() - t_ready;
                }
                const T Fx = gx[p] - (sp[p] + sn);
                fo[p] = Fx - bits_to<T>(df_lds64(ring_base + pn[p]));
                if (u[p] >= 0)
                    asm volatile("st.shared.b64 [%0], %1;" ::"r"(ring_base + (unsigned)((lo + 32 * p + lane) & a.ring_mask) * 8),
                                 "l"(df_bits<T>(Fx))
                                 : "memory");
            }
        }
        // passes beyond kNP (levels wider than 32 * kNP): serially, all deps done
        for (int32_t base = lo + 32 * kNP; base < hi; base += 32) {
            const int32_t e = base + lane;
            const int32_t ee = e < hi ? e : base;
            const unsigned st = stage_base + ((unsigned)(ee >> a.lg_ch) % ns) * sbytes;
            const unsigned off = (unsigned)(ee & (ch - 1));
            const unsigned row = st + off * (unsigned)a.kp * 2;
            const T g1 = bits_to<T>(df_lds64(st + dbytes + off * 8));
            int32_t u1;
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(u1) : "r"(st + dbytes + gbytes + off * 4));
            unsigned short p16;
            asm volatile("ld.shared.u16 %0, [%1];" : "=h"(p16) : "r"(row + 2 * (NN + NM + FE)));   // pads load zero
            const T Fx = g1 - (df_sum<T, FE>(ring_base, row + 2 * (NN + NM)) + df_sum<T, NM>(ring_base, row + 2 * NN) +
                               df_sum<T, NN>(ring_base, row));
            if (e < hi) {
                asm volatile("st.shared.b64 [%0], %1;" ::"r"(ring_base + (unsigned)(e & a.ring_mask) * 8),
                             "l"(df_bits<T>(Fx))
                             : "memory");
                f[(size_t)u1 * a.B + b] = Fx - bits_to<T>(df_lds64(ring_base + (unsigned)p16));
            }
        }
        long long t_pre = 0;
        if (PROF) t_pre = clock64();
        // publish: __syncwarp orders the lanes' ring stores before lane 0's
        // single release-arrive (one arrival per level: the sync unit
        // processes arrivals one at a time)
        __syncwarp();
        if (lane == 0)
            asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&lvlbar[L & (kLB - 1)]))
                         : "memory");
        if (lane == 0) {
            asm volatile("st.relaxed.cta.shared.s32 [%0], %1;" ::"r"(ctrl + 4), "r"(hi) : "memory");
            if (PROF && b == 0) {
                const long long t = clock64();
                prof[0] += t - t_ready;
                prof[4] += 1;
                prof[5] += t_pre - t_ready;
                prof[6] += np;
                prof_last = (unsigned long long)t;
            }
        }
#pragma unroll
        for (int p = 0; p < kNP; p++)
            if (p < np && u[p] >= 0) f[(size_t)u[p] * a.B + b] = fo[p];
    }
    if (PROF) {
        asm volatile("bar.sync 1, %0;" ::"r"(32 * kNWC));
        if (tid == 0 && b == 0)
            for (int i = 0; i < 8; i++) a.dbg[i] = prof[i];
    }
}

// ---------------------------------------------------------------------------
// Schedule RINGFR ("fresh warp"): the same tables, but the level-by-level
// critical path stays inside ONE warp (hand-off between levels = __syncwarp;
// the near dependencies, levels L-1 and L-2, were written by this warp
// itself), and kNH helper warps compute each element's far + mid sum
// S_old(x) ahead of time: helper h owns levels L ≡ h (mod kNH), sums the far
// part once level L-7 is done and the mid part once level L-3 is done, writes
// S_old into a shared buffer and arrives on sold_bar[L % kLB].  The fresh warp
// publishes level completion on lvl_bar[L % kLB] (arrive.release by its 32
// lanes) for the helpers; it normally finds sold_bar[L] already complete.
template <typename T, int NN, int NM, int FE, int kNH>
__global__ void __launch_bounds__(32 * (kNH + 3)) k_moeb_ringfr(RDFArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int RING = a.ring_mask + 1;
    const int ch = 1 << a.lg_ch;
    const unsigned ring_base = smem_u32(smem);
    u64 *bars = reinterpret_cast<u64 *>(smem + (size_t)(RING + 2) * 8);   // nstage + 2 * kLB
    u64 *lvlbar = bars + a.nstage, *soldbar = lvlbar + kLB;
    const unsigned ctrl = smem_u32(bars + ((a.nstage + 2 * kLB + 1) & ~1));   // ready, done_rank
    T *sold = reinterpret_cast<T *>(smem + (size_t)(RING + 2) * 8 + 8 * ((a.nstage + 2 * kLB + 1) & ~1) + 16);
    const int SB = a.sbuf;   // S_old entries (power of two), indexed by rank
    int *stag = reinterpret_cast<int *>(sold + SB);   // rank whose S_old is in the slot
    // f output buffer (fresh warp -> writer warp): value and user id per rank
    constexpr int FB = 1024;
    T *fbuf = reinterpret_cast<T *>(stag + SB);
    int *fusr = reinterpret_cast<int *>(fbuf + FB);
    unsigned char *stage0 = reinterpret_cast<unsigned char *>(fusr + FB);
    const unsigned stage_base = smem_u32(stage0);
    const unsigned dbytes = (unsigned)ch * a.kp * 2, gbytes = (unsigned)ch * 8, ubytes = (unsigned)ch * 4;
    const unsigned sbytes = dbytes + gbytes + ubytes;
    const int b = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const T *gcol = reinterpret_cast<const T *>(a.gP) + (size_t)b * a.npad;
    const int32_t nchunks = (int32_t)(a.npad >> a.lg_ch);
    const unsigned ns = (unsigned)a.nstage;

    for (int i = tid; i < SB; i += blockDim.x) stag[i] = -1;
    if (tid == 0) {
        asm volatile("st.shared.b64 [%0], %1;" ::"r"(ring_base + (unsigned)RING * 8), "l"(0ull) : "memory");
        for (int s2 = 0; s2 < a.nstage; s2++) mbar_init(&bars[s2], 1);
        for (int s2 = 0; s2 < 2 * kLB; s2++) mbar_init(&lvlbar[s2], 1);
        asm volatile("st.shared.s32 [%0], 0;\n\tst.shared.s32 [%0+4], 0;\n\tst.shared.s32 [%0+8], 0;" ::"r"(ctrl)
                     : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto wait_bar = [&](u64 *bar, int32_t Ld) {   // phase of level Ld complete
        if (Ld < 0) return;
        mbar_wait(&bar[Ld & (kLB - 1)], (unsigned)((Ld / kLB) & 1));
    };
    auto stage_row = [&](int32_t e, unsigned &st, unsigned &off) {
        st = stage_base + ((unsigned)(e >> a.lg_ch) % ns) * sbytes;
        off = (unsigned)(e & (ch - 1));
    };

    if (warp == kNH + 1) {
        // ------------------------------------------------------ producer --
        if (lane == 0) {
            auto issue = [&](int32_t c) {
                const int s2 = (int)((unsigned)c % ns);
                unsigned char *st = stage0 + (size_t)s2 * sbytes;
                const size_t r0 = (size_t)c << a.lg_ch;
                mbar_expect_tx(&bars[s2], sbytes);
                bulk_g2s(st, a.D + r0 * a.kp, dbytes, &bars[s2]);
                bulk_g2s(st + dbytes, gcol + r0, gbytes, &bars[s2]);
                bulk_g2s(st + dbytes + gbytes, a.ru + r0, ubytes, &bars[s2]);
            };
            int32_t issued = 0, arrived = 0;
            for (; issued < nchunks && issued < a.nstage; issued++) issue(issued);
            while (arrived < nchunks) {
                mbar_wait(&bars[(unsigned)arrived % ns], ((unsigned)arrived / ns) & 1u);
                arrived++;
                df_rel(ctrl, arrived << a.lg_ch);
                while (issued < nchunks) {
                    const int32_t done = df_acq(ctrl + 4);
                    if (((int64_t)(issued - a.nstage + 1) << a.lg_ch) > done) {
                        if (arrived < issued) break;
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

    if (warp == kNH + 2) {
        // -------------------------------------------------------- writer --
        // drains fbuf: ranks < done_rank (published with release by the
        // fresh warp) are final; publishes drained (ctrl + 8) for slot reuse
        T *f = reinterpret_cast<T *>(a.f);
        int32_t w = 0;
        while (w < a.n) {
            const int32_t done = df_acq(ctrl + 4);
            if (done <= w) { __nanosleep(32); continue; }
            for (int32_t r = w + lane; r < done; r += 32) {
                const int i = r & (FB - 1);
                f[(size_t)fusr[i] * a.B + b] = fbuf[i];
            }
            __syncwarp();
            w = done;
            if (lane == 0) df_rel(ctrl + 8, w);
        }
        return;
    }

    if (warp >= 1) {
        // ------------------------------------------------------- helpers --
        const int h = warp - 1;
        int32_t staged = 0;
        for (int32_t L = h; L < a.ell; L += kNH) {
            const int32_t lo = a.lvl_ptr[L], hi = a.lvl_ptr[L + 1];
            while (staged < hi) staged = df_acq(ctrl);
            // far deps: levels <= L-7 done.  This also frees the S_old slots
            // this level reuses: SB >= (kMid + 4) * max level width, so the
            // previous occupant of slot e & (SB-1) lies in a level <= L-8.
            wait_bar(lvlbar, L - kMid - 1);
            T sf[4];
            unsigned rows[4];
            const int np = min((hi - lo + 31) >> 5, 4);
#pragma unroll
            for (int p = 0; p < 4; p++) {
                if (p < np) {
                    const int32_t e = lo + 32 * p + lane, ee = e < hi ? e : lo + 32 * p;
                    unsigned st, off;
                    stage_row(ee, st, off);
                    rows[p] = st + off * (unsigned)a.kp * 2;
                    sf[p] = df_sum<T, FE>(ring_base, rows[p] + 2 * (NN + NM));
                }
            }
            wait_bar(lvlbar, L - kNear - 1);
#pragma unroll
            for (int p = 0; p < 4; p++) {
                if (p < np) {
                    const int32_t e = lo + 32 * p + lane;
                    const unsigned cn = (lds32u(rows[p] + 2 * (NN + NM + FE)) >> 16) >> 8;
                    uint4 mw[NM / 8];
#pragma unroll
                    for (int q = 0; q < NM / 8; q++) mw[q] = df_lds128(rows[p] + 2 * NN + 16 * q);
                    const T v = sf[p] + df_sum_wc<T, NM>(ring_base, mw, (int)cn);
                    if (e < hi) {
                        sold[e & (SB - 1)] = v;
                        df_rel(smem_u32(&stag[e & (SB - 1)]), e);   // value, then tag (release)
                    }
                }
            }
            for (int32_t base = lo + 128; base < hi; base += 32) {   // levels wider than 128: serial
                const int32_t e = base + lane, ee = e < hi ? e : base;
                unsigned st, off;
                stage_row(ee, st, off);
                const unsigned row = st + off * (unsigned)a.kp * 2;
                const T v = df_sum<T, FE>(ring_base, row + 2 * (NN + NM)) + df_sum<T, NM>(ring_base, row + 2 * NN);
                if (e < hi) {
                    sold[e & (SB - 1)] = v;
                    df_rel(smem_u32(&stag[e & (SB - 1)]), e);
                }
            }
        }
        return;
    }

    // ---------------------------------------------------------- fresh warp --
    // Level L's first pass uses row data loaded while level L-1's loads were
    // in flight; S_old(x) is taken when its tag shows x (written by a helper
    // with release semantics), so nothing but shared-memory loads, adds, the
    // ring store and __syncwarp sit between two levels.
    T *f = reinterpret_cast<T *>(a.f);
    int32_t staged = 0;
    int32_t cb = 0;
    int32_t clo = a.lvl_ptr[min(lane, a.ell)], cnx = a.lvl_ptr[min(31 + lane, a.ell)];
    auto bounds = [&](int32_t L, int32_t &lo, int32_t &hi) {
        if (L >= a.ell) { lo = hi = a.n; return; }
        if (L - cb >= 31) {
            cb += 31;
            clo = cnx;
            cnx = a.lvl_ptr[min(cb + 31 + lane, a.ell)];
        }
        lo = __shfl_sync(0xffffffffu, clo, L - cb);
        hi = __shfl_sync(0xffffffffu, clo, L - cb + 1);
    };
    struct Row { unsigned pc; uint4 nw[NN / 8]; T g; int32_t u; T so; };
    auto load_row = [&](int32_t e, int32_t hi_, Row &R) {
        const int32_t ee = e < hi_ ? e : hi_ - 1;
        unsigned st, off;
        stage_row(ee, st, off);
        const unsigned row = st + off * (unsigned)a.kp * 2;
        R.pc = lds32u(row + 2 * (NN + NM + FE));
#pragma unroll
        for (int q = 0; q < NN / 8; q++) R.nw[q] = df_lds128(row + 16 * q);
        R.g = bits_to<T>(df_lds64(st + dbytes + off * 8));
        R.u = e < hi_ ? (int32_t)lds32u(st + dbytes + gbytes + off * 4) : -1;
        const unsigned ta = smem_u32(&stag[ee & (SB - 1)]);
        while (df_acq(ta) != ee) {
        }
        R.so = sold[ee & (SB - 1)];
    };
    int32_t lo, hi;
    int32_t drained = 0;
    bounds(0, lo, hi);
    Row R;
    while (staged < hi) staged = df_acq(ctrl);
    load_row(lo + lane, hi, R);
    for (int32_t L = 0; L < a.ell; L++) {
        int32_t nlo, nhi;
        bounds(L + 1, nlo, nhi);
        // level L, first pass: issue the near loads and F(next) ...
        const T sn = df_sum_wc<T, NN>(ring_base, R.nw, (int)(R.pc >> 16) & 0xff);
        const T Fp = bits_to<T>(df_lds64(ring_base + (R.pc & 0xffffu)));
        // ... and prefetch level L+1's first pass while they are in flight
        Row Rn;
        if (L + 1 < a.ell) {
            while (staged < nhi) staged = df_acq(ctrl);
            load_row(nlo + lane, nhi, Rn);
        }
        {
            const T Fx = R.g - (R.so + sn);
            if (R.u >= 0) {
                const int e = lo + lane;
                asm volatile("st.shared.b64 [%0], %1;" ::"r"(ring_base + (unsigned)(e & a.ring_mask) * 8),
                             "l"(df_bits<T>(Fx))
                             : "memory");
                fbuf[e & (FB - 1)] = Fx - Fp;
                fusr[e & (FB - 1)] = R.u;
            }
        }
        for (int32_t base = lo + 32; base < hi; base += 32) {   // further passes of a wide level
            Row Rx;
            load_row(base + lane, hi, Rx);
            const T Fx = Rx.g - (Rx.so + df_sum_wc<T, NN>(ring_base, Rx.nw, (int)(Rx.pc >> 16) & 0xff));
            const T Fq = bits_to<T>(df_lds64(ring_base + (Rx.pc & 0xffffu)));
            if (Rx.u >= 0) {
                const int e = base + lane;
                asm volatile("st.shared.b64 [%0], %1;" ::"r"(ring_base + (unsigned)(e & a.ring_mask) * 8),
                             "l"(df_bits<T>(Fx))
                             : "memory");
                fbuf[e & (FB - 1)] = Fx - Fq;
                fusr[e & (FB - 1)] = Rx.u;
            }
        }
        __syncwarp();
        if (lane == 0) {
            asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&lvlbar[L & (kLB - 1)]))
                         : "memory");
            df_rel(ctrl + 4, hi);   // ranks < hi final (producer, writer)
        }
        R = Rn;
        // fbuf slots of the next level must have been drained
        if (nhi - FB > drained) {
            while ((drained = df_acq(ctrl + 8)) < nhi - FB) {
            }
        }
        lo = nlo;
        hi = nhi;
    }
}

// ------------------------------------------------------------- host -------
static constexpr size_t kSmemCapDF = 227 * 1024;
static constexpr int kNHPlan = 6;
static size_t ringfr_plan_smem(int ring, int sbuf, int kp, int ch, int nstage) {
    return (size_t)(ring + 2) * 8 + 8 * ((nstage + 2 * kLB + 1) & ~1) + 16 + (size_t)sbuf * 12 + 1024 * 12 +
           (size_t)nstage * ch * ((size_t)kp * 2 + 12);
}

static size_t ringdf_smem_bytes(int ring, int kp, int ch, int nstage) {
    return (size_t)(ring + 2) * 8 + 8 * ((nstage + kLB + 1) & ~1) + 16 + (size_t)nstage * ch * ((size_t)kp * 2 + 12);
}

void ringdf_plan(int32_t n, int32_t k, int32_t max_level_width, unsigned reach,
                 const unsigned counts2[2], RingDFPlan &R) {
    R.ok = false;
    if (n <= 0 || k > 256 || counts2[0] > 16 || counts2[1] > 32) return;
    R.nn = counts2[0] <= 8 ? 8 : 16;
    R.nm = counts2[1] <= 16 ? 16 : 32;
    R.fe = k <= 64 ? 64 : k <= 128 ? 128 : 256;
    int32_t kp = R.nn + R.nm + R.fe + 8;   // + next slot, counts, padding
    if ((kp / 8) % 2 == 0) kp += 8;
    const int64_t ahead = (int64_t)(8 + kMid + 4) * max_level_width;   // up to 8 consumer warps
    int64_t ring = 32;
    while (ring < (int64_t)reach + ahead + 1) ring <<= 1;
    if (ring > 4096) return;   // rows hold byte offsets: (RING + 1) * 8 must fit in 16 bits
    // the fewest stages of the largest chunk that hold 9 levels and fit
    for (int ch : {256, 128, 64, 32}) {
        for (int nstage = 2; nstage <= 8; nstage++) {
            if ((int64_t)(nstage - 1) * ch < (int64_t)(8 + 1) * max_level_width) continue;
            if (ringdf_smem_bytes((int)ring, kp, ch, nstage) > kSmemCapDF) break;
            {
                R.ok = true;
                R.kp = kp;
                R.ring = (int32_t)ring;
                R.ch = ch;
                R.nstage = nstage;
                R.npad = ((int64_t)n + ch - 1) / ch * ch;
                R.nwc = 8;
                // RINGFR: S_old buffer for the helpers' lead (kNH levels + slack)
                int64_t sb = 64;
                while (sb < (int64_t)(kNHPlan + 4) * max_level_width + 64) sb <<= 1;
                R.sbuf = (int32_t)sb;
                R.fr_ok = ringfr_plan_smem((int)ring, (int)sb, kp, ch, nstage) <= kSmemCapDF;
                return;
            }
        }
    }
}

cudaError_t launch_df_counts(const DevPoset &P, const int32_t *level, const int32_t *slot_rank,
                             unsigned *out2, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(out2, 0, 2 * sizeof(unsigned), s);
    if (e != cudaSuccess || P.n == 0) return e;
    k_df_counts<<<(P.n + 255) / 256, 256, 0, s>>>(P.M, P.n, P.k, P.chain, level, slot_rank, out2);
    launches_add(1);
    return cudaGetLastError();
}

cudaError_t launch_build_ringdf(const DevPoset &P, const RingDFPlan &R, const int32_t *level,
                                const int32_t *slot_rank, cudaStream_t s) {
    if (P.n == 0) return cudaSuccess;
    const size_t smem = (size_t)64 * (P.k + 1) * 2 + (size_t)32 * R.kp * 2;
    cudaError_t e = cudaFuncSetAttribute(k_build_ringdf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    k_build_ringdf<<<(unsigned)(R.npad / 32), 256, smem, s>>>(P.M, P.n, P.k, R.kp, R.nn, R.nm, R.fe,
                                                              R.ring, P.chain, P.slot, slot_rank,
                                                              level, R.D);
    launches_add(1);
    return cudaGetLastError();
}

static constexpr int kNH = 6;   // RINGFR helper warps

static size_t ringfr_smem_bytes(int ring, int sbuf, int kp, int ch, int nstage) {
    return (size_t)(ring + 2) * 8 + 8 * ((nstage + 2 * kLB + 1) & ~1) + 16 + (size_t)sbuf * 12 + 1024 * 12 +
           (size_t)nstage * ch * ((size_t)kp * 2 + 12);
}

cudaError_t launch_moebius_ringfr(const DevPoset &P, const RingDFPlan &R, const int32_t *ru_pad,
                                  int dtype, const void *gP, void *f, int64_t B, cudaStream_t s) {
    if (P.n == 0) return cudaSuccess;
    RDFArgs a{};
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
    a.lg_ch = 0;
    while ((1 << a.lg_ch) < R.ch) a.lg_ch++;
    a.nstage = R.nstage;
    a.sbuf = R.sbuf;
    const size_t smem = ringfr_smem_bytes(R.ring, R.sbuf, R.kp, R.ch, R.nstage);
    void *fn = nullptr;
#define RFR_FN(NN, NM, FE)                                                                     \
    if (R.nn == NN && R.nm == NM && R.fe == FE)                                                \
        fn = dtype == 0 ? (void *)k_moeb_ringfr<u64, NN, NM, FE, kNH> : (void *)k_moeb_ringfr<double, NN, NM, FE, kNH>;
    RFR_FN(8, 16, 64) RFR_FN(8, 32, 64) RFR_FN(16, 16, 64) RFR_FN(16, 32, 64)
    RFR_FN(8, 16, 128) RFR_FN(8, 32, 128) RFR_FN(16, 16, 128) RFR_FN(16, 32, 128)
    RFR_FN(8, 16, 256) RFR_FN(8, 32, 256) RFR_FN(16, 16, 256) RFR_FN(16, 32, 256)
#undef RFR_FN
    if (!fn || !R.fr_ok) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    void *args[] = {&a};
    launches_add(1);
    return cudaLaunchKernel(fn, dim3((unsigned)B), dim3(32 * (kNH + 3)), args, smem, s);
}

cudaError_t launch_moebius_ringdf(const DevPoset &P, const RingDFPlan &R, const int32_t *ru_pad,
                                  int dtype, const void *gP, void *f, int64_t B, cudaStream_t s) {
    if (P.n == 0) return cudaSuccess;
    RDFArgs a;
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
    a.lg_ch = 0;
    while ((1 << a.lg_ch) < R.ch) a.lg_ch++;
    a.nstage = R.nstage;
    a.dbg = R.dbg;
    a.skip_far = R.skip_far;
    const size_t smem = ringdf_smem_bytes(R.ring, R.kp, R.ch, R.nstage);
    void *fn = nullptr;
#define RDF_FN(NN, NM, FE, W)                                                                  \
    if (R.nn == NN && R.nm == NM && R.fe == FE && R.nwc == W)                                  \
        fn = R.prof ? (dtype == 0 ? (void *)k_moeb_ringdf<u64, NN, NM, FE, W, true>            \
                                  : (void *)k_moeb_ringdf<double, NN, NM, FE, W, true>)        \
                    : (dtype == 0 ? (void *)k_moeb_ringdf<u64, NN, NM, FE, W>                  \
                                  : (void *)k_moeb_ringdf<double, NN, NM, FE, W>);
#define RDF_W(NN, NM, FE) RDF_FN(NN, NM, FE, 4) RDF_FN(NN, NM, FE, 8)
    RDF_W(8, 16, 64) RDF_W(8, 32, 64) RDF_W(16, 16, 64) RDF_W(16, 32, 64)
    RDF_W(8, 16, 128) RDF_W(8, 32, 128) RDF_W(16, 16, 128) RDF_W(16, 32, 128)
    RDF_W(8, 16, 256) RDF_W(8, 32, 256) RDF_W(16, 16, 256) RDF_W(16, 32, 256)
#undef RDF_W
#undef RDF_FN
    if (!fn) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    void *args[] = {&a};
    launches_add(1);
    return cudaLaunchKernel(fn, dim3((unsigned)B), dim3(32 * (R.nwc + 1)), args, smem, s);
}

}  // namespace poset
