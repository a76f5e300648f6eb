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
//   rows [npad][kp] uint16: see k_build_ringdf (mid | near | pn | counts |
//   far, the far entries bank-coloured per half-warp)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <type_traits>

#include "kernels.cuh"
#include "ptx.cuh"

namespace poset {

typedef unsigned long long u64;

static constexpr int kNear = 2;    // level distance <= kNear: near
static constexpr int kMid = 6;     // kNear < distance <= kMid: mid; beyond: far
static constexpr int kLB = 16;     // level-completion mbarriers (ring), > kMid + 1
static constexpr int kNP = 3;      // passes of 32 elements kept in registers per level
static constexpr int kNWC = 8;     // consumer warps (levels round-robin)
static constexpr int kMaxStageCL = 32;   // RINGCL stage barriers
static constexpr int kNWH = 16;          // RINGCL block: 16 warps (helper: 2 per level group)

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

// Row layout (uint16 entries; all but the counts word are byte offsets into
// the ring, the zero entries RING .. RING+15 padding every segment):
//   [0, NM) mid | [NM, NM+NN) near | pn | counts | pad to 16 B | far (fe)
// counts = nnear | nmid << 5 | nf16 << 11, nf16 = far entries / 16 of the row's
// half-warp group (the kernel loops to the warp maximum).
__host__ __device__ constexpr int df_off_far(int nm, int nn) { return (2 * (nm + nn + 2) + 15) / 16 * 16; }

// Far entries are ORDERED so that a warp's shared-memory loads hit distinct
// banks: within each half-warp group (16 consecutive ranks of a level pass,
// the lanes of one wavefront of 8-byte loads) every position j holds 16
// distinct bank pairs (slot & 15).  This is an edge colouring of the
// lanes x banks bipartite multigraph, done first-fit with 64-bit position
// masks per bank -- except that lanes needing the same slot share a position
// when they can (one address = a broadcast, no conflict; far dependencies of
// one level's elements overlap heavily).  Free (lane, position) cells take
// the zero entry of a bank nobody uses there.  WRITE = false only measures
// the longest group (-> fe).
template <bool WRITE>
__global__ void __launch_bounds__(256) k_build_ringdf(
    const int32_t *__restrict__ M, int32_t n, int32_t k, const int32_t *__restrict__ lvl_ptr,
    int32_t kpn, int32_t kpf, int32_t nn, int32_t nm, int32_t fe, int32_t ring,
    const int32_t *__restrict__ chain, const int32_t *__restrict__ slot,
    const int32_t *__restrict__ slot_rank, const int32_t *__restrict__ level,
    uint16_t *__restrict__ Dn, uint16_t *__restrict__ Df, unsigned *__restrict__ jmax) {
    const int kp = kpn + kpf;   // tile rows: near table row | far table row
    extern __shared__ __align__(16) unsigned char dsm[];
    const int ks = k + 1;
    unsigned long long *posmask = reinterpret_cast<unsigned long long *>(dsm);   // [2][16][4]
    unsigned long long *taken = posmask + 2 * 16 * 4;                              // [32][4]
    uint16_t *raw = reinterpret_cast<uint16_t *>(taken + 32 * 4);                  // [32][ks] slots
    uint16_t *cls = raw + 32 * ks;                                                 // [32][ks] classes
    uint16_t *outr = cls + 32 * ks;                                                // [32][kp]
    uint16_t *slotpos = outr + 32 * kp;   // [2][4096]: position + 1 of a slot already placed
    for (int t = threadIdx.x; t < 2 * 4096; t += blockDim.x) slotpos[t] = 0;
    __shared__ int jh[2];
    const int L = blockIdx.x;
    const int lo = lvl_ptr[L], hi = lvl_ptr[L + 1];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int mask = ring - 1;
    const int ofar = kpn;
    for (int r0 = lo; r0 < hi; r0 += 32) {
        const int nr = min(32, hi - r0);
        const int r = r0 + lane;
        for (int j = w; j < k; j += nw) {
            int dep = -1;
            if (lane < nr) {
                const int32_t s = M[(size_t)j * n + r];
                if (s != n && chain[r] != j) dep = slot_rank[s];
            }
            raw[lane * ks + j] = (uint16_t)(dep >= 0 ? (dep & mask) : 0);
            int c = 3;   // 0 near, 1 mid, 2 far, 3 none
            if (dep >= 0) {
                const int32_t ld = level[r] - level[dep];
                c = ld <= kNear ? 0 : ld <= kMid ? 1 : 2;
            }
            cls[lane * ks + j] = (uint16_t)c;
        }
        __syncthreads();
        if (w == 1 && (lane & 15) == 0) {
            // first-fit colouring of half-warp group h (ranks r0+16h ..)
            const int h = lane >> 4, nh = min(16, nr - 16 * h);
            unsigned long long *pm = posmask + h * 64;
            uint16_t *sp = slotpos + h * 4096;
            for (int t = 0; t < 64; t++) pm[t] = 0ull;
            int J = 0;
            for (int i = 0; i < nh; i++) {
                const int ln = 16 * h + i;
                unsigned long long tk[4] = {0ull, 0ull, 0ull, 0ull};
                for (int j = 0; j < k; j++) {
                    if (cls[ln * ks + j] != 2) continue;
                    const int s = raw[ln * ks + j], b = s & 15;
                    int pos = (int)sp[s] - 1;
                    if (pos < 0 || ((tk[pos >> 6] >> (pos & 63)) & 1ull)) {
                        pos = 256;
#pragma unroll
                        for (int q = 0; q < 4; q++) {
                            const unsigned long long fr = ~(pm[b * 4 + q] | tk[q]);
                            if (pos == 256 && fr) pos = 64 * q + __ffsll((long long)fr) - 1;
                        }
                        if (pos >= 256) { J = 1 << 20; continue; }   // cannot happen for k <= 256
                        pm[b * 4 + (pos >> 6)] |= 1ull << (pos & 63);
                        if (!sp[s]) sp[s] = (uint16_t)(pos + 1);
                    }
                    tk[pos >> 6] |= 1ull << (pos & 63);
                    if (WRITE && pos < fe) outr[ln * kp + ofar + pos] = (uint16_t)s;
                    J = max(J, pos + 1);
                }
#pragma unroll
                for (int q = 0; q < 4; q++) taken[ln * 4 + q] = tk[q];
            }
            if (!WRITE) {
                atomicMax(jmax, (unsigned)J);
            } else {
                // free cells: the zero entry of a bank not used at that
                // position (one address for all of them: a broadcast)
                for (int pos = 0; pos < fe; pos++) {
                    unsigned used = 0;
                    for (int b = 0; b < 16; b++) used |= (unsigned)((pm[b * 4 + (pos >> 6)] >> (pos & 63)) & 1ull) << b;
                    const int t = used == 0xffffu ? 0 : __ffs(~used & 0xffffu) - 1;
                    for (int i = 0; i < nh; i++) {
                        const int ln = 16 * h + i;
                        if ((taken[ln * 4 + (pos >> 6)] >> (pos & 63)) & 1ull) continue;
                        outr[ln * kp + ofar + pos] = (uint16_t)(ring + t);
                    }
                }
                jh[h] = (J + 15) / 16;
            }
            for (int i = 0; i < nh; i++)   // clear the slot map for the next pass
                for (int j = 0; j < k; j++)
                    if (cls[(16 * h + i) * ks + j] == 2) sp[raw[(16 * h + i) * ks + j]] = 0;
        }
        if (WRITE && w == 0 && lane < nr) {
            const uint16_t *in = raw + lane * ks, *cl = cls + lane * ks;
            uint16_t *out = outr + lane * kp;
            int nnear = 0, nmid = 0;
            for (int j = 0; j < k; j++) {
                const int s = in[j];
                if (cl[j] == 0) { if (nnear < nn) out[nm + nnear] = (uint16_t)s; nnear++; }
                else if (cl[j] == 1) { if (nmid < nm) out[nmid] = (uint16_t)s; nmid++; }
            }
            for (int j = nnear; j < nn; j++) out[nm + j] = (uint16_t)ring;
            for (int j = nmid; j < nm; j++) out[j] = (uint16_t)ring;
            for (int j = nm + nn + 2; j < ofar; j++) out[j] = (uint16_t)ring;
            for (int j = ofar + fe; j < kp; j++) out[j] = (uint16_t)ring;
            int pn = -1;
            const int32_t s = slot[r];
            if (s > 0) {
                const int32_t p = slot_rank[s - 1];
                if (chain[p] == chain[r]) pn = p;
            }
            out[nm + nn] = (uint16_t)(pn >= 0 ? (pn & mask) : ring);
        }
        __syncthreads();
        if (WRITE) {
            if (w == 0 && lane < nr) {
                int nnear = 0, nmid = 0;
                for (int j = 0; j < k; j++) { nnear += cls[lane * ks + j] == 0; nmid += cls[lane * ks + j] == 1; }
                outr[lane * kp + nm + nn + 1] =
                    (uint16_t)(min(nnear, nn) | (min(nmid, nm) << 5) | (jh[lane >> 4] << 11));
                outr[lane * kp + ofar + fe] = (uint16_t)jh[lane >> 4];   // far chunks, in the far table
            }
            __syncthreads();
            // ring slots -> byte offsets (slot * 8; (RING + 16) * 8 <= 65536 by
            // the plan), except the two count words
            for (int t = threadIdx.x; t < nr * kp; t += blockDim.x) {
                const int j = t % kp, rr = r0 + t / kp;
                const uint16_t v = outr[t];
                const uint16_t o = (j == nm + nn + 1 || j == ofar + fe) ? v : (uint16_t)(v * 8);
                if (j < kpn) Dn[(int64_t)rr * kpn + j] = o;
                else Df[(int64_t)rr * kpf + (j - kpn)] = o;
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------ kernel ------
struct RDFArgs {
    const uint16_t *Dn;         // [npad][kpn] mid | near | pn | counts
    const uint16_t *Df;         // [npad][kpf] far (bank-coloured) | far chunks
    const void *gP;             // [B][npad]
    const int32_t *ru;          // [npad]
    const int32_t *lvl_ptr;     // [ell + 1]
    void *f;                    // [n][B]
    int64_t npad;
    int32_t n, kpn, kpf, fe, ell, B;
    int32_t ring_mask;
    int32_t lg_ch, nstage;
    int32_t lg_chh, nstage_h;   // RINGCL helper staging
    int32_t cw_sleep;           // RINGCW level warps: ns between level polls (0: try_wait)
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
// predicated 8-byte shared load (0 when p == 0) / store: no branch
__device__ __forceinline__ u64 df_ldp64(unsigned addr, unsigned p) {
    u64 v;
    asm volatile("{\n.reg .pred q;\nsetp.ne.u32 q, %2, 0;\nmov.b64 %0, 0;\n@q ld.shared.b64 %0, [%1];\n}"
                 : "=l"(v)
                 : "r"(addr), "r"(p)
                 : "memory");
    return v;
}
__device__ __forceinline__ void df_stp64(unsigned addr, u64 v, unsigned p) {
    asm volatile("{\n.reg .pred q;\nsetp.ne.u32 q, %2, 0;\n@q st.shared.b64 [%0], %1;\n}" ::"r"(addr), "l"(v), "r"(p)
                 : "memory");
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
    } else {
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

// value pinned in a register at this point of the program: the compiler may
// not recompute it later (used to keep address / partial-sum arithmetic off
// the post-wait critical path)
__device__ __forceinline__ void df_pin(unsigned &x) { asm volatile("" : "+r"(x)); }
__device__ __forceinline__ void df_pin(u64 &x) { asm volatile("" : "+l"(x)); }
__device__ __forceinline__ void df_pin(double &x) { asm volatile("" : "+d"(x)); }

// NN/2 words of near slots (two 16-bit byte offsets per word)
template <int NN>
__device__ __forceinline__ void df_near_words(unsigned addr, unsigned (&w)[NN / 2]) {
    if constexpr (NN == 4) {
        asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(w[0]), "=r"(w[1]) : "r"(addr));
    } else {
#pragma unroll
        for (int q = 0; q < NN / 8; q++) {
            const uint4 v = df_lds128(addr + 16 * q);
            w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
        }
    }
}
// Σ ring[slot] over E row entries, read one by one (the rare serial passes)
template <typename T, int E>
__device__ __forceinline__ T df_sum_u16(unsigned ring_base, unsigned row) {
    T acc = T(0);
#pragma unroll 4
    for (int j = 0; j < E; j++) {
        unsigned short o;
        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(o) : "r"(row + 2 * j));
        acc += bits_to<T>(df_lds64(ring_base + (unsigned)o));
    }
    return acc;
}

template <typename T, int NN, int NM, bool PROF = false>
__global__ void __launch_bounds__(32 * (kNWC + 1)) k_moeb_ringdf(RDFArgs a) {
    // near-table row (byte offsets): mid | near | pn, counts; the far row is separate
    constexpr unsigned OFF_NEAR = 2 * NM, OFF_PN = 2 * (NM + NN);
    extern __shared__ __align__(16) unsigned char smem[];
    const int RING = a.ring_mask + 1;
    const int ch = 1 << a.lg_ch;
    const unsigned ring_base = smem_u32(smem);                            // RING + 16 entries
    u64 *bars = reinterpret_cast<u64 *>(smem + (size_t)(RING + 16) * 8);
    const unsigned ctrl = smem_u32(bars + ((a.nstage + kLB + 1) & ~1));   // ready, done_rank
    unsigned char *stage0 = smem + (size_t)(RING + 16) * 8 + 8 * ((a.nstage + kLB + 1) & ~1) + 16;
    const unsigned stage_base = smem_u32(stage0);
    // stage: near rows | far rows | g | user ids
    const unsigned nbytes = (unsigned)ch * a.kpn * 2, fbytes = (unsigned)ch * a.kpf * 2;
    const unsigned dbytes = nbytes + fbytes, gbytes = (unsigned)ch * 8, ubytes = (unsigned)ch * 4;
    const unsigned sbytes = dbytes + gbytes + ubytes;
    const int b = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const T *gcol = reinterpret_cast<const T *>(a.gP) + (size_t)b * a.npad;
    const int32_t nchunks = (int32_t)(a.npad >> a.lg_ch);

    if (tid < 16)   // the zero entries, one per bank pair
        asm volatile("st.shared.b64 [%0], %1;" ::"r"(ring_base + (unsigned)(RING + tid) * 8), "l"(0ull) : "memory");
    if (tid == 0) {
        for (int s = 0; s < a.nstage; s++) mbar_init(&bars[s], 1);
        for (int s = 0; s < kLB; s++) mbar_init(&bars[a.nstage + s], 32);   // one arrival per lane
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
                bulk_g2s(st, a.Dn + r0 * a.kpn, nbytes, &bars[s]);
                bulk_g2s(st + nbytes, a.Df + r0 * a.kpf, fbytes, &bars[s]);
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
    // Level completion is published on a ring of kLB mbarriers: lane 0 of the
    // warp that owns level L arrives (release, after a __syncwarp that orders
    // the lanes' ring stores) on lvlbar[L % kLB]; a waiter for "level L done"
    // try_waits (acquire) on the phase (L / kLB) & 1.  Levels finish in
    // order, so "L done" means every level <= L is done, and no waiter ever
    // looks more than kMid + 1 < kLB levels back, so parities cannot alias.
    T *f = reinterpret_cast<T *>(a.f);
    u64 *lvlbar = bars + a.nstage;   // kLB barriers after the stage barriers
    const unsigned lvl_u32 = smem_u32(lvlbar);
    const unsigned zero_off = (unsigned)RING * 8u;   // byte offset of the zero entry
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
        // One level, NPX passes of 32 elements in registers (NPX = 1: the
        // common single-pass level, no code for other passes; NPX = kNP:
        // passes p < np, the rest serially after the near wait).
        auto level = [&](auto npx) {
            constexpr int NPX = decltype(npx)::value;
            auto act = [&](int p) { return NPX == 1 || p < np; };
            T gx[NPX], sp[NPX];
            int32_t u[NPX];
            unsigned rowa[NPX], rowf[NPX], pn[NPX], cnt[NPX];
            unsigned nw[NPX][NN / 2];
#pragma unroll
            for (int p = 0; p < NPX; p++) {
                if (act(p)) {
                    const int32_t e = lo + 32 * p + lane;
                    const int32_t ee = e < hi ? e : lo + 32 * p;
                    const unsigned st = stage_base + ((unsigned)(ee >> a.lg_ch) % ns) * sbytes;
                    const unsigned off = (unsigned)(ee & (ch - 1));
                    rowa[p] = st + off * (unsigned)a.kpn * 2;
                    rowf[p] = st + nbytes + off * (unsigned)a.kpf * 2;
                    gx[p] = bits_to<T>(df_lds64(st + dbytes + off * 8));
                    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(u[p]) : "r"(st + dbytes + gbytes + off * 4));
                    const unsigned pc = lds32u(rowa[p] + OFF_PN);
                    pn[p] = pc & 0xffffu;
                    cnt[p] = pc >> 16;   // near count | mid count << 5 | far chunks << 11
                    df_near_words<NN>(rowa[p] + OFF_NEAR, nw[p]);
                    u[p] = e < hi ? u[p] : -1;
                } else {
                    gx[p] = T(0);
                    u[p] = -1;
                    rowa[p] = rowf[p] = pn[p] = cnt[p] = 0;
#pragma unroll
                    for (int q = 0; q < NN / 2; q++) nw[p][q] = zero_off | (zero_off << 16);
                }
            }
            wait_level(L - kMid - 1);   // far: levels <= L-7
#pragma unroll
            for (int p = 0; p < NPX; p++) {
                if (act(p)) {
                    // far entries in chunks of 16, to the longest row of the warp
                    const unsigned nf = (a.skip_far & 1) ? 0u : __reduce_max_sync(0xffffffffu, cnt[p] >> 11);
                    T acc = T(0);
                    for (unsigned c = 0; c < nf; c++) acc += df_sum<T, 16>(ring_base, rowf[p] + 32 * c);
                    sp[p] = acc;
                }
            }
            wait_level(L - kNear - 1);  // mid: levels <= L-3
#pragma unroll
            for (int p = 0; p < NPX; p++) {
                if (act(p)) {
                    // mid entries in chunks of 8 (zero-entry padded), to the warp's longest
                    const unsigned nm8 =
                        (a.skip_far & 2) ? 0u : (__reduce_max_sync(0xffffffffu, (cnt[p] >> 5) & 63u) + 7) >> 3;
                    T acc = T(0);
                    for (unsigned c = 0; c < nm8; c++) acc += df_sum<T, 8>(ring_base, rowa[p] + 16 * c);
                    sp[p] += acc;
                }
            }
            // Everything the critical path needs is formed (and pinned in
            // registers) before the near wait: gx - (far + mid), the absolute
            // ring addresses of the near slots (padding = the zero entry, so
            // the loads need no predicates), the ring store address and
            // predicate and the barrier address.  After the wait: NN loads per
            // pass, the add tree, one subtract, a predicated store,
            // __syncwarp and the arrive.
            unsigned lvl_addr = lvl_u32 + (unsigned)(L & (kLB - 1)) * 8u;
            df_pin(lvl_addr);
            T gs[NPX], Fx[NPX];
            unsigned na[NPX][NN], sa[NPX], stp[NPX];
#pragma unroll
            for (int p = 0; p < NPX; p++) {
                gs[p] = act(p) ? gx[p] - sp[p] : T(0);
                df_pin(gs[p]);
                sa[p] = ring_base + (unsigned)((lo + 32 * p + lane) & a.ring_mask) * 8u;
                stp[p] = (act(p) && u[p] >= 0) ? 1u : 0u;
                df_pin(sa[p]);
                df_pin(stp[p]);
#pragma unroll
                for (int q = 0; q < NN / 2; q++) {
                    const unsigned w = (a.skip_far & 4) ? (zero_off | (zero_off << 16)) : nw[p][q];
                    na[p][2 * q] = ring_base + (w & 0xffffu);
                    na[p][2 * q + 1] = ring_base + (w >> 16);
                    df_pin(na[p][2 * q]);
                    df_pin(na[p][2 * q + 1]);
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
            T v[NPX][NN];
#pragma unroll
            for (int p = 0; p < NPX; p++)
#pragma unroll
                for (int j = 0; j < NN; j++) v[p][j] = bits_to<T>(df_lds64(na[p][j]));
#pragma unroll
            for (int p = 0; p < NPX; p++) {
#pragma unroll
                for (int st = 1; st < NN; st <<= 1)
#pragma unroll
                    for (int j = 0; j < NN; j += 2 * st) v[p][j] += v[p][j + st];
                Fx[p] = gs[p] - v[p][0];
                if (PROF && p == 0 && lane == 0 && b == 0) {
                    asm volatile("" ::"l"(df_bits<T>(Fx[0])));   // the near sum completes before the stamp
                    prof[7] += clock64() - t_ready;
                }
            }
#pragma unroll
            for (int p = 0; p < NPX; p++) df_stp64(sa[p], df_bits<T>(Fx[p]), stp[p]);
            if (NPX == kNP) {
                // passes beyond kNP (levels wider than 32 * kNP): serially, all deps done
                for (int32_t base = lo + 32 * kNP; base < hi; base += 32) {
                    const int32_t e = base + lane;
                    const int32_t ee = e < hi ? e : base;
                    const unsigned st = stage_base + ((unsigned)(ee >> a.lg_ch) % ns) * sbytes;
                    const unsigned off = (unsigned)(ee & (ch - 1));
                    const unsigned row = st + off * (unsigned)a.kpn * 2;
                    const unsigned row_f = st + nbytes + off * (unsigned)a.kpf * 2;
                    const T g1 = bits_to<T>(df_lds64(st + dbytes + off * 8));
                    int32_t u1;
                    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(u1) : "r"(st + dbytes + gbytes + off * 4));
                    const unsigned pc1 = lds32u(row + OFF_PN);
                    const unsigned p16 = pc1 & 0xffffu;
                    T s1 = df_sum<T, NM>(ring_base, row) + df_sum_u16<T, NN>(ring_base, row + OFF_NEAR);
                    for (unsigned c = 0; c < (pc1 >> 27); c++) s1 += df_sum<T, 16>(ring_base, row_f + 32 * c);
                    const T F1 = g1 - s1;
                    if (e < hi) {
                        asm volatile("st.shared.b64 [%0], %1;" ::"r"(ring_base + (unsigned)(e & a.ring_mask) * 8),
                                     "l"(df_bits<T>(F1))
                                     : "memory");
                        f[(size_t)u1 * a.B + b] = F1 - bits_to<T>(df_lds64(ring_base + p16));
                    }
                }
            }
            long long t_pre = 0;
            if (PROF) t_pre = clock64();
            // publish: every lane arrives (release: its own ring store is
            // ordered before its arrival; the phase needs all 32), so neither
            // a __syncwarp nor a branch sits on the critical path; lane 0 also
            // advances done_rank (producer)
            asm volatile(
                "{\n.reg .pred q;\nsetp.eq.u32 q, %0, 0;\n"
                "mbarrier.arrive.release.cta.shared::cta.b64 _, [%1];\n"
                "@q st.relaxed.cta.shared.s32 [%2], %3;\n}" ::"r"(lane),
                "r"(lvl_addr), "r"(ctrl + 4), "r"(hi)
                : "memory");
            if (PROF && lane == 0 && b == 0) {
                const long long t = clock64();
                prof[0] += t - t_ready;
                prof[4] += 1;
                prof[5] += t_pre - t_ready;
                prof[6] += np;
                prof_last = (unsigned long long)t;
            }
            // f(x) = F(x) - F(next below on the chain), after the publish, off
            // the critical path (the pn slot stays live: RING >= reach + 18 wmax)
#pragma unroll
            for (int p = 0; p < NPX; p++)
                if (stp[p]) f[(size_t)u[p] * a.B + b] = Fx[p] - bits_to<T>(df_lds64(ring_base + pn[p]));
        };
        if (np <= 1)
            level(std::integral_constant<int, 1>{});
        else
            level(std::integral_constant<int, kNP>{});
    }
    if (PROF) {
        asm volatile("bar.sync 1, %0;" ::"r"(32 * kNWC));
        if (tid == 0 && b == 0)
            for (int i = 0; i < 8; i++) a.dbg[i] = prof[i];
    }
}

// ------------------------------------------------------------- host -------
static constexpr size_t kSmemCapDF = 227 * 1024;

static size_t ringdf_smem_bytes(int ring, int kp, int ch, int nstage) {   // kp = kpn + kpf
    return (size_t)(ring + 16) * 8 + 8 * ((nstage + kLB + 1) & ~1) + 16 + (size_t)nstage * ch * ((size_t)kp * 2 + 12);
}
static int32_t odd16(int32_t e) { return (e / 8) % 2 == 0 ? e + 8 : e; }   // rows of 16 * odd bytes

void ringdf_plan(int32_t n, int32_t k, int32_t max_level_width, unsigned reach,
                 const unsigned counts3[3], RingDFPlan &R) {
    R.ok = false;
    if (n <= 0 || k > 256 || counts3[0] > 16 || counts3[1] > 32 || counts3[2] > 31 * 16) return;
    R.nn = counts3[0] <= 4 ? 4 : counts3[0] <= 8 ? 8 : 16;
    R.nm = counts3[1] <= 16 ? 16 : 32;
    R.fe = std::max(16, (int)(counts3[2] + 15) / 16 * 16);   // longest bank-coloured far group
    R.kpn = odd16(df_off_far(R.nm, R.nn) / 2);   // near-table rows (16 * odd bytes: rows spread banks)
    R.kpf = odd16(R.fe + 8);                      // far rows + chunk count
    const int32_t kp = R.kpn + R.kpf;
    const int64_t ahead = (int64_t)(kNWC + kMid + 4) * max_level_width;
    int64_t ring = 32;
    while (ring < (int64_t)reach + ahead + 1) ring <<= 1;
    if (ring > 4096) return;   // rows hold byte offsets: (RING + 16) * 8 must fit in 16 bits
    // the fewest stages of the largest chunk that hold 9 levels and fit
    for (int ch : {256, 128, 64, 32}) {
        for (int nstage = 2; nstage <= 8; nstage++) {
            if ((int64_t)(nstage - 1) * ch < (int64_t)(kNWC + 1) * max_level_width) continue;
            if (ringdf_smem_bytes((int)ring, kp, ch, nstage) > kSmemCapDF) break;
            R.ok = true;
            R.kp = kp;
            R.ring = (int32_t)ring;
            R.ch = ch;
            R.nstage = nstage;
            R.npad = ((int64_t)n + ch - 1) / ch * ch;
            R.nwc = kNWC;
            R.wmax = max_level_width;
            ringcl_plan(R);
            return;
        }
    }
}

static size_t build_smem(int k, int kp) { return 2048 + (size_t)64 * (k + 1) * 2 + (size_t)32 * kp * 2 + 2 * 4096 * 2; }

cudaError_t launch_df_counts(const DevPoset &P, const int32_t *level, const int32_t *slot_rank,
                             unsigned *out3, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(out3, 0, 3 * sizeof(unsigned), s);
    if (e != cudaSuccess || P.n == 0) return e;
    k_df_counts<<<(P.n + 255) / 256, 256, 0, s>>>(P.M, P.n, P.k, P.chain, level, slot_rank, out3);
    launches_add(1);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (P.k > 256 || P.ell <= 0) return cudaSuccess;   // no RINGDF plan (ringdf_plan)
    const size_t smem = build_smem(P.k, 0);
    e = cudaFuncSetAttribute(k_build_ringdf<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_build_ringdf<false><<<(unsigned)P.ell, 256, smem, s>>>(P.M, P.n, P.k, P.lvl_ptr, 0, 0, 0, 0, 0, 4096,
                                                          P.chain, P.slot, slot_rank, level, nullptr, nullptr,
                                                          out3 + 2);
    launches_add(1);
    return cudaGetLastError();
}

cudaError_t launch_build_ringdf(const DevPoset &P, const RingDFPlan &R, const int32_t *level,
                                const int32_t *slot_rank, cudaStream_t s) {
    if (P.n == 0) return cudaSuccess;
    const size_t smem = build_smem(P.k, R.kp);
    cudaError_t e = cudaFuncSetAttribute(k_build_ringdf<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    k_build_ringdf<true><<<(unsigned)P.ell, 256, smem, s>>>(P.M, P.n, P.k, P.lvl_ptr, R.kpn, R.kpf, R.nn, R.nm,
                                                         R.fe, R.ring, P.chain, P.slot, slot_rank, level, R.D,
                                                         R.D + R.npad * R.kpn, nullptr);
    launches_add(1);
    return cudaGetLastError();
}

cudaError_t launch_moebius_ringdf(const DevPoset &P, const RingDFPlan &R, const int32_t *ru_pad,
                                  int dtype, const void *gP, void *f, int64_t B, cudaStream_t s) {
    if (P.n == 0) return cudaSuccess;
    RDFArgs a;
    a.Dn = R.D;
    a.Df = R.D + R.npad * R.kpn;
    a.gP = gP;
    a.ru = ru_pad;
    a.lvl_ptr = P.lvl_ptr;
    a.f = f;
    a.npad = R.npad;
    a.n = P.n;
    a.kpn = R.kpn;
    a.kpf = R.kpf;
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
#define RDF_FN(NN, NM)                                                                         \
    if (R.nn == NN && R.nm == NM)                                                              \
        fn = R.prof ? (dtype == 0 ? (void *)k_moeb_ringdf<u64, NN, NM, true>                   \
                                  : (void *)k_moeb_ringdf<double, NN, NM, true>)               \
                    : (dtype == 0 ? (void *)k_moeb_ringdf<u64, NN, NM>                         \
                                  : (void *)k_moeb_ringdf<double, NN, NM>);
    RDF_FN(4, 16) RDF_FN(4, 32) RDF_FN(8, 16) RDF_FN(8, 32) RDF_FN(16, 16) RDF_FN(16, 32)
#undef RDF_FN
    if (!fn) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    void *args[] = {&a};
    launches_add(1);
    return cudaLaunchKernel(fn, dim3((unsigned)B), dim3(32 * (kNWC + 1)), args, smem, s);
}

// ---------------------------------------------------------------------------
// Schedule RINGCL: RINGDF over a thread-block cluster of 1 + NH CTAs per
// column (NH = 1..3 helpers; 2 by default), so that other SMs' shared-memory
// pipes and issue slots take the far sums.
//   owner  (cluster rank 0): the level pipeline of RINGDF -- rows (near
//          table), mid sums, the near wait, F into its ring -- but the far
//          sum of each element comes from the helpers through DSMEM (2 NH
//          partial sums in the sfar buffers, landing on farbar[L % kLB],
//          armed by the owner with 16 NH bytes per element).  After
//          publishing level L locally it forwards F to every helper's ring
//          with st.async, each store completing 8 bytes on that helper's
//          lvlbar[L % kLB].
//   helper (cluster ranks 1..NH): 16 warps; warps 2g and 2g+1 own the
//          levels L = g (mod 8) and the 16-entry far chunks c = qi (mod 2 NH)
//          of their rows (qi = 2 (rank - 1) + warp parity).  A warp arms
//          lvlbar[L % kLB] (8 bytes per element), loads its level's far-row
//          words from global memory into registers (their latency hides
//          behind the wait), waits for the owner's levels L-14 .. L-7 (they
//          are published out of order; older ones it saw at level L-8), sums
//          and st.async's its partial sums to the owner.
// Slack: the far sum of level L is needed when level L-1 completes, i.e.
// 6 level times after level L-7 completed (a DSMEM round trip is ~320
// cycles).  Waits are CTA-scope try_waits: the bytes are made visible by the
// complete_tx mechanism, and a cluster-scope acquire would cost an L1
// invalidate (CCTL.IVALL) per wait.
__device__ __forceinline__ unsigned cl_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cl_mapa(unsigned a, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void cl_st64(unsigned ra, u64 v) {
    asm volatile("st.shared::cluster.b64 [%0], %1;" ::"r"(ra), "l"(v) : "memory");
}
__device__ __forceinline__ void cl_arrive_remote(unsigned ra) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
// DSMEM store that signals its bytes on the destination CTA's mbarrier
__device__ __forceinline__ void cl_st_async64(unsigned ra, u64 v, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(ra), "l"(v),
                 "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void cl_expect(unsigned a, unsigned bytes) {   // the phase's single arrival
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cl_arrive_local(unsigned a) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
// wait for a phase completed by st.async complete_tx bytes (the transaction
// mechanism makes the bytes visible; CTA-scope acquire, so no L1 invalidate
// -- a cluster-scope acquire costs a CCTL.IVALL per wait)
__device__ __forceinline__ void cl_wait(unsigned a, unsigned parity) {
    asm volatile(
        "{\n.reg .pred p;\nWC_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WC_%=;\n}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void cl_wait_cta(unsigned a, unsigned parity) {
    asm volatile(
        "{\n.reg .pred p;\nWL_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WL_%=;\n}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <typename T, int NN, int NM, int FEC, bool PROF = false, int NH = 1, bool CW = false>
__global__ void __launch_bounds__(32 * kNWH) k_moeb_ringcl(RDFArgs a) {
    // NH helper CTAs (cluster of NH + 1); the far chunks of a row are split
    // over the 2 * NH helper warps of a level group (chunk c -> c mod 2NH)
    constexpr int S = 2 * NH, CPW = (FEC + S - 1) / S;
    constexpr unsigned OFF_NEAR = 2 * NM, OFF_PN = 2 * (NM + NN);
    extern __shared__ __align__(16) unsigned char smem[];
    const int RING = a.ring_mask + 1;
    const unsigned crank = cl_rank(), peer = 0u;   // helpers talk to the owner (rank 0)
    const bool owner = crank == 0;
    // role-specific staging (the helper's warps finish out of order, so it
    // keeps more rows in flight)
    const int lgc = owner ? a.lg_ch : a.lg_chh;
    const int ch = 1 << lgc;
    const unsigned ring_base = smem_u32(smem);                         // RING + 16 entries
    const unsigned sfar_base = ring_base + (unsigned)(RING + 16) * 8;   // 2 NH buffers of SB entries (owner)
    const int SB = RING >> (NH == 1 ? 0 : NH == 2 ? 1 : 2);   // 2 NH buffers fit in 2 RING entries
    u64 *bars = reinterpret_cast<u64 *>(smem + (size_t)(3 * RING + 16) * 8);
    constexpr int nb = kMaxStageCL + 2 * kLB;   // stage | lvlbar | farbar
    const unsigned lvl_u32 = smem_u32(bars + kMaxStageCL), far_u32 = lvl_u32 + kLB * 8;
    unsigned *ctrl_p = reinterpret_cast<unsigned *>(bars + nb);   // ready | done | prog[8]
    const unsigned ctrl = smem_u32(ctrl_p);
    unsigned char *stage0 = reinterpret_cast<unsigned char *>(ctrl_p + 12);
    const unsigned stage_base = smem_u32(stage0);
    // owner stage: near rows | g | user ids;  helper stage: far rows
    const unsigned nbytes = owner ? (unsigned)ch * a.kpn * 2 : 0u, fbytes = owner ? 0u : (unsigned)ch * a.kpf * 2;
    const unsigned gbytes = owner ? (unsigned)ch * 8 : 0u, ubytes = owner ? (unsigned)ch * 4 : 0u;
    const unsigned sbytes = nbytes + fbytes + gbytes + ubytes;
    const int b = blockIdx.x / (NH + 1);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const T *gcol = reinterpret_cast<const T *>(a.gP) + (size_t)b * a.npad;
    const int32_t nchunks = (int32_t)(a.npad >> lgc);
    const int nstage = owner ? a.nstage : a.nstage_h;
    const unsigned ns = (unsigned)nstage;
    T *f = reinterpret_cast<T *>(a.f);
    const unsigned zero_off = (unsigned)RING * 8u;
    __shared__ long long pubt[64];   // instrumentation (a.dbg): owner publish clock per level
    // CW: hand-off records [8 levels][kNP passes][32 lanes] x 32 bytes after the stages
    const unsigned hb_base = (stage_base + (unsigned)nstage * sbytes + 15u) & ~15u;
    static_assert(!CW || NN == 4, "the critical-warp records hold 4 near offsets");
    if (CW && owner)
        for (int t = tid; t < 8 * kNP * 256; t += blockDim.x)   // tags 4095 / -1: match no level < 8
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(hb_base + 4u * t), "r"(0xffffffffu) : "memory");

    if (tid < 16)
        asm volatile("st.shared.b64 [%0], %1;" ::"r"(ring_base + (unsigned)(RING + tid) * 8), "l"(0ull) : "memory");
    if (tid == 0) {
        for (int s = 0; s < nb; s++) mbar_init(&bars[s], 1);
        if (owner && !CW)   // the owner's level barriers take one arrival per lane (RINGCW: lane 0)
            for (int s = 0; s < kLB; s++) mbar_init(&bars[kMaxStageCL + s], 32);
        for (int i = 0; i < 10; i++) ctrl_p[i] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cl_sync();   // both CTAs' barriers initialised before any remote arrive

    auto wait_lvl = [&](int32_t Ld) {   // local level completion (owner)
        if (Ld < 0) return;
        cl_wait_cta(lvl_u32 + (unsigned)(Ld & (kLB - 1)) * 8u, (unsigned)((Ld / kLB) & 1));
    };
    // RINGCW level warps: poll with test_wait and sleep in between, so that
    // waiting warps do not crowd the shared-memory pipe the critical warp uses
    auto wait_lvl_sleep = [&](int32_t Ld) {
        if (Ld < 0) return;
        const unsigned ad = lvl_u32 + (unsigned)(Ld & (kLB - 1)) * 8u, par = (unsigned)((Ld / kLB) & 1);
        for (;;) {
            unsigned ok;
            asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                         : "=r"(ok)
                         : "r"(ad), "r"(par)
                         : "memory");
            if (ok) return;
            __nanosleep(a.cw_sleep);
        }
    };
    // owner roles.  RINGCW keeps the critical warp alone on its SM
    // sub-partition (warps 1, 5, 9, 13 share one): warp 1 is the critical
    // warp, 5 / 9 / 13 idle, the level warps are 0, 2, 3, 4, 6, 7, 8, 10 and
    // warp 11 the producer.  RINGCL: level warps 0..7, producer 8.
    constexpr int kCWarp = 1, kProd = CW ? 11 : kNWC;
    const int mid = !CW ? (warp < kNWC ? warp : -1)
                        : (warp == 0 ? 0 : warp == 2 ? 1 : warp == 3 ? 2 : warp == 4 ? 3 : warp == 6 ? 4
                           : warp == 7 ? 5 : warp == 8 ? 6 : warp == 10 ? 7 : -1);
    if (owner && warp == kProd) {
        // ------------------------------------------------------ producer --
        if (lane == 0) {
            auto issue = [&](int32_t c) {
                const int s = (int)((unsigned)c % ns);
                unsigned char *st = stage0 + (size_t)s * sbytes;
                const size_t r0 = (size_t)c << lgc;
                mbar_expect_tx(&bars[s], sbytes);
                if (owner) {
                    bulk_g2s(st, a.Dn + r0 * a.kpn, nbytes, &bars[s]);
                    bulk_g2s(st + nbytes, gcol + r0, gbytes, &bars[s]);
                    bulk_g2s(st + nbytes + gbytes, a.ru + r0, ubytes, &bars[s]);
                } else {
                    bulk_g2s(st, a.Df + r0 * a.kpf, fbytes, &bars[s]);
                }
            };
            // consumers' progress: owner levels finish in order (done word);
            // helper warps finish out of order (minimum of per-warp words)
            auto progress = [&]() -> int32_t {
                if (owner) return df_acq(ctrl + 4);
                int32_t m = 0x7fffffff;
                for (int w = 0; w < kNWC; w++) m = min(m, df_acq(ctrl + 8 + 4 * w));
                return m;
            };
            int32_t issued = 0, arrived = 0;
            for (; issued < nchunks && issued < nstage; issued++) issue(issued);
            while (arrived < nchunks) {
                mbar_wait(&bars[(unsigned)arrived % ns], ((unsigned)arrived / ns) & 1u);
                arrived++;
                df_rel(ctrl, arrived << lgc);
                while (issued < nchunks) {
                    const int32_t done = progress();
                    if (((int64_t)(issued - nstage + 1) << lgc) > done) {
                        if (arrived < issued) break;
                        __nanosleep(64);
                        continue;
                    }
                    issue(issued);
                    issued++;
                }
            }
        }
    } else if (!owner) {
        // -------------------------------------------------- helper warps --
        // Far rows come straight from global memory into registers, issued
        // before the wait for the owner's levels (their latency hides behind
        // it); no staging, so no coupling between the out-of-order helper
        // warps and a stage ring.
        // Two warps per level group and helper (kNWH = 16): warp (g, hh) =
        // (warp / 2, warp % 2) (the pair on different SM sub-partitions) owns
        // the levels L = g (mod 8) and the chunks c = qi (mod 2 NH) of their
        // far rows; the owner adds the 2 NH partial sums.
        const int g = warp >> 1, hh = warp & 1;   // the two warps of a pair on different SMSPs
        const int qi = ((int)crank - 1) * 2 + hh;   // this warp's chunk class (mod 2 NH)
        const unsigned sfar_h = sfar_base + (unsigned)(qi * SB) * 8u;
        int32_t hcb = 0, hlo, hhi;   // level bounds of this warp's next 32 levels, in registers
        hlo = a.lvl_ptr[min(g + lane * kNWC, a.ell)];
        hhi = a.lvl_ptr[min(g + lane * kNWC + 1, a.ell)];
        auto far_sum = [&](const uint4 (&w)[2 * CPW], unsigned nf) -> T {
            T acc = T(0);
#pragma unroll
            for (int j = 0; j < CPW; j++) {
                if ((unsigned)(qi + S * j) >= nf) break;   // warp-uniform: the group's colour count
                const unsigned ws[8] = {w[2 * j].x, w[2 * j].y, w[2 * j].z, w[2 * j].w,
                                        w[2 * j + 1].x, w[2 * j + 1].y, w[2 * j + 1].z, w[2 * j + 1].w};
                T v[16];
#pragma unroll
                for (int h = 0; h < 8; h++) {
                    v[2 * h] = bits_to<T>(df_lds64(ring_base + (ws[h] & 0xffffu)));
                    v[2 * h + 1] = bits_to<T>(df_lds64(ring_base + (ws[h] >> 16)));
                }
#pragma unroll
                for (int st2 = 1; st2 < 16; st2 <<= 1)
#pragma unroll
                    for (int j = 0; j < 16; j += 2 * st2) v[j] += v[j + st2];
                acc += v[0];
            }
            return acc;
        };
        auto load_row = [&](int32_t ee, uint4 (&w)[2 * CPW], unsigned &c16) {
            const uint4 *rg = reinterpret_cast<const uint4 *>(a.Df + (size_t)ee * a.kpf);
            const int nq = a.fe / 8;   // the row's 16-byte words (fe <= 16 * FEC)
#pragma unroll
            for (int j = 0; j < CPW; j++) {   // chunk qi + S j = words 2 (qi + S j), +1
                const int q = 2 * (qi + S * j);
                w[2 * j] = q < nq ? __ldg(rg + q) : make_uint4(0, 0, 0, 0);
                w[2 * j + 1] = q + 1 < nq ? __ldg(rg + q + 1) : make_uint4(0, 0, 0, 0);
            }
            c16 = __ldg(a.Df + (size_t)ee * a.kpf + a.fe);   // 16-entry chunks used by this row's group
        };
        uint4 w0[2 * CPW];
        unsigned c0 = 0;
        for (int32_t L = g, i = 0; L < a.ell; L += kNWC, i++) {
            if (i - hcb == 32) {
                hcb += 32;
                hlo = a.lvl_ptr[min(g + (hcb + lane) * kNWC, a.ell)];
                hhi = a.lvl_ptr[min(g + (hcb + lane) * kNWC + 1, a.ell)];
            }
            const int32_t lo = __shfl_sync(0xffffffffu, hlo, i - hcb), hi = __shfl_sync(0xffffffffu, hhi, i - hcb);
            // arm this level's phase: the owner's F values of level L land here
            // with st.async (8 bytes per element); phase L-16 is complete (this
            // warp waited for it at level L-8)
            if (hh == 0 && lane == 0) cl_expect(lvl_u32 + (unsigned)(L & (kLB - 1)) * 8u, 8u * (unsigned)(hi - lo));
            const int32_t e0 = lo + lane;
            // this level's first-pass row words: their latency hides behind
            // the wait for the owner's levels below (no second register set
            // for a prefetch -- registers go to loads in flight)
            load_row(e0 < hi ? e0 : lo, w0, c0);
            // owner levels <= L-7 in this CTA's ring: the owner warps publish
            // independently, so wait for every level this warp has not yet
            // seen (L-14 .. L-7; older ones were covered by its level L-8)
            if (PROF && (a.skip_far & 2)) {   // instrumentation: wait for this level's row words here
                unsigned x = 0;
#pragma unroll
                for (int q = 0; q < FEC; q++) x ^= w0[q].x ^ w0[q].y ^ w0[q].z ^ w0[q].w;
                asm volatile("st.shared.u32 [%0], %1;" ::"r"(ctrl + 40), "r"(x) : "memory");   // dummy word
            }
            const long long t0 = PROF ? clock64() : 0;
            if (L >= kMid + kNWC) {
                // the seven older phases are almost always complete: test them
                // together (non-blocking), fall back to waiting one by one
                unsigned ok;
                const int32_t X0 = L - kMid - kNWC;
                asm volatile(
                    "{\n.reg .pred p0, p1, p2, p3, p4, p5, p6;\n"
                    "mbarrier.test_wait.parity.shared::cta.b64 p0, [%1], %8;\n"
                    "mbarrier.test_wait.parity.shared::cta.b64 p1, [%2], %9;\n"
                    "mbarrier.test_wait.parity.shared::cta.b64 p2, [%3], %10;\n"
                    "mbarrier.test_wait.parity.shared::cta.b64 p3, [%4], %11;\n"
                    "mbarrier.test_wait.parity.shared::cta.b64 p4, [%5], %12;\n"
                    "mbarrier.test_wait.parity.shared::cta.b64 p5, [%6], %13;\n"
                    "mbarrier.test_wait.parity.shared::cta.b64 p6, [%7], %14;\n"
                    "and.pred p0, p0, p1;\nand.pred p2, p2, p3;\nand.pred p4, p4, p5;\n"
                    "and.pred p0, p0, p2;\nand.pred p4, p4, p6;\nand.pred p0, p0, p4;\n"
                    "selp.u32 %0, 1, 0, p0;\n}\n"
                    : "=r"(ok)
                    : "r"(lvl_u32 + (unsigned)((X0 + 0) & (kLB - 1)) * 8u), "r"(lvl_u32 + (unsigned)((X0 + 1) & (kLB - 1)) * 8u),
                      "r"(lvl_u32 + (unsigned)((X0 + 2) & (kLB - 1)) * 8u), "r"(lvl_u32 + (unsigned)((X0 + 3) & (kLB - 1)) * 8u),
                      "r"(lvl_u32 + (unsigned)((X0 + 4) & (kLB - 1)) * 8u), "r"(lvl_u32 + (unsigned)((X0 + 5) & (kLB - 1)) * 8u),
                      "r"(lvl_u32 + (unsigned)((X0 + 6) & (kLB - 1)) * 8u), "r"((unsigned)(((X0 + 0) / kLB) & 1)),
                      "r"((unsigned)(((X0 + 1) / kLB) & 1)), "r"((unsigned)(((X0 + 2) / kLB) & 1)),
                      "r"((unsigned)(((X0 + 3) / kLB) & 1)), "r"((unsigned)(((X0 + 4) / kLB) & 1)),
                      "r"((unsigned)(((X0 + 5) / kLB) & 1)), "r"((unsigned)(((X0 + 6) / kLB) & 1))
                    : "memory");
                if (!ok)
                    for (int32_t X = X0; X < L - kMid - 1; X++)
                        cl_wait(lvl_u32 + (unsigned)(X & (kLB - 1)) * 8u, (unsigned)((X / kLB) & 1));
                cl_wait(lvl_u32 + (unsigned)((L - kMid - 1) & (kLB - 1)) * 8u, (unsigned)(((L - kMid - 1) / kLB) & 1));
            } else {
                for (int32_t X = max(0, L - kMid - kNWC); X <= L - kMid - 1; X++)
                    cl_wait(lvl_u32 + (unsigned)(X & (kLB - 1)) * 8u, (unsigned)((X / kLB) & 1));
            }
            const long long t1 = PROF ? clock64() : 0;
            long long t1b = t1, t1s = t1;
            const unsigned fbar = cl_mapa(far_u32 + (unsigned)(L & (kLB - 1)) * 8u, peer);
            {
                const T acc = (a.skip_far & 1) ? T(0) : far_sum(w0, __reduce_max_sync(0xffffffffu, c0));
                if (PROF) {   // instrumentation: the sum is complete here
                    asm volatile("" ::"l"(df_bits<T>(acc)));
                    t1b = clock64();
                    if (a.skip_far & 4) {   // a second, identical far sum, timed on its own
                        const T acc2 = far_sum(w0, __reduce_max_sync(0xffffffffu, c0));
                        asm volatile("st.shared.b64 [%0], %1;" ::"r"(ctrl + 40), "l"(df_bits<T>(acc2)) : "memory");
                        t1s = t1b;
                        t1b = clock64();
                    }
                }
                if (e0 < hi) cl_st_async64(cl_mapa(sfar_h + (unsigned)(e0 & (SB - 1)) * 8u, peer), df_bits<T>(acc), fbar);
            }
            for (int32_t base = lo + 32; base < hi; base += 32) {   // wide levels: further passes
                const int32_t e = base + lane;
                uint4 w1[2 * CPW];
                unsigned c1;
                load_row(e < hi ? e : base, w1, c1);
                const T acc = (a.skip_far & 1) ? T(0) : far_sum(w1, __reduce_max_sync(0xffffffffu, c1));
                if (e < hi) cl_st_async64(cl_mapa(sfar_h + (unsigned)(e & (SB - 1)) * 8u, peer), df_bits<T>(acc), fbar);
            }
            if (PROF && b == 0 && lane == 0 && hh == 0) {
                const long long t2 = PROF ? clock64() : 0;
                atomicAdd(a.dbg + 4, (unsigned long long)(t1 - t0));
                atomicAdd(a.dbg + 5, (unsigned long long)(t2 - t1));
                atomicAdd(a.dbg + 6, 1ull);
                atomicAdd(a.dbg + 7, (unsigned long long)(t1b - t1s));
            }
        }
        // the owner's last stores into this CTA have landed before it may exit
        for (int32_t X = max(0, a.ell - kNWC); X < a.ell; X++)
            cl_wait(lvl_u32 + (unsigned)(X & (kLB - 1)) * 8u, (unsigned)((X / kLB) & 1));
    } else if (CW && warp == kCWarp) {
        // ------------------------------------------------- critical warp --
        // Every level's near step in ONE warp (lane = element): no
        // cross-warp hand-off on the chain.  The owner warps above hand each
        // level's g - mid - far and near offsets over in tagged 16-byte
        // records; this warp polls the record (a plain shared load: the tag
        // and the data are one 16-byte store), adds the <= 4 near values (the
        // previous two levels, written by this warp), stores F, publishes the
        // level on lvlbar and forwards F to the helpers.
        // The loop is kept short (it IS the critical path): one iteration per
        // 32-element pass, everything it needs in the pass's record (no level
        // bounds, no branches but the level end), the next record read
        // during the current pass's near loads.
        unsigned ln = (unsigned)lane;
        df_pin(ln);
        const unsigned my_rec = hb_base + ln * 32u, rb = ring_base;
        unsigned lvlb = lvl_u32, ctl = ctrl + 4;
        df_pin(lvlb);
        df_pin(ctl);
        const int32_t ell = a.ell;
        auto rec_ok = [](const uint4 &h0, const uint4 &h1, int32_t L) {
            const unsigned ez = ((unsigned)L & 7u) | (((unsigned)L >> 3) & 7u) << 16;
            const unsigned ew = (((unsigned)L >> 6) & 7u) | (((unsigned)L >> 9) & 7u) << 16;
            return ((h0.z & 0x70007u) == ez) & ((h0.w & 0x70007u) == ew) & (h1.z == (unsigned)L);
        };
        auto wait_rec = [&](unsigned ad, int32_t L, uint4 &h0, uint4 &h1) {
            for (unsigned spins = 0;; spins++) {
                if (spins > (1u << 28)) __trap();   // watchdog: a lost record is POSET_ECUDA, not a hang
                h0 = df_lds128(ad);
                h1 = df_lds128(ad + 16u);
                if (__all_sync(0xffffffffu, rec_ok(h0, h1, L))) return;
            }
        };
        const long long tstart = a.dbg ? clock64() : 0;
        unsigned long long nwait = 0;
        int32_t L = 0;
        unsigned ellu = (unsigned)ell;
        df_pin(ellu);
        const int32_t ellr = (int32_t)ellu;
        unsigned cur = my_rec;
        uint4 h0, h1;
        if (ellr > 0) wait_rec(cur, 0, h0, h1);
        const unsigned is0 = ln == 0 ? 1u : 0u;
        while (L < ellr) {
            // (1) near loads of this pass (addresses from the record in registers)
            const T v0 = bits_to<T>(df_lds64(rb + (h0.z & 0xfff8u)));
            const T v1 = bits_to<T>(df_lds64(rb + ((h0.z >> 16) & 0xfff8u)));
            const T v2 = bits_to<T>(df_lds64(rb + (h0.w & 0xfff8u)));
            const T v3 = bits_to<T>(df_lds64(rb + ((h0.w >> 16) & 0xfff8u)));
            // (2) the next pass's record (level L+1 after the last pass of L)
            const unsigned last = (h1.x >> 17) & 1u;   // warp-uniform
            const int32_t Ln = L + (int32_t)last;
            const unsigned nxt = last ? hb_base + (unsigned)(Ln & 7) * (kNP * 1024u) + ln * 32u : cur + 1024u;
            const uint4 n0 = df_lds128(nxt), n1 = df_lds128(nxt + 16u);
            // (3) off-chain arithmetic while the loads fly
            const unsigned barad = lvlb + (unsigned)(L & (kLB - 1)) * 8u, pub = last & is0;
            const unsigned ez = ((unsigned)Ln & 7u) | (((unsigned)Ln >> 3) & 7u) << 16;
            const unsigned ew = (((unsigned)Ln >> 6) & 7u) | (((unsigned)Ln >> 9) & 7u) << 16;
            const T gsv = bits_to<T>(((u64)h0.y << 32) | h0.x);
            // (4) the chain: F = g - mid - far - near, into the ring
            const T Fx = gsv - ((v0 + v1) + (v2 + v3));
            df_stp64(rb + (h1.x & 0xffffu), df_bits<T>(Fx), h1.x & (1u << 16));
            __syncwarp();   // the lanes' F stores before lane 0's release and this warp's next loads
            asm volatile(
                "{\n.reg .pred q;\nsetp.ne.u32 q, %3, 0;\n"
                "@q mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n"
                "@q st.relaxed.cta.shared.s32 [%1], %2;\n}" ::"r"(barad),
                "r"(ctl), "r"(h1.y), "r"(pub)
                : "memory");
            L = Ln;
            h0 = n0;
            h1 = n1;
            cur = nxt;
            const bool ok = ((n0.z & 0x70007u) == ez) & ((n0.w & 0x70007u) == ew) & (n1.z == (unsigned)Ln);
            if (__builtin_expect(!__all_sync(0xffffffffu, ok | (Ln >= ellr)), 0)) {   // not handed over yet
                wait_rec(cur, L, h0, h1);
                nwait++;
            }
        }
        if (a.dbg && b == 0 && ln == 0) {
            atomicAdd(a.dbg + 0, nwait);
            atomicAdd(a.dbg + 2, (unsigned long long)ell);
            atomicAdd(a.dbg + 4, (unsigned long long)(clock64() - tstart));
        }
    } else if (mid >= 0) {
        // --------------------------------------------------- owner warps --
        int32_t cb = 0;
        auto ld_bounds = [&](int32_t i0, int32_t &vlo, int32_t &vhi) {
            const int32_t L = mid + (i0 + lane) * kNWC;
            vlo = a.lvl_ptr[min(L, a.ell)];
            vhi = a.lvl_ptr[min(L + 1, a.ell)];
        };
        int32_t clo, chi;
        ld_bounds(0, clo, chi);
        int32_t staged = 0;
        for (int32_t i = 0;; i++) {
            const int32_t L = mid + i * kNWC;
            if (L >= a.ell) break;
            if (i - cb == 32) {
                cb += 32;
                ld_bounds(cb, clo, chi);
            }
            const int32_t lo = __shfl_sync(0xffffffffu, clo, i - cb);
            const int32_t hi = __shfl_sync(0xffffffffu, chi, i - cb);
            const int32_t np = min((hi - lo + 31) >> 5, kNP);
            // arm this level's far-sum phase (the helper's st.async land on it);
            // phase L-16 completed when this warp consumed level L-16
            if (lane == 0) cl_expect(far_u32 + (unsigned)(L & (kLB - 1)) * 8u, 16u * NH * (unsigned)(hi - lo));
            while (staged < hi) staged = df_acq(ctrl);
            auto level = [&](auto npx) {
                constexpr int NPX = decltype(npx)::value;
                auto act = [&](int p) { return NPX == 1 || p < np; };
                T gx[NPX], sp[NPX];
                int32_t u[NPX];
                unsigned rowa[NPX], pn[NPX], cnt[NPX];
                unsigned nw[NPX][NN / 2];
#pragma unroll
                for (int p = 0; p < NPX; p++) {
                    if (act(p)) {
                        const int32_t e = lo + 32 * p + lane;
                        const int32_t ee = e < hi ? e : lo + 32 * p;
                        const unsigned st = stage_base + ((unsigned)(ee >> lgc) % ns) * sbytes;
                        const unsigned off = (unsigned)(ee & (ch - 1));
                        rowa[p] = st + off * (unsigned)a.kpn * 2;
                        gx[p] = bits_to<T>(df_lds64(st + nbytes + off * 8));
                        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(u[p]) : "r"(st + nbytes + gbytes + off * 4));
                        const unsigned pc = lds32u(rowa[p] + OFF_PN);
                        pn[p] = pc & 0xffffu;
                        cnt[p] = pc >> 16;
                        df_near_words<NN>(rowa[p] + OFF_NEAR, nw[p]);
                        u[p] = e < hi ? u[p] : -1;
                    } else {
                        gx[p] = T(0);
                        u[p] = -1;
                        rowa[p] = pn[p] = cnt[p] = 0;
#pragma unroll
                        for (int q = 0; q < NN / 2; q++) nw[p][q] = zero_off | (zero_off << 16);
                    }
                }
                const bool mprof = CW && a.dbg != nullptr && b == 0 && lane == 0;
                const long long m0 = mprof ? clock64() : 0;
                long long m1 = m0, t2 = 0, t2b = 0, rtt = 0;
                if constexpr (CW) {
                    // RINGCW: everything that does not need levels L-6 .. L-3 first
                    // (far partials, the mid row words), then one wait and the mid
                    // sum in a single round of loads: the latency from level L-3's
                    // completion to this level's record is what paces the critical warp
                    t2 = clock64();
                    cl_wait(far_u32 + (unsigned)(L & (kLB - 1)) * 8u, (unsigned)((L / kLB) & 1));
                    t2b = clock64();
                    uint4 mw[NPX][NM / 8];
#pragma unroll
                    for (int p = 0; p < NPX; p++) {
                        sp[p] = T(0);
                        if (act(p)) {
#pragma unroll
                            for (int k2 = 0; k2 < 2 * NH; k2++)
                                sp[p] += bits_to<T>(df_lds64(sfar_base + (unsigned)(k2 * SB + ((lo + 32 * p + lane) & (SB - 1))) * 8u));
#pragma unroll
                            for (int q = 0; q < NM / 8; q++) mw[p][q] = df_lds128(rowa[p] + 16u * q);
                        }
                    }
                    if (a.cw_sleep) wait_lvl_sleep(L - kNear - 1); else wait_lvl(L - kNear - 1);   // mid: levels <= L-3
                    m1 = mprof ? clock64() : 0;
#pragma unroll
                    for (int p = 0; p < NPX; p++)
                        if (act(p) && !(a.skip_far & 2)) sp[p] += df_sum_w<T, NM>(ring_base, mw[p]);
                } else {
                wait_lvl(L - kNear - 1);   // mid: levels <= L-3
#pragma unroll
                for (int p = 0; p < NPX; p++) {
                    sp[p] = T(0);
                    if (act(p)) {
                        const unsigned nm8 = (__reduce_max_sync(0xffffffffu, (cnt[p] >> 5) & 63u) + 7) >> 3;
                        T acc = T(0);
                        for (unsigned c = 0; c < nm8; c++) acc += df_sum<T, 8>(ring_base, rowa[p] + 16 * c);
                        sp[p] = acc;
                    }
                }
                // far sums of this level, from the helper (as late as possible)
                t2 = PROF ? clock64() : 0;
                cl_wait(far_u32 + (unsigned)(L & (kLB - 1)) * 8u, (unsigned)((L / kLB) & 1));
                t2b = PROF ? clock64() : 0;
                rtt = PROF && L >= kMid + 1 ? t2b - pubt[(L - kMid - 1) & 63] : 0;
#pragma unroll
                for (int p = 0; p < NPX; p++)
                    if (act(p))
#pragma unroll
                        for (int k2 = 0; k2 < 2 * NH; k2++)
                            sp[p] += bits_to<T>(df_lds64(sfar_base + (unsigned)(k2 * SB + ((lo + 32 * p + lane) & (SB - 1))) * 8u));
                }
                unsigned lvl_addr = lvl_u32 + (unsigned)(L & (kLB - 1)) * 8u;
                df_pin(lvl_addr);
                T gs[NPX], Fx[NPX];
                unsigned na[NPX][NN], sa[NPX], stp[NPX];
#pragma unroll
                for (int p = 0; p < NPX; p++) {
                    gs[p] = act(p) ? gx[p] - sp[p] : T(0);
                    df_pin(gs[p]);
                    sa[p] = ring_base + (unsigned)((lo + 32 * p + lane) & a.ring_mask) * 8u;
                    stp[p] = (act(p) && u[p] >= 0) ? 1u : 0u;
                    df_pin(sa[p]);
                    df_pin(stp[p]);
#pragma unroll
                    for (int q = 0; q < NN / 2; q++) {
                        na[p][2 * q] = ring_base + (nw[p][q] & 0xffffu);
                        na[p][2 * q + 1] = ring_base + (nw[p][q] >> 16);
                        df_pin(na[p][2 * q]);
                        df_pin(na[p][2 * q + 1]);
                    }
                }
                if constexpr (CW) {
                    // hand the level to the critical warp, one 32-byte record per
                    // lane and pass: {g - mid - far, near offsets | tag bits},
                    // {ring offset | on << 16 | last pass << 17, hi, L, 0}; each
                    // 16-byte half is one store carrying the tag
                    const unsigned ez = (L & 7u) | (((unsigned)L >> 3) & 7u) << 16;
                    const unsigned ew = (((unsigned)L >> 6) & 7u) | (((unsigned)L >> 9) & 7u) << 16;
                    const unsigned hbL = hb_base + (unsigned)(L & 7) * (kNP * 1024u) + (unsigned)lane * 32u;
                    const int npl = (hi - lo + 31) >> 5;
#pragma unroll
                    for (int p = 0; p < NPX; p++)
                        if (act(p)) {
                            const u64 gb = df_bits<T>(gs[p]);
                            const int32_t e = lo + 32 * p + lane;
                            const unsigned w4 = (unsigned)(e & a.ring_mask) * 8u | (e < hi ? 1u << 16 : 0u) |
                                                (p == npl - 1 ? 1u << 17 : 0u);
                            asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(hbL + 1024u * p + 16u),
                                         "r"(w4), "r"(hi), "r"(L), "r"(0u)
                                         : "memory");
                            asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(hbL + 1024u * p),
                                         "r"((unsigned)gb), "r"((unsigned)(gb >> 32)), "r"(nw[p][0] | ez),
                                         "r"(nw[p][1] | ew)
                                         : "memory");
                        }
                    // outputs once the critical warp has completed level L
                    const long long m3 = mprof ? clock64() : 0;
                    if (a.cw_sleep) wait_lvl_sleep(L); else wait_lvl(L);
                    if constexpr (CW) {   // forward F to the helpers' rings (their lvlbar[L % kLB])
#pragma unroll
                        for (unsigned r = 1; r <= NH; r++) {
                            const unsigned rbar = cl_mapa(lvl_addr, r);
#pragma unroll
                            for (int p = 0; p < NPX; p++)
                                if (stp[p]) cl_st_async64(cl_mapa(sa[p], r), df_lds64(sa[p]), rbar);
                        }
                    }
                    if (mprof) {
                        const long long m4 = clock64();
                        atomicAdd(a.dbg + 6, (unsigned long long)(m4 - m3));
                        atomicAdd(a.dbg + 7, (unsigned long long)(m3 - m1));
                    }
#pragma unroll
                    for (int p = 0; p < NPX; p++)
                        if (stp[p])
                            f[(size_t)u[p] * a.B + b] = bits_to<T>(df_lds64(sa[p])) - bits_to<T>(df_lds64(ring_base + pn[p]));
                } else {
                    const long long t3 = PROF ? clock64() : 0;
                    wait_lvl(L - 1);   // near: the critical path
                    if (PROF && b == 0 && lane == 0) {
                        const long long t4 = clock64();
                        atomicAdd(a.dbg + 0, (unsigned long long)(t2b - t2));
                        atomicAdd(a.dbg + 1, (unsigned long long)(t4 - t3));
                        atomicAdd(a.dbg + 2, (unsigned long long)rtt);
                        atomicAdd(a.dbg + 3, 1ull);
                    }
                    T v[NPX][NN];
    #pragma unroll
                    for (int p = 0; p < NPX; p++)
    #pragma unroll
                        for (int j = 0; j < NN; j++) v[p][j] = bits_to<T>(df_lds64(na[p][j]));
    #pragma unroll
                    for (int p = 0; p < NPX; p++) {
    #pragma unroll
                        for (int st = 1; st < NN; st <<= 1)
    #pragma unroll
                            for (int j = 0; j < NN; j += 2 * st) v[p][j] += v[p][j + st];
                        Fx[p] = gs[p] - v[p][0];
                    }
    #pragma unroll
                    for (int p = 0; p < NPX; p++) df_stp64(sa[p], df_bits<T>(Fx[p]), stp[p]);
                    if (NPX == kNP) {
                        // passes beyond kNP: serially, all deps done (far sums in sfar)
                        for (int32_t base = lo + 32 * kNP; base < hi; base += 32) {
                            const int32_t e = base + lane;
                            const int32_t ee = e < hi ? e : base;
                            const unsigned st = stage_base + ((unsigned)(ee >> lgc) % ns) * sbytes;
                            const unsigned off = (unsigned)(ee & (ch - 1));
                            const unsigned row = st + off * (unsigned)a.kpn * 2;
                            const T g1 = bits_to<T>(df_lds64(st + nbytes + off * 8));
                            int32_t u1;
                            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(u1) : "r"(st + nbytes + gbytes + off * 4));
                            const unsigned p16 = lds32u(row + OFF_PN) & 0xffffu;
                            T sf1 = T(0);
    #pragma unroll
                            for (int k2 = 0; k2 < 2 * NH; k2++)
                                sf1 += bits_to<T>(df_lds64(sfar_base + (unsigned)(k2 * SB + (ee & (SB - 1))) * 8u));
                            const T s1 = sf1 +
                                         df_sum<T, NM>(ring_base, row) + df_sum_u16<T, NN>(ring_base, row + OFF_NEAR);
                            const T F1 = g1 - s1;
                            if (e < hi) {
                                const unsigned sl = ring_base + (unsigned)(e & a.ring_mask) * 8u;
                                asm volatile("st.shared.b64 [%0], %1;" ::"r"(sl), "l"(df_bits<T>(F1)) : "memory");
    #pragma unroll
                                for (unsigned r = 1; r <= NH; r++) cl_st_async64(cl_mapa(sl, r), df_bits<T>(F1), cl_mapa(lvl_addr, r));
                                f[(size_t)u1 * a.B + b] = F1 - bits_to<T>(df_lds64(ring_base + p16));
                            }
                        }
                    }
                    // publish locally (critical path): all 32 lanes arrive
                    asm volatile(
                        "{\n.reg .pred q;\nsetp.eq.u32 q, %0, 0;\n"
                        "mbarrier.arrive.release.cta.shared::cta.b64 _, [%1];\n"
                        "@q st.relaxed.cta.shared.s32 [%2], %3;\n}" ::"r"(lane),
                        "r"(lvl_addr), "r"(ctrl + 4), "r"(hi)
                        : "memory");
                    if (PROF && lane == 0) pubt[L & 63] = clock64();
                    // forward F to the helper's ring: each store completes its bytes
                    // on the helper's lvlbar[L % kLB] (armed there with 8 * width)
                    {
    #pragma unroll
                        for (unsigned r = 1; r <= NH; r++) {
                            const unsigned rbar = cl_mapa(lvl_addr, r);
    #pragma unroll
                            for (int p = 0; p < NPX; p++)
                                if (stp[p]) cl_st_async64(cl_mapa(sa[p], r), df_bits<T>(Fx[p]), rbar);
                        }
                    }
    #pragma unroll
                    for (int p = 0; p < NPX; p++)
                        if (stp[p]) f[(size_t)u[p] * a.B + b] = Fx[p] - bits_to<T>(df_lds64(ring_base + pn[p]));
                }
            };
            if (np <= 1)
                level(std::integral_constant<int, 1>{});
            else
                level(std::integral_constant<int, kNP>{});
        }
    }
    __syncwarp();
    cl_sync();   // neither CTA exits while its peer may still write into its shared memory
}

static size_t ringcl_smem_bytes(const RingDFPlan &R, bool cw = false) {   // owner stages; the helper stages nothing
    const size_t so = (size_t)R.nstage * R.ch * ((size_t)R.kpn * 2 + 12);
    return (size_t)(3 * R.ring + 16) * 8 + 8 * (size_t)(kMaxStageCL + 2 * kLB) + 48 + so +
           (cw ? 16 + (size_t)8 * kNP * 1024 : 0);   // RINGCW hand-off records
}

void ringcl_plan(RingDFPlan &R) {
    R.ch_h = R.ch;
    R.nstage_h = R.nstage;
    R.cl_ok = R.ok && R.fe <= 128 && ringcl_smem_bytes(R) <= kSmemCapDF;
    R.cw_ok = R.cl_ok && R.nn == 4 && R.wmax <= 32 * kNP && ringcl_smem_bytes(R, true) <= kSmemCapDF;
    // helper CTAs: 2 NH far-sum buffers of RING >> {0,1,2} entries, each
    // holding >= 10 level widths (the helpers run <= 8 levels ahead)
    R.nh_max = 1;
    if ((R.ring >> 1) >= 10 * R.wmax) R.nh_max = 2;
    if ((R.ring >> 2) >= 10 * R.wmax) R.nh_max = 3;
}

bool ringcl_fits(const RingDFPlan &R) { return R.cl_ok; }
bool ringcw_fits(const RingDFPlan &R) { return R.cw_ok; }

cudaError_t launch_moebius_ringcl(const DevPoset &P, const RingDFPlan &R, const int32_t *ru_pad,
                                  int dtype, const void *gP, void *f, int64_t B, int num_sms, cudaStream_t s,
                                  int *ctas_out) {
    // two helper CTAs per column when three SMs per column fit one wave
    // (measured on C5w: 1 helper 128.0 ms, 2 helpers 100.4, 3 helpers 103.7;
    // three stay available through the ringcl_helpers option)
    // (round 2, C5w B = 32: 3 helpers 94.9 ms vs 96.9 for int64, but 102.4 vs
    // 100.7 for fp64 -- so int64 takes three when four SMs per column fit)
    int nh = 1;
    if (R.nh_max >= 2 && 3 * B <= num_sms) nh = 2;
    if (R.nh_max >= 3 && dtype == 0 && 4 * B <= num_sms) nh = 3;
    if (R.nh_force > 0) nh = std::min(R.nh_force, R.nh_max);   // tuning option ringcl_helpers
    if (P.n == 0) return cudaSuccess;
    if (!ringcl_fits(R) || (R.cw && !ringcw_fits(R))) return cudaErrorInvalidConfiguration;
    if (R.ch_cl > 0 && R.ch_cl != R.ch) {   // tuning: another owner stage chunk (same tables)
        RingDFPlan R2 = R;
        R2.ch = R.ch_cl;
        R2.ch_h = R.ch_cl;
        R2.nstage = std::max(2, (int)(((int64_t)(kNWC + 1) * R.wmax + R.ch_cl - 1) / R.ch_cl) + 1);
        R2.nstage_h = R2.nstage;
        R2.ch_cl = 0;
        if (R2.nstage > kMaxStageCL || ringcl_smem_bytes(R2, R2.cw) > kSmemCapDF) return cudaErrorInvalidValue;
        return launch_moebius_ringcl(P, R2, ru_pad, dtype, gP, f, B, num_sms, s, ctas_out);
    }
    RDFArgs a{};
    a.Dn = R.D;
    a.Df = R.D + R.npad * R.kpn;
    a.gP = gP;
    a.ru = ru_pad;
    a.lvl_ptr = P.lvl_ptr;
    a.f = f;
    a.npad = R.npad;
    a.n = P.n;
    a.kpn = R.kpn;
    a.kpf = R.kpf;
    a.fe = R.fe;
    a.ell = P.ell;
    a.B = (int32_t)B;
    a.ring_mask = R.ring - 1;
    a.lg_ch = 0;
    while ((1 << a.lg_ch) < R.ch) a.lg_ch++;
    a.nstage = R.nstage;
    a.lg_chh = 0;
    while ((1 << a.lg_chh) < R.ch_h) a.lg_chh++;
    a.nstage_h = R.nstage_h;
    a.dbg = R.prof ? R.dbg : nullptr;   // ring_debug bit 3: wait-time counters
    a.skip_far = R.skip_far;            // timing experiments only
    a.cw_sleep = R.cw_sleep;
    const size_t smem = ringcl_smem_bytes(R, R.cw);
    void *fn = nullptr;
#define RCW_FN(NM, FEC)                                                                        \
    if (R.cw && R.nn == 4 && R.nm == NM && fec == FEC)                                         \
        fn = nh == 3 ? (dtype == 0 ? (void *)k_moeb_ringcl<u64, 4, NM, FEC, false, 3, true>    \
                                   : (void *)k_moeb_ringcl<double, 4, NM, FEC, false, 3, true>) \
           : nh == 2 ? (dtype == 0 ? (void *)k_moeb_ringcl<u64, 4, NM, FEC, false, 2, true>    \
                                   : (void *)k_moeb_ringcl<double, 4, NM, FEC, false, 2, true>) \
                     : (dtype == 0 ? (void *)k_moeb_ringcl<u64, 4, NM, FEC, false, 1, true>    \
                                   : (void *)k_moeb_ringcl<double, 4, NM, FEC, false, 1, true>);
#define RCL_FN(NN, NM, FEC)                                                                    \
    if (!R.cw && R.nn == NN && R.nm == NM && fec == FEC)                                       \
        fn = R.prof ? (dtype == 0 ? (void *)k_moeb_ringcl<u64, NN, NM, FEC, true>              \
                                  : (void *)k_moeb_ringcl<double, NN, NM, FEC, true>)          \
           : nh == 3 ? (dtype == 0 ? (void *)k_moeb_ringcl<u64, NN, NM, FEC, false, 3>         \
                                   : (void *)k_moeb_ringcl<double, NN, NM, FEC, false, 3>)     \
           : nh == 2 ? (dtype == 0 ? (void *)k_moeb_ringcl<u64, NN, NM, FEC, false, 2>         \
                                   : (void *)k_moeb_ringcl<double, NN, NM, FEC, false, 2>)     \
                     : (dtype == 0 ? (void *)k_moeb_ringcl<u64, NN, NM, FEC>                   \
                                   : (void *)k_moeb_ringcl<double, NN, NM, FEC>);
#define RCL_NM(NN, FEC) RCL_FN(NN, 16, FEC) RCL_FN(NN, 32, FEC)
#define RCL_FE(FEC) RCL_NM(4, FEC) RCL_NM(8, FEC) RCL_NM(16, FEC)
    const int fec = R.fe <= 64 ? 4 : R.fe <= 96 ? 6 : 8;   // chunks per row, split by parity
    RCL_FE(4) RCL_FE(6) RCL_FE(8)
    RCW_FN(16, 4) RCW_FN(16, 6) RCW_FN(16, 8) RCW_FN(32, 4) RCW_FN(32, 6) RCW_FN(32, 8)
#undef RCW_FN
#undef RCL_FE
#undef RCL_NM
#undef RCL_FN
    if (!fn) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    const int cdim = R.prof && !R.cw ? 2 : nh + 1;   // the instrumented build is the 1-helper kernel
    cfg.gridDim = dim3((unsigned)(cdim * B));
    cfg.blockDim = dim3(32 * kNWH);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)cdim;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // a cluster that cannot be placed at all (fewer SMs per GPC, MIG, ...)
    // falls back to fewer helpers before launching
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg) != cudaSuccess || nclusters == 0) {
        cudaGetLastError();
        if (nh > 1 && !R.prof) {
            RingDFPlan R2 = R;
            R2.nh_force = nh - 1;
            return launch_moebius_ringcl(P, R2, ru_pad, dtype, gP, f, B, num_sms, s, ctas_out);
        }
        return cudaErrorInvalidConfiguration;
    }
    void *args[] = {&a};
    if (ctas_out) *ctas_out = (int)(cdim * B);
    launches_add(1);
    return cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace poset
