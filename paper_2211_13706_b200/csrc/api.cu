// C-ABI of libposet.so -- see include/poset.h for the contract of every entry
// point.  Host setup (setup.cpp) + device residency + kernel launches
// (kernels.cu).  No compute step runs on the host: every transform step is a
// CUDA kernel; without a GPU every compute call returns POSET_ECUDA.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <initializer_list>
#include <string>
#include <vector>

#include "internal.h"
#include "kernels.cuh"

using namespace poset;

static thread_local std::string g_last_error;

static poset_status fail(poset_status s, const std::string &msg) {
    g_last_error = msg;
    return s;
}

struct poset_s {
    int device = 0;
    int num_sms = 148;
    HostPoset H;
    poset_info info{};
    int moeb_opt = MOEB_AUTO;
    cudaError_t sticky = cudaSuccess;
    // cross-stream ordering of calls on one handle, per scratch lane: a call
    // records lane_ev[l] on its stream for every lane l it uses, and a call on
    // a different stream first waits on those lanes' events -- so no scratch
    // buffer is shared by two calls in flight, while a zeta (lane Z) and a
    // ring-family Möbius (lane R) on two streams may run concurrently
    //   lane Z: d_F, d_scan, d_part, d_bar, the lazily built gather order;
    //   lanes R0 / R1: d_gPx[0] / [1] (rank-major g of the ring schedules,
    //   double-buffered: a ring-family call on another stream than the
    //   previous one takes the other buffer, so its permutation kernel runs
    //   while the previous solve still reads the first);  lane S: d_stage
    //   lanes R2 / R3: d_gPx[2] / [3], used only with option solves_inflight
    //   3 / 4 (the buffers rotate over max(2, solves_inflight) lanes)
    static constexpr int NLANES = 6;
    cudaEvent_t lane_ev[NLANES] = {};
    cudaStream_t lane_s[NLANES] = {};
    bool lane_used[NLANES] = {};
    // the ring-family solve kernels of a handle run one at a time (each
    // holds one cluster of SMs per column for the whole solve)
    cudaEvent_t solve_ev = nullptr;
    cudaStream_t solve_s = nullptr;
    bool solve_used = false;
    int solves_inflight = 1;          // option solves_inflight (1: one solve at a time; 2-4: no ordering)
    int gp_cur = 0;                   // d_gPx buffer of the current ring-family call
    cudaStream_t gp_last_s = nullptr;
    bool gp_any = false;
    int zeta_sms = 0;                 // option zeta_sms: SMs the zeta's persistent grids size for
    // device residency
    int32_t *d_rank_user = nullptr, *d_slot = nullptr, *d_chain = nullptr, *d_lvl = nullptr;
    int32_t *d_child = nullptr, *d_slot_user = nullptr, *d_M = nullptr;
    int64_t *d_child_ptr = nullptr;
    unsigned *d_bar = nullptr;
    unsigned long long *d_count = nullptr;
    RingPlan ring;                    // RING Möbius schedule (moebius_ring.cu)
    RingWSPlan rws;                   // RINGWS Möbius schedule (moebius_ringws.cu)
    RingDFPlan rdf;                   // RINGDF Möbius schedule (moebius_ringdf.cu)
    CsrRows csr;                      // sparse U-rows (moebius_csr.cu)
    bool zeta_csr = false;            // zeta gathers over the CSR rows (sparse table)
    bool sparse_only = false;         // no dense table M: rows built straight from the DAG (N1)
    unsigned setup_flags = 0;
    GatherPi gpi;                     // batched gather in the per-tile gather order (lazy)
    bool gpi_failed = false;
    // poset_shard_rows: only index rows [m_lo, m_hi) kept (d_M is then [k][m_hi - m_lo])
    bool sharded = false;
    int64_t m_lo = 0, m_hi = 0;
    bool gpi_delta_failed = false;
    void *d_gPx[4] = {};   // [B][npad] g in rank order (ring-family input)
    size_t gPx_bytes[4] = {};
    // scratch, grown on demand
    void *d_F = nullptr;
    size_t F_bytes = 0;
    void *d_scan = nullptr;
    size_t scan_bytes = 0;
    void *d_part = nullptr;
    size_t part_bytes = 0;
    void *d_stage[2] = {nullptr, nullptr};
    size_t stage_bytes[2] = {0, 0};
    // profiling: event pairs recorded on the caller's stream per kernel phase
    bool prof_on = false;
    struct Rec { int ph; cudaEvent_t a, b; };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    DevPoset dev() const {
        DevPoset P;
        P.n = H.n;
        P.k = H.k;
        P.ell = H.ell;
        P.rank_user = d_rank_user;
        P.slot = d_slot;
        P.chain = d_chain;
        P.lvl_ptr = d_lvl;
        P.child_ptr = d_child_ptr;
        P.child = d_child;
        P.slot_user = d_slot_user;
        P.M = sharded ? d_M - m_lo : d_M;
        P.ldm = sharded ? m_hi - m_lo : H.n;
        return P;
    }
};

// Errors that leave the CUDA context unusable (a fault inside a kernel) are
// sticky in the handle; recoverable ones (an allocation that does not fit, a
// launch configuration that cannot be placed, a bad argument) are returned
// once and cleared from the runtime's last-error slot so they do not leak into
// the next call on this or another handle.
static bool fatal_cuda_error(cudaError_t e) {
    switch (e) {
        case cudaErrorIllegalAddress: case cudaErrorLaunchFailure: case cudaErrorHardwareStackError:
        case cudaErrorIllegalInstruction: case cudaErrorMisalignedAddress:
        case cudaErrorInvalidAddressSpace: case cudaErrorInvalidPc: case cudaErrorLaunchTimeout:
        case cudaErrorECCUncorrectable: case cudaErrorAssert: case cudaErrorUnknown:
            return true;
        default:
            return false;
    }
}

#define CK(expr)                                                                              \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess) {                                                              \
            if (fatal_cuda_error(_e)) {                                                       \
                if (h) h->sticky = _e;                                                        \
            } else {                                                                          \
                cudaGetLastError();                                                           \
            }                                                                                 \
            return fail(_e == cudaErrorMemoryAllocation ? POSET_ENOMEM : POSET_ECUDA,         \
                        std::string(#expr) + ": " + cudaGetErrorString(_e));                  \
        }                                                                                     \
    } while (0)

static void free_all(poset_s *h) {
    if (!h) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(h->device);
    for (auto &r : h->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : h->pool) cudaEventDestroy(e);
    for (auto e : h->lane_ev)
        if (e) cudaEventDestroy(e);
    if (h->solve_ev) cudaEventDestroy(h->solve_ev);
    free_gather_pi(h->gpi);
    void *ptrs[] = {h->d_rank_user, h->d_slot, h->d_chain, h->d_lvl, h->d_child, h->d_slot_user,
                    h->d_M, h->d_child_ptr, h->d_bar, h->d_count, h->d_F, h->d_scan, h->d_part,
                    h->d_stage[0], h->d_stage[1], h->ring.D, h->ring.Pn, h->ring.ru_pad, h->rws.D, h->rdf.D, h->d_gPx[0], h->d_gPx[1], h->d_gPx[2], h->d_gPx[3], h->ring.dbg, h->csr.ptr, h->csr.idx};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    cudaSetDevice(prev);
}

template <typename T>
static cudaError_t upload(T **dst, const std::vector<T> &v) {
    size_t bytes = std::max<size_t>(v.size(), 1) * sizeof(T);
    cudaError_t e = cudaMalloc((void **)dst, bytes);
    if (e != cudaSuccess) return e;
    if (!v.empty()) e = cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
    return e;
}

// Sparse mode: the dense table does not fit (or the
// caller asked for POSET_SETUP_SPARSE) -- the U-rows are built straight from
// the DAG (build_csr_direct) and every transform runs over them: zeta by
// k_gather_csr, Möbius by the CSR schedule.  The schedules that need the
// dense table (ring family, LEVEL / GRID / WARP, the gather order) are off.
static poset_status finish_setup_sparse(poset_s *h, double t0, size_t table, size_t free_b) {
    HostPoset &H = h->H;
    CK(upload(&h->d_rank_user, H.rank_user));
    CK(upload(&h->d_slot, H.slot));
    CK(upload(&h->d_chain, H.chain));
    CK(upload(&h->d_lvl, H.lvl_ptr));
    CK(upload(&h->d_child_ptr, H.child_ptr));
    CK(upload(&h->d_child, H.child));
    CK(upload(&h->d_slot_user, H.slot_user));
    for (auto &e : h->lane_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->solve_ev, cudaEventDisableTiming));
    CK(cudaMalloc((void **)&h->d_bar, 64));
    CK(cudaMalloc((void **)&h->d_count, 64));
    int32_t *d_slot_chain = nullptr, *d_chain_off = nullptr;
    {
        std::vector<int32_t> sc((size_t)H.n);
        for (int32_t sl = 0; sl < H.n; sl++) sc[sl] = H.chain[H.slot_rank[sl]];
        CK(upload(&d_slot_chain, sc));
        CK(upload(&d_chain_off, H.chain_off));
    }
    CK(cudaDeviceSynchronize());
    double t1 = now_seconds();
    size_t fb = 0, tb = 0;
    CK(cudaMemGetInfo(&fb, &tb));
    // room left for F / g / f / staging of a batch: max(2 GiB, 1/8 of free)
    const size_t reserve = std::max<size_t>((size_t)2 << 30, fb / 8);
    DevPoset P = h->dev();
    cudaError_t e = build_csr_direct(P, H.lvl_ptr.data(), d_slot_chain, d_chain_off, h->csr,
                                     fb > reserve ? fb - reserve : 0, H.max_level_width, 0);
    cudaFree(d_slot_chain);
    cudaFree(d_chain_off);
    CK(e);
    if (!h->csr.ok) {
        char buf[256];
        snprintf(buf, sizeof buf,
                 "poset_setup: neither the dense table (%.2f GB, n=%d, k=%d) nor the sparse rows fit "
                 "(%.2f GB free)", table / 1e9, H.n, H.k, free_b / 1e9);
        return fail(POSET_ETOOBIG, buf);
    }
    h->sparse_only = true;
    h->zeta_csr = true;
    double t2 = now_seconds();
    poset_info &I = h->info;
    I.n = H.n;
    I.m = H.m;
    I.k = H.k;
    I.q = H.q;
    I.ell = H.ell;
    I.nnz = h->csr.nnz + H.n;   // + the self entries
    I.table_bytes = (int64_t)table;
    I.max_level_width = H.max_level_width;
    I.t_ingest = H.t_ingest;
    I.t_levels = H.t_levels;
    I.t_match = H.t_match;
    I.t_chains = H.t_chains;
    I.t_upload = t1 - t0;
    I.t_mtable = t2 - t1;   // the sparse rows take the dense table's place
    I.device = h->device;
    I.csr_bytes = h->csr.nnz * 4 + ((int64_t)H.n + 1) * 8;
    I.zeta_sparse = 1;
    I.moebius_kernel = MOEB_CSR;
    I.depth_u = -1;
    std::vector<int32_t>().swap(H.child);
    std::vector<int64_t>().swap(H.child_ptr);
    return POSET_OK;
}

static poset_status finish_setup(poset_s *h) {
    HostPoset &H = h->H;
    double t0 = now_seconds();
    CK(cudaSetDevice(h->device));
    CK(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device));
    // size guard: dense table + resident arrays + a B=1 F buffer
    size_t table = (size_t)H.n * (size_t)H.k * 4;
    size_t resident = table + (size_t)H.n * 4 * 6 + (size_t)H.m * 4 + (size_t)H.n * 8 + 4096;
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    h->info.table_bytes = (int64_t)table;
    h->info.k = H.k;
    const bool dense_fits = resident + (size_t)(H.n + 1) * 8 * 4 <= free_b;
    if (!dense_fits || (h->setup_flags & POSET_SETUP_SPARSE)) return finish_setup_sparse(h, t0, table, free_b);
    CK(upload(&h->d_rank_user, H.rank_user));
    CK(upload(&h->d_slot, H.slot));
    CK(upload(&h->d_chain, H.chain));
    CK(upload(&h->d_lvl, H.lvl_ptr));
    CK(upload(&h->d_child_ptr, H.child_ptr));
    CK(upload(&h->d_child, H.child));
    CK(upload(&h->d_slot_user, H.slot_user));
    for (auto &e : h->lane_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->solve_ev, cudaEventDisableTiming));
    CK(cudaMalloc((void **)&h->d_bar, 64));
    CK(cudaMalloc((void **)&h->d_count, 64));
    CK(cudaMalloc((void **)&h->d_M, std::max<size_t>(table, 4)));
    CK(cudaDeviceSynchronize());
    double t1 = now_seconds();
    DevPoset P = h->dev();
    {
        int64_t creach = 0;   // rank distance of the farthest child (host CSR, rank space)
        for (int32_t r = 0; r < H.n; r++)
            for (int64_t t = H.child_ptr[r]; t < H.child_ptr[r + 1]; t++)
                creach = std::max<int64_t>(creach, r - H.child[t]);
        CK(launch_mtable(P, h->d_M, 0, (int32_t)std::min<int64_t>(creach, INT32_MAX / 2), H.max_level_width));
    }
    CK(launch_count_nnz(h->d_M, (int64_t)H.n * H.k, H.n, h->d_count, 0));
    unsigned long long nnz = 0;
    CK(cudaMemcpy(&nnz, h->d_count, sizeof nnz, cudaMemcpyDeviceToHost));
    CK(cudaDeviceSynchronize());
    double t2 = now_seconds();
    // RING / RINGWS schedule data: reach of the dependencies, the plans, then
    // the rank-major ring-slot tables if they fit shared and device memory.
    {
        int32_t *d_slot_rank = nullptr, *d_level = nullptr;
        CK(upload(&d_slot_rank, H.slot_rank));
        CK(upload(&d_level, H.level));
        unsigned reach = 0, near3[3] = {0, 0, 0}, counts3[3] = {0, 0, 0};
        cudaError_t e = launch_reach_max(P, d_slot_rank, (unsigned *)h->d_count, 0);
        if (e == cudaSuccess) e = cudaMemcpy(&reach, h->d_count, sizeof reach, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) e = launch_near_max(P, d_level, d_slot_rank, (unsigned *)h->d_count, 0);
        if (e == cudaSuccess) e = cudaMemcpy(near3, h->d_count, sizeof near3, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) e = launch_df_counts(P, d_level, d_slot_rank, (unsigned *)h->d_count, 0);
        if (e == cudaSuccess) e = cudaMemcpy(counts3, h->d_count, sizeof counts3, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) { cudaFree(d_slot_rank); cudaFree(d_level); CK(e); }
        ring_plan(H.n, H.k, H.ell, H.max_level_width, reach, h->ring);
        ringws_plan(H.n, H.k, H.max_level_width, reach, near3, h->rws);
        ringdf_plan(H.n, H.k, H.max_level_width, reach, counts3, h->rdf);
        const int64_t npad = ((int64_t)H.n + 255) / 256 * 256;   // common to all plans
        h->ring.npad = npad;
        h->rws.npad = npad;
        h->rdf.npad = npad;
        size_t fb = 0, tb = 0;
        cudaMemGetInfo(&fb, &tb);
        const size_t reserve = (size_t)1 << 30;
        auto alloc = [&](void **p, size_t bytes) {
            if (bytes + reserve > fb || cudaMalloc(p, bytes) != cudaSuccess) { cudaGetLastError(); return false; }
            fb -= bytes;
            return true;
        };
        if ((h->ring.ok || h->rws.ok || h->rdf.ok) && !alloc((void **)&h->ring.ru_pad, (size_t)npad * 4)) {
            h->ring.ok = false;
            h->rws.ok = false;
            h->rdf.ok = false;
        }
        if (h->rdf.ok && !alloc((void **)&h->rdf.D, (size_t)npad * h->rdf.kp * 2)) h->rdf.ok = false;
        if (h->ring.ok && !(alloc((void **)&h->ring.D, (size_t)npad * h->ring.kp * 2) &&
                            alloc((void **)&h->ring.Pn, (size_t)npad * 2)))
            h->ring.ok = false;
        if (h->rws.ok && !alloc((void **)&h->rws.D, (size_t)npad * h->rws.kp * 2)) h->rws.ok = false;
        e = cudaSuccess;
        if (h->ring.ok || h->rws.ok || h->rdf.ok) {
            e = cudaMemset(h->ring.ru_pad, 0, (size_t)npad * 4);
            if (e == cudaSuccess)
                e = cudaMemcpy(h->ring.ru_pad, h->d_rank_user, (size_t)H.n * 4, cudaMemcpyDeviceToDevice);
        }
        if (e == cudaSuccess && h->ring.ok)
            e = launch_build_dist(P, d_slot_rank, h->ring.kp, h->ring.ring, npad, h->ring.D, h->ring.Pn, 0);
        if (e == cudaSuccess && h->rws.ok) e = launch_build_ringws(P, h->rws, d_level, d_slot_rank, 0);
        if (e == cudaSuccess && h->rdf.ok) e = launch_build_ringdf(P, h->rdf, d_level, d_slot_rank, 0);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        cudaFree(d_slot_rank);
        cudaFree(d_level);
        CK(e);
    }
    // sparse U-rows: for the Möbius solve when RING does not apply, and for
    // the zeta gather when the dense table is mostly ∞ (fill < 1/2)
    {
        const double fill = H.n && H.k ? (double)nnz / ((double)H.n * H.k) : 1.0;
        if (!h->ring.ok || fill < 0.5) {
            size_t fb = 0, tb = 0;
            CK(cudaMemGetInfo(&fb, &tb));
            const size_t reserve = (size_t)1 << 30;
            CK(build_csr(P, h->csr, fb > reserve ? fb - reserve : 0));
            h->zeta_csr = h->csr.ok && fill < 0.5;
        }
    }
    double t3 = now_seconds();
    poset_info &I = h->info;
    I.n = H.n;
    I.m = H.m;
    I.k = H.k;
    I.q = H.q;
    I.ell = H.ell;
    I.nnz = (int64_t)nnz;
    I.max_level_width = H.max_level_width;
    I.t_ingest = H.t_ingest;
    I.t_levels = H.t_levels;
    I.t_match = H.t_match;
    I.t_chains = H.t_chains;
    I.t_upload = t1 - t0;
    I.t_mtable = t2 - t1;
    I.device = h->device;
    I.reach = h->ring.reach;
    I.dist_bytes = (h->ring.ok ? (int64_t)h->ring.npad * (h->ring.kp * 2 + 2) : 0) +
                   (h->rws.ok ? (int64_t)h->rws.npad * h->rws.kp * 2 : 0) +
                   (h->rdf.ok ? (int64_t)h->rdf.npad * h->rdf.kp * 2 : 0);
    I.ringws = h->rws.ok ? 1 : 0;
    I.ringdf = h->rdf.ok ? (ringcl_fits(h->rdf) ? 3 : 1) | (ringcw_fits(h->rdf) ? 4 : 0) : 0;   // bit 1: RINGCL, 2: RINGCW
    I.ring_bytes = h->ring.ok ? (int64_t)h->ring.npad * (h->ring.kp * 2 + 2) : 0;
    I.rws_bytes = h->rws.ok ? (int64_t)h->rws.npad * h->rws.kp * 2 : 0;
    I.rdf_bytes = h->rdf.ok ? (int64_t)h->rdf.npad * h->rdf.kp * 2 : 0;
    I.t_dist = t3 - t2;
    I.depth_u = -1;
    I.csr_bytes = h->csr.ok ? h->csr.nnz * 4 + ((int64_t)H.n + 1) * 8 : 0;
    I.zeta_sparse = h->zeta_csr ? 1 : 0;
    I.moebius_kernel = ringcl_fits(h->rdf) ? MOEB_RINGCL   // (for a batch that fits 2 SMs per column)
                       : h->rdf.ok   ? MOEB_RINGDF
                       : h->rws.ok   ? MOEB_RINGWS
                       : h->ring.ok  ? MOEB_RING
                       : h->csr.ok ? MOEB_CSR
                                   : moebius_pick(P, 1, H.max_level_width, h->num_sms);
    // drop host arrays only the device needs
    std::vector<int32_t>().swap(H.child);
    std::vector<int64_t>().swap(H.child_ptr);
    return POSET_OK;
}

static poset_status setup_common(int64_t n, int64_t m, const int64_t *src, const int64_t *dst,
                                 int64_t k, const int64_t *cp, const int64_t *ce, bool inject,
                                 int device, poset_t *out, unsigned flags = 0) {
    if (!out) return fail(POSET_EINVAL, "poset_setup: out is null");
    *out = nullptr;
    int ndev = 0;
    cudaError_t ce_ = cudaGetDeviceCount(&ndev);
    if (ce_ != cudaSuccess || ndev == 0)
        return fail(POSET_ECUDA, std::string("poset_setup: no CUDA device: ") + cudaGetErrorString(ce_));
    if (device < 0 || device >= ndev) return fail(POSET_EINVAL, "poset_setup: bad device ordinal");
    poset_s *h = new (std::nothrow) poset_s();
    if (!h) return fail(POSET_ENOMEM, "poset_setup: out of host memory");
    h->device = device;
    h->setup_flags = flags;
    std::string err;
    poset_status st;
    try {
        st = host_ingest(n, m, src, dst, h->H, err);
        if (st == POSET_OK)
            st = inject ? host_chains_injected(h->H, k, cp, ce, err) : host_chains_matching(h->H, err);
    } catch (const std::bad_alloc &) {
        st = POSET_ENOMEM;
        err = "poset_setup: out of host memory";
    }
    if (st != POSET_OK) {
        delete h;
        return fail(st, err);
    }
    st = finish_setup(h);
    if (st != POSET_OK) {
        free_all(h);
        delete h;
        return st;
    }
    *out = h;
    return POSET_OK;
}

extern "C" {

poset_status poset_setup_ex(int64_t n, int64_t m, const int64_t *src, const int64_t *dst, int device,
                            uint32_t flags, poset_t *out) {
    if (flags & ~(uint32_t)POSET_SETUP_SPARSE) return fail(POSET_EINVAL, "poset_setup_ex: unknown flags");
    return setup_common(n, m, src, dst, 0, nullptr, nullptr, false, device, out, flags);
}

poset_status poset_setup(int64_t n, int64_t m, const int64_t *src, const int64_t *dst, int device,
                         poset_t *out) {
    return setup_common(n, m, src, dst, 0, nullptr, nullptr, false, device, out);
}

poset_status poset_setup_chains(int64_t n, int64_t m, const int64_t *src, const int64_t *dst,
                                int64_t k, const int64_t *chain_ptr, const int64_t *chain_elems,
                                int device, poset_t *out) {
    return setup_common(n, m, src, dst, k, chain_ptr, chain_elems, true, device, out);
}

}  // extern "C"

// ------------------------------------------------------------- helpers ----
static poset_status grow(poset_s *h, void **p, size_t *cap, size_t need) {
    if (need <= *cap) return POSET_OK;
    if (*p) {
        CK(cudaFree(*p));
        *p = nullptr;
        *cap = 0;
    }
    CK(cudaMalloc(p, need));
    *cap = need;
    return POSET_OK;
}

static poset_status check_call(poset_s *h, const void *a, const void *b, int64_t batch, int dt,
                               const char *fn) {
    if (!h) return fail(POSET_EINVAL, std::string(fn) + ": null handle");
    if (h->sticky != cudaSuccess)
        return fail(POSET_ECUDA, std::string(fn) + ": sticky CUDA error: " + cudaGetErrorString(h->sticky));
    if (batch <= 0) return fail(POSET_EINVAL, std::string(fn) + ": batch must be > 0");
    if (dt != POSET_I64 && dt != POSET_F64) return fail(POSET_EINVAL, std::string(fn) + ": bad dtype");
    if (h->H.n > 0 && (!a || !b)) return fail(POSET_EINVAL, std::string(fn) + ": null data pointer");
    if ((int64_t)h->H.n * batch > ((int64_t)1 << 40))
        return fail(POSET_EINVAL, std::string(fn) + ": n*batch too large");
    return POSET_OK;
}

static bool is_device_ptr(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// 32-byte aligned device memory: what the split-phase kernels' 256-bit
// vector loads and stores need (the transforms stage anything else).
static bool dev_aligned(const void *p) { return is_device_ptr(p) && ((uintptr_t)p % 32) == 0; }

enum : unsigned { LANE_Z = 1, LANE_R = 2, LANE_S = 4, LANE_R1 = 8, LANE_R2 = 16, LANE_R3 = 32, LANE_ALL = 63 };
static const unsigned LANE_OF_GP[4] = {LANE_R, LANE_R1, LANE_R2, LANE_R3};

static poset_status begin_call(poset_s *h, cudaStream_t s, unsigned lanes = LANE_ALL) {
    for (int l = 0; l < poset_s::NLANES; l++)
        if ((lanes >> l & 1) && h->lane_used[l] && s != h->lane_s[l])
            CK(cudaStreamWaitEvent(s, h->lane_ev[l], 0));
    return POSET_OK;
}

static poset_status end_call(poset_s *h, cudaStream_t s, poset_status st, unsigned lanes = LANE_ALL) {
    if (st != POSET_OK) return st;
    for (int l = 0; l < poset_s::NLANES; l++)
        if (lanes >> l & 1) {
            CK(cudaEventRecord(h->lane_ev[l], s));
            h->lane_s[l] = s;
            h->lane_used[l] = true;
        }
    return POSET_OK;
}

static poset_status ensure_F(poset_s *h, int64_t batch, cudaStream_t s) {
    size_t need = (size_t)(h->H.n + 1) * batch * 8;
    poset_status st = grow(h, &h->d_F, &h->F_bytes, need);
    if (st) return st;
    // row n is the all-zero target of ∞ entries (reading G12)
    CK(cudaMemsetAsync((char *)h->d_F + (size_t)h->H.n * batch * 8, 0, (size_t)batch * 8, s));
    return POSET_OK;
}

// CUDA-event timer around one kernel phase (only when profiling is on)
struct PhaseTimer {
    poset_s *h;
    int ph;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    static cudaEvent_t get(poset_s *h) {
        cudaEvent_t e = nullptr;
        if (!h->pool.empty()) { e = h->pool.back(); h->pool.pop_back(); }
        else cudaEventCreate(&e);
        return e;
    }
    PhaseTimer(poset_s *h_, int ph_, cudaStream_t s_) : h(h_), ph(ph_), s(s_) {
        if (h->prof_on) { a = get(h); cudaEventRecord(a, s); }
    }
    void end() {
        if (!a) return;
        cudaEvent_t b = get(h);
        cudaEventRecord(b, s);
        h->recs.push_back({ph, a, b});
        a = nullptr;
    }
    ~PhaseTimer() { end(); }
};

typedef poset_status (*device_fn)(poset_s *, const void *, void *, int64_t, int, cudaStream_t);

static int g_scan_mode = 0;   // option scan_mode (process-wide, tuning): 0 auto, 1 single pass, 2 three kernels

static poset_status zeta_dev(poset_s *h, const void *f, void *g, int64_t B, int dt, cudaStream_t s) {
    if (h->sharded)
        return fail(POSET_EINVAL, "poset_zeta: the index rows are sharded (poset_shard_rows); use the split phases");
    poset_status st = ensure_F(h, B, s);
    if (st) return st;
    st = grow(h, &h->d_scan, &h->scan_bytes, std::max(scan_scratch_bytes(h->H.n, B), scan1p_scratch_bytes(h->H.n, B)));
    if (st) return st;
    // persistent gather grids size for the zeta's SM budget (option zeta_sms:
    // the SMs a concurrent Möbius on another stream leaves free)
    const int zs = h->zeta_sms > 0 ? std::min(h->zeta_sms, h->num_sms) : h->num_sms;
    size_t pb = gather_partial_bytes(h->dev(), h->H.n, B, zs);
    if (pb) {
        st = grow(h, &h->d_part, &h->part_bytes, pb);
        if (st) return st;
    }
    DevPoset P = h->dev();
    // batched dense gather: build the gather-order table on first use (4nk
    // bytes more; if it does not fit, the rank-order kernels stay in use)
    const bool want_pi = !h->zeta_csr && B % 32 == 0 && gather_variant_get() == 0 && h->H.k > 0;
    if (want_pi && !h->gpi.ok && !h->gpi_failed) {
        size_t fb = 0, tb = 0;
        CK(cudaMemGetInfo(&fb, &tb));
        const size_t need = ((size_t)h->H.n + 256) * ((size_t)h->H.k + 2) * 4 + ((size_t)1 << 30);
        cudaError_t e = need < fb ? build_gather_pi(P, h->gpi, s) : cudaErrorMemoryAllocation;
        if (e != cudaSuccess) {
            if (fatal_cuda_error(e)) CK(e);
            cudaGetLastError();
            free_gather_pi(h->gpi);
            h->gpi_failed = true;
        }
    }
    // the delta list over the gather order (gather_delta.cu, option
    // gather_pi_cfg 4; measured slower than the default on C5w / C4w, DESIGN
    // §5.2), built on first use; if it does not fit, the default kernel serves
    if (want_pi && h->gpi.ok && !h->gpi.delta_ok && !h->gpi_delta_failed && gather_pi_cfg_get() == 4) {
        {
            int32_t *d_off = nullptr;
            cudaError_t e = cudaMalloc((void **)&d_off, ((size_t)h->H.k + 1) * 4);
            if (e == cudaSuccess)
                e = cudaMemcpy(d_off, h->H.chain_off.data(), ((size_t)h->H.k + 1) * 4, cudaMemcpyHostToDevice);
            if (e == cudaSuccess) e = build_gather_delta(P, d_off, h->gpi, s);
            cudaFree(d_off);
            if (e != cudaSuccess) {
                if (fatal_cuda_error(e)) CK(e);
                cudaGetLastError();
                h->gpi_delta_failed = true;
            }
        }
    }
    const bool use_pi = want_pi && h->gpi.ok;
    const bool use_delta = use_pi && h->gpi.delta_ok && gather_pi_cfg_get() == 4;
    h->info.gather_bytes = h->gpi.ok ? (int64_t)h->gpi.npad * (h->H.k + 1) * 4 + (h->gpi.npad / 256) * h->H.k * 8
                                           + h->gpi.nentries * 8 + (h->gpi.npad / 256 + 1) * 8
                                     : 0;
    h->info.gather_entries = h->gpi.nentries;
    h->info.gather_resets = h->gpi.nreset;
    {
        PhaseTimer t(h, POSET_PH_SCAN, s);
        if (g_scan_mode == 1 || (g_scan_mode == 0 && B <= 4))   // single pass (decoupled look-back)
            CK(launch_scan_1p(P, dt, f, h->d_F, B, h->d_scan, s));
        else
            CK(launch_scan(P, dt, f, h->d_F, 0, h->H.n, B, h->d_scan, nullptr, s));
    }
    {
        PhaseTimer t(h, POSET_PH_GATHER, s);
        if (h->zeta_csr)
            CK(launch_gather_csr(P, h->csr, dt, h->d_F, g, 0, h->H.n, B, 0, s));
        else if (use_delta)
            CK(launch_gather_delta(h->gpi, h->H.n, h->H.k, dt, h->d_F, g, B, zs, s));
        else if (use_pi)
            CK(launch_gather_pi(h->gpi, h->H.k, dt, h->d_F, g, B, zs, s));
        else
            CK(launch_gather(P, dt, h->d_F, g, 0, h->H.n, B, 0, pb ? h->d_part : nullptr, zs, s));
    }
    return POSET_OK;
}

// AUTO: the CTA-pair schedule when two SMs per column fit in one wave
static int moebius_which(const poset_s *h, int64_t B) {
    return h->moeb_opt != MOEB_AUTO ? h->moeb_opt
           : (ringcl_fits(h->rdf) && 2 * B <= h->num_sms) ? MOEB_RINGCL
           : h->rdf.ok  ? MOEB_RINGDF
           : h->rws.ok  ? MOEB_RINGWS
           : h->ring.ok ? MOEB_RING
           : h->csr.ok  ? MOEB_CSR
                        : moebius_pick(h->dev(), B, h->H.max_level_width, h->num_sms);
}

// the ring family reads only d_gP (lane R); the others use d_F / d_bar (lane Z)
static bool ring_family(int which) {
    return which == MOEB_RINGDF || which == MOEB_RINGCL || which == MOEB_RINGCW || which == MOEB_RINGWS ||
           which == MOEB_RING;
}

// one ring-family solve at a time per handle (see poset_s::solve_ev)
static poset_status solve_begin(poset_s *h, cudaStream_t s) {
    if (h->solves_inflight >= 2) return POSET_OK;   // option solves_inflight: two streams' solves overlap
    if (h->solve_used && h->solve_s != s) CK(cudaStreamWaitEvent(s, h->solve_ev, 0));
    return POSET_OK;
}
static poset_status solve_end(poset_s *h, cudaStream_t s) {
    CK(cudaEventRecord(h->solve_ev, s));
    h->solve_s = s;
    h->solve_used = true;
    return POSET_OK;
}

static poset_status moebius_dev(poset_s *h, const void *g, void *f, int64_t B, int dt, cudaStream_t s) {
    poset_status st = POSET_OK;
    void *&d_gP = h->d_gPx[h->gp_cur];
    size_t &gP_bytes = h->gPx_bytes[h->gp_cur];
    DevPoset P = h->dev();
    const int which = moebius_which(h, B);
    if (!ring_family(which) && (st = ensure_F(h, B, s))) return st;
    if (h->sharded && (which == MOEB_LEVEL || which == MOEB_GRID || which == MOEB_WARP))
        return fail(POSET_EINVAL, "poset_moebius: the index rows are sharded (poset_shard_rows); the LEVEL / "
                                  "GRID / WARP schedules read the whole table");
    if (h->sparse_only && which != MOEB_CSR)
        return fail(POSET_EINVAL, "poset_moebius: sparse-rows poset (no dense table): only the CSR schedule "
                                  "applies; use AUTO");
    if (which == MOEB_CSR) {
        if (!h->csr.ok)
            return fail(POSET_EINVAL, "poset_moebius: the CSR schedule has no sparse rows for this "
                                      "poset (not built: RING applies or memory); use AUTO");
        PhaseTimer t(h, POSET_PH_MSOLVE, s);
        h->info.moebius_sms = h->num_sms;
        CK(launch_moebius_csr(P, h->csr, dt, g, h->d_F, f, B, h->d_bar, h->num_sms, s));
        return POSET_OK;
    }
    h->info.moebius_kernel = which;
    h->info.moebius_sms = ring_family(which) ? std::min<int64_t>(B, h->num_sms) : h->num_sms;
    if (which == MOEB_RINGDF || which == MOEB_RINGCL || which == MOEB_RINGCW) {
        if (!h->rdf.ok)
            return fail(POSET_EINVAL, "poset_moebius: the RINGDF schedule does not fit this poset; use AUTO");
        if (which == MOEB_RINGCL && !ringcl_fits(h->rdf))
            return fail(POSET_EINVAL, "poset_moebius: the RINGCL schedule does not fit this poset; use AUTO");
        if (which == MOEB_RINGCW && !ringcw_fits(h->rdf))
            return fail(POSET_EINVAL, "poset_moebius: the RINGCW schedule does not fit this poset; use AUTO");
        st = grow(h, &d_gP, &gP_bytes, (size_t)B * h->rdf.npad * 8);
        if (st) return st;
        {
            PhaseTimer t(h, POSET_PH_PERM, s);
            CK(launch_to_rank_major(P, dt, g, B, h->rdf.npad, d_gP, s));
        }
        if ((st = solve_begin(h, s))) return st;
        PhaseTimer t(h, POSET_PH_MSOLVE, s);
        if (which == MOEB_RINGCL || which == MOEB_RINGCW) {
            h->rdf.cw = which == MOEB_RINGCW;
            int ctas = 0;
            cudaError_t ce = launch_moebius_ringcl(P, h->rdf, h->ring.ru_pad, dt, d_gP, f, B, h->num_sms, s,
                                                   &ctas);
            if (ce == cudaSuccess) h->info.moebius_sms = std::min(ctas, h->num_sms);
            if (ce == cudaErrorInvalidConfiguration && h->moeb_opt == MOEB_AUTO) {   // no cluster fits: RINGDF
                cudaGetLastError();
                h->info.moebius_kernel = MOEB_RINGDF;
                ce = launch_moebius_ringdf(P, h->rdf, h->ring.ru_pad, dt, d_gP, f, B, s);
            }
            CK(ce);
        } else
            CK(launch_moebius_ringdf(P, h->rdf, h->ring.ru_pad, dt, d_gP, f, B, s));
        return solve_end(h, s);
    }
    if (which == MOEB_RINGWS) {
        if (!h->rws.ok)
            return fail(POSET_EINVAL, "poset_moebius: the RINGWS schedule does not fit this poset; use AUTO");
        st = grow(h, &d_gP, &gP_bytes, (size_t)B * h->rws.npad * 8);
        if (st) return st;
        {
            PhaseTimer t(h, POSET_PH_PERM, s);
            CK(launch_to_rank_major(P, dt, g, B, h->rws.npad, d_gP, s));
        }
        if ((st = solve_begin(h, s))) return st;
        PhaseTimer t(h, POSET_PH_MSOLVE, s);
        CK(launch_moebius_ringws(P, h->rws, h->ring.ru_pad, dt, d_gP, f, B, s));
        return solve_end(h, s);
    }
    if (which == MOEB_RING) {
        if (!h->ring.ok)
            return fail(POSET_EINVAL, "poset_moebius: the RING schedule does not fit this poset "
                                      "(reach or rows too large); use AUTO");
        st = grow(h, &d_gP, &gP_bytes, (size_t)B * h->ring.npad * 8);
        if (st) return st;
        {
            PhaseTimer t(h, POSET_PH_PERM, s);
            CK(launch_to_rank_major(P, dt, g, B, h->ring.npad, d_gP, s));
        }
        if ((st = solve_begin(h, s))) return st;
        PhaseTimer t(h, POSET_PH_MSOLVE, s);
        CK(launch_moebius_ring(P, h->ring, dt, d_gP, f, B, s));
        return solve_end(h, s);
    }
    {
        PhaseTimer t(h, POSET_PH_MSOLVE, s);
        CK(launch_moebius_solve(P, h->H.lvl_ptr.data(), dt, g, h->d_F, B, which, h->d_bar,
                                h->num_sms, s));
    }
    {
        PhaseTimer t(h, POSET_PH_DIFF, s);
        CK(launch_chain_diff(P, dt, h->d_F, f, B, s));
    }
    return POSET_OK;
}

// Host buffers (and device buffers not 32-byte aligned, which the 256-bit
// vector loads/stores need) are staged through handle-owned device buffers:
// copy in, kernels, copy out -- all on `s`.
static poset_status run_staged(poset_s *h, device_fn fn, const void *in, void *out, int64_t B,
                               int dt, cudaStream_t s) {
    bool din = is_device_ptr(in) && ((uintptr_t)in % 32) == 0;
    bool dout = is_device_ptr(out) && ((uintptr_t)out % 32) == 0;
    size_t bytes = (size_t)h->H.n * B * 8;
    const void *src = in;
    void *dst = out;
    if (!din) {
        poset_status st = grow(h, &h->d_stage[0], &h->stage_bytes[0], bytes);
        if (st) return st;
        PhaseTimer t(h, POSET_PH_H2D, s);
        CK(cudaMemcpyAsync(h->d_stage[0], in, bytes, cudaMemcpyDefault, s));
        src = h->d_stage[0];
    }
    if (!dout) {
        poset_status st = grow(h, &h->d_stage[1], &h->stage_bytes[1], bytes);
        if (st) return st;
        dst = h->d_stage[1];
    }
    poset_status st = fn(h, src, dst, B, dt, s);
    if (st) return st;
    if (!dout) {
        PhaseTimer t(h, POSET_PH_D2H, s);
        CK(cudaMemcpyAsync(out, dst, bytes, cudaMemcpyDefault, s));
    }
    return POSET_OK;
}

static bool needs_staging(const void *in, const void *out) {
    return !(is_device_ptr(in) && ((uintptr_t)in % 32) == 0) || !(is_device_ptr(out) && ((uintptr_t)out % 32) == 0);
}

extern "C" {

poset_status poset_zeta(poset_t h, const void *f, void *g, int64_t batch, poset_dtype dt, void *stream) {
    poset_status st = check_call(h, f, g, batch, dt, "poset_zeta");
    if (st || h->H.n == 0) return st;
    CK(cudaSetDevice(h->device));
    cudaStream_t s = (cudaStream_t)stream;
    const unsigned lanes = LANE_Z | (needs_staging(f, g) ? LANE_S : 0);
    if ((st = begin_call(h, s, lanes))) return st;
    return end_call(h, s, run_staged(h, zeta_dev, f, g, batch, dt, s), lanes);
}

poset_status poset_moebius(poset_t h, const void *g, void *f, int64_t batch, poset_dtype dt,
                           void *stream) {
    poset_status st = check_call(h, g, f, batch, dt, "poset_moebius");
    if (st || h->H.n == 0) return st;
    CK(cudaSetDevice(h->device));
    cudaStream_t s = (cudaStream_t)stream;
    const bool ringf = ring_family(moebius_which(h, batch));
    if (ringf) {   // the other rank-major buffer when the stream changes (see poset_s::d_gPx)
        if (h->gp_any && s != h->gp_last_s) h->gp_cur = (h->gp_cur + 1) % std::max(2, h->solves_inflight);
        h->gp_last_s = s;
        h->gp_any = true;
    }
    const unsigned lanes = (ringf ? LANE_OF_GP[h->gp_cur] : LANE_Z) | (needs_staging(g, f) ? LANE_S : 0);
    if ((st = begin_call(h, s, lanes))) return st;
    return end_call(h, s, run_staged(h, moebius_dev, g, f, batch, dt, s), lanes);
}

// Split phases: caller pointers go straight to the kernels (no staging), so
// they must be device memory: [n][B] arrays 32-byte aligned (256-bit vector
// accesses), the small tail / carry arrays 8-byte aligned (scalar accesses).
static poset_status check_split(const char *fn, std::initializer_list<const void *> arrays,
                                std::initializer_list<const void *> small = {}) {
    for (const void *p : arrays)
        if (p && !dev_aligned(p))
            return fail(POSET_EINVAL, std::string(fn) + ": [n][B] arrays must be 32-byte aligned "
                                                        "device pointers (split phases do not stage)");
    for (const void *p : small)
        if (p && !(is_device_ptr(p) && (uintptr_t)p % 8 == 0))
            return fail(POSET_EINVAL, std::string(fn) + ": tail / carry must be 8-byte aligned "
                                                        "device pointers");
    return POSET_OK;
}

poset_status poset_scan_slots_mc(poset_t h, const void *f, void *F_mc, void *tail, int64_t lo, int64_t hi,
                                 int64_t batch, poset_dtype dt, void *stream) {
    poset_status st = check_call(h, f, F_mc, batch, dt, "poset_scan_slots_mc");
    if (st) return st;
    if (lo < 0 || hi > h->H.n || lo > hi || !tail) return fail(POSET_EINVAL, "poset_scan_slots_mc: bad range");
    CK(cudaSetDevice(h->device));
    if ((st = check_split("poset_scan_slots_mc", {f}, {tail}))) return st;
    if ((uintptr_t)F_mc % 8) return fail(POSET_EINVAL, "poset_scan_slots_mc: F_mc must be 8-byte aligned");
    cudaStream_t s = (cudaStream_t)stream;
    if ((st = begin_call(h, s))) return st;
    st = grow(h, &h->d_scan, &h->scan_bytes, scan_scratch_bytes(hi - lo, batch));
    if (st) return st;
    CK(launch_scan(h->dev(), dt, f, nullptr, lo, hi, batch, h->d_scan, tail, s, F_mc));
    return end_call(h, s, POSET_OK);
}

poset_status poset_scan_slots(poset_t h, const void *f, void *F, void *tail, int64_t lo, int64_t hi,
                              int64_t batch, poset_dtype dt, void *stream) {
    poset_status st = check_call(h, f, F, batch, dt, "poset_scan_slots");
    if (st) return st;
    if (lo < 0 || hi > h->H.n || lo > hi || !tail) return fail(POSET_EINVAL, "poset_scan_slots: bad range");
    CK(cudaSetDevice(h->device));
    if ((st = check_split("poset_scan_slots", {f, F}, {tail}))) return st;
    cudaStream_t s = (cudaStream_t)stream;
    if ((st = begin_call(h, s))) return st;
    st = grow(h, &h->d_scan, &h->scan_bytes, scan_scratch_bytes(hi - lo, batch));
    if (st) return st;
    CK(launch_scan(h->dev(), dt, f, F, lo, hi, batch, h->d_scan, tail, s));
    return end_call(h, s, POSET_OK);
}

poset_status poset_scan_carry(poset_t h, void *F, const void *carry, int64_t lo, int64_t hi,
                              int64_t batch, poset_dtype dt, void *stream) {
    poset_status st = check_call(h, F, carry, batch, dt, "poset_scan_carry");
    if (st) return st;
    if (lo < 0 || hi > h->H.n || lo > hi) return fail(POSET_EINVAL, "poset_scan_carry: bad range");
    // the carry reaches the rows before the first chain start at or after lo
    const std::vector<int32_t> &off = h->H.chain_off;
    auto itr = std::lower_bound(off.begin(), off.end() - 1, (int32_t)lo);
    int64_t end = itr == off.end() - 1 ? hi : std::min<int64_t>(hi, *itr);
    CK(cudaSetDevice(h->device));
    if ((st = check_split("poset_scan_carry", {F}, {carry}))) return st;
    cudaStream_t s = (cudaStream_t)stream;
    if ((st = begin_call(h, s))) return st;
    CK(launch_scan_carry(h->dev(), dt, F, carry, lo, end, batch, s));
    return end_call(h, s, POSET_OK);
}

poset_status poset_gather_rows(poset_t h, const void *F, void *g_rank, int64_t lo, int64_t hi,
                               int64_t batch, poset_dtype dt, void *stream) {
    poset_status st = check_call(h, F, g_rank, batch, dt, "poset_gather_rows");
    if (st) return st;
    if (lo < 0 || hi > h->H.n || lo > hi) return fail(POSET_EINVAL, "poset_gather_rows: bad range");
    if (h->sharded && hi > lo && (lo < h->m_lo || hi > h->m_hi))
        return fail(POSET_EINVAL, "poset_gather_rows: rows outside the kept shard (poset_shard_rows)");
    CK(cudaSetDevice(h->device));
    if ((st = check_split("poset_gather_rows", {F, g_rank}))) return st;
    cudaStream_t s = (cudaStream_t)stream;
    if ((st = begin_call(h, s))) return st;
    if (h->zeta_csr) {
        CK(launch_gather_csr(h->dev(), h->csr, dt, F, g_rank, lo, hi, batch, 1, s));
        return end_call(h, s, POSET_OK);
    }
    size_t pb = gather_partial_bytes(h->dev(), hi - lo, batch, h->num_sms);
    if (pb) {
        st = grow(h, &h->d_part, &h->part_bytes, pb);
        if (st) return st;
    }
    CK(launch_gather(h->dev(), dt, F, g_rank, lo, hi, batch, 1, pb ? h->d_part : nullptr, h->num_sms, s));
    return end_call(h, s, POSET_OK);
}

poset_status poset_shard_rows(poset_t h, int64_t lo, int64_t hi, uint32_t flags) {
    if (!h) return fail(POSET_EINVAL, "poset_shard_rows: null handle");
    const HostPoset &H = h->H;
    if (lo < 0 || hi > H.n || lo > hi) return fail(POSET_EINVAL, "poset_shard_rows: bad range");
    if (h->sparse_only || h->zeta_csr || !h->d_M)
        return fail(POSET_EINVAL, "poset_shard_rows: the zeta of this poset does not gather from the dense table");
    if (h->sharded) return fail(POSET_EINVAL, "poset_shard_rows: already sharded");
    CK(cudaSetDevice(h->device));
    CK(cudaDeviceSynchronize());   // no call may still read the whole table
    const int64_t w = hi - lo;
    int32_t *Mc = nullptr;
    cudaError_t e = cudaMalloc((void **)&Mc, std::max<size_t>((size_t)w * H.k * 4, 4));
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        return fail(POSET_ENOMEM, "poset_shard_rows: no room for the kept rows");
    }
    CK(e);
    if (w > 0 && H.k > 0)
        CK(cudaMemcpy2D(Mc, (size_t)w * 4, h->d_M + lo, (size_t)H.n * 4, (size_t)w * 4, (size_t)H.k,
                        cudaMemcpyDeviceToDevice));
    CK(cudaDeviceSynchronize());
    cudaFree(h->d_M);
    h->d_M = Mc;
    h->sharded = true;
    h->m_lo = lo;
    h->m_hi = hi;
    free_gather_pi(h->gpi);     // built from the whole table; zeta is refused from now on
    h->gpi_failed = true;
    if (flags & POSET_SHARD_DROP_MOEBIUS) {   // ranks that never run the Möbius solve
        void *ptrs[] = {h->ring.D, h->ring.Pn, h->rws.D, h->rdf.D, h->csr.ptr, h->csr.idx};
        for (void *p : ptrs)
            if (p) cudaFree(p);
        h->ring.D = nullptr; h->ring.Pn = nullptr; h->rws.D = nullptr; h->rdf.D = nullptr;
        h->csr.ptr = nullptr; h->csr.idx = nullptr;
        h->ring.ok = h->rws.ok = h->rdf.ok = h->csr.ok = false;
        h->rdf.cl_ok = h->rdf.cw_ok = false;
        h->info.dist_bytes = h->info.ring_bytes = h->info.rws_bytes = h->info.rdf_bytes = h->info.csr_bytes = 0;
        h->info.ringws = h->info.ringdf = 0;
    }
    h->info.table_bytes = w * H.k * 4;
    return POSET_OK;
}

poset_status poset_combine_tails(poset_t h, const void *tails_all, int64_t world, int64_t rank,
                                 void *carry_out, int64_t batch, poset_dtype dt, void *stream) {
    poset_status st = check_call(h, tails_all, carry_out, batch, dt, "poset_combine_tails");
    if (st) return st;
    if (world <= 0 || rank < 0 || rank >= world) return fail(POSET_EINVAL, "poset_combine_tails: bad rank");
    CK(cudaSetDevice(h->device));
    if ((st = check_split("poset_combine_tails", {}, {tails_all, carry_out}))) return st;
    cudaStream_t s = (cudaStream_t)stream;
    if ((st = begin_call(h, s))) return st;
    CK(launch_combine_tails(dt, tails_all, world, rank, carry_out, batch, s));
    return end_call(h, s, POSET_OK);
}

poset_status poset_rank_to_user(poset_t h, const void *g_rank, void *g_user, int64_t batch,
                                poset_dtype dt, void *stream) {
    poset_status st = check_call(h, g_rank, g_user, batch, dt, "poset_rank_to_user");
    if (st) return st;
    CK(cudaSetDevice(h->device));
    if ((st = check_split("poset_rank_to_user", {g_rank, g_user}))) return st;
    cudaStream_t s = (cudaStream_t)stream;
    if ((st = begin_call(h, s))) return st;
    CK(launch_rank_to_user(h->dev(), dt, g_rank, g_user, batch, s));
    return end_call(h, s, POSET_OK);
}

poset_status poset_analyze(int64_t n, int64_t m, const int64_t *src, const int64_t *dst,
                           poset_info *out, int64_t *chain, int64_t *pos, int64_t *level) {
    if (!out) return fail(POSET_EINVAL, "poset_analyze: out is null");
    HostPoset H;
    std::string err;
    poset_status st;
    try {
        st = host_ingest(n, m, src, dst, H, err);
        if (st == POSET_OK) st = host_chains_matching(H, err);
    } catch (const std::bad_alloc &) {
        st = POSET_ENOMEM;
        err = "poset_analyze: out of host memory";
    }
    if (st != POSET_OK) return fail(st, err);
    poset_info I{};
    I.n = H.n;
    I.m = H.m;
    I.k = H.k;
    I.q = H.q;
    I.ell = H.ell;
    I.nnz = -1;
    I.depth_u = -1;
    I.table_bytes = (int64_t)H.n * H.k * 4;
    I.max_level_width = H.max_level_width;
    I.t_ingest = H.t_ingest;
    I.t_levels = H.t_levels;
    I.t_match = H.t_match;
    I.t_chains = H.t_chains;
    I.device = -1;
    *out = I;
    for (int32_t r = 0; r < H.n; r++) {
        int32_t u = H.rank_user[r];
        if (chain) chain[u] = H.chain[r];
        if (pos) pos[u] = H.pos[r];
        if (level) level[u] = H.level[r];
    }
    return POSET_OK;
}

poset_status poset_query(poset_t h, poset_info *out) {
    if (!h || !out) return fail(POSET_EINVAL, "poset_query: null argument");
    *out = h->info;
    out->num_sms = h->num_sms;
    return POSET_OK;
}

poset_status poset_set_option(poset_t h, const char *key, int64_t value) {
    if (!h || !key) return fail(POSET_EINVAL, "poset_set_option: null argument");
    if (!strcmp(key, "moebius_kernel")) {
        if (value < MOEB_AUTO || value > MOEB_RINGCW) return fail(POSET_EINVAL, "poset_set_option: bad value");
        h->moeb_opt = (int)value;
        return POSET_OK;
    }
    if (!strcmp(key, "ring_lpe")) {   // lanes per element of the RING schedule (tuning)
        const int64_t E = h->ring.entries ? h->ring.entries / value : 0;
        if (!h->ring.ok || value < 1 || value > 32 || (value & (value - 1)) || E < 8 || E > 64)
            return fail(POSET_EINVAL, "poset_set_option: ring_lpe must be a power of two with "
                                      "8 <= entries/ring_lpe <= 64");
        h->ring.lpe = (int32_t)value;
        return POSET_OK;
    }
    if (!strcmp(key, "ringws_nwo") || !strcmp(key, "ringws_lpeo")) {   // RINGWS tuning
        if (!h->rws.ok) return fail(POSET_EINVAL, "poset_set_option: RINGWS is not available");
        if (!strcmp(key, "ringws_nwo")) {
            if (value != 4 && value != 8 && value != 12) return fail(POSET_EINVAL, "ringws_nwo is 4, 8 or 12");
            h->rws.nwo = (int32_t)value;
        } else {
            const int64_t E = h->rws.fe / (value > 0 ? value : 1);
            if (value < 4 || value > 32 || (value & (value - 1)) || (E != 8 && E != 16))
                return fail(POSET_EINVAL, "ringws_lpeo must leave 8 or 16 far entries per lane");
            h->rws.lpeo = (int32_t)value;
        }
        return POSET_OK;
    }
    if (!strcmp(key, "solves_inflight")) {   // 2: ring-family solves on two streams may overlap
        if (value < 1 || value > 4) return fail(POSET_EINVAL, "poset_set_option: solves_inflight is 1..4");
        h->solves_inflight = (int)value;
        h->gp_cur %= std::max(2, h->solves_inflight);
        return POSET_OK;
    }
    if (!strcmp(key, "zeta_sms")) {   // SMs the zeta's persistent grids size for (0 = all)
        if (value < 0 || value > 4096) return fail(POSET_EINVAL, "poset_set_option: zeta_sms is 0..4096");
        h->zeta_sms = (int)value;
        return POSET_OK;
    }
    if (!strcmp(key, "scan_mode")) {   // process-wide zeta scan choice (tuning)
        if (value < 0 || value > 2) return fail(POSET_EINVAL, "scan_mode is 0..2");
        g_scan_mode = (int)value;
        return POSET_OK;
    }
    if (!strcmp(key, "ringcl_chunk")) {   // RINGCL owner stage chunk, ranks (tuning; 0 = the plan's)
        if (value != 0 && value != 32 && value != 64 && value != 128 && value != 256)
            return fail(POSET_EINVAL, "ringcl_chunk is 0, 32, 64, 128 or 256");
        h->rdf.ch_cl = (int32_t)value;
        return POSET_OK;
    }
    if (!strcmp(key, "ringcl_helpers")) {   // RINGCL helper CTAs per column (tuning; 0 = auto)
        if (value < 0 || value > 3) return fail(POSET_EINVAL, "ringcl_helpers is 0..3");
        h->rdf.nh_force = (int32_t)value;
        return POSET_OK;
    }
    if (!strcmp(key, "ring_debug")) {   // timing experiments only (bit 0: results NOT valid,
                                         // bit 3: instrumented RINGDF -> poset_debug_read)
        h->ring.debug = (int32_t)(value & 1);
        if (!h->ring.dbg) CK(cudaMalloc((void **)&h->ring.dbg, 64));
        CK(cudaMemset(h->ring.dbg, 0, 64));
        h->rdf.prof = (value & 8) != 0;
        h->rdf.skip_far = (int32_t)((value >> 4) & 7);   // bits 4-6: RINGDF without far / mid / near sums
        h->rdf.dbg = h->ring.dbg;
        return POSET_OK;
    }
    if (!strcmp(key, "ringcw_sleep")) {   // RINGCW level warps: ns between level polls (tuning)
        if (value < 0 || value > 100000) return fail(POSET_EINVAL, "poset_set_option: ringcw_sleep is 0..100000");
        h->rdf.cw_sleep = (int32_t)value;
        return POSET_OK;
    }
    if (!strcmp(key, "gather_variant")) {   // process-wide dense-gather kernel choice (tuning)
        if (value < 0 || value > 4) return fail(POSET_EINVAL, "poset_set_option: gather_variant is 0..4");
        set_gather_variant((int)value);
        return POSET_OK;
    }
    if (!strcmp(key, "gather_pi_cfg")) {   // process-wide gather-order kernel configuration (tuning)
        if (value < 0 || value > 7) return fail(POSET_EINVAL, "poset_set_option: gather_pi_cfg is 0..7");
        set_gather_pi_cfg((int)value);
        return POSET_OK;
    }
    if (!strcmp(key, "compute_depth_u")) {
        if (h->sparse_only || h->sharded)
            return fail(POSET_EINVAL, "compute_depth_u: needs the whole dense table (sparse-rows or sharded poset)");
        CK(cudaSetDevice(h->device));
        double t0 = now_seconds();
        int32_t *d_sr = nullptr, *d_D = nullptr;
        cudaError_t e = upload(&d_sr, h->H.slot_rank);
        if (e == cudaSuccess) e = cudaMalloc((void **)&d_D, std::max<size_t>((size_t)h->H.n * 4, 4));
        if (e == cudaSuccess) e = launch_depth_u(h->dev(), d_sr, d_D, (unsigned *)h->d_count, 0);
        unsigned du = 0;
        if (e == cudaSuccess) e = cudaMemcpy(&du, h->d_count, sizeof du, cudaMemcpyDeviceToHost);
        cudaFree(d_sr);
        cudaFree(d_D);
        CK(e);
        h->info.depth_u = du;
        h->info.t_depth = now_seconds() - t0;
        return POSET_OK;
    }
    if (!strcmp(key, "profile")) {
        h->prof_on = value != 0;
        return POSET_OK;
    }
    return fail(POSET_EINVAL, std::string("poset_set_option: unknown key ") + key);
}

poset_status poset_profile_read(poset_t h, double *ms, int64_t *calls, int64_t *launches) {
    if (!h) return fail(POSET_EINVAL, "poset_profile_read: null handle");
    double acc[POSET_PH_COUNT] = {0};
    int64_t cnt[POSET_PH_COUNT] = {0};
    CK(cudaSetDevice(h->device));
    for (auto &r : h->recs) {
        CK(cudaEventSynchronize(r.b));
        float t = 0;
        CK(cudaEventElapsedTime(&t, r.a, r.b));
        acc[r.ph] += t;
        cnt[r.ph]++;
        h->pool.push_back(r.a);
        h->pool.push_back(r.b);
    }
    h->recs.clear();
    for (int i = 0; i < POSET_PH_COUNT; i++) {
        if (ms) ms[i] = acc[i];
        if (calls) calls[i] = cnt[i];
    }
    int64_t l = launches_take();
    if (launches) *launches = l;
    return POSET_OK;
}

poset_status poset_export_chains(poset_t h, int64_t *chain, int64_t *pos, int64_t *level, int64_t *rank) {
    if (!h || !chain || !pos || !level || !rank) return fail(POSET_EINVAL, "poset_export_chains: null argument");
    const HostPoset &H = h->H;
    for (int32_t r = 0; r < H.n; r++) {
        int32_t u = H.rank_user[r];
        chain[u] = H.chain[r];
        pos[u] = H.pos[r];
        level[u] = H.level[r];
        rank[u] = r;
    }
    return POSET_OK;
}

poset_status poset_debug_read(poset_t h, int64_t *out8) {
    if (!h || !out8) return fail(POSET_EINVAL, "poset_debug_read: null argument");
    CK(cudaSetDevice(h->device));
    if (!h->ring.dbg) { for (int i = 0; i < 8; i++) out8[i] = 0; return POSET_OK; }
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out8, h->ring.dbg, 64, cudaMemcpyDeviceToHost));
    return POSET_OK;
}

poset_status poset_export_mtable(poset_t h, int32_t *out) {
    if (!h || !out) return fail(POSET_EINVAL, "poset_export_mtable: null argument");
    if (h->sharded) return fail(POSET_EINVAL, "poset_export_mtable: the index rows are sharded");
    const HostPoset &H = h->H;
    if (h->sparse_only) {   // from the U-rows: own chain = pos(x), the rest from the row, ∞ = -1
        std::vector<int64_t> ptr((size_t)H.n + 1);
        std::vector<int32_t> idx((size_t)std::max<int64_t>(h->csr.nnz, 1));
        CK(cudaSetDevice(h->device));
        CK(cudaMemcpy(ptr.data(), h->csr.ptr, ptr.size() * 8, cudaMemcpyDeviceToHost));
        if (h->csr.nnz) CK(cudaMemcpy(idx.data(), h->csr.idx, (size_t)h->csr.nnz * 4, cudaMemcpyDeviceToHost));
        for (int32_t r = 0; r < H.n; r++) {
            int32_t *row = out + (size_t)H.rank_user[r] * H.k;
            for (int32_t j = 0; j < H.k; j++) row[j] = -1;
            row[H.chain[r]] = H.pos[r];
            for (int64_t e = ptr[r]; e < ptr[r + 1]; e++) {
                const int32_t sl = idx[e], q = H.slot_rank[sl];
                row[H.chain[q]] = H.pos[q];
            }
        }
        return POSET_OK;
    }
    std::vector<int32_t> M((size_t)H.n * H.k);
    CK(cudaSetDevice(h->device));
    if (!M.empty()) CK(cudaMemcpy(M.data(), h->d_M, M.size() * 4, cudaMemcpyDeviceToHost));
    for (int32_t j = 0; j < H.k; j++)
        for (int32_t r = 0; r < H.n; r++) {
            int32_t v = M[(size_t)j * H.n + r];
            out[(size_t)H.rank_user[r] * H.k + j] = v == H.n ? -1 : v - H.chain_off[j];
        }
    return POSET_OK;
}

poset_status poset_sync(poset_t h, void *stream) {
    if (!h) return fail(POSET_EINVAL, "poset_sync: null handle");
    CK(cudaSetDevice(h->device));
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    return POSET_OK;
}

void poset_destroy(poset_t h) {
    if (!h) return;
    free_all(h);
    delete h;
}

const char *poset_strerror(poset_status s) {
    switch (s) {
        case POSET_OK: return "ok";
        case POSET_EINVAL: return "invalid argument";
        case POSET_ESELFLOOP: return "self loop";
        case POSET_ECYCLE: return "cycle";
        case POSET_ENOTCHAIN: return "not a chain";
        case POSET_ENOTPARTITION: return "not a partition";
        case POSET_ETOOBIG: return "dense table too big for device memory";
        case POSET_ENOMEM: return "out of host memory";
        case POSET_ECUDA: return "CUDA error";
    }
    return "unknown";
}

const char *poset_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"

// ---------------------------------------------- NVLS multicast buffers ----
// Driver entry points fetched through the runtime (no link against libcuda).
namespace {
struct Drv {
    bool ok = false;
    decltype(&cuDeviceGet) DeviceGet;
    decltype(&cuMulticastCreate) McCreate;
    decltype(&cuMulticastGetGranularity) McGran;
    decltype(&cuMulticastAddDevice) McAdd;
    decltype(&cuMulticastBindMem) McBind;
    decltype(&cuMulticastUnbind) McUnbind;
    decltype(&cuMemGetAllocationGranularity) MemGran;
    decltype(&cuMemCreate) MemCreate;
    decltype(&cuMemRelease) MemRelease;
    decltype(&cuMemAddressReserve) AddrReserve;
    decltype(&cuMemAddressFree) AddrFree;
    decltype(&cuMemMap) Map;
    decltype(&cuMemUnmap) Unmap;
    decltype(&cuMemSetAccess) SetAccess;
    decltype(&cuDeviceGetAttribute) DevAttr;
};
template <class F>
bool entry(const char *name, F &fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion(name, &p, 12030, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p) {
        cudaGetLastError();
        return false;
    }
    fn = reinterpret_cast<F>(p);
    return true;
}
const Drv &drv() {
    static Drv d = [] {
        Drv x;
        x.ok = entry("cuDeviceGet", x.DeviceGet) && entry("cuMulticastCreate", x.McCreate) &&
               entry("cuMulticastGetGranularity", x.McGran) && entry("cuMulticastAddDevice", x.McAdd) &&
               entry("cuMulticastBindMem", x.McBind) && entry("cuMulticastUnbind", x.McUnbind) &&
               entry("cuMemGetAllocationGranularity", x.MemGran) && entry("cuMemCreate", x.MemCreate) &&
               entry("cuMemRelease", x.MemRelease) && entry("cuMemAddressReserve", x.AddrReserve) &&
               entry("cuMemAddressFree", x.AddrFree) && entry("cuMemMap", x.Map) && entry("cuMemUnmap", x.Unmap) &&
               entry("cuMemSetAccess", x.SetAccess) && entry("cuDeviceGetAttribute", x.DevAttr);
        return x;
    }();
    return d;
}
}  // namespace

struct poset_nvls_s {
    int ndev = 0;
    std::vector<int> dev;
    size_t size = 0;
    CUmemGenericAllocationHandle mc = 0;
    std::vector<CUmemGenericAllocationHandle> mem;
    std::vector<CUdeviceptr> uc;
    CUdeviceptr mcva = 0;
    std::vector<bool> bound, mapped;
    bool mc_mapped = false;
};

static void nvls_release(poset_nvls_s *b) {
    const Drv &d = drv();
    if (!b || !d.ok) return;
    if (b->mc_mapped) { d.Unmap(b->mcva, b->size); }
    if (b->mcva) d.AddrFree(b->mcva, b->size);
    for (int i = 0; i < b->ndev; i++) {
        if (b->mapped[i]) d.Unmap(b->uc[i], b->size);
        if (b->uc[i]) d.AddrFree(b->uc[i], b->size);
        if (b->bound[i]) {
            CUdevice cd;
            if (d.DeviceGet(&cd, b->dev[i]) == CUDA_SUCCESS) d.McUnbind(b->mc, cd, 0, b->size);
        }
        if (b->mem[i]) d.MemRelease(b->mem[i]);
    }
    if (b->mc) d.MemRelease(b->mc);
}

#define CU(expr, what)                                                                           \
    do {                                                                                         \
        CUresult _r = (expr);                                                                    \
        if (_r != CUDA_SUCCESS) {                                                                \
            nvls_release(b);                                                                     \
            delete b;                                                                            \
            return fail(_r == CUDA_ERROR_OUT_OF_MEMORY ? POSET_ENOMEM : POSET_ECUDA,             \
                        std::string("poset_nvls_create: ") + what + " failed (CUresult " +       \
                            std::to_string((int)_r) + ")");                                      \
        }                                                                                        \
    } while (0)

extern "C" {

poset_status poset_nvls_create(const int *devices, int ndev, int64_t bytes, poset_nvls_t *out) {
    if (!out || !devices || ndev < 1 || ndev > 64 || bytes <= 0)
        return fail(POSET_EINVAL, "poset_nvls_create: bad argument");
    *out = nullptr;
    const Drv &d = drv();
    if (!d.ok) return fail(POSET_ECUDA, "poset_nvls_create: driver multicast entry points unavailable");
    poset_nvls_s *b = new poset_nvls_s();
    b->ndev = ndev;
    b->dev.assign(devices, devices + ndev);
    b->mem.assign(ndev, 0);
    b->uc.assign(ndev, 0);
    b->bound.assign(ndev, false);
    b->mapped.assign(ndev, false);
    std::vector<CUdevice> cd(ndev);
    for (int i = 0; i < ndev; i++) {
        if (cudaSetDevice(devices[i]) != cudaSuccess || cudaFree(nullptr) != cudaSuccess) {   // context
            cudaGetLastError();
            delete b;
            return fail(POSET_EINVAL, "poset_nvls_create: bad device ordinal");
        }
        CU(d.DeviceGet(&cd[i], devices[i]), "cuDeviceGet");
        int sup = 0;
        CU(d.DevAttr(&sup, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cd[i]), "cuDeviceGetAttribute");
        if (!sup) {
            delete b;
            return fail(POSET_ECUDA, "poset_nvls_create: device does not support multicast (NVLS)");
        }
    }
    // the driver wants an exportable handle type on the object (the POSIX fd
    // type; nothing is exported here), NONE as a fallback
    CUmulticastObjectProp mp = {};
    mp.numDevices = (unsigned)ndev;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = (size_t)bytes;
    size_t mg = 0, ag = 0;
    CU(d.McGran(&mg, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity");
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = devices[0];
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CU(d.MemGran(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity");
    const size_t gran = std::max(mg, ag);
    b->size = ((size_t)bytes + gran - 1) / gran * gran;
    mp.size = b->size;
    if (d.McCreate(&b->mc, &mp) != CUDA_SUCCESS) {
        b->mc = 0;
        mp.handleTypes = CU_MEM_HANDLE_TYPE_NONE;
        ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_NONE;
        CU(d.McCreate(&b->mc, &mp), "cuMulticastCreate");
    }
    for (int i = 0; i < ndev; i++) CU(d.McAdd(b->mc, cd[i]), "cuMulticastAddDevice");
    std::vector<CUmemAccessDesc> acc(ndev);
    for (int i = 0; i < ndev; i++) {
        acc[i].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        acc[i].location.id = devices[i];
        acc[i].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    }
    for (int i = 0; i < ndev; i++) {
        cudaSetDevice(devices[i]);
        ap.location.id = devices[i];
        CU(d.MemCreate(&b->mem[i], b->size, &ap, 0), "cuMemCreate");
        CU(d.McBind(b->mc, 0, b->mem[i], 0, b->size, 0), "cuMulticastBindMem");
        b->bound[i] = true;
        CU(d.AddrReserve(&b->uc[i], b->size, gran, 0, 0), "cuMemAddressReserve");
        CU(d.Map(b->uc[i], b->size, 0, b->mem[i], 0), "cuMemMap");
        b->mapped[i] = true;
        CU(d.SetAccess(b->uc[i], b->size, &acc[i], 1), "cuMemSetAccess");
    }
    CU(d.AddrReserve(&b->mcva, b->size, gran, 0, 0), "cuMemAddressReserve (multicast)");
    CU(d.Map(b->mcva, b->size, 0, b->mc, 0), "cuMemMap (multicast)");
    b->mc_mapped = true;
    CU(d.SetAccess(b->mcva, b->size, acc.data(), ndev), "cuMemSetAccess (multicast)");
    cudaSetDevice(devices[0]);
    *out = b;
    return POSET_OK;
}

poset_status poset_nvls_ptrs(poset_nvls_t b, void **mc, void **uc, int64_t *bytes) {
    if (!b) return fail(POSET_EINVAL, "poset_nvls_ptrs: null buffer");
    if (mc) *mc = (void *)b->mcva;
    if (uc)
        for (int i = 0; i < b->ndev; i++) uc[i] = (void *)b->uc[i];
    if (bytes) *bytes = (int64_t)b->size;
    return POSET_OK;
}

void poset_nvls_destroy(poset_nvls_t b) {
    if (!b) return;
    cudaDeviceSynchronize();
    nvls_release(b);
    delete b;
}

int poset_abi_version(void) { return 2; }   // 2: poset_info.moebius_sms / num_sms

}  // extern "C"
