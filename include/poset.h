/*
 * poset.h -- C-ABI of the B200-native chain-decomposition zeta / Moebius
 * transforms (arXiv 2211.13706, "Fast Möbius and zeta transforms on posets";
 * paper text at /root/reference/PAPER.md, cited as P:Lnnn).
 *
 * Library: paper_2211_13706_b200/libposet.so (sm_100a CUDA + host C++).
 * Every step of the transforms runs in this library's CUDA kernels; there is
 * no CPU fallback.  A missing GPU makes every compute call return POSET_ECUDA.
 *
 * ---------------------------------------------------------------------------
 * Conventions
 * ---------------------------------------------------------------------------
 *  Vertices   dense user ids 0..n-1.  Ids are never renumbered at the ABI.
 *  Edges      (src[e], dst[e]) means dst ⪯ src: dst is a successor of src in
 *             the DAG.  Duplicates are ignored, isolated vertices
 *             are singleton chains, the DAG need not be connected (reading
 *             G11 of DESIGN.md).
 *  Functions  f, g are row-major [n][batch] arrays (batch contiguous), in
 *             USER vertex order.  dtype POSET_I64 computes in Z/2^64
 *             (two's-complement wraparound, reading G14); POSET_F64 uses
 *             IEEE binary64 adds/subtracts (no multiplies).
 *  Pointers   f, g may be device pointers (any CUDA allocation on the
 *             handle's device) or host pointers (pinned or pageable).  Host
 *             buffers are staged through device buffers owned by the handle
 *             (H2D copy, kernels, D2H copy, all on `stream`); the host result
 *             is valid once `stream` has synchronised.  f == g is allowed.
 *  Streams    `stream` is a cudaStream_t passed as void* (NULL = legacy
 *             default stream).  Compute calls are asynchronous and
 *             stream-ordered; setup is synchronous.
 *  Threads    a handle is not re-entrant: serialise calls per handle (host
 *             side).  Calls on DIFFERENT streams are ordered by the library
 *             wherever they share handle scratch: the scratch is split in
 *             lanes (Z: the zeta's scan / gather buffers and the non-ring
 *             Möbius schedules; R0 / R1: the ring-family Möbius input, double
 *             buffered -- a ring-family call on another stream than the
 *             previous one takes the other buffer; S: host staging); each
 *             call records an event per lane it uses on its stream, and a
 *             call on another stream first waits on the events of its own
 *             lanes.  So a zeta on one stream and a ring-family Möbius
 *             (poset_info.moebius_kernel RING / RINGWS / RINGDF / RINGCL /
 *             RINGCW) on another, both on device buffers, run concurrently,
 *             and two ring-family Möbius calls on two streams overlap the
 *             second one's permutation kernel with the first one's solve;
 *             the solve kernels of one handle run one at a time (the
 *             library orders them by an event) unless option
 *             "solves_inflight" is 2..4 (up to that many streams' solves
 *             then overlap, each with its own rank-major lane R0..R3);
 *             everything else is serialised.  Data
 *             dependencies between the caller's own buffers are the caller's
 *             to order (events).  A host result is valid once `stream` has
 *             synchronised (poset_sync).
 *  Errors     return codes, never exceptions; poset_last_error() gives the
 *             calling thread's last message.  CUDA faults inside a kernel
 *             (illegal address, launch failure, ...) are sticky in the handle
 *             (POSET_ECUDA); recoverable CUDA errors (a device allocation that
 *             does not fit -> POSET_ENOMEM, a launch that cannot be placed) are
 *             returned once and cleared.
 *  Alignment  split-phase entry points (poset_scan_slots .. poset_rank_to_user)
 *             take device pointers only: [n][B] arrays 32-byte aligned, tail /
 *             carry arrays 8-byte aligned; anything else is POSET_EINVAL.
 *             poset_zeta / poset_moebius accept any pointer (they stage).
 *
 * Internal layout: elements are ranked in level order
 * (Alg. 6 antichains, bottom-up, ties by user id); chains are
 * laid out contiguously ("slots"), chain j occupying slots off_j..off_j+len_j-1
 * bottom-up.  The reachability table is chain-major int32 M[k][n]:
 * M[j][r] = off_j + m(r, j) where m(x,j) = max{p : chain_j[p] ⪯ x}
 * (= the paper's niv_j(x), as a position), or n when
 * ↓x ∩ Z_j = ∅ (the paper's ∞, mapped to an all-zero row of F).
 */
#ifndef POSET_H
#define POSET_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct poset_s *poset_t;

typedef enum {
    POSET_OK = 0,
    POSET_EINVAL = 1,         /* bad argument: null pointer, id out of range, batch <= 0, range  */
    POSET_ESELFLOOP = 2,      /* an edge (u, u) (S:L48 SelfLoopError)                           */
    POSET_ECYCLE = 3,         /* the edges contain a directed cycle (S:L48 CycleError)           */
    POSET_ENOTCHAIN = 4,      /* injected chain with consecutive incomparable elements  */
    POSET_ENOTPARTITION = 5,  /* injected chains do not partition 0..n-1                */
    POSET_ETOOBIG = 6,        /* neither the dense n*k*4-byte table nor the sparse rows fit      */
    POSET_ENOMEM = 7,         /* host allocation, or a device scratch allocation, failed (not sticky) */
    POSET_ECUDA = 8           /* CUDA error (no device, launch failure, ...) -- sticky           */
} poset_status;

typedef enum { POSET_I64 = 0, POSET_F64 = 1 } poset_dtype;

/* Moebius U-solve strategies (kernel v). */
typedef enum {
    POSET_MOEB_AUTO = 0,      /* cost model picks one of the below                       */
    POSET_MOEB_LEVEL = 1,     /* one launch per antichain level (Alg. 5)     */
    POSET_MOEB_GRID = 2,      /* persistent cooperative kernel, grid barrier per level   */
    POSET_MOEB_WARP = 3,      /* one warp per column group sweeps all levels (no grid sync) */
    POSET_MOEB_RING = 4,      /* bounded-reach posets: one CTA per column, F in a shared-memory
                                 ring, U-solve and chain difference fused   */
    POSET_MOEB_CSR = 5,       /* sparse U-rows, persistent kernel with a grid barrier per
                                 level, one warp per (element, column group) */
    POSET_MOEB_RINGWS = 6,    /* RING with warp specialisation: one warp on the level-by-level
                                 critical path (near dependencies only), the others summing the
                                 far dependencies ahead of it                 */
    POSET_MOEB_RINGDF = 7,    /* barrier-free level pipeline: warps own levels round-robin and
                                 publish level completion through mbarriers; far / mid
                                 dependencies are summed levels ahead, near ones on the
                                 critical path                                               */
    POSET_MOEB_RINGCL = 8,    /* RINGDF over a CTA pair (cluster of 2) per column: the second
                                 SM sums the far dependencies and returns them through
                                 distributed shared memory                  */
    POSET_MOEB_RINGCW = 9     /* RINGCL with ONE critical warp taking every level's near step
                                 (no cross-warp hand-off on the dependency chain); the level
                                 warps hand it g - mid - far in tagged shared-memory records
                                                                             */
} poset_moebius_kernel;

typedef struct {
    int64_t n;            /* elements                                               */
    int64_t m;            /* distinct edges after de-duplication                    */
    int64_t k;            /* chains (minimum path cover of E, reading G1)           */
    int64_t q;            /* longest chain of the decomposition            */
    int64_t ell;          /* antichain levels = poset length (Thm. 5)       */
    int64_t nnz;          /* finite niv entries incl. self entries = nnz(N)*/
    int64_t table_bytes;  /* bytes of the dense chain-major int32 table (4*n*k)     */
    int64_t max_level_width;
    double t_ingest;      /* seconds: validate, de-duplicate, CSR                   */
    double t_levels;      /* seconds: Alg. 6 levels + ranks                         */
    double t_match;       /* seconds: Alg. 1 maximum matching (augmenting paths)    */
    double t_chains;      /* seconds: chain walk, slots                             */
    double t_upload;      /* seconds: host -> device copies                         */
    double t_mtable;      /* seconds: kernel (ii) + nnz count                       */
    int32_t device;
    int32_t moebius_kernel; /* strategy AUTO resolves to (poset_moebius_kernel)     */
    int64_t reach;        /* max rank distance from x to a dependency of its U-solve
                             row or to next(x) (level order); RING needs < 65535     */
    int64_t dist_bytes;   /* bytes of the RING distance table (0 = RING unavailable)*/
    double t_dist;        /* seconds: reach + distance table + sparse rows build    */
    int64_t csr_bytes;    /* bytes of the sparse U-rows (0 = not built)             */
    int64_t zeta_sparse;  /* 1 if zeta gathers over the sparse rows (fill < 1/2)    */
    int64_t ringws;       /* 1 if the RINGWS schedule is available                  */
    int64_t ringdf;       /* bit 0: RINGDF available, bit 1: RINGCL, bit 2: RINGCW  */
    int64_t rdf_bytes;    /* bytes of the RINGDF / RINGCL near + far tables         */
    int64_t ring_bytes;   /* bytes of the RING tables (dist + next slot)            */
    int64_t rws_bytes;    /* bytes of the RINGWS tables                             */
    int64_t depth_u;      /* D_U: longest dependency path of the U-solve (Alg. 4
                             first loop), the PRAM depth bound of P:L740-745;
                             -1 until poset_set_option("compute_depth_u", 1)   */
    double t_depth;       /* seconds of that computation                            */
    int64_t gather_bytes; /* bytes of the gather-order table + delta list (0 = not
                             built yet)                                             */
    int64_t gather_entries; /* entries of the zeta delta list (changed niv slots
                             between consecutive gather positions) */
    int64_t gather_resets;  /* positions summed from scratch in that list         */
    int64_t moebius_sms;  /* SMs the last poset_moebius launch occupied (ring family:
                             one CTA per SM; 0 = no call yet)                        */
    int64_t num_sms;      /* SMs of the handle's device                              */
} poset_info;

/*
 * poset_setup -- one-time precomputation for the poset given by the DAG
 * (n vertices, m edges src[e] -> dst[e], host int64 arrays).  Runs Alg. 6
 * levels, Alg. 1 chain decomposition by maximum matching on the
 * split graph (augmenting paths), and kernel (ii): the table M by
 * level-sequential max propagation, Thm. 4.  Synchronous.
 * device: CUDA ordinal.  On success *out owns all device memory of the poset.
 * Errors: EINVAL, ESELFLOOP, ECYCLE, ETOOBIG, ENOMEM, ECUDA.
 */
poset_status poset_setup(int64_t n, int64_t m, const int64_t *src, const int64_t *dst,
                         int device, poset_t *out);

/* poset_setup_ex flags */
enum {
    POSET_SETUP_SPARSE = 1    /* never build the dense table: the U-rows (the paper's sparse N,
                                 P:L292) are built straight from the DAG, level by level (Thm. 4,
                                 P:L356-367), and zeta / Möbius run over them.
                                 poset_setup does this on its own when the dense n*k table does
                                 not fit in device memory.                                  */
};

/*
 * poset_setup_ex -- poset_setup with flags (POSET_SETUP_SPARSE).  Errors as
 * poset_setup; EINVAL for unknown flags; ETOOBIG only when neither the dense
 * table nor the sparse rows fit.
 */
poset_status poset_setup_ex(int64_t n, int64_t m, const int64_t *src, const int64_t *dst, int device,
                            uint32_t flags, poset_t *out);

/*
 * poset_setup_chains -- as poset_setup, but with an injected chain
 * decomposition (SPEC decompose_explicit): chain c is
 * chain_elems[chain_ptr[c] .. chain_ptr[c+1]) listed TOP-DOWN (largest first),
 * user ids.  Consecutive elements must be comparable (ENOTCHAIN); the chains
 * must partition 0..n-1 (ENOTPARTITION).  Test hook: reproduces the paper's N.
 */
poset_status poset_setup_chains(int64_t n, int64_t m, const int64_t *src, const int64_t *dst,
                                int64_t k, const int64_t *chain_ptr, const int64_t *chain_elems,
                                int device, poset_t *out);

/*
 * poset_zeta -- g = Z f, g(x) = Σ_{y ⪯ x} f(y)  (Eq. inv-formula P:L13;
 * fast form Eq. zeta-fast P:L401-407 / Alg. 3, factorised as
 * Z = U V, Eq. zfac): kernel (iii) segmented chain scan F = V f,
 * then kernel (iv) gather-reduce g(x) = Σ_j F[M[j][x]].
 * f, g: [n][batch], see Conventions.  Errors: EINVAL, ECUDA.
 */
poset_status poset_zeta(poset_t h, const void *f, void *g, int64_t batch, poset_dtype dt,
                        void *stream);

/*
 * poset_moebius -- f = Z^{-1} g = M g, f(x) = Σ_{y ⪯ x} μ(y,x) g(y)
 * (Eq. inv-formula, Cor. 1 P:L143-151; fast form P:L499-502 / Alg. 4
 * P:L645-674): kernel (v) back-substitution x = U y' in level order
 * (F(x) = g(x) - Σ_{j≠id(x)} F[M[j][x]]), then the chain difference
 * f(x) = F(x) - F(next(x)) (V^{-1}).  g, f: [n][batch].
 * Errors: EINVAL, ECUDA.
 */
poset_status poset_moebius(poset_t h, const void *g, void *f, int64_t batch, poset_dtype dt,
                           void *stream);

/* ---- split phases for row-sharded single-function zeta ----
 * A rank owning slot range [slot_lo, slot_hi) and rank-row range
 * [row_lo, row_hi) runs:
 *   poset_scan_slots(f -> F[slot_lo:slot_hi], carry_in = 0, tail out)
 *   (all-gather the tails over NCCL, combine them -> carry_in)
 *   poset_scan_carry(F[slot_lo:slot_hi] += carry_in up to the first chain start)
 *   (all-gather F over NCCL)
 *   poset_gather_rows(F -> g rows [row_lo, row_hi) in rank order)
 * F is a device array [n+1][batch] in slot order; the caller owns it and must
 * keep row n zero.  tail: device [2][batch] (word 0 of column b = 1 if the
 * range contains a chain start else 0; word 1 = sum of the values after the
 * last chain start in the range, or of all values if none).
 */
poset_status poset_scan_slots(poset_t h, const void *f, void *F, void *tail, int64_t slot_lo,
                              int64_t slot_hi, int64_t batch, poset_dtype dt, void *stream);
poset_status poset_scan_carry(poset_t h, void *F, const void *carry_in, int64_t slot_lo,
                              int64_t slot_hi, int64_t batch, poset_dtype dt, void *stream);
poset_status poset_gather_rows(poset_t h, const void *F, void *g_rank, int64_t row_lo,
                               int64_t row_hi, int64_t batch, poset_dtype dt, void *stream);
/*
 * poset_shard_rows -- keep only index rows [row_lo, row_hi) (rank order) of the
 * dense table on this handle: 4*k*(row_hi - row_lo) bytes instead of 4*n*k
 * (the row-sharded index of SURVEY §8(f) N3; the setup still built the whole
 * table, this frees it).  Afterwards poset_gather_rows accepts only rows in
 * that range, poset_zeta / LEVEL / GRID / WARP Möbius / compute_depth_u /
 * poset_export_mtable return EINVAL; the ring and sparse-row Möbius schedules
 * keep working unless flags has POSET_SHARD_DROP_MOEBIUS (frees their tables
 * too: for ranks that never run the Möbius solve).  Synchronises the device.
 * Errors: EINVAL (bad range, sparse-row zeta, already sharded), ENOMEM, ECUDA.
 */
#define POSET_SHARD_DROP_MOEBIUS 1u
poset_status poset_shard_rows(poset_t h, int64_t row_lo, int64_t row_hi, uint32_t flags);

/* carry_out[b] = value of the segmented prefix of tails_all[0..rank-1]
 * (device [world][2][batch] as written by poset_scan_slots on each rank), the
 * carry into rank `rank`'s slot range. */
poset_status poset_combine_tails(poset_t h, const void *tails_all, int64_t world, int64_t rank,
                                 void *carry_out, int64_t batch, poset_dtype dt, void *stream);
/* g_user[user(r)] = g_rank[r] for all ranks r (device arrays [n][batch]). */
poset_status poset_rank_to_user(poset_t h, const void *g_rank, void *g_user, int64_t batch,
                                poset_dtype dt, void *stream);

/*
 * poset_analyze -- HOST-ONLY part of the setup (no GPU needed): ingest,
 * Alg. 6 levels, Alg. 1 chain decomposition.  Fills out->n, m, k, q, ell,
 * max_level_width, table_bytes (= 4*n*k, the dense table poset_setup would
 * allocate) and the host timings; nnz = -1.  chain/pos/level (nullable, host
 * int64 [n]): per user vertex chain id, bottom-up position, level.  Used to
 * report the literal configs' k and table size (POSET_ETOOBIG decision)
 * without a device, and by the CPU test-suite.
 */
poset_status poset_analyze(int64_t n, int64_t m, const int64_t *src, const int64_t *dst,
                           poset_info *out, int64_t *chain, int64_t *pos, int64_t *level);

/* poset_query -- sizes, timings and the resolved Moebius strategy. */
poset_status poset_query(poset_t h, poset_info *out);

/* poset_set_option -- "moebius_kernel" (poset_moebius_kernel value);
 * "ring_lpe" (lanes per element of the RING schedule, tuning);
 * "ringws_nwo" / "ringws_lpeo" (RINGWS warps / lanes per element, tuning);
 * "gather_variant" (process-wide dense zeta gather for batch % 32 == 0:
 * 0 = per-tile gather order with per-lane row reuse (default; its table,
 * 4*n*k bytes, is built on the first such call), 1 = lanes over columns,
 * 2 = lanes over ranks, 3 / 4 = rank-order per-lane row reuse with 4 / 2
 * chains per step);
 * "gather_pi_cfg" (process-wide, tuning: 0 = the gather-order kernel with
 * per-lane row reuse (default), 1..3 = its alternatives measured in
 * DESIGN.md §5.2, 4 = the delta-list gather: g carried from one gather
 * position to the next, only the changed chains' rows loaded, with an fp64
 * error certificate; its list is built on first use -- measured slower;
 * 5..7 = 4 / 16 / 4 positions per lane, measured slower);
 * "zeta_sms" (0 = all SMs): the SM count the zeta's persistent gather grids
 * size for -- set it to the SMs a concurrent ring-family Möbius on another
 * stream leaves free (num_sms - poset_info.moebius_sms), so the gather does
 * not queue CTAs behind the Möbius (the batched pipeline);
 * "solves_inflight" (1 = default: the ring-family solve kernels of a handle
 * run one at a time; 2..4: calls on that many streams overlap their solves
 * -- a throughput option for a stream of batches: each solve holds its own
 * CTAs / clusters of SMs and its own rank-major input buffer (the buffers
 * rotate over max(2, solves_inflight) lanes on every stream change), so the
 * caller keeps at most that many streams' Möbius calls in flight and sizes
 * the schedule so they fit side by side);
 * "ringcl_helpers" (RINGCL / RINGCW helper CTAs per column 1..3, 0 = auto);
 * "ringcl_chunk" (RINGCL owner stage chunk 32..256 ranks, 0 = the plan's; tuning);
 * "ringcw_sleep" (RINGCW level warps: ns between level polls, 0 = try_wait; tuning);
 * "compute_depth_u" (1: compute D_U now, synchronously, into poset_info.depth_u);
 * "profile" (0/1): record a CUDA event pair on the call's stream around every
 * kernel phase of subsequent calls (see poset_profile_read);
 * "ring_debug" (timing experiments only): bit 0 RING without the f store,
 * bit 3 the instrumented RINGDF / RINGCL instantiation (counters through
 * poset_debug_read), bits 4-6 RINGDF / RINGCL with the far / mid / near sums
 * skipped -- bits 0 and 4-6 make the results INVALID. */
poset_status poset_set_option(poset_t h, const char *key, int64_t value);

/* Profiling phases. */
enum {
    POSET_PH_SCAN = 0,      /* kernel (iii)   */
    POSET_PH_GATHER = 1,    /* kernel (iv)    */
    POSET_PH_MSOLVE = 2,    /* kernel (v)     */
    POSET_PH_DIFF = 3,      /* chain difference */
    POSET_PH_H2D = 4,       /* host staging in  */
    POSET_PH_D2H = 5,       /* host staging out */
    POSET_PH_PERM = 6,      /* RING: g permuted to rank-major columns */
    POSET_PH_COUNT = 8
};

/* poset_profile_read -- synchronise the recorded events, return per phase the
 * summed milliseconds (ms[POSET_PH_COUNT]), the number of timed calls
 * (calls[POSET_PH_COUNT]) and the number of kernel launches the library made
 * since the last read (*launches), then reset.  Any pointer may be NULL. */
poset_status poset_profile_read(poset_t h, double *ms, int64_t *calls, int64_t *launches);

/*
 * Test / inspection hooks (copy device state to caller-owned HOST arrays):
 *  poset_export_chains: per user vertex x: chain[x] (0..k-1), pos[x] (bottom-up
 *    position, 0 = lowest), level[x] (0 = leaves), rank[x].
 *  poset_export_mtable: out[x*k + j] = m(x, j) (position, -1 = ∞), user order;
 *    n*k int32 host array.
 */
poset_status poset_export_chains(poset_t h, int64_t *chain, int64_t *pos, int64_t *level,
                                 int64_t *rank);
poset_status poset_export_mtable(poset_t h, int32_t *out);
/* poset_debug_read -- tuning hook: the 8 int64 counters of the last RING call
 * made with option "ring_debug" bit 1 (clock64 per-phase sums of CTA 0:
 * [0] row data + ring loads + tree, [1] lane reduction, [2] tail,
 * [3] next-level prefetch, [4] barrier, [5] levels). */
poset_status poset_debug_read(poset_t h, int64_t *out8);

/*
 * NVLS multicast (the row-sharded zeta's all-gather of F
 * fused into the scan epilogue, P:L738-745 row sharding).
 *
 * poset_nvls_create -- one buffer of `bytes` (rounded up to the multicast
 *   granularity) on each of the ndev CUDA ordinals `devices` (this process
 *   drives all of them), bound to one NVLS multicast object: a store through
 *   the multicast address lands at the same offset of every device's buffer
 *   (NVSwitch replicates it).  The library owns the memory; free it with
 *   poset_nvls_destroy (which synchronises the device).  ECUDA when the
 *   driver or the device has no multicast support (the caller falls back to
 *   the NCCL all-gather path), ENOMEM when the memory does not fit.
 *   (Sharing the object across processes -- one process per GPU -- needs a
 *   shareable-handle exchange that is not built: the pool has one GPU.)
 * poset_nvls_ptrs -- *mc: the multicast address (device-visible on every
 *   listed device; only multimem.* instructions may use it); uc[i]: the
 *   plain (unicast) address of device i's buffer; *bytes: the rounded size.
 *
 * poset_scan_slots_mc -- poset_scan_slots (Eq. zeta_cache P:L390-400 over
 *   slots [lo, hi)), but every F row is stored with multimem.st through the
 *   multicast address F_mc (F_mc + slot * batch * 8 is slot's row): all
 *   devices bound to the object receive the rank's rows, so no separate
 *   all-gather of F follows.  The kernel ends with a system-scope fence;
 *   a peer may read the rows after its stream is ordered after this call's
 *   completion (an event, or a collective that follows it on this stream).
 *   tail: as poset_scan_slots.  F_mc: 8-byte aligned multicast address of
 *   a buffer of >= n * batch * 8 bytes; f: 32-byte aligned device memory.
 */
typedef struct poset_nvls_s *poset_nvls_t;
poset_status poset_nvls_create(const int *devices, int ndev, int64_t bytes, poset_nvls_t *out);
poset_status poset_nvls_ptrs(poset_nvls_t b, void **mc, void **uc, int64_t *bytes);
void poset_nvls_destroy(poset_nvls_t b);
poset_status poset_scan_slots_mc(poset_t h, const void *f, void *F_mc, void *tail, int64_t slot_lo,
                                 int64_t slot_hi, int64_t batch, poset_dtype dt, void *stream);

/* poset_sync -- cudaStreamSynchronize(stream) on the handle's device (host
 * results of poset_zeta / poset_moebius are valid after it). */
poset_status poset_sync(poset_t h, void *stream);

void poset_destroy(poset_t h);
const char *poset_strerror(poset_status s);
const char *poset_last_error(void);
int poset_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* POSET_H */
