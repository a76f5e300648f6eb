// Kernel launchers (kernels.cu) used by the C-ABI (api.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace poset {

// Number of kernel launches issued by this library (all handles, all
// threads); read and reset by poset_profile_read.
int64_t launches_take();
void launches_add(int64_t c);

// Device view of one poset (all arrays in device memory, rank space).
struct DevPoset {
    int32_t n, k, ell;
    const int32_t *rank_user;   // [n]  rank -> user id
    const int32_t *slot;        // [n]  rank -> slot
    const int32_t *chain;       // [n]  rank -> chain id
    const int32_t *lvl_ptr;     // [ell+1]
    const int64_t *child_ptr;   // [n+1] rank-space CSR
    const int32_t *child;       // [m]
    const int32_t *slot_user;   // [n]  slot -> user | start flag (bit 31)
    const int32_t *M;           // [k][n] chain-major slot table (n = none)
    int64_t ldm = 0;            // row stride of M (n; hi - lo after poset_shard_rows, M then
                                // points lo entries before the kept rows)
};

// ---- kernel (ii): reachability table ----
// child_reach = max over DAG edges of rank(parent) - rank(child) (-1:
// unknown): with the widest level it sizes the shared-memory ring of the
// fast path; the one-warp-per-chain global-memory sweep otherwise.
cudaError_t launch_mtable(const DevPoset &P, int32_t *M, cudaStream_t s, int32_t child_reach = -1,
                          int32_t max_level_width = 0);
cudaError_t launch_count_nnz(const int32_t *M, int64_t total, int32_t n,
                             unsigned long long *out, cudaStream_t s);

// ---- D_U, the dependency depth of the Möbius U-solve (diagnostic) ----
cudaError_t launch_depth_u(const DevPoset &P, const int32_t *slot_rank, int32_t *D, unsigned *out,
                           cudaStream_t s);

// ---- kernel (iii): segmented chain scan F[slot] = prefix of f[user(slot)] ----
// Scans slots [slot_lo, slot_hi).  carry-in of the first rows is 0 (the
// split-phase API adds remote carries with launch_scan_carry).  tail (nullable):
// [2][batch] words: flag (0/1) and value of the whole range's segmented sum.
// scratch must hold scan_scratch_bytes(...) bytes.
size_t scan_scratch_bytes(int64_t rows, int64_t batch);
cudaError_t launch_scan(const DevPoset &P, int dtype, const void *f, void *F, int64_t slot_lo,
                        int64_t slot_hi, int64_t batch, void *scratch, void *tail,
                        cudaStream_t s, void *F_mc = nullptr);   // F_mc: NVLS multicast stores
// The whole slot range in one pass (decoupled look-back, f read once): the
// zeta transform's scan.  scratch: scan1p_scratch_bytes(n, batch) bytes.
size_t scan1p_scratch_bytes(int64_t rows, int64_t batch);
cudaError_t launch_scan_1p(const DevPoset &P, int dtype, const void *f, void *F, int64_t batch, void *scratch,
                           cudaStream_t s);
cudaError_t launch_scan_carry(const DevPoset &P, int dtype, void *F, const void *carry,
                              int64_t slot_lo, int64_t slot_hi, int64_t batch, cudaStream_t s);

cudaError_t launch_combine_tails(int dtype, const void *tails, int64_t world, int64_t rank,
                                void *carry, int64_t batch, cudaStream_t s);

// ---- kernel (iv): zeta gather-reduce g[user(r)] = Σ_j F[M[j][r]] ----
// rows [row_lo, row_hi).  out_rank != 0: write g_rank[r - row_lo] (rank order)
// instead of g[user(r)].  partial: scratch for j-slicing (may be null if
// gather_partial_bytes() == 0).
void set_gather_variant(int v);   // 0 r4 (default), 1 cols, 2 lanes over ranks (B % 32 == 0)
size_t gather_partial_bytes(const DevPoset &P, int64_t rows, int64_t batch, int num_sms);
cudaError_t launch_gather(const DevPoset &P, int dtype, const void *F, void *g, int64_t row_lo,
                          int64_t row_hi, int64_t batch, int out_rank, void *partial,
                          int num_sms, cudaStream_t s);

// ---- kernel (iv), batched form (gather_pi.cu): B % 32 == 0, the index table
// re-laid in a per-tile greedy gather order (built lazily on the first such
// call) ----
struct GatherPi {
    bool ok = false;
    int64_t npad = 0;            // n rounded up to the 256-element tile
    int32_t *Mg = nullptr;       // [k][npad] F slots in gather order (n = ∞ / padding)
    int32_t *out_user = nullptr; // [npad] user id of each position (-1 = padding)
    void *Fr = nullptr;          // [npad/256][k] int2 F-slot range per (tile, chain) (L2 prefetch)
    // delta list (gather_delta.cu): per tile, per position in gather order,
    // the chains whose niv slot differs from the previous position's
    bool delta_ok = false;
    int64_t nentries = 0;        // entries of D
    int64_t nreset = 0;          // positions summed from scratch (tile starts + magnitude guard)
    void *D = nullptr;           // [nentries] int2 {new slot | LAST<<31, old slot | RESET<<31}
    int64_t *Dptr = nullptr;     // [npad/256 + 1] first entry of each tile
    int64_t *redo = nullptr;     // fp64: (position, column group) pairs to sum directly
    int64_t redo_cap = 0;
    unsigned long long *nredo = nullptr;
};
cudaError_t build_gather_pi(const DevPoset &P, GatherPi &G, cudaStream_t s);
// Build the delta list from G.Mg (chain_off: device [k+1]); fails with
// cudaErrorMemoryAllocation (nothing kept) when it does not fit.
cudaError_t build_gather_delta(const DevPoset &P, const int32_t *chain_off, GatherPi &G, cudaStream_t s);
// fp64 also runs k_gather_redo over the positions its error certificate
// rejected (the redo list is grown here on first use for a batch size).
cudaError_t launch_gather_delta(GatherPi &G, int32_t n, int32_t k, int dtype, const void *F, void *g,
                                int64_t B, int num_sms, cudaStream_t s);
void free_gather_pi(GatherPi &G);
cudaError_t launch_gather_pi(const GatherPi &G, int32_t k, int dtype, const void *F, void *g, int64_t B,
                             int num_sms, cudaStream_t s);
int gather_variant_get();
void set_gather_pi_cfg(int c);   // tuning: kernel configuration of the gather-order kernel
int gather_pi_cfg_get();         //   0 = default, 1-3 = alternatives, 4 = the delta list

// ---- kernel (v): Moebius U-solve F[slot(r)] = g[user(r)] - Σ_{j≠id} F[M[j][r]] ----
enum MoebKernel { MOEB_AUTO = 0, MOEB_LEVEL = 1, MOEB_GRID = 2, MOEB_WARP = 3, MOEB_RING = 4, MOEB_CSR = 5,
                  MOEB_RINGWS = 6, MOEB_RINGDF = 7, MOEB_RINGCL = 8, MOEB_RINGCW = 9 };
int moebius_pick(const DevPoset &P, int64_t batch, int max_level_width, int num_sms);
cudaError_t launch_moebius_solve(const DevPoset &P, const int32_t *h_lvl_ptr, int dtype,
                                 const void *g, void *F, int64_t batch, int which,
                                 unsigned *barrier, int num_sms, cudaStream_t s);

// ---- chain difference f[user(s)] = F[s] - F[s-1] (0 at a chain start) ----
cudaError_t launch_chain_diff(const DevPoset &P, int dtype, const void *F, void *f,
                              int64_t batch, cudaStream_t s);

// ---- g_user[user(r)] = g_rank[r] ----
cudaError_t launch_rank_to_user(const DevPoset &P, int dtype, const void *g_rank, void *g_user,
                                int64_t batch, cudaStream_t s);

// ---- kernel (v), RING schedule (moebius_ring.cu) ----
// Bounded-reach posets: U-solve + chain difference fused, one CTA per column,
// F kept in a shared-memory ring, dependency rows streamed by bulk copies.
struct RingPlan {
    bool ok = false;
    unsigned reach = 0;         // max rank distance to a dependency (incl. next)
    int32_t kp = 0;             // padded row length of D (uint16 words): entries + 8
    int32_t ring = 0;           // ring entries (power of two >= reach + max level width)
    int32_t ch = 0, nstage = 0; // ranks per staged chunk, pipeline depth
    int32_t entries = 0;        // row entries (64, 128 or 256 >= k)
    int32_t lpe = 1;            // lanes per element; entries / lpe per lane (8..64)
    int32_t debug = 0;          // tuning experiments (poset_set_option "ring_debug")
    unsigned long long *dbg = nullptr;   // [8] device, clock64 breakdown (debug bit 1)
    int64_t npad = 0;           // n rounded up to a multiple of ch
    uint16_t *D = nullptr;      // [npad][kp]
    uint16_t *Pn = nullptr;     // [npad] ring slot of next(r)
    int32_t *ru_pad = nullptr;  // [npad]
};
// Fills everything but the device pointers; ok = false if the poset does not
// fit the schedule (reach >= 65535, rows or ring too large for shared memory).
void ring_plan(int32_t n, int32_t k, int32_t ell, int32_t max_level_width, unsigned reach,
               RingPlan &R);
size_t ring_smem_bytes(int ring, int kp, int ch, int nstage);
cudaError_t launch_reach_max(const DevPoset &P, const int32_t *slot_rank, unsigned *out,
                             cudaStream_t s);
cudaError_t launch_build_dist(const DevPoset &P, const int32_t *slot_rank, int32_t kp, int32_t ring,
                              int64_t npad, uint16_t *D, uint16_t *Pn, cudaStream_t s);
cudaError_t launch_to_rank_major(const DevPoset &P, int dtype, const void *g, int64_t B,
                                 int64_t npad, void *gP, cudaStream_t s);
cudaError_t launch_moebius_ring(const DevPoset &P, const RingPlan &R, int dtype, const void *gP,
                                void *f, int64_t B, cudaStream_t s);

// ---- kernel (v), RINGWS schedule (moebius_ringws.cu): RING with a fresh
// warp on the level-by-level critical path and old warps summing the far
// dependencies ahead of it ----
struct RingWSPlan {
    bool ok = false;
    int32_t ld = 0;             // near = dependencies at level distance <= ld
    int32_t nn = 0, fe = 0;     // near / far row entries
    int32_t kp = 0;             // row stride (uint16 words)
    int32_t ring = 0, sbuf = 0; // ring entries, S_old buffer entries (powers of two)
    int32_t ch = 0, nstage = 0;
    int32_t lpeo = 0;           // old-warp lanes per element
    int32_t nwo = 0;            // old warps per CTA (4, 8, 12)
    int64_t npad = 0;
    uint16_t *D = nullptr;      // [npad][kp]
};
void ringws_plan(int32_t n, int32_t k, int32_t max_level_width, unsigned reach,
                 const unsigned near_max[3], RingWSPlan &R);
cudaError_t launch_near_max(const DevPoset &P, const int32_t *level, const int32_t *slot_rank,
                            unsigned *out3, cudaStream_t s);
cudaError_t launch_build_ringws(const DevPoset &P, const RingWSPlan &R, const int32_t *level,
                                const int32_t *slot_rank, cudaStream_t s);
cudaError_t launch_moebius_ringws(const DevPoset &P, const RingWSPlan &R, const int32_t *ru_pad,
                                  int dtype, const void *gP, void *f, int64_t batch, cudaStream_t s);

// ---- kernel (v), RINGDF schedule (moebius_ringdf.cu): barrier-free level
// pipeline, near / mid / far dependencies ----
struct RingDFPlan {
    bool ok = false;
    int32_t nn = 0, nm = 0, fe = 0;   // near / mid / far row entries (far: bank-coloured, /16)
    int32_t kp = 0, ring = 0, ch = 0, nstage = 0;   // kp = kpn + kpf
    int32_t kpn = 0, kpf = 0;         // near-table / far-table row entries (D = near | far tables)
    int32_t wmax = 0;                 // widest level
    int32_t ch_h = 0, nstage_h = 0;   // RINGCL helper staging
    bool cl_ok = false;               // RINGCL fits shared memory
    bool cw_ok = false;               // RINGCW (critical warp) applies: 4 near entries, <= 3 passes, fits
    bool cw = false;                  // launch_moebius_ringcl runs the RINGCW variant
    int32_t cw_sleep = 0;             // RINGCW level warps' poll interval, ns (option ringcw_sleep; 0 = try_wait)
    int32_t nh_max = 1;               // RINGCL helper CTAs per column (1..3) the buffers allow
    int32_t nh_force = 0;             // RINGCL helpers forced (option ringcl_helpers; 0 = auto)
    int32_t ch_cl = 0;                // RINGCL owner stage chunk (option ringcl_chunk; 0 = the plan's)
    int32_t nwc = 8;                  // consumer warps
    bool prof = false;                // instrumented instantiation (tuning)
    int32_t skip_far = 0;             // timing experiment only
    unsigned long long *dbg = nullptr;
    int64_t npad = 0;
    uint16_t *D = nullptr;
};
void ringdf_plan(int32_t n, int32_t k, int32_t max_level_width, unsigned reach,
                 const unsigned counts3[3], RingDFPlan &R);
cudaError_t launch_df_counts(const DevPoset &P, const int32_t *level, const int32_t *slot_rank,
                             unsigned *out3, cudaStream_t s);   // near max, mid max, far colours
cudaError_t launch_build_ringdf(const DevPoset &P, const RingDFPlan &R, const int32_t *level,
                                const int32_t *slot_rank, cudaStream_t s);
cudaError_t launch_moebius_ringdf(const DevPoset &P, const RingDFPlan &R, const int32_t *ru_pad,
                                  int dtype, const void *gP, void *f, int64_t batch, cudaStream_t s);
// RINGCL: the same tables over a CTA pair per column (far sums on the second SM)
bool ringcl_fits(const RingDFPlan &R);
bool ringcw_fits(const RingDFPlan &R);
void ringcl_plan(RingDFPlan &R);
cudaError_t launch_moebius_ringcl(const DevPoset &P, const RingDFPlan &R, const int32_t *ru_pad,
                                  int dtype, const void *gP, void *f, int64_t batch, int num_sms, cudaStream_t s,
                                  int *ctas_out = nullptr);   // CTAs (one per SM) of the launch

// ---- sparse U-rows (moebius_csr.cu): zeta gather + Möbius over CSR rows ----
struct CsrRows {
    bool ok = false;
    int64_t nnz = 0;            // entries (U-rows: niv_j(r), j ≠ id(r), ∞ omitted)
    int64_t *ptr = nullptr;     // [n+1] rank order
    int32_t *idx = nullptr;     // [nnz] F slots
};
// Builds the rows from the dense table if they fit in free_budget bytes
// (C.ok = false otherwise; not an error).
cudaError_t build_csr(const DevPoset &P, CsrRows &C, size_t free_budget);
// The same rows straight from the DAG, level by level, without M (N1):
// budget = device bytes the rows may take; C.ok = false if they do not fit.
// slot_chain[s] = chain of slot s; chain_off[k+1] = chain starts (device);
// h_lvl_ptr = host level bounds.
cudaError_t build_csr_direct(const DevPoset &P, const int32_t *h_lvl_ptr, const int32_t *slot_chain,
                             const int32_t *chain_off, CsrRows &C, size_t budget, int32_t max_level_width,
                             cudaStream_t s);
cudaError_t launch_gather_csr(const DevPoset &P, const CsrRows &C, int dtype, const void *F,
                              void *g, int64_t row_lo, int64_t row_hi, int64_t batch,
                              int out_rank, cudaStream_t s);
cudaError_t launch_moebius_csr(const DevPoset &P, const CsrRows &C, int dtype, const void *g,
                               void *F, void *f, int64_t batch, unsigned *barrier, int num_sms,
                               cudaStream_t s);

}  // namespace poset
