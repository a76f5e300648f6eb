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
};

// ---- kernel (ii): reachability table ----
cudaError_t launch_mtable(const DevPoset &P, int32_t *M, cudaStream_t s);
cudaError_t launch_count_nnz(const int32_t *M, int64_t total, int32_t n,
                             unsigned long long *out, cudaStream_t s);

// ---- kernel (iii): segmented chain scan F[slot] = prefix of f[user(slot)] ----
// Scans slots [slot_lo, slot_hi).  carry-in of the first rows is 0 (the
// split-phase API adds remote carries with launch_scan_carry).  tail (nullable):
// [2][batch] words: flag (0/1) and value of the whole range's segmented sum.
// scratch must hold scan_scratch_bytes(...) bytes.
size_t scan_scratch_bytes(int64_t rows, int64_t batch);
cudaError_t launch_scan(const DevPoset &P, int dtype, const void *f, void *F, int64_t slot_lo,
                        int64_t slot_hi, int64_t batch, void *scratch, void *tail,
                        cudaStream_t s);
cudaError_t launch_scan_carry(const DevPoset &P, int dtype, void *F, const void *carry,
                              int64_t slot_lo, int64_t slot_hi, int64_t batch, cudaStream_t s);

cudaError_t launch_combine_tails(int dtype, const void *tails, int64_t world, int64_t rank,
                                void *carry, int64_t batch, cudaStream_t s);

// ---- kernel (iv): zeta gather-reduce g[user(r)] = Σ_j F[M[j][r]] ----
// rows [row_lo, row_hi).  out_rank != 0: write g_rank[r - row_lo] (rank order)
// instead of g[user(r)].  partial: scratch for j-slicing (may be null if
// gather_partial_bytes() == 0).
size_t gather_partial_bytes(const DevPoset &P, int64_t rows, int64_t batch, int num_sms);
cudaError_t launch_gather(const DevPoset &P, int dtype, const void *F, void *g, int64_t row_lo,
                          int64_t row_hi, int64_t batch, int out_rank, void *partial,
                          int num_sms, cudaStream_t s);

// ---- kernel (v): Moebius U-solve F[slot(r)] = g[user(r)] - Σ_{j≠id} F[M[j][r]] ----
enum MoebKernel { MOEB_AUTO = 0, MOEB_LEVEL = 1, MOEB_GRID = 2, MOEB_WARP = 3 };
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

}  // namespace poset
