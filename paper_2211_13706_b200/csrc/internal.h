// Internal declarations shared by the host setup (setup.cpp), the kernels
// (kernels.cu) and the C-ABI (api.cu).  Not part of the public ABI.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/poset.h"

namespace poset {

// Host-side result of the one-time precomputation.
// All per-element arrays are indexed by RANK r (level order)
// unless the name says otherwise.
struct HostPoset {
    int32_t n = 0, k = 0, q = 0, ell = 0;
    int64_t m = 0;
    int32_t max_level_width = 0;
    std::vector<int32_t> rank_user;   // rank -> user id
    std::vector<int32_t> user_rank;   // user id -> rank
    std::vector<int32_t> level;       // rank -> level (0 = leaves)
    std::vector<int32_t> lvl_ptr;     // level L holds ranks [lvl_ptr[L], lvl_ptr[L+1])
    std::vector<int64_t> child_ptr;   // rank-space CSR of children (covered-by edges)
    std::vector<int32_t> child;       //   sorted ascending rank
    std::vector<int32_t> chain;       // rank -> chain id
    std::vector<int32_t> pos;         // rank -> bottom-up position in its chain
    std::vector<int32_t> slot;        // rank -> off[chain] + pos
    std::vector<int32_t> chain_off;   // k + 1
    std::vector<int32_t> slot_user;   // slot -> user id | (chain start ? 1<<31 : 0)
    std::vector<int32_t> slot_rank;   // slot -> rank
    double t_ingest = 0, t_levels = 0, t_match = 0, t_chains = 0;
};

// S0 + S1: validate and de-duplicate the edges, Alg. 6 levels, ranks and the
// rank-space CSR.  Returns POSET_OK / EINVAL / ESELFLOOP / ECYCLE / ENOMEM.
poset_status host_ingest(int64_t n, int64_t m, const int64_t *src, const int64_t *dst,
                         HostPoset &P, std::string &err);

// S2: Alg. 1 by augmenting-path maximum matching (Pothen-Fan) on the split graph; fills next -> chains.
poset_status host_chains_matching(HostPoset &P, std::string &err);

// S2 (injected): validate and adopt caller chains (top-down user ids).
poset_status host_chains_injected(HostPoset &P, int64_t k, const int64_t *chain_ptr,
                                  const int64_t *chain_elems, std::string &err);

double now_seconds();

}  // namespace poset
