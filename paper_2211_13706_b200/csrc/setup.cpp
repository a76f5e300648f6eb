// Host one-time precomputation, C++.
//
//  S0  ingest: validate ids, reject self loops, de-duplicate,
//      user-space CSR of children.
//  S1  Alg. 6 antichain decomposition: peel leaves by
//      out-degree; level 0 = leaves.  ell = number of levels = poset length
//      (Thm. 5 Mirsky).  Elements are then RANKED in level order
//      (ties by user id): every kernel works in rank space.
//  S2  Alg. 1 chain decomposition: maximum matching on the split
//      graph G' = (P1 ∪ P2, {(v1,u2) : (v,u) ∈ E}) by augmenting paths; the
//      matched edge (v1,u2) is next(v) = u.  k = n - |matching| is a
//      minimum PATH cover of E (reading G1 of DESIGN.md).
//      Chains are laid out bottom-up in "slots": chain j owns slots
//      off_j .. off_j+len_j-1, slot(x) = off_{id(x)} + pos(x).
#include <algorithm>
#include <chrono>
#include <cstring>
#include <numeric>

#include "internal.h"

namespace poset {

double now_seconds() {
    using namespace std::chrono;
    return duration<double>(steady_clock::now().time_since_epoch()).count();
}

poset_status host_ingest(int64_t n, int64_t m, const int64_t *src, const int64_t *dst,
                         HostPoset &P, std::string &err) {
    double t0 = now_seconds();
    if (n < 0 || n >= INT32_MAX - 1 || m < 0 || (m > 0 && (!src || !dst))) {
        err = "poset_setup: invalid n/m or null edge arrays";
        return POSET_EINVAL;
    }
    for (int64_t e = 0; e < m; e++) {
        if (src[e] < 0 || src[e] >= n || dst[e] < 0 || dst[e] >= n) {
            err = "poset_setup: edge " + std::to_string(e) + " has a vertex id out of range";
            return POSET_EINVAL;
        }
        if (src[e] == dst[e]) {
            err = "poset_setup: self loop at vertex " + std::to_string(src[e]);
            return POSET_ESELFLOOP;
        }
    }
    const int32_t N = (int32_t)n;
    P.n = N;
    // user-space CSR (counting sort by src), then sort + unique each row
    std::vector<int64_t> uptr((size_t)N + 1, 0);
    for (int64_t e = 0; e < m; e++) uptr[src[e] + 1]++;
    for (int32_t v = 0; v < N; v++) uptr[v + 1] += uptr[v];
    std::vector<int32_t> uch((size_t)std::max<int64_t>(m, 1));
    {
        std::vector<int64_t> fill(uptr.begin(), uptr.end() - 1);
        for (int64_t e = 0; e < m; e++) uch[fill[src[e]]++] = (int32_t)dst[e];
    }
    int64_t w = 0;
    std::vector<int64_t> dptr((size_t)N + 1, 0);
    for (int32_t v = 0; v < N; v++) {
        int32_t *a = uch.data() + uptr[v], *b = uch.data() + uptr[v + 1];
        if (b - a > 1) std::sort(a, b);
        for (int32_t *p = a; p < b; p++)
            if (p == a || *p != p[-1]) uch[w++] = *p;
        dptr[v + 1] = w;
    }
    P.m = w;
    P.t_ingest = now_seconds() - t0;

    // ---- S1: Alg. 6, peel leaves level by level ----
    t0 = now_seconds();
    std::vector<int32_t> delta((size_t)N);                 // out-degree
    std::vector<int64_t> pptr((size_t)N + 1, 0);           // parents CSR
    for (int32_t v = 0; v < N; v++) {
        delta[v] = (int32_t)(dptr[v + 1] - dptr[v]);
        for (int64_t t = dptr[v]; t < dptr[v + 1]; t++) pptr[uch[t] + 1]++;
    }
    for (int32_t v = 0; v < N; v++) pptr[v + 1] += pptr[v];
    std::vector<int32_t> par((size_t)std::max<int64_t>(w, 1));
    {
        std::vector<int64_t> fill(pptr.begin(), pptr.end() - 1);
        for (int32_t v = 0; v < N; v++)
            for (int64_t t = dptr[v]; t < dptr[v + 1]; t++) par[fill[uch[t]]++] = v;
    }
    std::vector<int32_t> ulevel((size_t)N, -1);
    std::vector<int32_t> cur, nxt;
    cur.reserve(1024);
    for (int32_t v = 0; v < N; v++)
        if (delta[v] == 0) cur.push_back(v);            // L_1 = leaves
    int32_t L = 0, done = 0, maxw = 0;
    while (!cur.empty()) {
        nxt.clear();
        for (int32_t v : cur) {
            ulevel[v] = L;
            for (int64_t t = pptr[v]; t < pptr[v + 1]; t++) {
                int32_t u = par[t];
                if (--delta[u] == 0) nxt.push_back(u);
            }
        }
        done += (int32_t)cur.size();
        maxw = std::max<int32_t>(maxw, (int32_t)cur.size());
        L++;
        std::swap(cur, nxt);
    }
    if (done != N) {
        err = "poset_setup: the edges contain a directed cycle";
        return POSET_ECYCLE;
    }
    P.ell = L;
    P.max_level_width = maxw;
    // ranks: counting sort by level, stable in user id
    P.lvl_ptr.assign((size_t)L + 1, 0);
    for (int32_t v = 0; v < N; v++) P.lvl_ptr[ulevel[v] + 1]++;
    for (int32_t l = 0; l < L; l++) P.lvl_ptr[l + 1] += P.lvl_ptr[l];
    P.rank_user.resize(N);
    P.user_rank.resize(N);
    P.level.resize(N);
    {
        std::vector<int32_t> fill(P.lvl_ptr.begin(), P.lvl_ptr.end() - 1);
        for (int32_t v = 0; v < N; v++) {
            int32_t r = fill[ulevel[v]]++;
            P.rank_user[r] = v;
            P.user_rank[v] = r;
            P.level[r] = ulevel[v];
        }
    }
    // rank-space CSR of children, ascending rank
    P.child_ptr.assign((size_t)N + 1, 0);
    P.child.resize((size_t)std::max<int64_t>(w, 1));
    for (int32_t r = 0; r < N; r++) {
        int32_t v = P.rank_user[r];
        P.child_ptr[r + 1] = P.child_ptr[r] + (dptr[v + 1] - dptr[v]);
    }
    for (int32_t r = 0; r < N; r++) {
        int32_t v = P.rank_user[r];
        int32_t *o = P.child.data() + P.child_ptr[r];
        int64_t len = dptr[v + 1] - dptr[v];
        for (int64_t t = 0; t < len; t++) o[t] = P.user_rank[uch[dptr[v] + t]];
        if (len > 1) std::sort(o, o + len);
    }
    P.t_levels = now_seconds() - t0;
    return POSET_OK;
}

// chain arrays from next (rank space; nextr[r] = lower neighbour or -1).
// A chain successor is a child, so nextr[r] < r in level order: one forward
// pass over the ranks gives the bottom-up position and the chain id (chains
// numbered by the rank of their bottom element) without pointer chasing.
static void layout_chains(HostPoset &P, const std::vector<int32_t> &nextr) {
    const int32_t N = P.n;
    P.chain.assign(N, -1);
    P.pos.assign(N, 0);
    int32_t K = 0;
    for (int32_t r = 0; r < N; r++) {
        int32_t d = nextr[r];
        if (d >= 0) {
            P.chain[r] = P.chain[d];
            P.pos[r] = P.pos[d] + 1;
        } else {
            P.chain[r] = K++;
            P.pos[r] = 0;
        }
    }
    P.k = K;
    std::vector<int32_t> len((size_t)K, 0);
    for (int32_t r = 0; r < N; r++) len[P.chain[r]] = std::max(len[P.chain[r]], P.pos[r] + 1);
    P.chain_off.assign((size_t)K + 1, 0);
    int32_t q = 0;
    for (int32_t c = 0; c < K; c++) {
        P.chain_off[c + 1] = P.chain_off[c] + len[c];
        q = std::max(q, len[c]);
    }
    P.q = q;
    P.slot.assign(N, 0);
    P.slot_user.assign(N, 0);
    P.slot_rank.assign(N, 0);
    for (int32_t r = 0; r < N; r++) {
        int32_t sl = P.chain_off[P.chain[r]] + P.pos[r];
        P.slot[r] = sl;
        P.slot_rank[sl] = r;
        P.slot_user[sl] = P.rank_user[r] | (P.pos[r] == 0 ? (int32_t)0x80000000u : 0);
    }
}

poset_status host_chains_matching(HostPoset &P, std::string &err) {
    double t0 = now_seconds();
    const int32_t N = P.n;
    const int64_t *cp = P.child_ptr.data();
    const int32_t *ch = P.child.data();
    std::vector<int32_t> mate_l((size_t)N, -1), mate_r((size_t)N, -1);
    // Maximum matching of the split graph by augmenting paths: Pothen-Fan
    // phases (one DFS per free left vertex, right vertices visited at most
    // once per phase) with a persistent lookahead pointer per left vertex
    // (a free right vertex found by lookahead stays matched afterwards).
    // Ends when a phase finds no augmenting path => maximum (Berge).
    std::vector<int64_t> look(cp, cp + N), it((size_t)N);
    std::vector<int32_t> visited((size_t)N, 0), su((size_t)N + 1), sv((size_t)N + 1);
    int32_t phase = 0;
    for (;;) {
        phase++;
        int64_t aug = 0;
        for (int32_t u0 = 0; u0 < N; u0++) {
            if (mate_l[u0] >= 0) continue;
            int32_t sp = 0;
            su[0] = u0;
            it[u0] = cp[u0];
            while (sp >= 0) {
                int32_t u = su[sp];
                // lookahead for a free right vertex
                int32_t freev = -1;
                while (look[u] < cp[u + 1]) {
                    int32_t v = ch[look[u]++];
                    if (mate_r[v] < 0) { freev = v; break; }
                }
                if (freev >= 0) {
                    sv[sp] = freev;
                    for (int32_t i = sp; i >= 0; i--) { mate_l[su[i]] = sv[i]; mate_r[sv[i]] = su[i]; }
                    aug++;
                    break;
                }
                // depth-first through matched right vertices
                bool pushed = false;
                while (it[u] < cp[u + 1]) {
                    int32_t v = ch[it[u]++];
                    if (visited[v] == phase) continue;
                    visited[v] = phase;
                    int32_t w = mate_r[v];
                    sv[sp] = v;
                    su[++sp] = w;
                    it[w] = cp[w];
                    pushed = true;
                    break;
                }
                if (!pushed) sp--;
            }
        }
        if (aug == 0) break;
    }
    P.t_match = now_seconds() - t0;
    t0 = now_seconds();
    layout_chains(P, mate_l);
    P.t_chains = now_seconds() - t0;
    (void)err;
    return POSET_OK;
}

// a ⪰ b ?  BFS over children restricted to levels above level(b)
static bool reaches(const HostPoset &P, int32_t a, int32_t b, std::vector<int32_t> &stamp,
                    int32_t tag, std::vector<int32_t> &stk) {
    if (a == b) return true;
    if (P.level[a] <= P.level[b]) return false;
    stk.clear();
    stk.push_back(a);
    stamp[a] = tag;
    while (!stk.empty()) {
        int32_t v = stk.back();
        stk.pop_back();
        for (int64_t t = P.child_ptr[v]; t < P.child_ptr[v + 1]; t++) {
            int32_t u = P.child[t];
            if (u == b) return true;
            if (stamp[u] != tag && P.level[u] > P.level[b]) { stamp[u] = tag; stk.push_back(u); }
        }
    }
    return false;
}

poset_status host_chains_injected(HostPoset &P, int64_t k, const int64_t *chain_ptr,
                                  const int64_t *chain_elems, std::string &err) {
    double t0 = now_seconds();
    const int32_t N = P.n;
    if (k < 0 || (k > 0 && (!chain_ptr || !chain_elems)) || (N > 0 && k == 0)) {
        err = "poset_setup_chains: invalid chain arrays";
        return POSET_EINVAL;
    }
    std::vector<int32_t> nextr((size_t)N, -1);
    std::vector<char> seen((size_t)N, 0);
    std::vector<int32_t> stamp((size_t)N, 0), stk;
    int32_t tag = 0;
    for (int64_t c = 0; c < k; c++) {
        int64_t a = chain_ptr[c], b = chain_ptr[c + 1];
        if (b <= a || a < 0) { err = "poset_setup_chains: empty or malformed chain " + std::to_string(c); return POSET_ENOTPARTITION; }
        for (int64_t t = a; t < b; t++) {
            int64_t u = chain_elems[t];
            if (u < 0 || u >= N) { err = "poset_setup_chains: vertex id out of range"; return POSET_EINVAL; }
            if (seen[u]) { err = "poset_setup_chains: vertex " + std::to_string(u) + " in two chains"; return POSET_ENOTPARTITION; }
            seen[u] = 1;
            if (t + 1 < b) {
                int64_t d = chain_elems[t + 1];
                if (d < 0 || d >= N) { err = "poset_setup_chains: vertex id out of range"; return POSET_EINVAL; }
                int32_t ra = P.user_rank[u], rb = P.user_rank[d];
                if (!reaches(P, ra, rb, stamp, ++tag, stk)) {
                    err = "poset_setup_chains: " + std::to_string(u) + " and " + std::to_string(d) +
                          " are not comparable in chain order";
                    return POSET_ENOTCHAIN;
                }
                nextr[ra] = rb;
            }
        }
    }
    for (int32_t v = 0; v < N; v++)
        if (!seen[v]) { err = "poset_setup_chains: vertex " + std::to_string(v) + " in no chain"; return POSET_ENOTPARTITION; }
    P.t_match = now_seconds() - t0;
    t0 = now_seconds();
    // keep the caller's chain order: layout_chains sorts by bottom rank, so
    // re-sort here by caller index instead
    layout_chains(P, nextr);
    {
        // remap chain ids to caller order
        std::vector<int32_t> caller_of((size_t)P.k, -1);
        for (int64_t c = 0; c < k; c++) {
            int32_t top = P.user_rank[chain_elems[chain_ptr[c]]];
            caller_of[P.chain[top]] = (int32_t)c;
        }
        HostPoset Q = P;
        // rebuild slots in caller order
        int32_t off = 0;
        std::vector<int32_t> new_off((size_t)k + 1, 0);
        for (int64_t c = 0; c < k; c++) {
            new_off[c] = off;
            off += (int32_t)(chain_ptr[c + 1] - chain_ptr[c]);
        }
        new_off[k] = off;
        for (int32_t r = 0; r < N; r++) {
            int32_t c = caller_of[Q.chain[r]];
            P.chain[r] = c;
            P.slot[r] = new_off[c] + Q.pos[r];
            P.slot_rank[P.slot[r]] = r;
            P.slot_user[P.slot[r]] = P.rank_user[r] | (Q.pos[r] == 0 ? (int32_t)0x80000000u : 0);
        }
        P.chain_off = new_off;
    }
    P.t_chains = now_seconds() - t0;
    return POSET_OK;
}

}  // namespace poset
