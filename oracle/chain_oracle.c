/*
 * ORACLE O2 -- TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with paper_2211_13706_b200/.
 *
 * The paper's plain sequential chain algorithm, step by step, in the paper's
 * order and notation (arXiv 2211.13706, /root/reference/PAPER.md, "P:Lnnn"):
 *
 *   numbering  descending topological numbering x_1 (largest) .. x_n
 *              ("x_1 is a largest, and x_n a smallest element")
 *   Alg. 1     chain decomposition = maximum matching on the split graph
 *              G' = (P1 u P2, {(v1,u2) : (v,u) in E}), result "next"
 *              (P:L557-578).  Matching by plain augmenting paths (Kuhn).
 *   Alg. 6     antichain decomposition by peeling leaves
 *   Alg. 2     niv computation (Klaus-Simon) with the pruning test
 *              "w < niv_j[id[w]]"; readings G3/G4 of DESIGN.md:
 *              the self entry niv_id(v)(v) = v is stored, children visited in
 *              ascending paper index.
 *   Alg. 3     fast zeta
 *   Alg. 4     fast Moebius, reading G5: y'[next[i]].
 *
 * Arithmetic: int64 functions are computed in Z/2^64 (uint64_t wraparound,
 * reading G14); fp64 functions with IEEE double adds in the algorithms' order.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define INF_IDX 0x7fffffff

typedef struct {
    int32_t n, k, q, ell;
    int64_t m;
    int32_t *user_of;    /* paper index i (1..n) -> user id            */
    int32_t *paper_of;   /* user id -> paper index                      */
    int64_t *adj_ptr;    /* children of paper vertex v, ascending index */
    int32_t *adj;
    int32_t *next;       /* Alg. 1 output, next[i] = i at a chain end   */
    int32_t *id;         /* chain id 1..k                               */
    int32_t *level;      /* Alg. 6 level (1 = leaves)                   */
    int64_t *niv_ptr;    /* Alg. 2 output: row of paper vertex v        */
    int32_t *niv;        /*   entries = paper indices, incl. self entry */
    int64_t nnz;
} oracle_poset;

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

void oracle_free(oracle_poset *P) {
    if (!P) return;
    free(P->user_of); free(P->paper_of); free(P->adj_ptr); free(P->adj);
    free(P->next); free(P->id); free(P->level); free(P->niv_ptr); free(P->niv);
    free(P);
}

/* ---------------- numbering: descending topological sort ---------------- */
/* Kahn's algorithm from the maximal elements (no parent); ties by smallest
 * user id (a fixed topological sort).  Returns 0 or -1 on a cycle,
 * -2 on a self loop, -3 on bad input. */
static int number_vertices(oracle_poset *P, const int64_t *src, const int64_t *dst) {
    int32_t n = P->n;
    int64_t m = P->m;
    for (int64_t e = 0; e < m; e++) {
        if (src[e] < 0 || src[e] >= n || dst[e] < 0 || dst[e] >= n) return -3;
        if (src[e] == dst[e]) return -2;
    }
    /* user-space CSR of children, deduplicated */
    int64_t *cp = calloc((size_t)n + 1, sizeof(int64_t));
    int32_t *ci = malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
    for (int64_t e = 0; e < m; e++) cp[src[e] + 1]++;
    for (int32_t v = 0; v < n; v++) cp[v + 1] += cp[v];
    int64_t *fill = malloc(sizeof(int64_t) * (size_t)(n + 1));
    memcpy(fill, cp, sizeof(int64_t) * (size_t)(n + 1));
    for (int64_t e = 0; e < m; e++) ci[fill[src[e]]++] = (int32_t)dst[e];
    int64_t w = 0;
    int64_t *np_ = calloc((size_t)n + 1, sizeof(int64_t));
    for (int32_t v = 0; v < n; v++) {
        int64_t a = cp[v], b = cp[v + 1];
        qsort(ci + a, (size_t)(b - a), sizeof(int32_t), cmp_i32);
        for (int64_t t = a; t < b; t++)
            if (t == a || ci[t] != ci[t - 1]) ci[w++] = ci[t];
        np_[v + 1] = w;
    }
    P->m = w;
    /* in-degree (number of parents) */
    int32_t *indeg = calloc((size_t)n, sizeof(int32_t));
    for (int64_t t = 0; t < w; t++) indeg[ci[t]]++;
    /* min-heap on user id for deterministic tie-break */
    int32_t *heap = malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    int32_t hs = 0;
#define HPUSH(x) do { int32_t _i = hs++; heap[_i] = (x); \
        while (_i > 0 && heap[(_i - 1) / 2] > heap[_i]) { int32_t _p = (_i - 1) / 2, _t = heap[_p]; heap[_p] = heap[_i]; heap[_i] = _t; _i = _p; } } while (0)
    for (int32_t v = 0; v < n; v++) if (indeg[v] == 0) HPUSH(v);
    P->user_of = malloc(sizeof(int32_t) * ((size_t)n + 1));
    P->paper_of = malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    int32_t cnt = 0;
    while (hs > 0) {
        int32_t v = heap[0];
        heap[0] = heap[--hs];
        int32_t i = 0;
        for (;;) {
            int32_t l = 2 * i + 1, r = l + 1, s = i;
            if (l < hs && heap[l] < heap[s]) s = l;
            if (r < hs && heap[r] < heap[s]) s = r;
            if (s == i) break;
            int32_t t = heap[s]; heap[s] = heap[i]; heap[i] = t; i = s;
        }
        cnt++;
        P->user_of[cnt] = v;
        P->paper_of[v] = cnt;
        for (int64_t t = np_[v]; t < np_[v + 1]; t++)
            if (--indeg[ci[t]] == 0) HPUSH(ci[t]);
    }
#undef HPUSH
    free(heap); free(indeg);
    if (cnt != n) { free(cp); free(ci); free(fill); free(np_); return -1; }
    /* children lists in paper numbering, ascending paper index (reading G4) */
    P->adj_ptr = calloc((size_t)n + 2, sizeof(int64_t));
    P->adj = malloc(sizeof(int32_t) * (size_t)(w ? w : 1));
    for (int32_t i = 1; i <= n; i++) {
        int32_t v = P->user_of[i];
        P->adj_ptr[i + 1] = P->adj_ptr[i] + (np_[v + 1] - np_[v]);
    }
    for (int32_t i = 1; i <= n; i++) {
        int32_t v = P->user_of[i];
        int64_t o = P->adj_ptr[i];
        for (int64_t t = np_[v]; t < np_[v + 1]; t++) P->adj[o++] = P->paper_of[ci[t]];
        qsort(P->adj + P->adj_ptr[i], (size_t)(P->adj_ptr[i + 1] - P->adj_ptr[i]), sizeof(int32_t), cmp_i32);
    }
    free(cp); free(ci); free(fill); free(np_);
    return 0;
}

/* ---------------- Alg. 1: maximum matching on G' (Kuhn) ----------------- */
/* Left vertex v1 may match right vertex u2 iff (v,u) in E.  mate_l[v] = u,
 * mate_r[u] = v; next[v] = mate_l[v] or v when unmatched. */
static void alg1_matching(oracle_poset *P) {
    int32_t n = P->n;
    int32_t *mate_l = malloc(sizeof(int32_t) * ((size_t)n + 1));
    int32_t *mate_r = malloc(sizeof(int32_t) * ((size_t)n + 1));
    for (int32_t i = 0; i <= n; i++) mate_l[i] = mate_r[i] = 0;
    /* plain augmenting-path search from each free left vertex; iterative DFS
     * with a per-search visited stamp on right vertices */
    int32_t *stamp = calloc((size_t)n + 1, sizeof(int32_t));
    int32_t *stk_v = malloc(sizeof(int32_t) * ((size_t)n + 1));
    int64_t *stk_e = malloc(sizeof(int64_t) * ((size_t)n + 1));
    for (int32_t s = 1; s <= n; s++) {
        /* greedy first: a free child */
        for (int64_t t = P->adj_ptr[s]; t < P->adj_ptr[s + 1]; t++)
            if (!mate_r[P->adj[t]]) { mate_l[s] = P->adj[t]; mate_r[P->adj[t]] = s; break; }
        if (mate_l[s]) continue;
        int32_t sp = 0;
        stk_v[0] = s; stk_e[0] = P->adj_ptr[s];
        int found = 0;
        while (sp >= 0 && !found) {
            int32_t v = stk_v[sp];
            if (stk_e[sp] >= P->adj_ptr[v + 1]) { sp--; continue; }
            int32_t u = P->adj[stk_e[sp]++];
            if (stamp[u] == s) continue;
            stamp[u] = s;
            if (!mate_r[u]) {
                /* augment along the stack: stk_v[t] takes the edge it came through */
                int32_t cu = u;
                for (int32_t t = sp; t >= 0; t--) {
                    int32_t cv = stk_v[t];
                    int32_t prev = mate_l[cv];
                    mate_l[cv] = cu; mate_r[cu] = cv;
                    cu = prev;
                }
                found = 1;
            } else {
                sp++;
                stk_v[sp] = mate_r[u];
                stk_e[sp] = P->adj_ptr[mate_r[u]];
            }
        }
    }
    P->next = malloc(sizeof(int32_t) * ((size_t)n + 1));
    for (int32_t v = 1; v <= n; v++) P->next[v] = mate_l[v] ? mate_l[v] : v;
    free(mate_l); free(mate_r); free(stamp); free(stk_v); free(stk_e);
}

/* chain ids from next: a chain starts at a vertex nobody's next points to */
static void chains_from_next(oracle_poset *P) {
    int32_t n = P->n;
    char *has_pred = calloc((size_t)n + 1, 1);
    for (int32_t v = 1; v <= n; v++) if (P->next[v] != v) has_pred[P->next[v]] = 1;
    P->id = calloc((size_t)n + 1, sizeof(int32_t));
    int32_t k = 0, q = 0;
    for (int32_t v = 1; v <= n; v++) {
        if (has_pred[v]) continue;
        k++;
        int32_t len = 0, x = v;
        for (;;) { P->id[x] = k; len++; if (P->next[x] == x) break; x = P->next[x]; }
        if (len > q) q = len;
    }
    P->k = k; P->q = q;
    free(has_pred);
}

/* ---------------- Alg. 6: antichain decomposition ------------------------ */
static void alg6_levels(oracle_poset *P) {
    int32_t n = P->n;
    int32_t *delta = calloc((size_t)n + 1, sizeof(int32_t));   /* out-degree */
    int64_t *pp = calloc((size_t)n + 2, sizeof(int64_t));        /* parents    */
    for (int32_t v = 1; v <= n; v++) {
        delta[v] = (int32_t)(P->adj_ptr[v + 1] - P->adj_ptr[v]);
        for (int64_t t = P->adj_ptr[v]; t < P->adj_ptr[v + 1]; t++) pp[P->adj[t] + 1]++;
    }
    for (int32_t v = 1; v <= n + 0; v++) pp[v + 1] += pp[v];
    int32_t *par = malloc(sizeof(int32_t) * (size_t)(P->m ? P->m : 1));
    int64_t *fill = malloc(sizeof(int64_t) * ((size_t)n + 2));
    memcpy(fill, pp, sizeof(int64_t) * ((size_t)n + 2));
    for (int32_t v = 1; v <= n; v++)
        for (int64_t t = P->adj_ptr[v]; t < P->adj_ptr[v + 1]; t++) par[fill[P->adj[t]]++] = v;
    P->level = calloc((size_t)n + 1, sizeof(int32_t));
    int32_t *cur = malloc(sizeof(int32_t) * ((size_t)n + 1));
    int32_t *nxt = malloc(sizeof(int32_t) * ((size_t)n + 1));
    int32_t nc = 0, li = 0;
    for (int32_t v = 1; v <= n; v++) if (delta[v] == 0) cur[nc++] = v;   /* L_1 = leaves */
    while (nc > 0) {
        li++;
        int32_t nn = 0;
        for (int32_t a = 0; a < nc; a++) {
            int32_t v = cur[a];
            P->level[v] = li;
            for (int64_t t = pp[v]; t < pp[v + 1]; t++) {
                int32_t w = par[t];
                if (--delta[w] == 0) nxt[nn++] = w;
            }
        }
        int32_t *tmp = cur; cur = nxt; nxt = tmp; nc = nn;
    }
    P->ell = li;
    free(delta); free(pp); free(par); free(fill); free(cur); free(nxt);
}

/* ---------------- Alg. 2: niv computation -------------------------------- */
static int alg2_niv(oracle_poset *P) {
    int32_t n = P->n, k = P->k;
    int32_t *nivj = malloc(sizeof(int32_t) * ((size_t)k + 1));      /* niv_j as an array */
    for (int32_t s = 0; s <= k; s++) nivj[s] = INF_IDX;
    int64_t cap = (int64_t)n * 4 + 16, used = 0;
    int32_t *ent = malloc(sizeof(int32_t) * (size_t)cap);
    int64_t *start = malloc(sizeof(int64_t) * ((size_t)n + 2));
    int64_t *len = malloc(sizeof(int64_t) * ((size_t)n + 2));
    if (!nivj || !ent || !start || !len) return -4;
    for (int32_t v = n; v >= 1; v--) {                    /* for v <- n to 1 */
        for (int64_t t = P->adj_ptr[v]; t < P->adj_ptr[v + 1]; t++) {   /* w in adj(v) */
            int32_t w = P->adj[t];
            if (w < nivj[P->id[w]]) {                     /* pruning test */
                for (int64_t e = start[w]; e < start[w] + len[w]; e++) {  /* p in niv[w] */
                    int32_t p = ent[e];
                    if (p < nivj[P->id[p]]) nivj[P->id[p]] = p;   /* min(...) */
                }
            }
        }
        nivj[P->id[v]] = v;                               /* self entry (reading G3) */
        if (used + k > cap) {
            while (used + k > cap) cap *= 2;
            int32_t *ne = realloc(ent, sizeof(int32_t) * (size_t)cap);
            if (!ne) { free(ent); return -4; }
            ent = ne;
        }
        start[v] = used;
        for (int32_t s = 1; s <= k; s++) {                /* for s <- 1 to k */
            if (nivj[s] != INF_IDX) ent[used++] = nivj[s];
            nivj[s] = INF_IDX;
        }
        len[v] = used - start[v];
    }
    /* rows were appended for v = n..1; re-index as a CSR in paper order */
    P->niv_ptr = malloc(sizeof(int64_t) * ((size_t)n + 2));
    P->niv = malloc(sizeof(int32_t) * (size_t)(used ? used : 1));
    P->niv_ptr[1] = 0;
    for (int32_t v = 1; v <= n; v++) {
        memcpy(P->niv + P->niv_ptr[v], ent + start[v], sizeof(int32_t) * (size_t)len[v]);
        P->niv_ptr[v + 1] = P->niv_ptr[v] + len[v];
    }
    P->nnz = used;
    free(ent); free(start); free(len); free(nivj);
    return 0;
}

/* reachability check a ⪰ b by DFS, for validating injected chains */
static int reaches(oracle_poset *P, int32_t a, int32_t b, int32_t *stk, char *seen) {
    if (a == b) return 1;
    int32_t sp = 0, found = 0;
    stk[sp++] = a; seen[a] = 1;
    int32_t *touched = malloc(sizeof(int32_t) * ((size_t)P->n + 1));
    int32_t nt = 0; touched[nt++] = a;
    while (sp && !found) {
        int32_t v = stk[--sp];
        for (int64_t t = P->adj_ptr[v]; t < P->adj_ptr[v + 1]; t++) {
            int32_t u = P->adj[t];
            if (u == b) { found = 1; break; }
            if (!seen[u] && u < b) { seen[u] = 1; touched[nt++] = u; stk[sp++] = u; }
        }
    }
    for (int32_t i = 0; i < nt; i++) seen[touched[i]] = 0;
    free(touched);
    return found;
}

/*
 * Build.  chain_ptr/chain_elems (nullable): an injected decomposition
 * (SPEC decompose_explicit), chain c = chain_elems[chain_ptr[c]..chain_ptr[c+1])
 * listed top-down (largest first) in user ids.  Returns 0, -1 cycle,
 * -2 self loop, -3 bad input, -4 out of memory, -5 not a chain,
 * -6 not a partition.
 */
int oracle_build(int64_t n, int64_t m, const int64_t *src, const int64_t *dst,
                 int64_t kin, const int64_t *chain_ptr, const int64_t *chain_elems,
                 oracle_poset **out) {
    *out = NULL;
    if (n < 0 || n >= INF_IDX || m < 0) return -3;
    oracle_poset *P = calloc(1, sizeof(oracle_poset));
    P->n = (int32_t)n; P->m = m;
    int rc = number_vertices(P, src, dst);
    if (rc) { oracle_free(P); return rc; }
    if (chain_ptr) {
        P->next = malloc(sizeof(int32_t) * ((size_t)n + 1));
        P->id = calloc((size_t)n + 1, sizeof(int32_t));
        int32_t *stk = malloc(sizeof(int32_t) * ((size_t)n + 1));
        char *seen = calloc((size_t)n + 1, 1);
        P->k = (int32_t)kin; P->q = 0;
        int bad = 0;
        for (int64_t c = 0; c < kin && !bad; c++) {
            int64_t a = chain_ptr[c], b = chain_ptr[c + 1];
            if (b <= a) { bad = -6; break; }
            if (b - a > P->q) P->q = (int32_t)(b - a);
            for (int64_t t = a; t < b; t++) {
                int64_t u = chain_elems[t];
                if (u < 0 || u >= n) { bad = -3; break; }
                int32_t i = P->paper_of[u];
                if (P->id[i]) { bad = -6; break; }
                P->id[i] = (int32_t)(c + 1);
                P->next[i] = (t + 1 < b) ? P->paper_of[chain_elems[t + 1]] : i;
                if (t + 1 < b && !reaches(P, i, P->next[i], stk, seen)) { bad = -5; break; }
            }
        }
        for (int32_t i = 1; i <= n && !bad; i++) if (!P->id[i]) bad = -6;
        free(stk); free(seen);
        if (bad) { oracle_free(P); return bad; }
    } else {
        alg1_matching(P);
        chains_from_next(P);
    }
    alg6_levels(P);
    rc = alg2_niv(P);
    if (rc) { oracle_free(P); return rc; }
    *out = P;
    return 0;
}

/* n, m (deduplicated), k, q, ell, nnz */
void oracle_info(const oracle_poset *P, int64_t *o) {
    o[0] = P->n; o[1] = P->m; o[2] = P->k; o[3] = P->q; o[4] = P->ell; o[5] = P->nnz;
}

/* per user vertex: chain id (0-based), next (user id), level (1-based), paper index */
void oracle_export_chains(const oracle_poset *P, int64_t *chain, int64_t *next,
                          int64_t *level, int64_t *paper) {
    for (int32_t i = 1; i <= P->n; i++) {
        int32_t u = P->user_of[i];
        chain[u] = P->id[i] - 1;
        next[u] = P->user_of[P->next[i]];
        level[u] = P->level[i];
        paper[u] = i;
    }
}

/* dense niv: out[u*k + j] = user id of niv_{j+1}(u) or -1 (infinity) */
void oracle_export_niv(const oracle_poset *P, int64_t *out) {
    int32_t k = P->k;
    for (int64_t t = 0; t < (int64_t)P->n * k; t++) out[t] = -1;
    for (int32_t i = 1; i <= P->n; i++) {
        int32_t u = P->user_of[i];
        for (int64_t e = P->niv_ptr[i]; e < P->niv_ptr[i + 1]; e++) {
            int32_t p = P->niv[e];
            out[(int64_t)u * k + (P->id[p] - 1)] = P->user_of[p];
        }
    }
}

/* ---------------- Alg. 3: fast zeta transform ----------------------------- */
/* x, y are [n][B] row-major in USER order; dtype 0 = int64 (Z/2^64), 1 = fp64 */
int oracle_zeta(const oracle_poset *P, const void *xin, void *yout, int64_t B, int dtype) {
    int32_t n = P->n;
    size_t row = (size_t)B;
    if (dtype == 0) {
        const uint64_t *x = xin; uint64_t *y = yout;
        uint64_t *xp = calloc(((size_t)n + 1) * row, sizeof(uint64_t));    /* x' <- 0 */
        if (!xp) return -4;
        for (int32_t i = n; i >= 1; i--) {                                 /* for i <- n to 1 */
            const uint64_t *xi = x + (size_t)P->user_of[i] * row;
            uint64_t *xpi = xp + (size_t)i * row, *xpn = xp + (size_t)P->next[i] * row;
            for (size_t b = 0; b < row; b++) xpi[b] = xpn[b] + xi[b];      /* x'[i] <- x'[next[i]] + x[i] */
            uint64_t *yi = y + (size_t)P->user_of[i] * row;
            for (size_t b = 0; b < row; b++) yi[b] = 0;
            for (int64_t e = P->niv_ptr[i]; e < P->niv_ptr[i + 1]; e++) {   /* j in niv[i] */
                const uint64_t *xpj = xp + (size_t)P->niv[e] * row;
                for (size_t b = 0; b < row; b++) yi[b] += xpj[b];          /* y[i] <- y[i] + x'[j] */
            }
        }
        free(xp);
    } else {
        const double *x = xin; double *y = yout;
        double *xp = calloc(((size_t)n + 1) * row, sizeof(double));
        if (!xp) return -4;
        for (int32_t i = n; i >= 1; i--) {
            const double *xi = x + (size_t)P->user_of[i] * row;
            double *xpi = xp + (size_t)i * row, *xpn = xp + (size_t)P->next[i] * row;
            for (size_t b = 0; b < row; b++) xpi[b] = xpn[b] + xi[b];
            double *yi = y + (size_t)P->user_of[i] * row;
            for (size_t b = 0; b < row; b++) yi[b] = 0.0;
            for (int64_t e = P->niv_ptr[i]; e < P->niv_ptr[i + 1]; e++) {
                const double *xpj = xp + (size_t)P->niv[e] * row;
                for (size_t b = 0; b < row; b++) yi[b] += xpj[b];
            }
        }
        free(xp);
    }
    return 0;
}

/* ---------------- Alg. 4: fast Moebius transform -------------------------- */
int oracle_moebius(const oracle_poset *P, const void *xin, void *yout, int64_t B, int dtype) {
    int32_t n = P->n;
    size_t row = (size_t)B;
    if (dtype == 0) {
        const uint64_t *x = xin; uint64_t *y = yout;
        uint64_t *yp = calloc(((size_t)n + 1) * row, sizeof(uint64_t));   /* y' <- 0 */
        if (!yp) return -4;
        for (int32_t i = n; i >= 1; i--) {                                 /* first loop */
            uint64_t *ypi = yp + (size_t)i * row;
            const uint64_t *xi = x + (size_t)P->user_of[i] * row;
            for (size_t b = 0; b < row; b++) ypi[b] = xi[b];               /* y'[i] <- x[i] */
            for (int64_t e = P->niv_ptr[i]; e < P->niv_ptr[i + 1]; e++) {
                int32_t j = P->niv[e];
                if (j == i) continue;                                     /* niv[i] \ i */
                const uint64_t *ypj = yp + (size_t)j * row;
                for (size_t b = 0; b < row; b++) ypi[b] -= ypj[b];         /* y'[i] <- y'[i] - y'[j] */
            }
        }
        for (int32_t i = n; i >= 1; i--) {                                 /* second loop */
            uint64_t *yi = y + (size_t)P->user_of[i] * row;
            const uint64_t *ypi = yp + (size_t)i * row;
            if (P->next[i] != i) {
                const uint64_t *ypn = yp + (size_t)P->next[i] * row;
                for (size_t b = 0; b < row; b++) yi[b] = ypi[b] - ypn[b];  /* y'[i] - y'[next[i]] */
            } else {
                for (size_t b = 0; b < row; b++) yi[b] = ypi[b];
            }
        }
        free(yp);
    } else {
        const double *x = xin; double *y = yout;
        double *yp = calloc(((size_t)n + 1) * row, sizeof(double));
        if (!yp) return -4;
        for (int32_t i = n; i >= 1; i--) {
            double *ypi = yp + (size_t)i * row;
            const double *xi = x + (size_t)P->user_of[i] * row;
            for (size_t b = 0; b < row; b++) ypi[b] = xi[b];
            for (int64_t e = P->niv_ptr[i]; e < P->niv_ptr[i + 1]; e++) {
                int32_t j = P->niv[e];
                if (j == i) continue;
                const double *ypj = yp + (size_t)j * row;
                for (size_t b = 0; b < row; b++) ypi[b] -= ypj[b];
            }
        }
        for (int32_t i = n; i >= 1; i--) {
            double *yi = y + (size_t)P->user_of[i] * row;
            const double *ypi = yp + (size_t)i * row;
            if (P->next[i] != i) {
                const double *ypn = yp + (size_t)P->next[i] * row;
                for (size_t b = 0; b < row; b++) yi[b] = ypi[b] - ypn[b];
            } else {
                for (size_t b = 0; b < row; b++) yi[b] = ypi[b];
            }
        }
        free(yp);
    }
    return 0;
}

/* ---------------- brute-force sampled zeta (for full-size sampled parity) --
 * g(x) = sum_{y ⪯ x} f(y) for the listed user vertices only, by a DFS of ↓x
 * over the children lists ("transitive closure ... computed").
 * abs_out (nullable, fp64 only): sum_{y ⪯ x} |f(y)| for the tolerance. */
int oracle_zeta_sampled(const oracle_poset *P, const void *fin, int64_t B, int dtype,
                        int64_t ns, const int64_t *xs, void *gout, double *abs_out) {
    int32_t n = P->n;
    int32_t *stk = malloc(sizeof(int32_t) * ((size_t)n + 1));
    int32_t *seen = calloc((size_t)n + 1, sizeof(int32_t));
    if (!stk || !seen) return -4;
    for (int64_t s = 0; s < ns; s++) {
        int32_t root = P->paper_of[xs[s]];
        int32_t sp = 0;
        stk[sp++] = root; seen[root] = (int32_t)(s + 1);
        if (dtype == 0) {
            const uint64_t *f = fin; uint64_t *g = (uint64_t *)gout + (size_t)s * B;
            for (int64_t b = 0; b < B; b++) g[b] = 0;
            while (sp) {
                int32_t v = stk[--sp];
                const uint64_t *fv = f + (size_t)P->user_of[v] * B;
                for (int64_t b = 0; b < B; b++) g[b] += fv[b];
                for (int64_t t = P->adj_ptr[v]; t < P->adj_ptr[v + 1]; t++)
                    if (seen[P->adj[t]] != s + 1) { seen[P->adj[t]] = (int32_t)(s + 1); stk[sp++] = P->adj[t]; }
            }
        } else {
            const double *f = fin; double *g = (double *)gout + (size_t)s * B;
            double *ga = abs_out ? abs_out + (size_t)s * B : NULL;
            for (int64_t b = 0; b < B; b++) { g[b] = 0; if (ga) ga[b] = 0; }
            while (sp) {
                int32_t v = stk[--sp];
                const double *fv = f + (size_t)P->user_of[v] * B;
                for (int64_t b = 0; b < B; b++) { g[b] += fv[b]; if (ga) ga[b] += fv[b] < 0 ? -fv[b] : fv[b]; }
                for (int64_t t = P->adj_ptr[v]; t < P->adj_ptr[v + 1]; t++)
                    if (seen[P->adj[t]] != s + 1) { seen[P->adj[t]] = (int32_t)(s + 1); stk[sp++] = P->adj[t]; }
            }
        }
    }
    free(stk); free(seen);
    return 0;
}

/* ---------------- brute-force sampled zeta straight from the edge list ----
 * For full-size sampled parity (no matching, no niv): builds the children
 * CSR and sums f over ↓x by DFS for each listed x (definition).
 * dtype 0 int64 (Z/2^64), 1 fp64 (+ Σ|f| into abs_out if non-null). */
int oracle_zeta_sampled_edges(int64_t n, int64_t m, const int64_t *src, const int64_t *dst,
                              const void *fin, int64_t B, int dtype, int64_t ns,
                              const int64_t *xs, void *gout, double *abs_out) {
    int64_t *cp = calloc((size_t)n + 1, sizeof(int64_t));
    int64_t *ci = malloc(sizeof(int64_t) * (size_t)(m ? m : 1));
    int64_t *stk = malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    int64_t *seen = malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    if (!cp || !ci || !stk || !seen) return -4;
    for (int64_t e = 0; e < m; e++) cp[src[e] + 1]++;
    for (int64_t v = 0; v < n; v++) cp[v + 1] += cp[v];
    int64_t *fill = malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    memcpy(fill, cp, sizeof(int64_t) * (size_t)n);
    for (int64_t e = 0; e < m; e++) ci[fill[src[e]]++] = dst[e];
    free(fill);
    for (int64_t v = 0; v < n; v++) seen[v] = -1;
    for (int64_t s = 0; s < ns; s++) {
        int64_t sp = 0;
        stk[sp++] = xs[s];
        seen[xs[s]] = s;
        if (dtype == 0) {
            const uint64_t *f = fin; uint64_t *g = (uint64_t *)gout + (size_t)s * B;
            for (int64_t b = 0; b < B; b++) g[b] = 0;
            while (sp) {
                int64_t v = stk[--sp];
                for (int64_t b = 0; b < B; b++) g[b] += f[(size_t)v * B + b];
                for (int64_t t = cp[v]; t < cp[v + 1]; t++)
                    if (seen[ci[t]] != s) { seen[ci[t]] = s; stk[sp++] = ci[t]; }
            }
        } else {
            const double *f = fin; double *g = (double *)gout + (size_t)s * B;
            double *ga = abs_out ? abs_out + (size_t)s * B : NULL;
            for (int64_t b = 0; b < B; b++) { g[b] = 0; if (ga) ga[b] = 0; }
            while (sp) {
                int64_t v = stk[--sp];
                for (int64_t b = 0; b < B; b++) {
                    double x = f[(size_t)v * B + b];
                    g[b] += x;
                    if (ga) ga[b] += x < 0 ? -x : x;
                }
                for (int64_t t = cp[v]; t < cp[v + 1]; t++)
                    if (seen[ci[t]] != s) { seen[ci[t]] = s; stk[sp++] = ci[t]; }
            }
        }
    }
    free(cp); free(ci); free(stk); free(seen);
    return 0;
}

/* ---------------- parallel CPU baseline (OpenMP) ---------------------------
 * The same Algs. 3 and 4 scheduled as the paper's parallel CPU code: zeta
 * with the chain prefix sums x' computed chain by chain (chains in parallel)
 * and the rows y_i = sum_{j in niv(i)} x'_j in parallel ("for
 * y = U x we can execute all dot products in parallel"); Moebius by Alg. 5
 * (P:L692-705): the antichains L_1..L_ell of Alg. 6 in order, the elements of
 * one antichain in parallel, a barrier between antichains; then the n - k
 * subtractions y = y' - y'[next] in parallel (depth 1).  Every value
 * is the same sum of the same terms as the sequential code, so int64 results
 * are bit-identical (Z/2^64); fp64 sums each y_i in the same order too.
 * Compiled with -fopenmp when available (oracle/chain.py); without it the
 * loops run on one thread.  oracle_threads() reports the thread count. */
#ifdef _OPENMP
#include <omp.h>
#endif

int oracle_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* chains bottom-up: order[cptr[c] .. cptr[c+1]) lists chain c from its lowest
 * element (next[i] == i) to its top, paper indices */
static int chain_lists(const oracle_poset *P, int32_t **order_out, int64_t **cptr_out, int32_t *kc_out) {
    int32_t n = P->n;
    char *pointed = calloc((size_t)n + 1, 1);
    int32_t *order = malloc(sizeof(int32_t) * ((size_t)n + 1));
    int64_t *cptr = malloc(sizeof(int64_t) * ((size_t)n + 2));
    int32_t *stk = malloc(sizeof(int32_t) * ((size_t)n + 1));
    if (!pointed || !order || !cptr || !stk) { free(pointed); free(order); free(cptr); free(stk); return -4; }
    for (int32_t i = 1; i <= n; i++) if (P->next[i] != i) pointed[P->next[i]] = 1;
    int32_t kc = 0;
    int64_t w = 0;
    for (int32_t top = 1; top <= n; top++) {
        if (pointed[top]) continue;
        int32_t len = 0, v = top;                 /* walk top -> bottom */
        for (;;) { stk[len++] = v; if (P->next[v] == v) break; v = P->next[v]; }
        cptr[kc++] = w;
        while (len) order[w++] = stk[--len];      /* store bottom -> top */
    }
    cptr[kc] = w;
    free(pointed); free(stk);
    *order_out = order; *cptr_out = cptr; *kc_out = kc;
    return 0;
}

#define OMP_ZETA(T)                                                                      \
    do {                                                                                 \
        const T *x = xin; T *y = yout;                                                   \
        T *xp = calloc(((size_t)n + 1) * row, sizeof(T));                                \
        if (!xp) { free(order); free(cptr); return -4; }                                 \
        _Pragma("omp parallel for schedule(dynamic, 1)")                                 \
        for (int32_t c = 0; c < kc; c++) {                                               \
            for (int64_t t = cptr[c]; t < cptr[c + 1]; t++) {                            \
                int32_t i = order[t];                                                    \
                const T *xi = x + (size_t)P->user_of[i] * row;                           \
                T *xpi = xp + (size_t)i * row;                                           \
                if (t == cptr[c]) { for (size_t b = 0; b < row; b++) xpi[b] = xi[b]; }   \
                else {                                                                   \
                    const T *xpn = xp + (size_t)P->next[i] * row;                        \
                    for (size_t b = 0; b < row; b++) xpi[b] = xpn[b] + xi[b];            \
                }                                                                        \
            }                                                                            \
        }                                                                                \
        _Pragma("omp parallel for schedule(static, 1024)")                               \
        for (int32_t i = n; i >= 1; i--) {                                               \
            T *yi = y + (size_t)P->user_of[i] * row;                                     \
            for (size_t b = 0; b < row; b++) yi[b] = 0;                                  \
            for (int64_t e = P->niv_ptr[i]; e < P->niv_ptr[i + 1]; e++) {                \
                const T *xpj = xp + (size_t)P->niv[e] * row;                             \
                for (size_t b = 0; b < row; b++) yi[b] += xpj[b];                        \
            }                                                                            \
        }                                                                                \
        free(xp);                                                                        \
    } while (0)

int oracle_zeta_omp(const oracle_poset *P, const void *xin, void *yout, int64_t B, int dtype) {
    int32_t n = P->n, kc = 0;
    size_t row = (size_t)B;
    int32_t *order = NULL;
    int64_t *cptr = NULL;
    if (chain_lists(P, &order, &cptr, &kc)) return -4;
    if (dtype == 0) OMP_ZETA(uint64_t);
    else OMP_ZETA(double);
    free(order); free(cptr);
    return 0;
}

#define OMP_MOEB(T)                                                                      \
    do {                                                                                 \
        const T *x = xin; T *y = yout;                                                   \
        T *yp = calloc(((size_t)n + 1) * row, sizeof(T));                                \
        if (!yp) { free(lv); free(lptr); return -4; }                                    \
        _Pragma("omp parallel")                                                          \
        for (int32_t L = 0; L < P->ell; L++) {          /* Alg. 5: antichain by antichain */ \
            _Pragma("omp for schedule(static)")         /* implicit barrier = line 5 */  \
            for (int64_t t = lptr[L]; t < lptr[L + 1]; t++) {                            \
                int32_t i = lv[t];                                                       \
                T *ypi = yp + (size_t)i * row;                                           \
                const T *xi = x + (size_t)P->user_of[i] * row;                           \
                for (size_t b = 0; b < row; b++) ypi[b] = xi[b];                         \
                for (int64_t e = P->niv_ptr[i]; e < P->niv_ptr[i + 1]; e++) {            \
                    int32_t j = P->niv[e];                                               \
                    if (j == i) continue;                                                \
                    const T *ypj = yp + (size_t)j * row;                                 \
                    for (size_t b = 0; b < row; b++) ypi[b] -= ypj[b];                   \
                }                                                                        \
            }                                                                            \
        }                                                                                \
        _Pragma("omp parallel for schedule(static, 1024)")                               \
        for (int32_t i = n; i >= 1; i--) {                                               \
            T *yi = y + (size_t)P->user_of[i] * row;                                     \
            const T *ypi = yp + (size_t)i * row;                                         \
            if (P->next[i] != i) {                                                       \
                const T *ypn = yp + (size_t)P->next[i] * row;                            \
                for (size_t b = 0; b < row; b++) yi[b] = ypi[b] - ypn[b];                \
            } else {                                                                     \
                for (size_t b = 0; b < row; b++) yi[b] = ypi[b];                         \
            }                                                                            \
        }                                                                                \
        free(yp);                                                                        \
    } while (0)

int oracle_moebius_omp(const oracle_poset *P, const void *xin, void *yout, int64_t B, int dtype) {
    int32_t n = P->n;
    size_t row = (size_t)B;
    /* antichains of Alg. 6 as buckets: bucket L (0-based) = level L + 1
     * (P->level is 1 for the leaves), elements of a bucket in ascending
     * paper index */
    int64_t *lptr = calloc((size_t)P->ell + 1, sizeof(int64_t));
    int64_t *fill = calloc((size_t)P->ell + 1, sizeof(int64_t));
    int32_t *lv = malloc(sizeof(int32_t) * ((size_t)n + 1));
    if (!lptr || !fill || !lv) { free(lptr); free(fill); free(lv); return -4; }
    for (int32_t i = 1; i <= n; i++) lptr[P->level[i]]++;
    for (int32_t L = 0; L < P->ell; L++) lptr[L + 1] += lptr[L];
    for (int32_t L = 0; L < P->ell; L++) fill[L] = lptr[L];
    for (int32_t i = 1; i <= n; i++) lv[fill[P->level[i] - 1]++] = i;
    free(fill);
    if (dtype == 0) OMP_MOEB(uint64_t);
    else OMP_MOEB(double);
    free(lv); free(lptr);
    return 0;
}
