/*
 * metro_oracle.c -- CPU restatement of the reference's METRO / EPLB routing path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the sm_100a
 * kernels in paper_2512_09277_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The product
 * path never calls it (and has no CPU fallback).
 *
 * Parity is pinned: tests/test_oracle_golden.py checks every function below
 * against golden vectors produced by the unmodified reference package
 * (tests/golden/make_golden.py imports /root/reference/pkg/src/eproute).
 *
 * Each function restates one reference function literally (no shortcuts such
 * as the forced single-replica prefix the CUDA kernel uses), so that the
 * kernel's algebraic shortcuts are checked, not assumed:
 *   oracle_aggregate_loads   <- pkg/src/eproute/core.py:236-244
 *   oracle_route_metro       <- pkg/src/eproute/routing.py:75-113 (+ :41-52)
 *   oracle_route_metro_order <- pkg/src/eproute/routing.py:90-102 (explicit order,
 *                               used by route_metro_parallel :116-128)
 *   oracle_route_eplb        <- pkg/src/eproute/routing.py:55-72
 *   oracle_pair_rank_metro   <- routing.py:49 (x[i, choice[i]] = T[i]: every
 *                               (token, expert) pair of expert i goes to choice[i])
 *   oracle_pair_rank_eplb    <- convention of SURVEY.md §8(b): the o-th
 *                               row-major occurrence of expert i goes to its
 *                               (o mod r_i)-th replica in ascending GPU id,
 *                               which reproduces route_eplb's x exactly.
 *   oracle_gate_topk         <- the top-k selection of the reference's batch
 *                               generator (core.py:319-326: argpartition of the
 *                               negated scores, then descending by score) -- the
 *                               gating step fused into metro_route_scores_v1.
 *                               Ties (measure zero for the reference's continuous
 *                               scores) go to the lower expert id.
 *   oracle_dispatch_layout   <- the dispatch layout after routing (SURVEY.md
 *                               §8(f) rank 1; include/dispatch_layout.h): rows of
 *                               replica (i, g) number x[i, g] (routing.py:41-52,
 *                               :64-69); rows grouped by (rank, local slot), pairs
 *                               in row-major order inside a replica.  Written as
 *                               the obvious sequential counting pass.
 *
 * Integer-only; no floating point anywhere on this path.
 */
#include <stdint.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

enum {
    ORACLE_OK = 0,
    ORACLE_ERR_ID_RANGE = 1,      /* ValidationError("token t: expert id e out of range") */
    ORACLE_ERR_NO_REPLICA = 2,    /* AssertionError("placement invariant: ...") */
    ORACLE_ERR_ARG = 3,
};

int oracle_abi_version(void) { return 1; }

/* core.py:236-244.  Counts (token, slot) selections per expert; stops at the
 * first out-of-range id (row-major scan order == the reference's loop order). */
int oracle_aggregate_loads(const int32_t *ids, int64_t npairs, int32_t N,
                           int64_t *loads, int64_t *bad_pair) {
    if (N < 0 || npairs < 0) return ORACLE_ERR_ARG;
    memset(loads, 0, sizeof(int64_t) * (size_t)N);
    for (int64_t p = 0; p < npairs; ++p) {
        int32_t e = ids[p];
        if (e < 0 || e >= N) {
            if (bad_pair) *bad_pair = p;
            return ORACLE_ERR_ID_RANGE;
        }
        loads[e] += 1;
    }
    return ORACLE_OK;
}

/* ---- _active_order (routing.py:75-87) -------------------------------- */
typedef struct {
    int64_t r;    /* replica count = row sum of A (routing.py:82) */
    int64_t t;    /* load T[i] */
    int32_t id;
} order_key;

static int cmp_order_key(const void *pa, const void *pb) {
    const order_key *a = (const order_key *)pa, *b = (const order_key *)pb;
    /* key = (replica_counts[i], -T[i], i), ascending (routing.py:84-86) */
    if (a->r != b->r) return a->r < b->r ? -1 : 1;
    if (a->t != b->t) return a->t > b->t ? -1 : 1;
    if (a->id != b->id) return a->id < b->id ? -1 : 1;
    return 0;
}

/* _greedy_assign (routing.py:90-102) + _assignment_from_choice (:41-52).
 * choice[i] = GPU chosen for expert i, -1 if expert i is not in `order`.
 * rank_counts[g] = column sums of y; *lam = max_g rank_counts (0 when no
 * expert was assigned, routing.py:51). */
int oracle_route_metro_order(const int64_t *loads, const int8_t *A, int32_t N,
                             int32_t G, const int32_t *order, int32_t m,
                             int32_t *choice, int64_t *rank_counts, int64_t *lam) {
    (void)loads;
    if (N < 0 || G < 0 || m < 0) return ORACLE_ERR_ARG;
    for (int32_t i = 0; i < N; ++i) choice[i] = -1;
    for (int32_t g = 0; g < G; ++g) rank_counts[g] = 0;
    for (int32_t s = 0; s < m; ++s) {
        int32_t i = order[s];
        int32_t best = -1;
        /* A.replicas(i) = ascending GPU ids with A[i,g] != 0 (core.py:104-106);
         * replace only on strict '<', so the lowest id wins ties (:96-98). */
        for (int32_t g = 0; g < G; ++g) {
            if (A[(int64_t)i * G + g] == 0) continue;
            if (best < 0 || rank_counts[g] < rank_counts[best]) best = g;
        }
        if (best < 0) return ORACLE_ERR_NO_REPLICA;
        choice[i] = best;
        rank_counts[best] += 1;
    }
    int64_t mx = 0;
    for (int32_t g = 0; g < G; ++g)
        if (rank_counts[g] > mx) mx = rank_counts[g];
    *lam = (m > 0) ? mx : 0;
    return ORACLE_OK;
}

/* route_metro (routing.py:105-113): canonical order then greedy. */
int oracle_route_metro(const int64_t *loads, const int8_t *A, int32_t N, int32_t G,
                       int32_t *choice, int64_t *rank_counts, int64_t *lam) {
    if (N < 0 || G < 0) return ORACLE_ERR_ARG;
    order_key *keys = (order_key *)malloc(sizeof(order_key) * (size_t)(N > 0 ? N : 1));
    int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N > 0 ? N : 1));
    if (!keys || !order) { free(keys); free(order); return ORACLE_ERR_ARG; }
    int32_t m = 0;
    for (int32_t i = 0; i < N; ++i) {
        if (loads[i] == 0) continue;               /* np.flatnonzero(T.loads) */
        int64_t r = 0;
        for (int32_t g = 0; g < G; ++g) r += A[(int64_t)i * G + g];
        keys[m].r = r;
        keys[m].t = loads[i];
        keys[m].id = i;
        ++m;
    }
    qsort(keys, (size_t)m, sizeof(order_key), cmp_order_key);
    for (int32_t s = 0; s < m; ++s) order[s] = keys[s].id;
    int rc = oracle_route_metro_order(loads, A, N, G, order, m, choice, rank_counts, lam);
    free(keys);
    free(order);
    return rc;
}

/* route_eplb (routing.py:55-72).  x is dense int64 [N, G]. */
int oracle_route_eplb(const int64_t *loads, const int8_t *A, int32_t N, int32_t G,
                      int64_t *x, int64_t *rank_counts, int64_t *lam) {
    if (N < 0 || G < 0) return ORACLE_ERR_ARG;
    memset(x, 0, sizeof(int64_t) * (size_t)N * (size_t)G);
    for (int32_t i = 0; i < N; ++i) {
        if (loads[i] == 0) continue;
        int64_t r = 0;
        for (int32_t g = 0; g < G; ++g) r += (A[(int64_t)i * G + g] != 0);
        if (r == 0) return ORACLE_ERR_NO_REPLICA;   /* routing.py:66 */
        int64_t base = loads[i] / r, rem = loads[i] % r;
        int64_t rank = 0;
        for (int32_t g = 0; g < G; ++g) {
            if (A[(int64_t)i * G + g] == 0) continue;
            x[(int64_t)i * G + g] = base + (rank < rem ? 1 : 0);
            ++rank;
        }
    }
    int64_t mx = 0;
    for (int32_t g = 0; g < G; ++g) {
        int64_t c = 0;
        for (int32_t i = 0; i < N; ++i) c += (x[(int64_t)i * G + g] > 0);  /* y = x > 0 */
        rank_counts[g] = c;
        if (c > mx) mx = c;
    }
    *lam = (N && G) ? mx : 0;
    return ORACLE_OK;
}

/* Per-pair METRO replica: pair p of expert e goes to choice[e] (routing.py:49). */
void oracle_pair_rank_metro(const int32_t *ids, int64_t npairs, const int32_t *choice,
                            int32_t *out) {
    for (int64_t p = 0; p < npairs; ++p) out[p] = choice[ids[p]];
}

/* Per-pair EPLB replica (SURVEY.md §8(b) convention).  occ[] is caller
 * scratch of N int64.  Returns ORACLE_ERR_NO_REPLICA if a selected expert has
 * no replica. */
int oracle_pair_rank_eplb(const int32_t *ids, int64_t npairs, const int8_t *A,
                          int32_t N, int32_t G, int32_t *out) {
    int64_t *occ = (int64_t *)calloc((size_t)(N > 0 ? N : 1), sizeof(int64_t));
    if (!occ) return ORACLE_ERR_ARG;
    for (int64_t p = 0; p < npairs; ++p) {
        int32_t e = ids[p];
        int64_t r = 0;
        for (int32_t g = 0; g < G; ++g) r += (A[(int64_t)e * G + g] != 0);
        if (r == 0) { free(occ); return ORACLE_ERR_NO_REPLICA; }
        int64_t q = occ[e] % r;
        occ[e] += 1;
        int64_t seen = 0;
        for (int32_t g = 0; g < G; ++g) {
            if (A[(int64_t)e * G + g] == 0) continue;
            if (seen == q) { out[p] = g; break; }
            ++seen;
        }
    }
    free(occ);
    return ORACLE_OK;
}

/* Whole hot path for one MoE layer, as bench.py's CPU baseline times it:
 * aggregate_loads -> route_metro -> per-pair replica.  Scratch-free for the
 * caller; returns the first error code. */
int oracle_metro_layer(const int32_t *ids, int64_t npairs, const int8_t *A, int32_t N,
                       int32_t G, int64_t *loads, int32_t *choice, int64_t *rank_counts,
                       int64_t *lam, int32_t *pair_rank) {
    int64_t bad = -1;
    int rc = oracle_aggregate_loads(ids, npairs, N, loads, &bad);
    if (rc) return rc;
    rc = oracle_route_metro(loads, A, N, G, choice, rank_counts, lam);
    if (rc) return rc;
    if (pair_rank) oracle_pair_rank_metro(ids, npairs, choice, pair_rank);
    return ORACLE_OK;
}

/* Dispatch layout, sequentially.  Replica ids are rank-major, by local slot
 * (the i-th expert hosted on rank g in ascending expert id); rep_off [nrep + 1]
 * is the exclusive prefix of rows per replica; pair_row[p] is the row of pair p
 * counted from the first row of its serving rank.  Returns ORACLE_ERR_ID_RANGE /
 * ORACLE_ERR_NO_REPLICA (with *bad = pair index) when a pair has an id out of
 * range / a serving rank without a replica of its expert. */
int oracle_dispatch_layout(const int32_t *ids, const int32_t *pair_rank, int64_t npairs, const int8_t *A,
                           int32_t N, int32_t G, int32_t *pair_row, int32_t *rep_off, int64_t *bad) {
    int32_t *rid = (int32_t *)malloc(sizeof(int32_t) * (size_t)N * (size_t)G + 4);
    int32_t *rank_first = (int32_t *)malloc(sizeof(int32_t) * ((size_t)G + 1));
    if (!rid || !rank_first) return ORACLE_ERR_ARG;
    int32_t nrep = 0;
    for (int32_t g = 0; g < G; ++g) {
        rank_first[g] = nrep;
        for (int32_t i = 0; i < N; ++i) rid[(int64_t)i * G + g] = A[(int64_t)i * G + g] ? nrep++ : -1;
    }
    rank_first[G] = nrep;
    int64_t *cnt = (int64_t *)calloc((size_t)nrep + 1, sizeof(int64_t));
    int rc = ORACLE_OK;
    for (int64_t p = 0; p < npairs && rc == ORACLE_OK; ++p) {
        const int32_t e = ids[p], g = pair_rank[p];
        if (e < 0 || e >= N) {
            rc = ORACLE_ERR_ID_RANGE;
            *bad = p;
        } else if (g < 0 || g >= G || rid[(int64_t)e * G + g] < 0) {
            rc = ORACLE_ERR_NO_REPLICA;
            *bad = p;
        } else {
            cnt[rid[(int64_t)e * G + g]]++;
        }
    }
    if (rc == ORACLE_OK) {
        int64_t run = 0;
        for (int32_t r = 0; r < nrep; ++r) {
            rep_off[r] = (int32_t)run;
            run += cnt[r];
            cnt[r] = 0; /* reused: rows handed out so far */
        }
        rep_off[nrep] = (int32_t)run;
        for (int64_t p = 0; p < npairs; ++p) {
            const int32_t e = ids[p], g = pair_rank[p];
            const int32_t r = rid[(int64_t)e * G + g];
            pair_row[p] = (int32_t)(rep_off[r] - rep_off[rank_first[g]] + cnt[r]++);
        }
    }
    free(cnt);
    free(rank_first);
    free(rid);
    return rc;
}

/* Top-k of each token's scores, largest first; equal scores -> lower expert id
 * (-0.0 == +0.0 under float compare).  NaN ranks below every number (numpy's
 * "NaN sorts last" in the reference generator's argsort(-keys), core.py:322-326),
 * ties among NaNs -> lower id.  Written as k rounds of "first maximum" over the
 * not-yet-taken experts. */
void oracle_gate_topk(const float *scores, int64_t T, int32_t N, int32_t k, int32_t *ids) {
    unsigned char *taken = (unsigned char *)malloc((size_t)N + 1);
    for (int64_t t = 0; t < T; ++t) {
        const float *row = scores + t * N;
        memset(taken, 0, (size_t)N);
        for (int32_t r = 0; r < k; ++r) {
            int32_t best = -1;
            for (int32_t e = 0; e < N; ++e)
                if (!taken[e] && (best < 0 || (!isnan(row[e]) && (isnan(row[best]) || row[e] > row[best]))))
                    best = e;
            taken[best] = 1;
            ids[t * k + r] = best;
        }
    }
    free(taken);
}
