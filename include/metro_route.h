/*
 * metro_route.h -- C ABI of the B200-native (sm_100a) METRO / EPLB routing path.
 *
 * Library: paper_2512_09277_b200/_lib/libmetro_b200.so (built by
 * __graft_entry__.build() / `make -C paper_2512_09277_b200/csrc`).
 *
 * Plain pointers and sizes only (no torch types).  Device pointers are CUDA
 * global-memory pointers; `stream` is a cudaStream_t passed as void*.  All
 * device entry points are asynchronous and stream-ordered, graph-capturable,
 * and never synchronise except metro_route_host_v1 (the end-to-end call).
 *
 * Each entry point replaces one function of the reference package
 * (/root/reference/pkg/src/eproute, pure Python):
 *
 *   metro_route_v1            <- core.py:236-244 aggregate_loads  +
 *                                routing.py:105-113 route_metro  (+ :41-52 x/y/lam)
 *                                fused, from the all-gathered top-k ids
 *   metro_route_from_loads_v1 <- routing.py:105-113 route_metro(T, A)  (T given)
 *   metro_route_ordered_v1    <- routing.py:90-102 _greedy_assign with a caller
 *                                order (route_metro_parallel, routing.py:116-128)
 *   eplb_route_v1             <- core.py:236-244 + routing.py:55-72 route_eplb
 *   eplb_route_from_loads_v1  <- routing.py:55-72 route_eplb(T, A)
 *   metro_aggregate_loads_v1  <- core.py:236-244 aggregate_loads alone
 *   metro_route_scores_v1     <- the gating top-k (core.py:319-326, the
 *                                reference's generator of top-k ids) fused with
 *                                metro_route_v1
 *   metro_pack_placement      <- core.py:84-119 PlacementMap (binary A -> bitmasks)
 *   metro_route_host_v1       <- the same as metro_route_v1 from HOST buffers
 *                                (H2D, kernel, D2H, sync) -- the e2e call
 *
 * Error behaviour (mirrors the reference's exceptions):
 *   return value < 0  : host-detectable argument error (ValidationError in Python:
 *                       dimension mismatch routing.py:29-33, sizes, alignment)
 *   status[0] (device): written by the kernel at the end of every launch
 *       METRO_OK              0
 *       METRO_ERR_ID_RANGE    1  status[1..2] = first bad pair index (lo, hi),
 *                                status[3] = the bad id
 *                                (ValidationError "token t: expert id e out of
 *                                range", core.py:241-242; t = pair / k)
 *       METRO_ERR_NO_REPLICA  2  status[1] = lowest active expert without a
 *                                replica (AssertionError, routing.py:66, :99)
 *       METRO_ERR_LOAD_RANGE  3  a load does not fit 32 bits on the loads path
 *                                (the host wrapper rank-compresses loads first)
 *   Outputs are unspecified when status[0] != 0.
 *
 * Layouts (all row-major, int32 unless noted):
 *   topk_ids   [num_pairs]           = [B, k] global (all-gathered) batch
 *   rank_mask  [N, W] uint32         bit (g % 32) of word g / 32 set iff expert
 *                                    i has a replica on EP rank g; W = ceil(G/32)
 *   loads      [N]                   T[i] (aggregate_loads)
 *   choice     [N]                   METRO: the single rank serving expert i,
 *                                    -1 if T[i] == 0
 *   x          [N, G]                EPLB token split (int32; int64 on the
 *                                    from_loads entry point)
 *   rank_counts[G]                   activated replicas per EP rank (column sums of y)
 *   lam        [1]                   max_g rank_counts[g]  (0 if no expert active)
 *   pair_rank  [num_pairs] (nullable) EP rank serving each (token, slot) pair
 *   status     [4]
 *
 * Limits: 1 <= G <= 128, 1 <= N <= 4096, num_pairs < 2^31 (and the per-launch
 * shared-memory plan must fit 227 KB; every BASELINE shape does).
 */
#ifndef METRO_ROUTE_H
#define METRO_ROUTE_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define METRO_API __attribute__((visibility("default")))
#else
#define METRO_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define METRO_ABI_VERSION 1

enum {
    METRO_OK = 0,
    METRO_ERR_ID_RANGE = 1,
    METRO_ERR_NO_REPLICA = 2,
    METRO_ERR_LOAD_RANGE = 3,
    METRO_ERR_PAIR_RANK = 4,  /* dispatch layout: pair_rank[p] hosts no replica of ids[p] */
    METRO_EARG = -1,       /* null pointer / negative size */
    METRO_EDIMS = -2,      /* N or G outside the supported range */
    METRO_ECUDA = -3,      /* CUDA launch / copy error (see metro_last_cuda_error) */
    METRO_ENOTBINARY = -4, /* placement matrix not binary */
    METRO_ENOMEM = -5,     /* host allocation failed (launch plans) */
};

METRO_API int metro_abi_version(void);
METRO_API const char *metro_strerror(int code);
/* cudaError_t of the last failing CUDA call in this thread (0 if none). */
METRO_API int metro_last_cuda_error(void);
/* Words per expert in rank_mask: ceil(G / 32). */
METRO_API int metro_mask_words(int32_t num_ranks);

/* Host-side: pack a binary int8 placement A[N, G] into rank_mask[N, W].
 * Returns METRO_ENOTBINARY if an entry is not 0/1.  (PlacementMap, core.py:84-119) */
METRO_API int metro_pack_placement(const int8_t *A, int32_t num_experts, int32_t num_ranks,
                         uint32_t *rank_mask_out);

/* METRO from all-gathered top-k ids.  cluster_ctas: CTAs in the thread-block
 * cluster that stages/histograms the ids (1,2,4,8,16; 0 = auto). */
METRO_API int metro_route_v1(const int32_t *topk_ids, int64_t num_pairs, const uint32_t *rank_mask,
                   int32_t num_experts, int32_t num_ranks, int32_t *loads, int32_t *choice,
                   int32_t *rank_counts, int32_t *lam, int32_t *pair_rank, int32_t *status,
                   int32_t cluster_ctas, void *stream);

/* Gating top-k fused with METRO.  scores [num_tokens, N]
 * fp32 router scores of the all-gathered tokens; each token's top_k experts --
 * largest score first, ties to the lower expert id, the descending-key order of
 * the reference's generator (core.py:319-326) -- are written to topk_ids
 * [num_tokens, top_k] and counted as they are chosen (no separate pass over the
 * ids), then routed.  Other outputs as metro_route_v1.
 * ws: metro_scores_workspace_bytes(N) bytes of device memory, ZEROED ONCE by the
 * caller; the kernel leaves it zeroed (one workspace per stream).  Two variants:
 *   whole GPU   -- 32 tokens' top-k per CTA on every SM, partial counts added into
 *                  ws with atomics; a programmatically dependent launch of
 *                  routing CTAs (resident while the top-k runs) routes from ws,
 *                  each writing a share of the pair ranks (needs ws; two launches);
 *   one cluster -- the routing cluster also takes the top-k (one launch, no ws).
 * cluster_ctas: 0 = auto (one cluster up to 512 tokens, whole GPU above when ws
 * is given), -1 = whole GPU, 1/2/4/8/16 = one cluster of that size.
 * Order: larger score first, equal scores (incl. -0.0 == +0.0) to the lower
 * expert id, NaN below every number (taken last; ties among NaNs to the lower id).
 * Limits: N <= 512, G <= 32, top_k <= 32, top_k <= N. */
METRO_API size_t metro_scores_workspace_bytes(int32_t num_experts);
METRO_API int metro_route_scores_v1(const float *scores, int64_t num_tokens, int32_t top_k,
                                    const uint32_t *rank_mask, int32_t num_experts, int32_t num_ranks,
                                    int32_t *topk_ids, int32_t *loads, int32_t *choice, int32_t *rank_counts,
                                    int32_t *lam, int32_t *pair_rank, int32_t *status, void *ws,
                                    int32_t cluster_ctas, void *stream);

/* aggregate_loads only (core.py:236-244): loads[N] from the ids; status as above. */
METRO_API int metro_aggregate_loads_v1(const int32_t *topk_ids, int64_t num_pairs,
                                       int32_t num_experts, int32_t *loads, int32_t *status,
                                       int32_t cluster_ctas, void *stream);

/* METRO from a given load vector T (int64).  Loads must be < 2^32 (host
 * wrappers rank-compress larger values; the greedy only compares them). */
METRO_API int metro_route_from_loads_v1(const int64_t *loads, const uint32_t *rank_mask,
                              int32_t num_experts, int32_t num_ranks, int32_t *choice,
                              int32_t *rank_counts, int32_t *lam, int32_t *status,
                              void *stream);

/* Greedy over a caller-supplied order of `m` expert ids (metro-parallel's
 * seeded serialisation).  Experts not in `order` stay unassigned (-1). */
METRO_API int metro_route_ordered_v1(const int32_t *order, int32_t m, const uint32_t *rank_mask,
                           int32_t num_experts, int32_t num_ranks, int32_t *choice,
                           int32_t *rank_counts, int32_t *lam, int32_t *status,
                           void *stream);

/* EPLB even split from all-gathered top-k ids.  x and pair_rank are nullable.
 * pair_rank convention: the o-th row-major occurrence of expert i goes to its
 * (o mod r_i)-th replica in ascending rank id (reproduces x exactly). */
METRO_API int eplb_route_v1(const int32_t *topk_ids, int64_t num_pairs, const uint32_t *rank_mask,
                  int32_t num_experts, int32_t num_ranks, int32_t *loads, int32_t *x,
                  int32_t *rank_counts, int32_t *lam, int32_t *pair_rank, int32_t *status,
                  int32_t cluster_ctas, void *stream);

/* EPLB from a given load vector (int64 x output, any non-negative int64 loads). */
METRO_API int eplb_route_from_loads_v1(const int64_t *loads, const uint32_t *rank_mask,
                             int32_t num_experts, int32_t num_ranks, int64_t *x,
                             int32_t *rank_counts, int32_t *lam, int32_t *status,
                             void *stream);

/* End-to-end METRO from HOST buffers, synchronous.  Two transfer modes:
 *   flags = 0                    : cudaMemcpyAsync H2D of the ids into dev_workspace
 *                                  (metro_host_workspace_bytes() bytes), the kernel,
 *                                  D2H of the results, stream synchronise;
 *   flags & METRO_HOST_ZEROCOPY  : the kernel reads the ids from and writes the
 *                                  results to pinned (device-mapped) host memory
 *                                  directly over PCIe; dev_workspace unused.
 * host_out [8 + G + N] int32 receives: status[4], lam, pad[3], rank_counts[G],
 * choice[N].  pair_rank_host [num_pairs] is nullable. */
#define METRO_HOST_ZEROCOPY 1
/* flag: the host buffers stay allocated (pinned) across calls, so their
 * device-accessibility check is done once and cached */
#define METRO_HOST_STABLE_BUFFERS 2
METRO_API size_t metro_host_workspace_bytes(int64_t num_pairs, int32_t num_experts, int32_t num_ranks);
METRO_API int metro_route_host_v1(const int32_t *topk_ids_host, int64_t num_pairs,
                                  const uint32_t *rank_mask_dev, int32_t num_experts, int32_t num_ranks,
                                  void *dev_workspace, int32_t *host_out, int32_t *pair_rank_host,
                                  int32_t cluster_ctas, int32_t flags, void *stream);

/* Launch plans for eager callers (no CUDA graph): the argument checks, the
 * cluster / shared-memory plan and the kernel choice of metro_route_v1 /
 * eplb_route_v1 done ONCE for fixed buffers, so each layer's launch is one call
 * with two arguments.  kind: METRO_PLAN_METRO (metro_route_v1's arguments; x
 * unused) or METRO_PLAN_EPLB (eplb_route_v1's; choice unused).  The buffers must
 * stay allocated while the plan is used; num_pairs is fixed (a new batch size
 * needs a new plan).  Same outputs, status words and parity as the one-shot
 * entry points (routing.py:105-113 / :55-72). */
#define METRO_PLAN_METRO 0
#define METRO_PLAN_EPLB 1
typedef struct metro_route_plan metro_route_plan;
METRO_API int metro_route_plan_create_v1(int32_t kind, const int32_t *topk_ids, int64_t num_pairs,
                                         const uint32_t *rank_mask, int32_t num_experts, int32_t num_ranks,
                                         int32_t *loads, int32_t *choice, int32_t *x, int32_t *rank_counts,
                                         int32_t *lam, int32_t *pair_rank, int32_t *status, int32_t cluster_ctas,
                                         metro_route_plan **plan_out);
METRO_API int metro_route_plan_launch_v1(const metro_route_plan *plan, void *stream);
METRO_API int metro_route_plan_destroy_v1(metro_route_plan *plan);

/* Programmatic dependent launch of the routing kernels (default on; METRO_PDL=0
 * in the environment or metro_set_pdl(0) turns it off).  With it a routing
 * kernel launched behind another kernel in the stream (the gating kernel in a
 * decode step) runs its shared-memory prologue while that kernel finishes and
 * waits (griddepcontrol.wait) for its completion before the first global
 * access; it also lets the next kernel do the same. */
METRO_API void metro_set_pdl(int32_t enable);

/* Debug / tuning: per-phase clock64 stamps of CTA 0 of the next metro_route_v1
 * launch in this process are written to `stamps` (device, >= 16 int64) when set;
 * pass NULL to disable.  Not for production use. */
METRO_API void metro_debug_set_stamps(int64_t *stamps);

#ifdef __cplusplus
}
#endif
#endif /* METRO_ROUTE_H */
