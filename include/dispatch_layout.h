/*
 * dispatch_layout.h -- C ABI of the dispatch layout that follows routing
 * (SURVEY.md §8(f) rank 1): where every (token, slot) pair lands in the receive
 * buffer of the EP rank that serves it, and the per-replica row ranges the
 * grouped expert GEMM (include/moe_gemm.h) consumes.
 *
 * The reference stops at the routing decision; its row counts are the entries
 * of the assignment matrix x (routing.py:41-52 for METRO, x[i, choice[i]] = T[i];
 * routing.py:64-69 for EPLB) and simulate.py:87-88 prices the rank's tokens.
 * This layout materialises exactly those counts: rank g's rows for expert i
 * number x[i, g].
 *
 * Replica numbering ("rid"), fixed per placement: replicas are numbered
 * rank-major and, within a rank, by local slot, where the local slot of expert i
 * on rank g is the number of experts < i hosted on g (the order a rank's expert
 * weight tensor is laid out in).  slot_base[g] = first rid of rank g,
 * slot_base[G] = total replicas (nrep).
 *
 * Row order (deterministic, the convention the parity tests pin): a rank's rows
 * are grouped by local slot ascending; inside a slot, by pair index ascending
 * (row-major over the all-gathered [B, k] ids).
 */
#ifndef DISPATCH_LAYOUT_H
#define DISPATCH_LAYOUT_H

#include <stdint.h>

#include "metro_route.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Host, once per placement.  A [N, G] binary int8 (core.py:84-119 PlacementMap).
 * rid_tab [N, G] int32: rid of (i, g), -1 if rank g hosts no replica of i.
 * slot_base [G + 1] int32.  Returns METRO_ENOTBINARY on a non-binary entry. */
METRO_API int metro_replica_table(const int8_t *A, int32_t num_experts, int32_t num_ranks, int32_t *rid_tab,
                                  int32_t *slot_base);

/* Device.  For every pair p (expert topk_ids[p], serving rank pair_rank[p] as
 * written by metro_route_v1 / eplb_route_v1):
 *   pair_row[p]  row of p inside rank pair_rank[p]'s receive buffer
 *   rep_off[nrep + 1]  exclusive prefix of rows per replica in rid order, so
 *                rank g's rows of its local slot s are
 *                [rep_off[slot_base[g] + s], rep_off[slot_base[g] + s + 1]) minus
 *                rep_off[slot_base[g]], and rank g receives
 *                rep_off[slot_base[g + 1]] - rep_off[slot_base[g]] rows.
 * rid_tab / slot_base are device copies of metro_replica_table's outputs.
 * status [4]: METRO_OK; METRO_ERR_ID_RANGE (status[1..2] = first bad pair, lo/hi,
 * status[3] = the id); METRO_ERR_PAIR_RANK (status[1..2] = first pair whose rank
 * hosts no replica of its expert, status[3] = that rank).
 * cluster_ctas: CTAs of the thread-block cluster sharing the pairs (0 = auto).
 * Limits: nrep <= 4096, num_pairs <= 8192 * 16, 1 <= G <= 128, 1 <= N <= 4096. */
METRO_API int metro_dispatch_layout_v1(const int32_t *topk_ids, const int32_t *pair_rank, int64_t num_pairs,
                                       const int32_t *rid_tab, const int32_t *slot_base,
                                       int32_t num_experts, int32_t num_ranks,
                                       int32_t nrep, int32_t *pair_row, int32_t *rep_off, int32_t *status,
                                       int32_t cluster_ctas, void *stream);

/* METRO routing fused with its dispatch layout in ONE launch: the outputs of
 * metro_route_v1 (loads, choice, rank_counts, lam, pair_rank, status) and of
 * metro_dispatch_layout_v1 on that routing (pair_row, rep_off), identical to the
 * two launches chained.  A METRO expert has one active replica (e, choice[e])
 * with T[e] rows (routing.py:46-50), so the layout needs only the histogram the
 * routing already builds plus row-major occurrence ranks, which the kernel's
 * idle warps compute while the serial greedy runs.  Falls back to the two
 * launches when no fused plan fits shared memory (or for an empty batch).
 * pair_rank and pair_row are required when num_pairs > 0. */
METRO_API int metro_route_layout_v1(const int32_t *topk_ids, int64_t num_pairs, const uint32_t *rank_mask,
                                    int32_t num_experts, int32_t num_ranks, const int32_t *rid_tab,
                                    const int32_t *slot_base, int32_t nrep, int32_t *loads, int32_t *choice,
                                    int32_t *rank_counts, int32_t *lam, int32_t *pair_rank, int32_t *pair_row,
                                    int32_t *rep_off, int32_t *status, int32_t cluster_ctas, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* DISPATCH_LAYOUT_H */
