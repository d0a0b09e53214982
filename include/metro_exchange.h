/*
 * metro_exchange.h -- all-gather of global top-k knowledge fused with METRO
 * routing in ONE kernel per EP rank, over peer memory (NVLink / NVSwitch P2P).
 *
 * The reference's design point (costed as an ALL_GATHER at
 * costmodel.py:102-129, chosen for the greedy routers at simulate.py:33, :69-70)
 * is that every EP rank sees the global top-k ids and runs the identical
 * deterministic router, so no broadcast of the routing is needed.  The
 * unfused form is an NCCL all-gather of the ids followed by metro_route_v1
 * (dist.DistributedRouter).  This entry point replaces both with one launch:
 *
 *   1. stage this rank's local ids [local_pairs] (TMA) and histogram them;
 *   2. store the histogram row (N counts + the first bad pair) -- and, when
 *      `gathered_ids` is given, the local ids -- straight into every peer's
 *      exchange buffer (P2P stores), then release a per-(parity, source) flag
 *      word on each peer (st.release.sys);
 *   3. wait for the P-1 peer flags of this call (ld.acquire.sys, bounded: a peer
 *      that never arrives gives METRO_ERR_PEER_TIMEOUT instead of a hang);
 *   4. T = sum of the P rows; the METRO decision (routing.py:105-113) -- the
 *      same integer computation on every rank, so identical outputs;
 *   5. write loads / choice / rank_counts / lam / status, pair_rank of the LOCAL
 *      pairs and (optionally) the all-gathered ids, rank-major [P * local_pairs].
 *
 * Routing outputs depend only on T, so exchanging P histogram rows (N * 4 bytes
 * each) carries the same global knowledge as all-gathering B * k ids; the ids
 * are gathered only when a consumer (dispatch layout of all pairs) needs them.
 *
 * Exchange buffers: one per rank, metro_exchange_bytes() bytes, ZEROED once at
 * allocation, identical size on every rank, device memory that every peer can
 * address (cudaIpc / symmetric memory).  peer_exchange[q] is rank q's buffer as
 * addressable from THIS device (peer_exchange[rank] = own).  Calls must be
 * issued in the same order on every rank, on one stream per rank; the buffers
 * are double-buffered by call parity, so a rank may run at most one call ahead
 * of its slowest peer.  Every rank must pass the same local_pairs.
 *
 * Status (device, status[4]) as metro_route_v1, plus
 *   METRO_ERR_PEER_TIMEOUT (5): status[1] = the first peer that did not arrive.
 * Out-of-range ids anywhere in the global batch are reported identically on
 * every rank, with the global (rank-major) pair index.
 */
#ifndef METRO_EXCHANGE_H
#define METRO_EXCHANGE_H

#include <stddef.h>
#include <stdint.h>

#include "metro_route.h"

#ifdef __cplusplus
extern "C" {
#endif

#define METRO_ERR_PEER_TIMEOUT 5
#define METRO_MAX_WORLD 32

/* Bytes of one rank's exchange buffer. */
METRO_API size_t metro_exchange_bytes(int32_t num_experts, int32_t world, int64_t max_local_pairs);

METRO_API int metro_allgather_route_v1(const int32_t *local_ids, int64_t local_pairs, int32_t rank, int32_t world,
                                       void *const *peer_exchange, int64_t max_local_pairs,
                                       const uint32_t *rank_mask, int32_t num_experts, int32_t num_ranks,
                                       int32_t *loads, int32_t *choice, int32_t *rank_counts, int32_t *lam,
                                       int32_t *local_pair_rank, int32_t *gathered_ids, int32_t *status,
                                       void *stream);

/* The same exchange + METRO launch fused with the dispatch layout of the GLOBAL
 * (rank-major) batch (include/dispatch_layout.h semantics): besides the routing
 * outputs, local_pair_row [local_pairs] receives the row of each of this rank's
 * pairs in its serving rank's receive buffer and rep_off [nrep + 1] the rows per
 * replica (identical on every rank).  A pair's row needs only the exchanged
 * per-rank histograms (occurrences of its expert in earlier ranks' slices) and
 * the rank's own ids: no ids are gathered.  rid_tab / slot_base / nrep as
 * metro_replica_table (dispatch_layout.h).  Limits: nrep <= 4096, local_pairs
 * <= 65535.  Reference: the x[i, g] row counts of routing.py:41-52 charged by
 * simulate.py:87-88. */
METRO_API int metro_allgather_route_layout_v1(const int32_t *local_ids, int64_t local_pairs, int32_t rank,
                                              int32_t world, void *const *peer_exchange, int64_t max_local_pairs,
                                              const uint32_t *rank_mask, int32_t num_experts, int32_t num_ranks,
                                              const int32_t *rid_tab, const int32_t *slot_base, int32_t nrep,
                                              int32_t *loads, int32_t *choice, int32_t *rank_counts, int32_t *lam,
                                              int32_t *local_pair_rank, int32_t *local_pair_row, int32_t *rep_off,
                                              int32_t *status, void *stream);

/* An exchange buffer of `bytes` (cudaMalloc'd as its own allocation, so a CUDA
 * IPC handle maps exactly it; zeroed, synchronous) and its release. */
METRO_API int metro_exchange_alloc(size_t bytes, void **dev_ptr_out);
METRO_API int metro_exchange_free(void *dev_ptr);
/* Debug / tuning: globaltimer ns at the phases of every following launch are
 * written to dev_stamps[rank * 8 + phase] (0 start, 1 counted, 2 pushed,
 * 3 received, 4 routed, 5 end); NULL disables.  Not for production use. */
METRO_API void metro_allgather_debug_stamps(int64_t *dev_stamps);
/* CUDA IPC plumbing for the exchange buffers (64-byte cudaIpcMemHandle_t). */
METRO_API int metro_ipc_get_handle(void *dev_ptr, void *handle_out64);
METRO_API int metro_ipc_open_handle(const void *handle64, void **dev_ptr_out);
METRO_API int metro_ipc_close_handle(void *dev_ptr);

#ifdef __cplusplus
}
#endif
#endif /* METRO_EXCHANGE_H */
