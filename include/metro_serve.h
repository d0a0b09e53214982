/*
 * metro_serve.h -- persistent end-to-end METRO router (sm_100a) for HOST callers.
 *
 * Same computation and output layout as metro_route_host_v1 (metro_route.h):
 * the reference's aggregate_loads + route_metro (core.py:236-244,
 * routing.py:105-113) from top-k ids in host memory, results back in host
 * memory.  The difference is the transport: instead of a kernel launch and a
 * stream synchronise per call (~9 us of launch + sync latency on the B200 box
 * before any work happens), ONE resident CTA waits on a doorbell word in
 * pinned host memory.  A call writes its arguments and rings the doorbell; the
 * CTA reads the ids over PCIe (zero-copy, system-scope loads), routes them with
 * the same device phases as metro_route_v1 (metro_core.cuh), writes the results
 * straight into the caller's pinned buffers, fences at system scope and
 * publishes a completion word the caller spins on.
 *
 *   metro_server_create_v1   start a server for one placement (device rank masks)
 *   metro_server_route_v1    one routing call (synchronous; thread-safe per server
 *                            only under the caller's own lock)
 *   metro_server_destroy_v1  stop the resident CTA and free the server
 *
 * The resident CTA occupies one SM while it runs.  It exits by itself after
 * `idle_timeout_us` without a request (so a cudaDeviceSynchronize elsewhere in
 * the process waits at most that long) and is relaunched transparently by the
 * next call.  Placement changes (rebalance windows) need a new server: the
 * rank masks are read once per launch of the resident CTA.
 *
 * Buffers: ids_host [num_pairs] int32, host_out [8 + G + N] int32
 * ([status 4 | lam | pad 3 | rank_counts G | choice N], as metro_route_host_v1)
 * and pair_rank_host [num_pairs] (nullable) must be pinned, device-mapped host
 * memory (cudaHostAlloc / cudaHostRegister / torch pin_memory) and 16-byte
 * aligned.  num_pairs <= max_pairs given at creation.
 *
 * Return codes: METRO_OK, METRO_EARG (bad pointer / alignment / size),
 * METRO_EDIMS (N, G or max_pairs outside the supported range), METRO_ECUDA
 * (launch failure or the resident CTA stopped answering: the call times out
 * after 2 s instead of hanging).  Data errors (id out of range, expert without
 * replica) come back in host_out's status words exactly as metro_route_host_v1.
 */
#ifndef METRO_SERVE_H
#define METRO_SERVE_H

#include <stddef.h>
#include <stdint.h>

#include "metro_route.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct metro_server metro_server;

METRO_API int metro_server_create_v1(const uint32_t *rank_mask_dev, int32_t num_experts, int32_t num_ranks,
                                     int64_t max_pairs, int32_t idle_timeout_us, metro_server **out);
METRO_API int metro_server_route_v1(metro_server *server, const int32_t *ids_host, int64_t num_pairs,
                                    int32_t *host_out, int32_t *pair_rank_host);
/* Launches of the resident CTA so far (1 + relaunches after idle exits). */
METRO_API int64_t metro_server_launches(const metro_server *server);
METRO_API int metro_server_destroy_v1(metro_server *server);
/* Debug / tuning: phase times of the last completed request, from the resident
 * CTA's %globaltimer (ns): [0] doorbell seen (absolute), [1] ids staged,
 * [2] routed, [3] results stored, [4] system fence, [5] SM cycles over [1..4],
 * [6] total ns over [1..4], [7] PCIe round trip of the doorbell load that saw
 * the request (ns). */
METRO_API int metro_server_debug_stamps(const metro_server *server, int64_t *out8);

#ifdef __cplusplus
}
#endif
#endif /* METRO_SERVE_H */
