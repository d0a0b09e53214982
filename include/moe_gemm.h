/*
 * moe_gemm.h -- C ABI of K3, the grouped expert GEMM (tcgen05, sm_100a) that
 * streams the weights of the activated expert replicas of one EP rank.
 *
 * It replaces the reference's analytical weight-traffic model
 *   memory_time = (lambda * expert_weight_bytes + dense + tokens*2*hidden*dtype) / HBM
 * (/root/reference/pkg/src/eproute/costmodel.py:83-94) by the measured kernel.
 *
 * Layouts (bf16, row-major):
 *   W     [E, M, K]   weights of E expert slots (M rows of K inputs each)
 *   X     [T, K]      token activations, grouped so each item's tokens are contiguous
 *   Y     [T, M]      outputs (Y[t, m] = sum_k W[e][m, k] * X[t, k])
 *   items [n_items, 4] int32 device array: {e, m_block (128-row block of W),
 *                     t0 (first token row in X / Y), n (tokens, 1..256)}
 * Constraints: M % 128 == 0, K % 64 == 0 (FP8: K % 128 == 0), 16-byte aligned bases.
 *
 * Two tilings: items of <= moe_item_tokens() tokens run the narrow one (8-stage
 * TMA ring, 128 KB of weights in flight per SM), larger items the wide one (4
 * stages).  The *_v2 / FP8 entry points take the bound on the items' token
 * counts; the v1 entry points assume 256 (wide).
 *
 * FP8 (DeepSeek-V3 ships FP8 expert weights): E4M3 weights with one f32 scale
 * per (expert slot, 128-row block) [E, M / 128], E4M3 activations with one f32
 * scale per token row [T]; tcgen05.mma kind::f8f6f4, f32 accumulators, the
 * scales applied in the epilogue, bf16 out.  (DeepSeek's checkpoints scale per
 * 128 x 128 block, i.e. also along K; this kernel scales per 128-row block.)
 */
#ifndef MOE_GEMM_H
#define MOE_GEMM_H

#include <stdint.h>

#include "metro_route.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Y = per-item W[e] . X[t0:t0+n]^T for every item (persistent, one CTA per SM by
 * default; num_ctas > 0 overrides).  Stream-ordered, graph-capturable. */
METRO_API int moe_grouped_gemm_v1(const void *W, int32_t E, int32_t M, int32_t K, const void *X, int32_t T,
                                  const int32_t *items, int32_t n_items, void *Y, int32_t num_ctas,
                                  void *stream);
/* Tokens per item of the items moe_layout_items_v1 builds (the narrow tiling's bound). */
METRO_API int32_t moe_item_tokens(void);
/* v1 with the bound on the items' token counts (<= moe_item_tokens(): narrow tiling). */
METRO_API int moe_grouped_gemm_v2(const void *W, int32_t E, int32_t M, int32_t K, const void *X, int32_t T,
                                  const int32_t *items, int32_t n_items, int32_t max_item_tokens, void *Y,
                                  int32_t num_ctas, void *stream);

/* The same with the item count read on device (*n_items_dev, clamped to
 * items_cap) -- e.g. written by moe_layout_items_v1 -- so route -> layout ->
 * items -> GEMM runs without a host round trip (graph-capturable).  T_cap =
 * rows allocated in X / Y. */
METRO_API int moe_grouped_gemm_dev_v1(const void *W, int32_t E, int32_t M, int32_t K, const void *X,
                                      int32_t T_cap, const int32_t *items, int32_t items_cap,
                                      const int32_t *n_items_dev, void *Y, int32_t num_ctas, void *stream);
METRO_API int moe_grouped_gemm_dev_v2(const void *W, int32_t E, int32_t M, int32_t K, const void *X,
                                      int32_t T_cap, const int32_t *items, int32_t items_cap,
                                      const int32_t *n_items_dev, int32_t max_item_tokens, void *Y, int32_t num_ctas,
                                      void *stream);

/* FP8: W8 [E, M, K] E4M3 + w_scale [E, M / 128], X8 [T, K] E4M3 + x_scale [T]
 * -> Y [T, M] bf16.  n_items_dev nullable (device item count, clamped to n_items). */
METRO_API int moe_grouped_gemm_fp8_v1(const void *W8, const float *w_scale, int32_t E, int32_t M, int32_t K,
                                      const void *X8, const float *x_scale, int32_t T, const int32_t *items,
                                      int32_t n_items, const int32_t *n_items_dev, int32_t max_item_tokens, void *Y,
                                      int32_t num_ctas, void *stream);
/* bf16 rows -> E4M3 rows with one scale per row (max |x| / 448): X [T, K] -> X8, x_scale.
 * rows_dev nullable (device row count, clamped to T). */
METRO_API int moe_quantize_rows_fp8_v1(const void *X, int32_t T, int32_t K, void *X8, float *x_scale,
                                       const int32_t *rows_dev, void *stream);
/* H = silu(GU[:, :I]) * GU[:, I:] straight to E4M3 rows + per-row scales. */
METRO_API int moe_silu_mul_fp8_v1(const void *GU, int32_t T, int32_t I, void *H8, float *h_scale,
                                  const int32_t *rows_dev, void *stream);

/* Work items of EP rank `rank` from a dispatch layout (include/dispatch_layout.h:
 * rep_off [nrep + 1], slot_base [G + 1], device): for each local slot with rows,
 * each 128-row block of an M1-row (and, if M2 > 0, M2-row) weight matrix and each
 * <= moe_item_tokens()-row chunk, {slot, m_block, first row, rows} -- slot-major, then (m_block,
 * chunk).  counts[3] (device) = {items1, items2, rows of the rank}; item counts
 * beyond cap1 / cap2 are not written (the GEMM clamps; check counts on the host). */
METRO_API int moe_layout_items_v1(const int32_t *rep_off, const int32_t *slot_base, int32_t rank, int32_t M1,
                                  int32_t M2, int32_t *items1, int32_t cap1, int32_t *items2, int32_t cap2,
                                  int32_t *counts, void *stream);

/* The rank's receive buffer: dst[pair_row[p]] = src[p / top_k] (row_bytes each)
 * for every pair p with pair_rank[p] == rank (rows >= rows_cap are skipped).
 * row_bytes % 16 == 0, 16-byte aligned src / dst. */
METRO_API int moe_gather_rows_v1(const void *src, int32_t row_bytes, int32_t top_k, const int32_t *pair_rank,
                                 const int32_t *pair_row, int64_t num_pairs, int32_t rank, void *dst,
                                 int32_t rows_cap, void *stream);

/* H[t, i] = silu(GU[t, i]) * GU[t, I + i]  (GU [T, 2I] -> H [T, I], bf16) */
METRO_API int moe_silu_mul_v1(const void *GU, int32_t T, int32_t I, void *H, void *stream);
/* The same over min(T_cap, *rows_dev) rows (device row count). */
METRO_API int moe_silu_mul_dev_v1(const void *GU, int32_t T_cap, int32_t I, void *H, const int32_t *rows_dev,
                                  void *stream);

/* cudaError_t of the last failing CUDA call of the MoE entry points (0 if none). */
METRO_API int moe_last_cuda_error(void);
/* Tuning only: per-CTA {start, end} globaltimer stamps (ns) of the next grouped-GEMM
 * launches in this process, written to `stamps` (device, >= 2 x grid int64); NULL
 * disables.  Not for production use. */
METRO_API void moe_debug_set_stamps(int64_t *stamps);


#ifdef __cplusplus
}
#endif
#endif /* MOE_GEMM_H */
