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
 * Constraints: M % 128 == 0, K % 64 == 0, 16-byte aligned bases.
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

/* H[t, i] = silu(GU[t, i]) * GU[t, I + i]  (GU [T, 2I] -> H [T, I], bf16) */
METRO_API int moe_silu_mul_v1(const void *GU, int32_t T, int32_t I, void *H, void *stream);

/* cudaError_t of the last failing CUDA call of the MoE entry points (0 if none). */
METRO_API int moe_last_cuda_error(void);

#ifdef __cplusplus
}
#endif
#endif /* MOE_GEMM_H */
