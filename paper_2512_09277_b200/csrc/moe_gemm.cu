// moe_gemm.cu -- K3: grouped expert GEMM for the memory-bound MoE decode FFN
// on 5th-generation tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
// Purpose on this path (BASELINE.json north_star (4)):
// show that fewer activated replicas means fewer weight bytes pulled from HBM.
// The reference only models it: memory_time = (lambda * expert_bytes + ...) / HBM
// (/root/reference/pkg/src/eproute/costmodel.py:83-94).
//
// Swap-AB: in decode the token count per expert is small, so the weight matrix
// is the MMA "A" operand on M (128 rows per tile) and the tokens are "B" on N:
//     Y[t, m] = sum_k W[e][m, k] * X[t, k]      (D[m, n] = A[m, k] * B[n, k], both K-major)
// One work item = (expert slot e, 128-row block of W, up to 256 tokens of e).
// Persistent CTAs (one per SM), warp-specialised:
//   warp 4: TMA producer (W tile 128x64, X tile nb x 64, 128B swizzle, mbarrier ring)
//   warp 5: MMA issuer (one thread; tcgen05.mma kind::f16, fp32 accumulators in TMEM,
//           double-buffered so the epilogue of item i overlaps the MMAs of item i+1)
//   warps 0-3: epilogue (tcgen05.ld 32x32b -> bf16 -> coalesced stores)
// Weights are streamed exactly once per item; the kernel is HBM-bound.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "../../include/moe_gemm.h"

namespace moe {

constexpr int BM = 128;        // weight rows per tile (UMMA M)
constexpr int BK = 64;         // bf16 elements per 128-byte swizzled row
constexpr int MAXN = 256;      // tokens per item, wide variant (UMMA N <= 256)
constexpr int kItemTokens = 64;  // the item chunk of moe_layout_items / build_items
constexpr int kThreads = 192;  // 4 epilogue warps + TMA warp + MMA warp
constexpr int A_BYTES = BM * BK * 2;    // 16 KB
constexpr int NMAPS = 5;                // X maps with box heights 16, 32, 64, 128, 256
// Two tilings of the same kernel.  Decode items carry few tokens, so the narrow
// variant spends the shared memory on pipeline depth instead of token rows:
// 8 stages of (16 KB weights + 8 KB tokens) keep 128 KB of weights in flight per
// SM (the HBM latency x per-SM bandwidth product under load), where the wide one
// keeps 64 KB.  Both use 197,888 bytes of shared memory.
template <int NT, int ST>
struct Tile {
    static constexpr int kN = NT;                      // tokens per item (UMMA N)
    static constexpr int kStages = ST;
    static constexpr int kBBytes = NT * BK * 2;
    static constexpr int kSmem = 1024 + ST * (A_BYTES + kBBytes) + 256;
    static constexpr int kTmemCols = 2 * NT < 32 ? 32 : 2 * NT;  // 2 accumulators x NT fp32 columns
};
using WideTile = Tile<256, 4>;
using NarrowTile = Tile<kItemTokens, 8>;

struct Item {
    int e, m_blk, t0, n;
};
// This CTA's item `it` (16-byte load) or an empty item past the end.  Every role
// loads the NEXT item while it works on the current one, so no role starts an
// item with a descriptor round trip on its critical path (~1 % on the FP8 down
// projection, whose 2016 items carry 16 k-blocks each).
// Memory-safety guard: a token count outside [0, max_n] (the tiling's B stage and
// TMEM accumulator width) is clamped, so a malformed item can never overrun shared
// memory or TMEM.  Host items are checked before launch (moe.py); device items
// from moe_layout_items_v1 respect the bound by construction.
__device__ __forceinline__ Item load_item(const Item *items, int it, int n_items, int max_n) {
    if (it >= n_items) return Item{0, 0, 0, 0};
    const int4 v = __ldg(reinterpret_cast<const int4 *>(items + it));
    return Item{v.x, v.y, v.z, min(max(v.w, 0), max_n)};
}

struct Params {
    const float *w_scale;  // FP8: per (expert slot, 128-row block) dequantisation scale [E][M / 128]
    const float *x_scale;  // FP8: per token row [T]
    int mblocks;           // M / 128
    const Item *items;
    int n_items;                // capacity when n_items_dev is set
    const int32_t *n_items_dev; // nullable: item count produced on device (moe_layout_items_v1)
    int K;
    __nv_bfloat16 *Y;
    int ldy;
    int rows;  // rows of X / Y: epilogue stores past it are dropped (memory-safety guard)
    int64_t *stamps;  // tuning only (moe_debug_set_stamps): per CTA {start ns, end ns}
};

struct Maps {
    CUtensorMap w;          // [E][M][K]
    CUtensorMap x[NMAPS];   // [T][K], box heights 16 << i
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, uint64_t *b) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(b))
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *b) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(b))
        : "memory");
}
// UMMA shared-memory descriptor, K-major, 128-byte swizzle: rows of 128 B, 8-row
// atoms of 1024 B (SBO), LBO unused (1), version 1 (sm100), layout type 2.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
           (2ull << 61);
}
// instruction descriptor: D f32, A/B bf16, both K-major, M = 128, N = n
__device__ __forceinline__ uint32_t idesc_bf16(int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
           (static_cast<uint32_t>(BM >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
// FP8 (E4M3 A and B, f32 accumulate): same descriptors, K = 32 elements per MMA
// (32 bytes, as bf16's K = 16), a/b format fields 0 = E4M3
__device__ __forceinline__ uint32_t idesc_e4m3(int n) {
    return (1u << 4) | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(BM >> 4) << 24);
}
__device__ __forceinline__ void umma_e4m3(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t *b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

#define TMEM_LD_X32(taddr, v)                                                                                    \
    asm volatile(                                                                                                \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "   \
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"       \
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),        \
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),   \
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),              \
          "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),              \
          "=r"(v[30]), "=r"(v[31])                                                                                \
        : "r"(taddr))

__device__ __forceinline__ int map_index(int n) {  // smallest box height >= n
    int i = 0;
    while (i < NMAPS - 1 && (16 << i) < n) ++i;
    return i;
}

// PDL (programmatic dependent launch): every kernel here signals its dependents
// first and waits (griddepcontrol.wait) for its predecessors before the first
// global access that may depend on them.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// FP8: a 128-byte swizzled row holds 128 E4M3 elements (64 bf16), so one k-block
// is 128 elements; the shared-memory bytes per stage and the descriptors are the
// same as bf16's.
template <typename TL, bool FP8 = false>
__global__ void __launch_bounds__(kThreads, 1) moe_gemm_kernel(const __grid_constant__ Maps maps, const Params p) {
    constexpr int STAGES = TL::kStages, B_BYTES = TL::kBBytes, MAXN_T = TL::kN, TMEM_COLS = TL::kTmemCols;
    constexpr int BKE = FP8 ? 2 * BK : BK;  // elements per k-block
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char *sA = smem;
    unsigned char *sB = smem + STAGES * A_BYTES;
    uint64_t *full = reinterpret_cast<uint64_t *>(sB + STAGES * B_BYTES);
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;   // [2]
    uint64_t *tempty = tfull + 2;       // [2]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kblocks = p.K / BKE;
    if (warp == 4 && lane == 0)  // the tensor map is a kernel parameter: prefetch before the wait
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.w)) : "memory");
    pdl_wait();
    pdl_launch_dependents();  // only once this kernel runs: at most one dependent waits
    const int n_items = p.n_items_dev ? min(p.n_items, *p.n_items_dev) : p.n_items;

    if (warp == 4 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4);  // one arrival per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 5) {  // TMEM allocation by one full warp
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (p.stamps && threadIdx.x == 0) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.stamps[2 * blockIdx.x] = static_cast<int64_t>(t);
    }

    if (warp == 4) {
        // ---------------- TMA producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            Item nxt = load_item(p.items, blockIdx.x, n_items, TL::kN);
            for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
                const Item item = nxt;
                nxt = load_item(p.items, it + gridDim.x, n_items, TL::kN);
                const int mi = map_index(item.n);
                const uint32_t bbytes = static_cast<uint32_t>((16 << mi) * BK * 2);
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], A_BYTES + bbytes);
                    tma_load_3d(sA + stage * A_BYTES, &maps.w, kb * BKE, item.m_blk * BM, item.e, &full[stage]);
                    tma_load_2d(sB + stage * B_BYTES, &maps.x[mi], kb * BKE, item.t0, &full[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 5) {
        // ---------------- MMA issuer (one thread)
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int local = 0;
            Item nxt = load_item(p.items, blockIdx.x, n_items, TL::kN);
            for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++local) {
                const Item item = nxt;
                nxt = load_item(p.items, it + gridDim.x, n_items, TL::kN);
                const int acc = local & 1;
                const uint32_t aphase = (local >> 1) & 1;
                mbar_wait(&tempty[acc], aphase ^ 1);
                tc_fence_after();
                const int nmma = (item.n + 15) & ~15;
                const uint32_t idesc = FP8 ? idesc_e4m3(nmma) : idesc_bf16(nmma);
                const uint32_t dcol = tmem_base + static_cast<uint32_t>(acc * MAXN_T);
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + stage * A_BYTES), b0 = smem_u32(sB + stage * B_BYTES);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {  // 4 x 32 bytes of K per 128-byte row
                        if (FP8)
                            umma_e4m3(dcol, sw128_desc(a0 + k * 32), sw128_desc(b0 + k * 32), idesc,
                                      (kb | k) != 0 ? 1u : 0u);
                        else
                            umma_bf16(dcol, sw128_desc(a0 + k * 32), sw128_desc(b0 + k * 32), idesc,
                                      (kb | k) != 0 ? 1u : 0u);
                    }
                    umma_commit(&empty[stage]);  // frees the smem slot when these MMAs finish
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit(&tfull[acc]);  // accumulator ready for the epilogue
            }
        }
    } else {
        // ---------------- epilogue: warps 0-3 own TMEM lanes 32w .. 32w+31 (= W rows)
        int local = 0;
        Item nxt = load_item(p.items, blockIdx.x, n_items, TL::kN);
        for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++local) {
            const Item item = nxt;
            nxt = load_item(p.items, it + gridDim.x, n_items, TL::kN);
            const int acc = local & 1;
            const uint32_t aphase = (local >> 1) & 1;
            mbar_wait(&tfull[acc], aphase);
            tc_fence_after();
            const float ws = FP8 ? __ldg(p.w_scale + item.e * p.mblocks + item.m_blk) : 1.0f;
            const uint32_t tbase = tmem_base + static_cast<uint32_t>(acc * MAXN_T) + (static_cast<uint32_t>(warp * 32) << 16);
            for (int c = 0; c < item.n; c += 32) {
                uint32_t v[32];
                // FP8: lane j fetches token c + j's activation scale once (issued before
                // the TMEM load completes); every lane then takes it by shuffle
                float sc = 1.0f;
                if (FP8 && c + lane < item.n && item.t0 + c + lane < p.rows)
                    sc = ws * __ldg(p.x_scale + item.t0 + c + lane);
                TMEM_LD_X32(tbase + static_cast<uint32_t>(c), v);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                const int lim = min(min(32, item.n - c), p.rows - (item.t0 + c));
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    float y = __uint_as_float(v[j]);
                    if (FP8) y *= __shfl_sync(0xffffffffu, sc, j);
                    if (j < lim)
                        p.Y[static_cast<int64_t>(item.t0 + c + j) * p.ldy + item.m_blk * BM + warp * 32 + lane] =
                            __float2bfloat16_rn(y);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (p.stamps && threadIdx.x == 0) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.stamps[2 * blockIdx.x + 1] = static_cast<int64_t>(t);
    }
    if (warp == 5)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                     : "memory");
}

// H[t, i] = silu(GU[t, i]) * GU[t, I + i]   (gate | up halves of the first projection)
// One CTA per row (grid-stride over rows), bf16 pairs: no per-element division.
__global__ void silu_mul_kernel(const __nv_bfloat16 *__restrict__ gu, int T, int I, __nv_bfloat16 *__restrict__ h,
                                const int32_t *rows_dev) {
    pdl_wait();
    pdl_launch_dependents();  // only once this kernel runs: at most one dependent waits
    if (rows_dev) T = min(T, *rows_dev);
    const int pairs = I / 2;
    for (int64_t t = blockIdx.x; t < T; t += gridDim.x) {
        const __nv_bfloat162 *g = reinterpret_cast<const __nv_bfloat162 *>(gu + t * 2 * I);
        const __nv_bfloat162 *u = reinterpret_cast<const __nv_bfloat162 *>(gu + t * 2 * I + I);
        __nv_bfloat162 *o = reinterpret_cast<__nv_bfloat162 *>(h + t * I);
        for (int i = threadIdx.x; i < pairs; i += blockDim.x) {
            const float2 a = __bfloat1622float2(g[i]), b = __bfloat1622float2(u[i]);
            o[i] = __floats2bfloat162_rn(a.x / (1.0f + __expf(-a.x)) * b.x, a.y / (1.0f + __expf(-a.y)) * b.y);
        }
    }
}

// FP8 (E4M3) rows with one scale per row: q[t, :] = e4m3(v[t, :] / s_t),
// s_t = max |v[t, :]| / 448 (1 for an all-zero row).  One 256-thread CTA per row
// (grid-stride over rows): each thread keeps its <= kQPairs element pairs in
// registers, the row's max is a block reduction, and the E4M3 pairs are written
// from registers -- one read of the row.
constexpr int kQThreads = 256, kQPairs = 16;
__device__ __forceinline__ uint16_t e4m3x2(float a, float b) {
    return static_cast<uint16_t>(__nv_cvt_float2_to_fp8x2(make_float2(a, b), __NV_SATFINITE, __NV_E4M3));
}
__device__ __forceinline__ float block_max(float v, float *red) {
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, d));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();  // red is reused row after row
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float m = red[0];
#pragma unroll
    for (int w = 1; w < kQThreads / 32; ++w) m = fmaxf(m, red[w]);
    return m;
}
// MODE 0: v = x[t, :] (bf16 [T, K]); MODE 1: v = silu(gu[t, :K]) * gu[t, K:] (bf16 [T, 2K])
template <int MODE>
__global__ void __launch_bounds__(kQThreads) quantize_fp8_kernel(const __nv_bfloat16 *__restrict__ src, int T, int K,
                                                                 uint8_t *__restrict__ q, float *__restrict__ qs,
                                                                 const int32_t *rows_dev) {
    __shared__ float red[kQThreads / 32];
    pdl_wait();
    pdl_launch_dependents();  // only once this kernel runs: at most one dependent waits
    if (rows_dev) T = min(T, *rows_dev);
    const int pairs = K / 2;
    auto value = [&](int64_t t, int i) -> float2 {
        if (MODE == 0) return __bfloat1622float2(reinterpret_cast<const __nv_bfloat162 *>(src + t * K)[i]);
        const float2 g = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162 *>(src + t * 2 * K)[i]);
        const float2 u = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162 *>(src + t * 2 * K + K)[i]);
        return make_float2(g.x / (1.0f + __expf(-g.x)) * u.x, g.y / (1.0f + __expf(-g.y)) * u.y);
    };
    for (int64_t t = blockIdx.x; t < T; t += gridDim.x) {
        float2 v[kQPairs];
        float m = 0.0f;
#pragma unroll
        for (int j = 0; j < kQPairs; ++j) {
            const int i = threadIdx.x + j * kQThreads;
            v[j] = i < pairs ? value(t, i) : make_float2(0.0f, 0.0f);
            m = fmaxf(m, fmaxf(fabsf(v[j].x), fabsf(v[j].y)));
        }
        for (int i = threadIdx.x + kQPairs * kQThreads; i < pairs; i += kQThreads) {  // rows beyond the registers
            const float2 w = value(t, i);
            m = fmaxf(m, fmaxf(fabsf(w.x), fabsf(w.y)));
        }
        m = block_max(m, red);
        const float sc = m > 0.0f ? m / 448.0f : 1.0f, inv = 1.0f / sc;
        uint16_t *out = reinterpret_cast<uint16_t *>(q + t * K);
#pragma unroll
        for (int j = 0; j < kQPairs; ++j) {
            const int i = threadIdx.x + j * kQThreads;
            if (i < pairs) out[i] = e4m3x2(v[j].x * inv, v[j].y * inv);
        }
        for (int i = threadIdx.x + kQPairs * kQThreads; i < pairs; i += kQThreads) {
            const float2 w = value(t, i);
            out[i] = e4m3x2(w.x * inv, w.y * inv);
        }
        if (threadIdx.x == 0) qs[t] = sc;
    }
}

// Work items of one EP rank from a dispatch layout (include/dispatch_layout.h):
// for every local slot s with rows, every 128-row block of the weight matrix and
// every <= 256-row chunk -> {s, m_blk, t0, n}; slot-major, then (m_blk, chunk) --
// the order of moe.build_items.  Two projections (mb1 / mb2 row blocks) in one
// pass.  One CTA; counts = {items1, items2, rows of the rank}.
constexpr int kItThreads = 512;
__global__ void __launch_bounds__(kItThreads) layout_items_kernel(const int32_t *__restrict__ rep_off,
                                                                  const int32_t *__restrict__ slot_base, int rank,
                                                                  int mb1, int mb2, Item *items1, Item *items2,
                                                                  int cap1, int cap2, int32_t *counts) {
    __shared__ int32_t s_w[32];
    // per slot of the current chunk of kItThreads slots: first chunk (exclusive
    // prefix within the chunk; [kItThreads] = the chunk's total), first row, rows
    __shared__ int32_t s_pre[kItThreads + 1], s_t0[kItThreads], s_n[kItThreads];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    pdl_wait();
    pdl_launch_dependents();  // only once this kernel runs: at most one dependent waits
    const int b0 = slot_base[rank], S = slot_base[rank + 1] - b0;
    const int base_row = rep_off[b0];
    int run = 0;  // chunks of the slots already done
    for (int s0 = 0; s0 < S; s0 += kItThreads) {
        const int s = s0 + tid;
        const int n = (s < S) ? rep_off[b0 + s + 1] - rep_off[b0 + s] : 0;
        const int c = (n + kItemTokens - 1) / kItemTokens;
        int x = c;  // inclusive scan of chunk counts
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += y;
        }
        if (lane == 31) s_w[warp] = x;
        __syncthreads();
        if (warp == 0) {
            int w = lane < kItThreads / 32 ? s_w[lane] : 0;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, w, d);
                if (lane >= d) w += y;
            }
            s_w[lane] = w;
        }
        __syncthreads();
        const int chunk_total = s_w[kItThreads / 32 - 1];
        s_pre[tid] = x - c + (warp > 0 ? s_w[warp - 1] : 0);
        s_t0[tid] = (s < S) ? rep_off[b0 + s] - base_row : 0;
        s_n[tid] = n;
        if (tid == 0) s_pre[kItThreads] = chunk_total;
        __syncthreads();
        // every thread writes items: item q of this chunk belongs to the last slot
        // whose first item (s_pre * mb) is <= q (binary search); items are slot-major,
        // then (m_block, chunk) -- the order of moe.build_items
        auto emit = [&](Item *items, int mb, int cap) {
            const int tot = chunk_total * mb;
            for (int q = tid; q < tot; q += kItThreads) {
                int lo = 0, hi = kItThreads - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (s_pre[mid] * mb <= q) lo = mid;
                    else hi = mid - 1;
                }
                // skip empty slots that share the prefix (their range is empty)
                const int cc = s_pre[lo + 1] - s_pre[lo];
                const int local = q - s_pre[lo] * mb, m_blk = local / cc, j = local - m_blk * cc;
                const int idx = (run + s_pre[lo]) * mb + local;
                if (idx < cap)
                    items[idx] = Item{s0 + lo, m_blk, s_t0[lo] + j * kItemTokens,
                                      min(kItemTokens, s_n[lo] - j * kItemTokens)};
            }
        };
        emit(items1, mb1, cap1);
        if (mb2 > 0) emit(items2, mb2, cap2);
        run += chunk_total;
        __syncthreads();
    }
    if (tid == 0) {
        counts[0] = run * mb1;  // may exceed the capacity: the GEMM clamps, the host checks
        counts[1] = run * mb2;
        counts[2] = rep_off[b0 + S] - base_row;
    }
}

// dst[pair_row[p]] = src[p / k] for the pairs served by `rank` (one warp per pair,
// 16-byte vectors): the rank's receive buffer in dispatch-layout order.
__global__ void gather_rows_kernel(const uint4 *__restrict__ src, int row_vecs, int k,
                                   const int32_t *__restrict__ pair_rank, const int32_t *__restrict__ pair_row,
                                   int64_t num_pairs, int rank, uint4 *__restrict__ dst, int rows_cap) {
    pdl_wait();
    pdl_launch_dependents();  // only once this kernel runs: at most one dependent waits
    const int64_t warp_id = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t p = warp_id; p < num_pairs; p += nwarps) {
        if (pair_rank[p] != rank) continue;
        const int r = pair_row[p];
        if (r < 0 || r >= rows_cap) continue;
        const uint4 *s = src + (p / k) * row_vecs;
        uint4 *d = dst + static_cast<int64_t>(r) * row_vecs;
        // eight independent 16-byte loads in flight per lane before the stores
        constexpr int U = 8;
        int v0 = lane;
        for (; v0 + (U - 1) * 32 < row_vecs; v0 += U * 32) {
            uint4 t[U];
#pragma unroll
            for (int u = 0; u < U; ++u) t[u] = __ldg(s + v0 + u * 32);
#pragma unroll
            for (int u = 0; u < U; ++u) d[v0 + u * 32] = t[u];
        }
        for (int v = v0; v < row_vecs; v += 32) d[v] = __ldg(s + v);
    }
}

// ---------------------------------------------------------------- host
static thread_local int g_err = 0;
static int64_t *g_stamps = nullptr;  // moe_debug_set_stamps

// launch with programmatic stream serialisation (every kernel above waits with
// griddepcontrol.wait before touching its predecessors' outputs)
template <typename K, typename... Args>
static cudaError_t launch_pdl(K kernel, int grid, int block, int smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(block, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}

static bool encode(CUtensorMap *m, void *base, int rank, const cuuint64_t *dims, const cuuint64_t *strides,
                   const cuuint32_t *box, bool fp8 = false) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint32_t es[3] = {1, 1, 1};
    return fn(m, fp8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, base, dims, strides,
              box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace moe

using namespace moe;

extern "C" {

static int launch_gemm(const void *W, int32_t E, int32_t M, int32_t K, const void *X, int32_t T,
                       const int32_t *items, int32_t n_items, const int32_t *n_items_dev, int32_t max_item_tokens,
                       void *Y, int32_t num_ctas, void *stream, const float *w_scale = nullptr,
                       const float *x_scale = nullptr) {
    if (n_items > 0 && (reinterpret_cast<uintptr_t>(items) & 15)) return METRO_EARG;  // 16-byte item loads
    const bool fp8 = w_scale != nullptr;
    const cuuint64_t es = fp8 ? 1 : 2;             // bytes per element
    const cuuint32_t bke = fp8 ? 2 * BK : BK;      // elements per 128-byte row
    Maps maps;
    const cuuint64_t wdims[3] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(M), static_cast<cuuint64_t>(E)};
    const cuuint64_t wstr[2] = {static_cast<cuuint64_t>(K) * es, static_cast<cuuint64_t>(M) * K * es};
    const cuuint32_t wbox[3] = {bke, BM, 1};
    if (!encode(&maps.w, const_cast<void *>(W), 3, wdims, wstr, wbox, fp8)) return METRO_ECUDA;
    const cuuint64_t xdims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(T)};
    const cuuint64_t xstr[1] = {static_cast<cuuint64_t>(K) * es};
    for (int i = 0; i < NMAPS; ++i) {
        const cuuint32_t xbox[2] = {bke, static_cast<cuuint32_t>(16 << i)};
        if (!encode(&maps.x[i], const_cast<void *>(X), 2, xdims, xstr, xbox, fp8)) return METRO_ECUDA;
    }
    static std::once_flag attr;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(attr, [] {
        const void *ks[4] = {reinterpret_cast<const void *>(moe_gemm_kernel<WideTile, false>),
                             reinterpret_cast<const void *>(moe_gemm_kernel<NarrowTile, false>),
                             reinterpret_cast<const void *>(moe_gemm_kernel<WideTile, true>),
                             reinterpret_cast<const void *>(moe_gemm_kernel<NarrowTile, true>)};
        const int sm[4] = {WideTile::kSmem, NarrowTile::kSmem, WideTile::kSmem, NarrowTile::kSmem};
        for (int i = 0; i < 4 && attr_err == cudaSuccess; ++i)
            attr_err = cudaFuncSetAttribute(ks[i], cudaFuncAttributeMaxDynamicSharedMemorySize, sm[i]);
    });
    if (attr_err != cudaSuccess) {
        g_err = attr_err;
        return METRO_ECUDA;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // persistent CTAs, round-robin items.  Balanced grid: the fewest CTAs that keep
    // the minimal number of waves (items per CTA), so every CTA gets the same item
    // count (e.g. 2016 items: 144 CTAs x 14 instead of 148 with 92 x 14 + 56 x 13).
    // A/B on one B200 (tools/k3_grid_ab.sh): EPLB rank FFN -2 %, METRO rank within
    // 0.4 %.  MOE_BALANCED_GRID=0 restores one CTA per SM.  (Device item counts --
    // moe_grouped_gemm_dev -- are unknown here: one CTA per SM.)
    static const int balanced = [] {
        const char *v = getenv("MOE_BALANCED_GRID");
        return v ? atoi(v) : 1;
    }();
    int grid = num_ctas > 0 ? num_ctas : (n_items < sms ? n_items : sms);
    if (num_ctas <= 0 && balanced && n_items > sms && !n_items_dev) {
        const int waves = (n_items + sms - 1) / sms;
        grid = (n_items + waves - 1) / waves;
    }
    Params prm;
    prm.items = reinterpret_cast<const Item *>(items);
    prm.n_items = n_items;
    prm.n_items_dev = n_items_dev;
    prm.K = K;
    prm.Y = static_cast<__nv_bfloat16 *>(Y);
    prm.ldy = M;
    prm.rows = T;
    prm.w_scale = w_scale;
    prm.x_scale = x_scale;
    prm.mblocks = M / BM;
    prm.stamps = g_stamps;

    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool narrow = max_item_tokens <= NarrowTile::kN;
    cudaError_t e;
    if (fp8)
        e = narrow ? launch_pdl(moe_gemm_kernel<NarrowTile, true>, grid, kThreads, NarrowTile::kSmem, s, maps, prm)
                   : launch_pdl(moe_gemm_kernel<WideTile, true>, grid, kThreads, WideTile::kSmem, s, maps, prm);
    else
        e = narrow ? launch_pdl(moe_gemm_kernel<NarrowTile, false>, grid, kThreads, NarrowTile::kSmem, s, maps, prm)
                   : launch_pdl(moe_gemm_kernel<WideTile, false>, grid, kThreads, WideTile::kSmem, s, maps, prm);
    if (e != cudaSuccess) {
        g_err = e;
        return METRO_ECUDA;
    }
    return METRO_OK;
}

METRO_API int32_t moe_item_tokens(void) { return kItemTokens; }
// tuning only: per-CTA {start, end} globaltimer stamps of the next grouped-GEMM launches
METRO_API void moe_debug_set_stamps(int64_t *stamps) { g_stamps = stamps; }

METRO_API int moe_grouped_gemm_v2(const void *W, int32_t E, int32_t M, int32_t K, const void *X, int32_t T,
                                  const int32_t *items, int32_t n_items, int32_t max_item_tokens, void *Y,
                                  int32_t num_ctas, void *stream) {
    if (!W || !X || !Y || (!items && n_items > 0) || E < 1 || M < BM || K < BK || T < 1 || n_items < 0 ||
        max_item_tokens < 1 || max_item_tokens > MAXN)
        return METRO_EARG;
    if (M % BM || K % BK) return METRO_EDIMS;
    if (n_items == 0) return METRO_OK;
    return launch_gemm(W, E, M, K, X, T, items, n_items, nullptr, max_item_tokens, Y, num_ctas, stream);
}

METRO_API int moe_grouped_gemm_v1(const void *W, int32_t E, int32_t M, int32_t K, const void *X, int32_t T,
                        const int32_t *items, int32_t n_items, void *Y, int32_t num_ctas, void *stream) {
    return moe_grouped_gemm_v2(W, E, M, K, X, T, items, n_items, MAXN, Y, num_ctas, stream);
}

METRO_API int moe_grouped_gemm_dev_v2(const void *W, int32_t E, int32_t M, int32_t K, const void *X,
                                      int32_t T_cap, const int32_t *items, int32_t items_cap,
                                      const int32_t *n_items_dev, int32_t max_item_tokens, void *Y, int32_t num_ctas,
                                      void *stream) {
    if (!W || !X || !Y || !items || !n_items_dev || E < 1 || M < BM || K < BK || T_cap < 1 || items_cap < 1 ||
        max_item_tokens < 1 || max_item_tokens > MAXN)
        return METRO_EARG;
    if (M % BM || K % BK) return METRO_EDIMS;
    return launch_gemm(W, E, M, K, X, T_cap, items, items_cap, n_items_dev, max_item_tokens, Y, num_ctas, stream);
}

METRO_API int moe_grouped_gemm_dev_v1(const void *W, int32_t E, int32_t M, int32_t K, const void *X,
                                      int32_t T_cap, const int32_t *items, int32_t items_cap,
                                      const int32_t *n_items_dev, void *Y, int32_t num_ctas, void *stream) {
    return moe_grouped_gemm_dev_v2(W, E, M, K, X, T_cap, items, items_cap, n_items_dev, MAXN, Y, num_ctas, stream);
}

METRO_API int moe_grouped_gemm_fp8_v1(const void *W8, const float *w_scale, int32_t E, int32_t M, int32_t K,
                                      const void *X8, const float *x_scale, int32_t T, const int32_t *items,
                                      int32_t n_items, const int32_t *n_items_dev, int32_t max_item_tokens, void *Y,
                                      int32_t num_ctas, void *stream) {
    if (!W8 || !w_scale || !X8 || !x_scale || !Y || !items || E < 1 || M < BM || K < 2 * BK || T < 1 ||
        n_items < 0 || max_item_tokens < 1 || max_item_tokens > MAXN)
        return METRO_EARG;
    if (M % BM || K % (2 * BK)) return METRO_EDIMS;
    if (n_items == 0) return METRO_OK;
    return launch_gemm(W8, E, M, K, X8, T, items, n_items, n_items_dev, max_item_tokens, Y, num_ctas, stream, w_scale,
                       x_scale);
}

METRO_API int moe_quantize_rows_fp8_v1(const void *X, int32_t T, int32_t K, void *X8, float *x_scale,
                                       const int32_t *rows_dev, void *stream) {
    if (!X || !X8 || !x_scale || T < 0 || K < 2 || (K & 1)) return METRO_EARG;
    if (T == 0) return METRO_OK;
    const int grid = T < 148 * 8 ? T : 148 * 8;  // one CTA per row, grid-stride
    const cudaError_t e = launch_pdl(quantize_fp8_kernel<0>, grid, kQThreads, 0, static_cast<cudaStream_t>(stream),
                                     static_cast<const __nv_bfloat16 *>(X), static_cast<int>(T), static_cast<int>(K),
                                     static_cast<uint8_t *>(X8), x_scale, rows_dev);
    if (e != cudaSuccess) {
        g_err = e;
        return METRO_ECUDA;
    }
    return METRO_OK;
}

METRO_API int moe_silu_mul_fp8_v1(const void *GU, int32_t T, int32_t I, void *H8, float *h_scale,
                                  const int32_t *rows_dev, void *stream) {
    if (!GU || !H8 || !h_scale || T < 0 || I < 2 || (I & 1)) return METRO_EARG;
    if (T == 0) return METRO_OK;
    const int grid = T < 148 * 8 ? T : 148 * 8;
    const cudaError_t e = launch_pdl(quantize_fp8_kernel<1>, grid, kQThreads, 0, static_cast<cudaStream_t>(stream),
                                     static_cast<const __nv_bfloat16 *>(GU), static_cast<int>(T), static_cast<int>(I),
                                     static_cast<uint8_t *>(H8), h_scale, rows_dev);
    if (e != cudaSuccess) {
        g_err = e;
        return METRO_ECUDA;
    }
    return METRO_OK;
}

METRO_API int moe_layout_items_v1(const int32_t *rep_off, const int32_t *slot_base, int32_t rank, int32_t M1,
                                  int32_t M2, int32_t *items1, int32_t cap1, int32_t *items2, int32_t cap2,
                                  int32_t *counts, void *stream) {
    if (!rep_off || !slot_base || !items1 || !counts || rank < 0 || M1 < BM || cap1 < 0 || cap2 < 0 ||
        (M2 > 0 && !items2))
        return METRO_EARG;
    if (M1 % BM || (M2 > 0 && M2 % BM)) return METRO_EDIMS;
    const cudaError_t e = launch_pdl(layout_items_kernel, 1, kItThreads, 0, static_cast<cudaStream_t>(stream),
                                     rep_off, slot_base, static_cast<int>(rank), static_cast<int>(M1 / BM),
                                     static_cast<int>(M2 > 0 ? M2 / BM : 0), reinterpret_cast<Item *>(items1),
                                     reinterpret_cast<Item *>(items2), static_cast<int>(cap1),
                                     static_cast<int>(cap2), counts);
    if (e != cudaSuccess) {
        g_err = e;
        return METRO_ECUDA;
    }
    return METRO_OK;
}

METRO_API int moe_gather_rows_v1(const void *src, int32_t row_bytes, int32_t top_k, const int32_t *pair_rank,
                                 const int32_t *pair_row, int64_t num_pairs, int32_t rank, void *dst,
                                 int32_t rows_cap, void *stream) {
    if (!src || !dst || top_k < 1 || row_bytes < 16 || num_pairs < 0 || rows_cap < 0 ||
        (num_pairs > 0 && (!pair_rank || !pair_row)))
        return METRO_EARG;
    if (row_bytes % 16 || (reinterpret_cast<uintptr_t>(src) & 15) || (reinterpret_cast<uintptr_t>(dst) & 15))
        return METRO_EDIMS;
    if (num_pairs == 0) return METRO_OK;
    const int64_t blocks = (num_pairs + 7) / 8;
    const int grid = static_cast<int>(blocks < 148 * 16 ? blocks : 148 * 16);
    const cudaError_t e = launch_pdl(gather_rows_kernel, grid, 256, 0, static_cast<cudaStream_t>(stream),
                                     static_cast<const uint4 *>(src), static_cast<int>(row_bytes / 16),
                                     static_cast<int>(top_k), pair_rank, pair_row, num_pairs,
                                     static_cast<int>(rank), static_cast<uint4 *>(dst), static_cast<int>(rows_cap));
    if (e != cudaSuccess) {
        g_err = e;
        return METRO_ECUDA;
    }
    return METRO_OK;
}

static int launch_silu(const void *GU, int32_t T, int32_t I, void *H, const int32_t *rows_dev, void *stream);

METRO_API int moe_silu_mul_v1(const void *GU, int32_t T, int32_t I, void *H, void *stream) {
    return launch_silu(GU, T, I, H, nullptr, stream);
}

METRO_API int moe_silu_mul_dev_v1(const void *GU, int32_t T_cap, int32_t I, void *H, const int32_t *rows_dev,
                                  void *stream) {
    if (!rows_dev) return METRO_EARG;
    return launch_silu(GU, T_cap, I, H, rows_dev, stream);
}

static int launch_silu(const void *GU, int32_t T, int32_t I, void *H, const int32_t *rows_dev, void *stream) {
    if (!GU || !H || T < 0 || I < 2 || (I & 1)) return METRO_EARG;
    if (T == 0) return METRO_OK;
    const int grid = T < 148 * 8 ? T : 148 * 8;  // one CTA per row, grid-stride
    const cudaError_t e = launch_pdl(silu_mul_kernel, grid, 256, 0, static_cast<cudaStream_t>(stream),
                                     static_cast<const __nv_bfloat16 *>(GU), static_cast<int>(T),
                                     static_cast<int>(I), static_cast<__nv_bfloat16 *>(H), rows_dev);
    if (e != cudaSuccess) {
        g_err = e;
        return METRO_ECUDA;
    }
    return METRO_OK;
}

METRO_API int moe_last_cuda_error(void) { return g_err; }

}  // extern "C"
