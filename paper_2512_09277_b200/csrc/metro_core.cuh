// metro_core.cuh -- device-side phases of the METRO / EPLB routing kernels shared
// by the translation units of libmetro_b200.so (metro_route.cu: one launch per
// layer; metro_serve.cu: the persistent host-doorbell router).  Parameters,
// the shared-memory layout, staging, the lane-striped histogram + cluster
// exchange, the METRO decision (order + greedy) and the gating top-k.
// Reference semantics: see metro_route.cu's header.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/metro_route.h"
#include "sm100_ptx.cuh"
namespace metro {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxG = 128;
constexpr int kMaxN = 4096;
constexpr int kMaxCluster = 16;
constexpr int kMaxSmem = 232448;  // 227 KB opt-in on sm_100
constexpr int64_t kNoBad = INT64_MAX;
constexpr uint32_t kBadLo = 0xffffffffu, kBadHi = 0x7fffffffu;  // kNoBad split

enum Kind { kMetroIds = 0, kEplbIds = 1, kMetroLoads = 2, kEplbLoads = 3, kMetroOrdered = 4 };
enum Mode { kFromIds = 0, kFromLoads = 1, kFromOrder = 2 };

struct Params {
    const int32_t *ids;
    int64_t num_pairs;
    int64_t slice;  // ids per CTA (multiple of 4)
    const uint32_t *mask;
    const int64_t *loads_in;
    const int32_t *order;
    int32_t order_len;
    int32_t N, G, C;  // C = lane-striped histogram copies (power of two <= 32)
    int32_t staged;   // 1: slice staged in smem; 0: stream ids from global twice
    int32_t *loads;
    int32_t *choice;
    int32_t *rank_counts;
    int32_t *lam;
    int32_t *pair_rank;
    int32_t *status;
    int32_t *x32;
    int64_t *x64;
    int64_t *stamps;
    // gating mode (metro_route_scores_v1): router scores [num_tokens, N] fp32 in,
    // top-k ids [num_tokens, top_k] out; ids = nullptr
    const float *scores;
    int64_t num_tokens;
    int32_t top_k;
    int32_t *ids_out;
    int32_t score_bytes;  // > 0: the CTA's score rows are staged in smem (bytes per CTA)
    void *gate_ws;        // whole-GPU gating: int64 T[N] + routing-CTA counter, zero between launches
    int32_t gate_tokens;  // metro_gate_topk_kernel: tokens per CTA (<= kGateTokens)
    int32_t private_scratch;  // one-CTA plan: the sort scratch has its own shared memory (no alias of hist)
    // fused dispatch layout (metro_route_layout_v1; include/dispatch_layout.h semantics)
    const int32_t *rid_tab;    // [N, G] replica ids (-1: no replica), device
    const int32_t *slot_base;  // [G + 1]
    int32_t nrep;              // replicas; 0 = no fused layout
    int32_t *pair_row;         // [num_pairs] row in the serving rank's receive buffer
    int32_t *rep_off;          // [nrep + 1] exclusive row prefix per replica
    int32_t dbg_skip;          // tuning only (METRO_DBG_SKIP): bit mask of fused-layout phases to skip
};
// walk warps of the fused layout: the warps NOT on warp 0's SM sub-partition (warp w
// issues on SMSP w % 4; warp 0 runs the serial greedy meanwhile and keeps its SMSP)
#ifndef METRO_LAY_ALL_WARPS
constexpr int kLayWarps = (kThreads / 32) * 3 / 4;
__host__ __device__ constexpr int lay_index(int warp) { return (warp & 3) ? warp - 1 - (warp >> 2) : -1; }
#else  // A/B: every warp but warp 0 walks
constexpr int kLayWarps = kThreads / 32 - 1;
__host__ __device__ constexpr int lay_index(int warp) { return warp - 1; }
#endif
constexpr int kGateTokens = 2 * kThreads / 32;  // tokens per CTA in metro_gate_topk_kernel
// auto policy of metro_route_scores_v1: above this many tokens the whole GPU takes
// the top-k (measured crossover on B200: ~600 tokens at N = 256)
constexpr int64_t kGateWholeGpuMin = 512;

// CTA barrier over the kThreads routing threads (named barrier 1).  The same as
// __syncthreads() in the one-launch kernels (blockDim == kThreads); the
// persistent router (metro_serve.cu) runs doorbell warps outside this count.
__device__ __forceinline__ void cta_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory"); }

// ---------------------------------------------------------------- smem layout
// mbar | misc | mask | ids (staged slice) | T | choice | aux | hist | part
// The METRO sort/greedy scratch (keys, cand, smask, sid) aliases hist + part:
// both are dead once the partial histograms have been reduced into T.
struct Layout {
    int mbar, misc, mask, ids, T, choice, aux, hist, part, keys, cand, smask, sid, ent, rpart, sc, total;
    // fused dispatch layout: replica table, slot bases, walk-warp occurrence counts /
    // prefixes, per-pair in-warp ranks, CTA prefixes, rows / offsets per replica
    int lrtab, lsb, lhw, locc, lpre, lrows, loff, lbase, lwsum;
    int NP;  // partial-row stride (words): N + 2 (bad pair lo/hi) rounded to 4
    bool sync_part;  // the aliased sort scratch overlaps the partial rows (see make_layout)
};

__host__ __device__ inline int align_up(int x, int a) { return (x + a - 1) / a * a; }

// packed greedy entry sizes (words): r = 2 / r = 3 / generic
constexpr int kES = 12;  // packed greedy entry stride (words)

__host__ __device__ inline Layout make_layout(int kind, int N, int W, int R, int64_t slice,
                                              int C, int staged, bool warp_hist = false, int score_bytes = 0,
                                              bool private_scratch = false, int lay_G = 0, int lay_nrep = 0) {
    Layout L;
    int o = 0;
    L.mbar = o; o += 32;  // staging | partial exchange | fused-layout tables
    L.misc = o; o += 64 * 4;
    L.mask = o; o = align_up(o + N * W * 4, 16);
    L.NP = align_up(N + 2, 4);
    const bool ids_mode = (kind == kMetroIds || kind == kEplbIds);
    const bool metro = (kind == kMetroIds || kind == kMetroLoads || kind == kMetroOrdered);
    L.ids = o;
    if (ids_mode && staged) o = align_up(o + (int)slice * 4, 16);
    L.T = o; o = align_up(o + N * (kind == kEplbIds ? 8 : 4), 16);  // EPLB: + CTA base
    L.choice = o;
    if (metro) o = align_up(o + (N + 4) * 4, 16);  // + dummy slot for padded entries
    L.aux = o; o = align_up(o + 2 * kMaxG * 4, 16);  // L0 / EPLB counts | active-per-rank
    L.hist = o;
    int hist_bytes = 0;
    if (ids_mode) hist_bytes = warp_hist ? kWarps * N * 4 : N * C * 4;
    L.part = align_up(o + hist_bytes, 16);
    const int end1 = ids_mode ? align_up(L.part + R * L.NP * 4, 16) : L.part;
    // The METRO sort scratch aliases the histogram counters + partial rows (dead
    // once T is reduced), unless the plan gives it its own space: then no barrier
    // is needed between the last counter read and the first scratch write
    // (one-CTA plans, histogram_push).  Classify reads the partial rows (every
    // CTA's row of expert e, in passes of kThreads experts) while other threads
    // already write sort keys, so when the keys can reach the partial rows
    // (small C, large N) the rows are reduced into T behind a barrier first.
    auto scratch_at = [&](int keys) {
        L.keys = keys;
        L.cand = align_up(L.keys + (N + 16) * 8, 16);
        L.smask = L.cand;  // (unused: the warp greedy reads masks through sid)
        L.sid = align_up(L.cand + N * 4, 16);
        L.ent = align_up(L.sid + N * 4, 16);
        // packed-greedy entries (W == 1 only), one slot per rank + readable padding
        L.rpart = align_up(L.ent + (W == 1 ? (N + 16) * kES * 4 : 0), 16);  // [4][N] partial ranks
        return align_up(L.rpart + (4 * N + 16) * 4, 16);                    // + prefetch slack
    };
    const bool priv = private_scratch && ids_mode && metro;
    const int scratch_end = scratch_at(priv ? end1 : o);
    // aliased scratch reaching into the partial rows: classify first sums every
    // expert's rows into T, then a barrier, then the key writes (metro_decide)
    L.sync_part = ids_mode && metro && !priv && scratch_end > L.part;
    const int end2 = metro ? scratch_end : o;
    L.total = end1 > end2 ? end1 : end2;
    // fused dispatch layout: regions of their own (live across the decide phase)
    L.lrtab = L.lsb = L.lhw = L.locc = L.lpre = L.lrows = L.loff = L.lbase = L.lwsum = L.total;
    if (lay_nrep > 0) {
        int q = align_up(L.total, 16);
        L.lrtab = q; q = align_up(q + N * lay_G * 4, 16);
        L.lsb = q;   q = align_up(q + (lay_G + 1) * 4, 16);
        L.lhw = q;   q = align_up(q + kLayWarps * N * 4, 16);
        L.lrows = q; q = align_up(q + max(lay_nrep + 1, lay_G) * 4, 16);  // zeroed with lhw (contiguous)
        L.locc = q;  q = align_up(q + static_cast<int>(slice) * 2, 16);
        L.lpre = q;  q = align_up(q + N * 4, 16);
        L.loff = q;  q = align_up(q + (lay_nrep + 1) * 4, 16);
        L.lbase = q; q = align_up(q + N * 4, 16);
        L.lwsum = q; q += 32 * 4;
        L.total = q;
    }
    // gating mode: the CTA's fp32 score rows, staged by TMA bulk copies
    L.sc = align_up(L.total, 128);
    if (score_bytes > 0) L.total = L.sc + score_bytes;
    return L;
}

// misc word indices
enum {
    M_BAD_LO = 0, M_BAD_HI = 1,        // this CTA's min bad pair index (int64)
    M_NOREP = 2,                       // min active expert without replica
    M_LOADERR = 3,
    M_BADALL_LO = 4, M_BADALL_HI = 5,  // cluster-wide min bad pair index
    M_M2 = 6,                          // replicated active experts (compaction cursor)
    M_N2 = 7, M_N3 = 8,                // end of the r == 2 / r <= 3 segments (sorted order)
    M_PACKED_LO = 9, M_PACKED_HI = 10, M_PACKED_OK = 11,
};

// PTX helpers (mbarrier, bulk copy, cluster, DSMEM): sm100_ptx.cuh
__device__ __forceinline__ void stamp(const Params &p, int i) {
    if (p.stamps && threadIdx.x == 0 && cluster_ctarank() == 0) p.stamps[i] = clock64();
}
__device__ __forceinline__ int64_t join64(uint32_t lo, uint32_t hi) {
    return static_cast<int64_t>((static_cast<uint64_t>(hi) << 32) | lo);
}

// position of the (q+1)-th set bit of a W-word mask (q < popcount); short loops:
// q < r <= G and r is 2..3 in practice
template <int W>
__device__ __forceinline__ int nth_set_bit(const uint32_t *mw, int q) {
#pragma unroll
    for (int j = 0; j < W; ++j) {
        const int c = __popc(mw[j]);
        if (q < c) {
            uint32_t m = mw[j];
            for (int i = 0; i < q; ++i) m &= m - 1;
            return 32 * j + __ffs(m) - 1;
        }
        q -= c;
    }
    return -1;
}

// ---------------------------------------------------------------- phase A
struct StagePlan {
    int mask_words;
    bool mask_bulk, ids_bulk;
    int body;
};

template <int W>
__device__ __forceinline__ StagePlan stage_plan(const Params &p, int64_t beg, int n_local, bool stage_ids) {
    StagePlan s;
    s.mask_words = p.mask ? p.N * W : 0;  // aggregate-only launches carry no mask
    s.mask_bulk = s.mask_words > 0 && ((reinterpret_cast<uintptr_t>(p.mask) & 15) == 0) && (s.mask_words % 4 == 0);
    s.body = stage_ids ? (n_local & ~3) : 0;
    s.ids_bulk = stage_ids && s.body > 0 && ((reinterpret_cast<uintptr_t>(p.ids + beg) & 15) == 0);
    return s;
}

// fused layout: the replica table goes by one TMA bulk copy when it can
__device__ __forceinline__ bool layout_rtab_bulk(const Params &p) {
    return ((reinterpret_cast<uintptr_t>(p.rid_tab) & 15) == 0) && ((p.N * p.G) & 3) == 0;
}

// thread 0, first thing in the kernel: arm the mbarrier and launch the TMA copies
__device__ __forceinline__ void stage_issue(const Params &p, const Layout &L, unsigned char *smem, int64_t beg,
                                            const StagePlan &s) {
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + L.mbar);
    mbar_init(bar + 2, 1);  // fused layout: the replica table (read only after the decide phase)
    mbar_init(bar + 1, 1);  // partial-histogram exchange (st.async from the peer CTAs)
    mbar_init(bar, 1);      // TMA staging (its init fence covers all three)
    if (p.nrep > 0 && layout_rtab_bulk(p)) {
        const uint32_t rb = static_cast<uint32_t>(p.N * p.G * 4);
        mbar_arrive_expect_tx(bar + 2, rb);
        for (uint32_t o = 0; o < rb; o += 32768u)
            bulk_g2s(smem + L.lrtab + o, reinterpret_cast<const unsigned char *>(p.rid_tab) + o, min(32768u, rb - o),
                     bar + 2);
    }
    uint32_t sc_bytes = 0;
    const float *sc_src = nullptr;
    if (p.score_bytes > 0) {  // gating mode: this CTA's rows of the score matrix
        const int64_t t0 = beg / p.top_k;
        const int64_t nt = min(static_cast<int64_t>(p.slice / p.top_k), p.num_tokens - t0);
        sc_bytes = nt > 0 ? static_cast<uint32_t>(nt * p.N * 4) : 0u;
        sc_src = p.scores + t0 * p.N;
    }
    const uint32_t bytes = (s.mask_bulk ? s.mask_words * 4u : 0u) + (s.ids_bulk ? s.body * 4u : 0u) + sc_bytes;
    mbar_arrive_expect_tx(bar, bytes);
    if (s.mask_bulk) bulk_g2s(smem + L.mask, p.mask, s.mask_words * 4u, bar);
    if (s.ids_bulk) bulk_g2s(smem + L.ids, p.ids + beg, s.body * 4u, bar);
    for (uint32_t o = 0; o < sc_bytes; o += 32768u) {
        const uint32_t n = min(32768u, sc_bytes - o);
        bulk_g2s(smem + L.sc + o, reinterpret_cast<const unsigned char *>(sc_src) + o, n, bar);
    }
}

// all threads: whatever the TMA could not take (unaligned / ragged tail)
__device__ __forceinline__ void stage_rest(const Params &p, const Layout &L, unsigned char *smem, int64_t beg,
                                           int n_local, bool stage_ids, const StagePlan &s) {
    uint32_t *s_mask = reinterpret_cast<uint32_t *>(smem + L.mask);
    int32_t *s_ids = reinterpret_cast<int32_t *>(smem + L.ids);
    if (!s.mask_bulk)
        for (int i = threadIdx.x; i < s.mask_words; i += kThreads) s_mask[i] = __ldg(p.mask + i);
    if (stage_ids)
        for (int i = (s.ids_bulk ? s.body : 0) + threadIdx.x; i < n_local; i += kThreads)
            s_ids[i] = __ldg(p.ids + beg + i);
}

__device__ __forceinline__ void init_misc(int32_t *misc) {
    if (threadIdx.x < 64) {
        const int i = threadIdx.x;
        int32_t v = 0;
        if (i == M_BAD_LO || i == M_BADALL_LO) v = static_cast<int32_t>(kBadLo);
        if (i == M_BAD_HI || i == M_BADALL_HI) v = static_cast<int32_t>(kBadHi);
        if (i == M_NOREP) v = INT32_MAX;
        misc[i] = v;
    }
}

__device__ __forceinline__ void zero_smem(unsigned char *smem, int from, int to) {
    for (int i = from / 16 + threadIdx.x; i < to / 16; i += kThreads)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0, 0, 0, 0);
}

// ---------------------------------------------------------------- phase B + C
// Histogram this CTA's slice, then push the per-expert partial (and the CTA's
// min bad pair index) into row `rank` of every CTA's partial table.  Ends with
// the cluster barrier; afterwards part[r][e] holds CTA r's count of expert e.
template <bool PRIV, bool COUNT = true>
__device__ void histogram_push(const Params &p, const Layout &L, unsigned char *smem, int64_t beg, int n_local,
                               uint32_t R, uint32_t rank) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int N = p.N;
    int32_t *misc = reinterpret_cast<int32_t *>(smem + L.misc);
    int32_t *s_hist = reinterpret_cast<int32_t *>(smem + L.hist);
    int32_t *s_part = reinterpret_cast<int32_t *>(smem + L.part);
    const int32_t *src = p.staged ? reinterpret_cast<const int32_t *>(smem + L.ids) : (p.ids + beg);
    int64_t my_bad = kNoBad;
    int bad_i = INT32_MAX;  // first bad pair of this thread, relative to beg (32-bit min on the hot path)

    if (!COUNT) {
        // the gating stage already counted its ids into hist (gate_topk)
    } else if (!PRIV) {
        const int cm = p.C - 1;
        const int n4 = n_local & ~3;
        const bool vec = p.staged || ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
        if (vec) {
            for (int i = tid * 4; i < n4; i += kThreads * 4) {
                const int4 v = *reinterpret_cast<const int4 *>(src + i);
                const int ev[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int e = ev[q];
                    if (static_cast<unsigned>(e) < static_cast<unsigned>(N))
                        atomicAdd(&s_hist[e * p.C + (lane & cm)], 1);
                    else
                        bad_i = min(bad_i, i + q);
                }
            }
        }
        for (int i = (vec ? n4 : 0) + tid; i < n_local; i += kThreads) {
            const int e = src[i];
            if (static_cast<unsigned>(e) < static_cast<unsigned>(N))
                atomicAdd(&s_hist[e * p.C + (lane & cm)], 1);
            else
                bad_i = min(bad_i, i);
        }
        if (bad_i != INT32_MAX) my_bad = beg + bad_i;
    } else {
        // warp-private histograms over contiguous warp sub-slices; match_any groups
        // equal ids so one lane does a plain read-modify-write.  The same walk later
        // yields deterministic row-major occurrence ranks (EPLB pair_rank).
        const int ws = align_up((n_local + kWarps - 1) / kWarps, 32);
        const int wb = min(n_local, warp * ws), we = min(n_local, wb + ws);
        int32_t *hw = s_hist + warp * N;
        for (int p0 = wb; p0 < we; p0 += 32) {
            const int i = p0 + lane;
            int e = (i < we) ? src[i] : -1;
            if (i < we && static_cast<unsigned>(e) >= static_cast<unsigned>(N)) {
                my_bad = min(my_bad, beg + i);
                e = -1;
            }
            const unsigned m = __match_any_sync(kFull, e);
            if (e >= 0 && lane == __ffs(m) - 1) hw[e] += __popc(m);
            __syncwarp();
        }
    }
    if (my_bad != kNoBad)
        atomicMin(reinterpret_cast<unsigned long long *>(&misc[M_BAD_LO]), static_cast<unsigned long long>(my_bad));
    cta_sync();
    stamp(p, 2);

    // The peers' exchange mbarriers are initialised (every CTA arrived, with release
    // semantics, after its thread 0 initialised them) before anyone stores into a
    // peer.  Each partial goes out as st.async completing bytes on the receiver's
    // mbarrier: no release fence round trip and no cluster barrier; a CTA only
    // waits for the bytes it receives.
    uint64_t *xbar = reinterpret_cast<uint64_t *>(smem + L.mbar) + 1;
    if (R > 1) {
        cluster_wait();
        if (tid == 0) mbar_arrive_expect_tx(xbar, (R - 1) * static_cast<uint32_t>(L.NP) * 4u);
    }
    stamp(p, 20);
    int32_t *row = s_part + rank * L.NP;
    for (int e = tid; e < N; e += kThreads) {
        int s = 0;
        if (!PRIV) {
            const int C = p.C;
            if (C >= 4) {
                // bank-rotated 128-bit loads: the 8 lanes of a quarter-warp phase hit
                // 8 distinct 16-byte bank groups
                const int q4 = C / 4;
                const int4 *h4 = reinterpret_cast<const int4 *>(s_hist + e * C);
                for (int q = 0; q < q4; ++q) {
                    const int4 v = h4[(q + lane) & (q4 - 1)];
                    s += v.x + v.y + v.z + v.w;
                }
            } else {
                for (int c = 0; c < C; ++c) s += s_hist[e * C + c];
            }
        } else {
#pragma unroll 4
            for (int w = 0; w < kWarps; ++w) s += s_hist[w * N + e];
        }
        row[e] = s;
    }
    if (R > 1) {
        // ship the finished row in 16-byte st.async pieces (4x fewer DSMEM ops than
        // per-expert words; the row carries the CTA's bad-pair words at [N, N+2))
        if (tid < 2) row[N + tid] = misc[M_BAD_LO + tid];
        for (int e = N + 2 + tid; e < L.NP; e += kThreads) row[e] = 0;
        cta_sync();
        const int nv = L.NP / 4;
        for (uint32_t k = 1; k < R; ++k) {  // peers in rank order after this CTA (no division)
            const uint32_t d = (rank + k < R) ? rank + k : rank + k - R;
#pragma unroll 1
            for (int v = tid; v < nv; v += kThreads)
                st_async_v4(row + 4 * v, d, reinterpret_cast<const uint4 *>(row)[v], xbar);
        }
    } else if (!p.private_scratch) {
        // every thread's reads of the histogram counters are done before the decide
        // phase writes its sort scratch over them (keys / cand alias hist)
        cta_sync();
    }
    stamp(p, 18);
    if (R > 1) mbar_wait(xbar, 0);
    stamp(p, 3);
}

// cluster-wide min over the R rows' bad words; warp 0 only; publishes to misc
__device__ __forceinline__ void bad_min_warp0(const Layout &L, unsigned char *smem, uint32_t R, int N) {
    if ((threadIdx.x >> 5) != kWarps - 1) return;  // the last warp: idle in classify for N <= 480
    int32_t *misc = reinterpret_cast<int32_t *>(smem + L.misc);
    const int32_t *s_part = reinterpret_cast<const int32_t *>(smem + L.part);
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    uint32_t lo = kBadLo, hi = kBadHi;
    if (static_cast<uint32_t>(lane) == rank) {  // own partial: never written to the row
        lo = static_cast<uint32_t>(misc[M_BAD_LO]);
        hi = static_cast<uint32_t>(misc[M_BAD_HI]);
    } else if (static_cast<uint32_t>(lane) < R) {
        lo = static_cast<uint32_t>(s_part[lane * L.NP + N]);
        hi = static_cast<uint32_t>(s_part[lane * L.NP + N + 1]);
    }
    const bool bad = (lo != kBadLo) || (hi != kBadHi);
    if (!__any_sync(kFull, bad)) return;  // common path: one vote
    const uint32_t mhi = __reduce_min_sync(kFull, hi);
    const uint32_t mlo = __reduce_min_sync(kFull, hi == mhi ? lo : 0xffffffffu);
    if (lane == 0) {
        misc[M_BADALL_LO] = static_cast<int32_t>(mlo);
        misc[M_BADALL_HI] = static_cast<int32_t>(mhi);
    }
}

// after a __syncthreads: report an out-of-range id (status by CTA 0) and bail
__device__ __forceinline__ bool bad_after_sync(const Params &p, const Layout &L, unsigned char *smem,
                                               uint32_t rank) {
    const int32_t *misc = reinterpret_cast<const int32_t *>(smem + L.misc);
    const uint32_t lo = static_cast<uint32_t>(misc[M_BADALL_LO]), hi = static_cast<uint32_t>(misc[M_BADALL_HI]);
    if (lo == kBadLo && hi == kBadHi) return false;
    if (rank == 0 && threadIdx.x == 0) {
        const int64_t bad = join64(lo, hi);
        p.status[0] = METRO_ERR_ID_RANGE;
        p.status[1] = static_cast<int32_t>(lo);
        p.status[2] = static_cast<int32_t>(hi);
        p.status[3] = p.ids[bad];
    }
    return true;
}

__device__ __forceinline__ void write_error(const Params &p, bool writer, int code, int32_t a) {
    if (writer && threadIdx.x == 0) {
        p.status[0] = code;
        p.status[1] = a;
        p.status[2] = 0;
        p.status[3] = 0;
    }
}

// ---------------------------------------------------------------- phase D (METRO)
// Packed single-thread greedy for G <= 8 ranks while every rank hosts at most
// 126 active experts (so every L[g] <= 126 < 127): the 8 counters live as bytes
// in two registers.  Measured on B200 (tools/latency_probe.cu): a compare that
// produces a predicate costs 12-18 cycles on a dependent chain while PRMT / IADD
// cost 3-4, so the chain is predicate-free:
//   v_g   = PRMT(lo, sel_g, hi)       byte g zero-extended (sign-fill of a byte < 128)
//   m     = sign(v_b - v_a)           all ones iff b wins strictly (PRMT sign replicate)
//   L    += inc_a ^ ((inc_a ^ inc_b) & m)   (one LOP3 per half, then IADD)
// Candidates arrive in ascending rank id, so "first minimum" (routing.py:96-98,
// strict '<') means a later candidate wins only on strictly smaller L.
struct PackedL {
    uint32_t lo, hi;
};

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t sel, uint32_t b) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}
// zero-extended byte g of {lo, hi}: nibble0 = g, nibbles1..3 = sign-fill of byte g
__host__ __device__ constexpr uint32_t zsel(uint32_t g) {
    return g | ((8u | g) << 4) | ((8u | g) << 8) | ((8u | g) << 12);
}
// byte g of {lo, hi} moved to byte 1, other bytes zero (sign-fill of a byte < 128)
__host__ __device__ constexpr uint32_t zsel1(uint32_t g) {
    return (8u | g) | (g << 4) | ((8u | g) << 8) | ((8u | g) << 12);
}
// PTX shl clamps shift amounts >= 32 to 32 (result 0); unsigned wrap of sh - 32 included
__device__ __forceinline__ uint32_t shl_clamp(uint32_t v, uint32_t sh) {
    uint32_t d;
    asm("shl.b32 %0, %1, %2;" : "=r"(d) : "r"(v), "r"(sh));
    return d;
}
__device__ __forceinline__ uint32_t sgn(uint32_t d) { return prmt(d, 0xBBBBu, 0u); }  // 0 or ~0
__device__ __forceinline__ uint32_t pick(uint32_t a, uint32_t x, uint32_t m) {
    uint32_t d;  // a ^ (x & m)
    asm("lop3.b32 %0, %1, %2, %3, 0x78;" : "=r"(d) : "r"(a), "r"(x), "r"(m));
    return d;
}
__device__ __forceinline__ uint4 lds4(const uint32_t *p) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(smem_u32(p)));
    return v;
}
__host__ __device__ constexpr uint32_t inc_lo(uint32_t g) { return g < 4 ? (1u << (8 * g)) : 0u; }
__host__ __device__ constexpr uint32_t inc_hi(uint32_t g) { return g >= 4 ? (1u << (8 * (g - 4))) : 0u; }

// Below this many replicated active experts (m2, an upper bound of the r = 2
// steps) the greedy takes the r = 2 steps one at a time and the CTA skips the
// block-of-four delta table (its pass + barrier cost more than the blocks save on
// a short segment).  A/B on B200 (tools/ab_libs.sh, two boxes): Qwen3-30B shape
// (m2 = 39) -0.08..-0.29 us per layer with single steps; DeepSeek-V3 B = 64
// (m2 = 63..76) +0.03 us and B = 1024 (m2 = 85) +0.13..0.2 us, so they keep blocks.
#ifndef METRO_R2_BLOCK_MIN
#define METRO_R2_BLOCK_MIN 48
#endif
// Entry layouts (words):
//   r=2  {selA, selB, incA_lo, incA_hi, xAB_lo, xAB_hi, ga | gb << 8, id}
//   r=3  {selA, selB, selC, 0, incA_lo, incA_hi, xAB_lo, xAB_hi, incC_lo, incC_hi,
//         ga | gb << 8 | gc << 16, id}
//   r>=4 {c0..c7 (8g, + 0x7f00 for non-candidates), id, 0, 0, 0}
__device__ __forceinline__ void packed_entry(uint32_t *dst, int r, uint32_t m, int e) {
    if (r == 2 || r == 3) {
        const uint32_t m1 = m & (m - 1), m2 = m1 & (m1 - 1);
        const uint32_t g[3] = {static_cast<uint32_t>(__ffs(m) - 1), static_cast<uint32_t>(__ffs(m1) - 1),
                               static_cast<uint32_t>(__ffs(m2) - 1)};
        const uint32_t xlo = inc_lo(g[0]) ^ inc_lo(g[1]), xhi = inc_hi(g[0]) ^ inc_hi(g[1]);
        if (r == 2) {
            reinterpret_cast<uint4 *>(dst)[0] = make_uint4(zsel(g[0]), zsel(g[1]), inc_lo(g[0]), inc_hi(g[0]));
            reinterpret_cast<uint4 *>(dst)[1] = make_uint4(xlo, xhi, g[0] | (g[1] << 8), static_cast<uint32_t>(e));
        } else {
            reinterpret_cast<uint4 *>(dst)[0] = make_uint4(zsel(g[0]), zsel(g[1]), zsel(g[2]), 0u);
            reinterpret_cast<uint4 *>(dst)[1] = make_uint4(inc_lo(g[0]), inc_hi(g[0]), xlo, xhi);
            reinterpret_cast<uint4 *>(dst)[2] =
                make_uint4(inc_lo(g[2]), inc_hi(g[2]), g[0] | (g[1] << 8) | (g[2] << 16), static_cast<uint32_t>(e));
        }
    } else {
        // key offsets: 8g in the low byte (tie-break on the lower rank id, and the
        // increment's shift); non-candidates pushed above every valid counter
        uint32_t nc[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) nc[g] = (((m >> g) & 1u) ? 0u : 0x7f00u) | (8u * g);
        reinterpret_cast<uint4 *>(dst)[0] = make_uint4(nc[0], nc[1], nc[2], nc[3]);
        reinterpret_cast<uint4 *>(dst)[1] = make_uint4(nc[4], nc[5], nc[6], nc[7]);
        reinterpret_cast<uint4 *>(dst)[2] = make_uint4(static_cast<uint32_t>(e), 0u, 0u, 0u);
    }
}

// One thread.  Entries live at slot = rank (stride kES words) and are grouped
// by r because the canonical order sorts by r first: [0, n2) r=2,
// [n2, n2 + n3) r=3, [n2 + n3, m2) r>=4.  Slots up to m2 + 8 are readable (the
// r=2 prefetch may touch them; they are never applied).
__device__ __forceinline__ PackedL packed_greedy(const Params &p, const uint32_t *ent, const uint32_t *dlt, int n2,
                                                 int n3, int m2, int32_t *choice, PackedL L) {
    // every step stores its expert's choice (off the dependency chain: the store
    // only reads the decision)
    auto step2 = [&](const uint4 &a, const uint4 &b) {
        const uint32_t va = prmt(L.lo, a.x, L.hi), vb = prmt(L.lo, a.y, L.hi);
        const uint32_t m = sgn(vb - va);
        L.lo += pick(a.z, b.x, m);
        L.hi += pick(a.w, b.y, m);
        choice[b.w] = static_cast<int32_t>((b.z >> (m & 8u)) & 0xffu);
    };
    // Four consecutive r=2 steps in one dependency chain.  All eight candidate loads
    // are extracted from the same L; step j corrects its difference by
    // sum_i<j ([b_j == w_i] - [a_j == w_i]) for the winners w_i of the earlier
    // steps: the "step i took candidate A" terms dA are added up front (off the
    // chain) and step i's mask m_i (0 / ~0) then adds m_i * (dA - dB) -- one IMAD
    // per term (delta block: {dA, dA - dB} for the pairs 01 02 03 12 13 23).  The
    // chain per step is IMAD -> sgn (measured on B200: -230 cycles per DS layer
    // against the round-1 pick -> add -> sgn) instead of the full single-step chain.
    auto block4 = [&](const uint4 (&a)[4], const uint4 (&b)[4], const uint4 (&d)[3]) {
        uint32_t va[4], vb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            va[i] = prmt(L.lo, a[i].x, L.hi);
            vb[i] = prmt(L.lo, a[i].y, L.hi);
        }
        // table {dA_ij, c_ij = dA_ij - dB_ij} (ij = 01 02 03 12 13 23): d_j starts at its
        // "every earlier step took candidate A" value (the dA terms, off the chain) and
        // each earlier decision m_i (0 / ~0) adds m_i * c_ij: ONE IMAD per term on the
        // dependency chain (pick + add before)
        uint32_t d1 = vb[1] - va[1] + d[0].x;
        uint32_t d2 = (vb[2] - va[2] + d[0].z) + d[1].z;
        uint32_t d3 = (vb[3] - va[3] + d[1].x) + (d[2].x + d[2].z);
        const uint32_t m0 = sgn(vb[0] - va[0]);
        d1 = m0 * d[0].y + d1;
        d2 = m0 * d[0].w + d2;
        d3 = m0 * d[1].y + d3;
        const uint32_t m1 = sgn(d1);
        d2 = m1 * d[1].w + d2;
        d3 = m1 * d[2].y + d3;
        const uint32_t m2 = sgn(d2);
        d3 = m2 * d[2].w + d3;
        const uint32_t m3 = sgn(d3);
        const uint32_t m[4] = {m0, m1, m2, m3};
        uint32_t ilo = 0, ihi = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            ilo += pick(a[i].z, b[i].x, m[i]);
            ihi += pick(a[i].w, b[i].y, m[i]);
        }
        L.lo += ilo;
        L.hi += ihi;
#pragma unroll
        for (int i = 0; i < 4; ++i) choice[b[i].w] = static_cast<int32_t>((b[i].z >> (m[i] & 8u)) & 0xffu);
    };
    int s = 0;
    if (m2 < METRO_R2_BLOCK_MIN) {  // one step at a time, the next entry prefetched (no delta table)
        if (n2 > 0) {
            uint4 a = lds4(ent), b = lds4(ent + 4);
            for (; s < n2; ++s) {
                const uint4 an = lds4(ent + (s + 1) * kES), bn = lds4(ent + (s + 1) * kES + 4);
                step2(a, b);
                a = an;
                b = bn;
            }
        }
    } else {
        uint4 a[4], b[4], d[3];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            a[i] = lds4(ent + i * kES);
            b[i] = lds4(ent + i * kES + 4);
        }
#pragma unroll
        for (int i = 0; i < 3; ++i) d[i] = lds4(dlt + i * 4);
        for (; s + 4 <= n2; s += 4) {
            uint4 an[4], bn[4], dn[3];
            const uint32_t *nx = ent + (s + 4) * kES;         // readable even past n2
            const uint32_t *nd = dlt + ((s >> 2) + 1) * 12;   // idem
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                an[i] = lds4(nx + i * kES);
                bn[i] = lds4(nx + i * kES + 4);
            }
#pragma unroll
            for (int i = 0; i < 3; ++i) dn[i] = lds4(nd + i * 4);
            block4(a, b, d);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                a[i] = an[i];
                b[i] = bn[i];
            }
#pragma unroll
            for (int i = 0; i < 3; ++i) d[i] = dn[i];
        }
    }
    for (; s < n2; ++s) step2(lds4(ent + s * kES), lds4(ent + s * kES + 4));
    stamp(p, 8);
    // r = 3 steps, next entry prefetched (slots past m2 stay readable)
    if (s < n2 + n3) {
        uint4 a = lds4(ent + s * kES), b = lds4(ent + s * kES + 4), c = lds4(ent + s * kES + 8);
        for (; s < n2 + n3; ++s) {
            const uint4 an = lds4(ent + (s + 1) * kES), bn = lds4(ent + (s + 1) * kES + 4),
                        cn = lds4(ent + (s + 1) * kES + 8);
            const uint32_t va = prmt(L.lo, a.x, L.hi), vb = prmt(L.lo, a.y, L.hi), vc = prmt(L.lo, a.z, L.hi);
            const uint32_t m1 = sgn(vb - va);
            const uint32_t vab = pick(va, va ^ vb, m1);
            const uint32_t ilo = pick(b.x, b.z, m1), ihi = pick(b.y, b.w, m1);
            const uint32_t m2v = sgn(vc - vab);
            L.lo += pick(ilo, ilo ^ c.x, m2v);
            L.hi += pick(ihi, ihi ^ c.y, m2v);
            // winner: c if it beat the a/b winner, else b if it beat a, else a
            const uint32_t sh = (m2v & 16u) | (~m2v & m1 & 8u);
            choice[c.w] = static_cast<int32_t>((c.z >> sh) & 0xffu);
            a = an;
            b = bn;
            c = cn;
        }
    }
    stamp(p, 9);
    // r >= 4: key_g = L[g] << 8 | 8g (+ 0x7f00 off-replica); the unsigned min is
    // "smallest L, then lowest g" and its low byte is the increment's shift.
    // Next entry prefetched.
    if (s < m2) {
        uint4 n0 = lds4(ent + s * kES), n1 = lds4(ent + s * kES + 4);
        uint32_t id = ent[s * kES + 8];
        for (; s < m2; ++s) {
            const uint4 q0 = lds4(ent + (s + 1) * kES), q1 = lds4(ent + (s + 1) * kES + 4);
            const uint32_t qid = ent[(s + 1) * kES + 8];
            const uint32_t c[8] = {n0.x, n0.y, n0.z, n0.w, n1.x, n1.y, n1.z, n1.w};
            uint32_t k[8];
#pragma unroll
            for (int g = 0; g < 8; ++g) k[g] = prmt(L.lo, zsel1(g), L.hi) + c[g];
            const uint32_t kmin = min(min(min(k[0], k[1]), min(k[2], k[3])), min(min(k[4], k[5]), min(k[6], k[7])));
            const uint32_t sh = kmin & 0x38u;
            L.lo += shl_clamp(1u, sh);
            L.hi += shl_clamp(1u, sh - 32u);
            choice[id] = static_cast<int32_t>(sh >> 3);
            n0 = q0;
            n1 = q1;
            id = qid;
        }
    }
    stamp(p, 10);
    return L;
}

// Serial greedy in one warp for any G <= 128 (routing.py:94-101): lane owns ranks
// g = lane + 32 k as packed keys (L << 8 | g): the warp-wide min over candidate
// lanes is "smallest L, then smallest g" -- the reference's ascending scan with
// strict '<'.  Per chunk of 32 steps the candidacy bits are transposed with
// ballots (lane g gets bit s of step s), so the chain SEL -> redux.min -> ISETP ->
// IADD touches no memory.  Warp 0 only; kept out of line (__noinline__).
template <int W>
__device__ __noinline__ void warp_greedy(const uint32_t *s_mask, int32_t *s_choice, const int32_t *s_sid,
                                         const int32_t *s_L0, int G, int m2, int32_t *rank_counts, int32_t *lam,
                                         bool writer) {
    // (pointers and scalars only: a reference to the kernel's Params / Layout would
    // put them on the stack)
    const int lane = threadIdx.x & 31;
        uint32_t Lk[W];
#pragma unroll
    for (int k = 0; k < W; ++k) {
        const int g = lane + 32 * k;
        Lk[k] = (g < G) ? ((static_cast<uint32_t>(s_L0[g]) << 8) | static_cast<uint32_t>(g)) : 0xffffffffu;
    }
    for (int base = 0; base < m2; base += 32) {
        const int j = base + lane;
        const bool v = j < m2;
        const int myid = v ? s_sid[j] : 0;
        uint32_t cb[W];
#pragma unroll
        for (int k = 0; k < W; ++k) {
            const uint32_t m = v ? s_mask[myid * W + k] : 0u;
            cb[k] = 0;
            const int gk = min(32, G - 32 * k);
            for (int b = 0; b < gk; ++b) {
                const unsigned bb = __ballot_sync(kFull, (m >> b) & 1u);
                if (lane == b) cb[k] = bb;
            }
        }
        const int steps = min(32, m2 - base);
        uint32_t wmine = 0;
#pragma unroll
        for (int s = 0; s < 32; ++s) {
            if (s >= steps) break;
            uint32_t val = 0xffffffffu;
#pragma unroll
            for (int k = 0; k < W; ++k) val = ((cb[k] >> s) & 1u) ? min(val, Lk[k]) : val;
            const uint32_t win = __reduce_min_sync(kFull, val);
#pragma unroll
            for (int k = 0; k < W; ++k) Lk[k] += (Lk[k] == win) ? 256u : 0u;
            wmine = (lane == s) ? win : wmine;
        }
        if (v) s_choice[myid] = static_cast<int32_t>(wmine & 0xffu);
    }
    uint32_t mx = 0;
#pragma unroll
    for (int k = 0; k < W; ++k) {
        const int g = lane + 32 * k;
        if (g < G) {
            const uint32_t c = Lk[k] >> 8;
            if (writer) rank_counts[g] = static_cast<int32_t>(c);
            mx = max(mx, c);
        }
    }
    mx = __reduce_max_sync(kFull, mx);
    if (writer && lane == 0) *lam = static_cast<int32_t>(mx);
}

// Classify + sort + greedy.  MODE selects where T comes from: the cluster's
// partial rows (kFromIds), the int64 loads argument (kFromLoads), or nowhere
// (kFromOrder: a caller order, every listed expert goes through the greedy).
// Returns false on error (status written by the writer CTA).
struct NoOverlap {
    __device__ __forceinline__ void operator()() const {}
};
// OV: work for warps 1.. while warp 0 runs the serial greedy (called once, by whole
// warps, before the barrier that ends the greedy; e.g. the fused layout's walk)
template <int W, int MODE, typename OV = NoOverlap>
__device__ bool metro_decide(const Params &p, const Layout &L, unsigned char *smem, bool writer, uint32_t R,
                             uint32_t rank, const OV &overlap = OV()) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int N = p.N, G = p.G;
    int32_t *misc = reinterpret_cast<int32_t *>(smem + L.misc);
    const uint32_t *s_mask = reinterpret_cast<const uint32_t *>(smem + L.mask);
    uint32_t *s_T = reinterpret_cast<uint32_t *>(smem + L.T);
    int32_t *s_choice = reinterpret_cast<int32_t *>(smem + L.choice);
    const int32_t *s_part = reinterpret_cast<const int32_t *>(smem + L.part);
    uint64_t *s_keys = reinterpret_cast<uint64_t *>(smem + L.keys);
    int32_t *s_cand = reinterpret_cast<int32_t *>(smem + L.cand);
    int32_t *s_sid = reinterpret_cast<int32_t *>(smem + L.sid);
    int32_t *s_L0 = reinterpret_cast<int32_t *>(smem + L.aux);
    uint32_t *s_ent = reinterpret_cast<uint32_t *>(smem + L.ent);
    const bool try_packed = (W == 1) && G <= 8;

    int m2 = 0;
    if (MODE != kFromOrder) {
        if (MODE == kFromIds) bad_min_warp0(L, smem, R, N);
        if (MODE == kFromIds && L.sync_part) {  // T before any key write (make_layout)
            for (int e = tid; e < N; e += kThreads) {
                uint32_t t = 0;
                for (uint32_t q = 0; q < R; ++q) t += static_cast<uint32_t>(s_part[q * L.NP + e]);
                s_T[e] = t;
            }
            cta_sync();
        }
        for (int base = 0; base < N; base += kThreads) {
            if (base + warp * 32 >= N) break;  // warp-uniform: no experts for this warp
            const int e = base + tid;
            const bool valid = e < N;
            uint32_t t = 0;
            uint32_t mw[W];
            int r = 0;
#pragma unroll
            for (int j = 0; j < W; ++j) {
                mw[j] = valid ? s_mask[e * W + j] : 0u;
                r += __popc(mw[j]);
            }
            if (valid) {
                if (MODE == kFromIds && L.sync_part) {
                    t = s_T[e];
                } else if (MODE == kFromIds) {
#pragma unroll 4
                    for (uint32_t q = 0; q < R; ++q) t += static_cast<uint32_t>(s_part[q * L.NP + e]);
                } else {
                    const int64_t tl = p.loads_in[e];
                    if (tl < 0 || tl > 0xffffffffLL) misc[M_LOADERR] = 1;
                    t = static_cast<uint32_t>(tl);
                }
                s_T[e] = t;
            }
            const bool active = t > 0;
            const bool multi = active && r >= 2;
            // compact replicated active experts first (any order: the sort ranks
            // them); the segment atomic's latency overlaps the classification below
            const unsigned bm = __ballot_sync(kFull, multi);
            int seg = 0;
            if (lane == 0 && bm) seg = atomicAdd(&misc[M_M2], __popc(bm));
            if (base == 0) stamp(p, 14);
            if (active && r == 0) atomicMin(&misc[M_NOREP], e);
            const bool forced = active && r == 1;
            int g1 = -1;
            if (forced) {
#pragma unroll
                for (int j = W - 1; j >= 0; --j)
                    if (mw[j]) g1 = 32 * j + __ffs(mw[j]) - 1;
                // forced prefix: the single-replica experts' order is irrelevant
                // (SURVEY.md App. A): each lands on its only replica
                atomicAdd(&s_L0[g1], 1);
            }
            if (valid) s_choice[e] = g1;
            seg = __shfl_sync(kFull, seg, 0);
            if (multi) {
                const int off = seg + __popc(bm & lanemask_lt());
                // canonical key (routing.py:84-86): r asc, T desc, id asc
                s_keys[off] = (static_cast<uint64_t>(r) << 56) | (static_cast<uint64_t>(0xffffffffu - t) << 24) |
                              static_cast<uint64_t>(e);
                s_cand[off] = e;
            }
            if (base == 0) stamp(p, 17);
        }
        stamp(p, 11);
        cta_sync();
        stamp(p, 12);
        if (MODE == kFromIds && bad_after_sync(p, L, smem, rank)) return false;
        if (MODE == kFromLoads && misc[M_LOADERR]) {
            write_error(p, writer, METRO_ERR_LOAD_RANGE, 0);
            return false;
        }
        if (misc[M_NOREP] != INT32_MAX) {
            write_error(p, writer, METRO_ERR_NO_REPLICA, misc[M_NOREP]);
            return false;
        }
        m2 = misc[M_M2];
        if (tid < 16) s_keys[m2 + tid] = ~0ull;  // pad for the paired scan
        cta_sync();
        stamp(p, 4);
        // ---- rank-by-count sort.  Four warps per 32 candidates: lane = candidate,
        // warp & 3 = a quarter of the key array.  Every lane of a warp reads the same
        // key pair (a true broadcast: one shared-memory wavefront per load); the four
        // quarter counts meet in shared memory.  Entries are written at slot = rank
        // (packed layout for G <= 8, SoA masks always).
        int32_t *s_rpart = reinterpret_cast<int32_t *>(smem + L.rpart);  // [4][N]
        {
            const int grp = warp >> 2, part = warp & 3;
            for (int c0 = grp * 32; c0 < m2; c0 += (kWarps / 4) * 32) {
                const int c = c0 + lane;
                const uint64_t kc = (c < m2) ? s_keys[c] : 0ull;
                int r0 = 0, r1 = 0, r2 = 0, r3 = 0;
#pragma unroll 2
                for (int c2 = 2 * part; c2 < m2; c2 += 16) {
                    const ulonglong2 k0 = *reinterpret_cast<const ulonglong2 *>(s_keys + c2);
                    const ulonglong2 k1 = *reinterpret_cast<const ulonglong2 *>(s_keys + c2 + 8);
                    r0 += k0.x < kc;
                    r1 += k0.y < kc;
                    r2 += k1.x < kc;
                    r3 += k1.y < kc;
                }
                if (c < m2) s_rpart[part * N + c] = (r0 + r1) + (r2 + r3);
            }
        }
        cta_sync();
        stamp(p, 13);
        for (int c = tid; c < m2; c += kThreads) {
            const int rk = (s_rpart[c] + s_rpart[N + c]) + (s_rpart[2 * N + c] + s_rpart[3 * N + c]);
            const int e = s_cand[c];
            const int r = static_cast<int>(s_keys[c] >> 56);
            s_sid[rk] = e;
            if (try_packed) packed_entry(s_ent + rk * kES, r, s_mask[e], e);
            if (r == 2) atomicMax(&misc[M_N2], rk + 1);
            if (r <= 3) atomicMax(&misc[M_N3], rk + 1);  // end of the r=3 segment
        }
        if (try_packed && m2 >= METRO_R2_BLOCK_MIN) {
            // block-of-four corrections for the r=2 lookahead: for steps i < j of a
            // block with candidates (a_i, b_i), dX_ij = [b_j == X] - [a_j == X]; stored
            // as {dA_ij, dA_ij - dB_ij} for ij = 01 02 03 12 13 23 (12 words per block).
            // With fewer replicated experts (m2 < METRO_R2_BLOCK_MIN) the greedy steps
            // one at a time and this pass and its barrier are skipped.
            cta_sync();
            const int n2 = misc[M_N2];
            uint32_t *dlt = reinterpret_cast<uint32_t *>(smem + L.rpart);
            for (int q = tid; q < (n2 >> 2) * 6; q += kThreads) {
                const int blk = q / 6, pr = q - blk * 6;
                const int i = pr < 3 ? 0 : (pr < 5 ? 1 : 2);
                const int j = pr < 3 ? pr + 1 : (pr < 5 ? pr - 1 : 3);
                const uint32_t gi = s_ent[(4 * blk + i) * kES + 6], gj = s_ent[(4 * blk + j) * kES + 6];
                const int ai = gi & 0xff, bi = (gi >> 8) & 0xff, aj = gj & 0xff, bj = (gj >> 8) & 0xff;
                const int dA = static_cast<int>(bj == ai) - static_cast<int>(aj == ai);
                const int dB = static_cast<int>(bj == bi) - static_cast<int>(aj == bi);
                dlt[blk * 12 + 2 * pr] = static_cast<uint32_t>(dA);
                dlt[blk * 12 + 2 * pr + 1] = static_cast<uint32_t>(dA - dB);
            }
        }
    } else {
        // caller-supplied order (metro-parallel): single-replica experts included
        m2 = p.order_len;
        for (int s = tid; s < m2; s += kThreads) {
            const int e = p.order[s];
            int r = 0;
            if (e >= 0 && e < N) {
#pragma unroll
                for (int j = 0; j < W; ++j) r += __popc(s_mask[e * W + j]);
                s_sid[s] = e;
            }
            if (e < 0 || e >= N || r == 0) atomicMin(&misc[M_NOREP], (e < 0 || e >= N) ? -1 : e);
        }
        for (int e = tid; e < N; e += kThreads) s_choice[e] = -1;
        cta_sync();
        if (misc[M_NOREP] != INT32_MAX) {
            write_error(p, writer, METRO_ERR_NO_REPLICA, misc[M_NOREP]);
            return false;
        }
    }
    cta_sync();
    stamp(p, 5);

    bool done = false, overlap_done = false;
    if (MODE != kFromOrder && try_packed) {
        // Packed greedy (thread 0).  Valid iff every final counter is <= 126: the
        // counters only grow, so no byte ever crossed into the sign bit.
        if (tid == 0) {
            PackedL Lp;
            Lp.lo = Lp.hi = 0;
            int assigned = m2;
            bool ok = true;
            for (int g = 0; g < G; ++g) {
                const int c = s_L0[g];
                ok = ok && c <= 126;
                assigned += c;
                const uint32_t v = static_cast<uint32_t>(c) << (8 * (g & 3));
                if (g < 4) Lp.lo += v;
                else Lp.hi += v;
            }
            const int n2 = misc[M_N2], n3 = misc[M_N3] - n2;
            if (ok)
                Lp = packed_greedy(p, s_ent, reinterpret_cast<const uint32_t *>(smem + L.rpart), n2, n3, m2,
                                   s_choice, Lp);
            // every final counter <= 126 (no byte reached the sign bit; counters only
            // grow) and the byte sum equals the assignments (no byte wrapped past 255)
            ok = ok && ((Lp.lo | Lp.hi) & 0x80808080u) == 0 && ((Lp.lo + 0x01010101u) & 0x80808080u) == 0 &&
                 ((Lp.hi + 0x01010101u) & 0x80808080u) == 0 &&
                 __dp4a(Lp.lo, 0x01010101u, __dp4a(Lp.hi, 0x01010101u, 0u)) == static_cast<uint32_t>(assigned);
            misc[M_PACKED_OK] = ok ? 1 : 0;
            misc[M_PACKED_LO] = static_cast<int32_t>(Lp.lo);
            misc[M_PACKED_HI] = static_cast<int32_t>(Lp.hi);
        }
        if (warp != 0) overlap();
        overlap_done = true;
        cta_sync();
        done = misc[M_PACKED_OK] != 0;
        if (done) {  // the greedy thread stored every choice as it went
            stamp(p, 6);
            if (writer && warp == 0) {  // counts and lambda off the greedy thread's chain
                const uint32_t w = static_cast<uint32_t>(misc[lane < 4 ? M_PACKED_LO : M_PACKED_HI]);
                const uint32_t c = lane < G ? (w >> (8 * (lane & 3))) & 0xffu : 0u;
                if (lane < G) p.rank_counts[lane] = static_cast<int32_t>(c);
                const uint32_t mx = __reduce_max_sync(kFull, c);
                if (lane == 0) *p.lam = static_cast<int32_t>(mx);
            }
            return true;
        }
    }
    if (!done) {
        // ---- serial greedy (routing.py:94-101) in warp 0, any G <= 128 (out of
        // line: its unrolled code stays out of the packed path's instruction stream)
        if (warp == 0) {
            warp_greedy<W>(s_mask, s_choice, s_sid, s_L0, G, m2, p.rank_counts, p.lam, writer);
        } else if (!overlap_done) {
            overlap();
        }
    }
    cta_sync();
    stamp(p, 6);
    return true;
}

// exclusive scan of v[0..n) into out[0..n], out[n] = total, over the kThreads
// routing threads (three barriers)
static __device__ __forceinline__ void block_exscan(const int32_t *v, int32_t *out, int n, int32_t *wsum) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (n + kThreads - 1) / kThreads;
    const int b = min(n, tid * per), e = min(n, b + per);
    int32_t s = 0;
    for (int i = b; i < e; ++i) s += v[i];
    int32_t x = s;  // inclusive warp scan
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int32_t y = __shfl_up_sync(kFull, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    cta_sync();
    if (warp == 0) {
        int32_t w = lane < kWarps ? wsum[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int32_t y = __shfl_up_sync(kFull, w, d);
            if (lane >= d) w += y;
        }
        if (lane < kWarps) wsum[lane] = w;  // inclusive warp totals
    }
    cta_sync();
    int32_t run = x - s + (warp > 0 ? wsum[warp - 1] : 0);
    for (int i = b; i < e; ++i) {
        out[i] = run;
        run += v[i];
    }
    if (tid == kThreads - 1) out[n] = wsum[kWarps - 1];
    cta_sync();
}

// ---------------------------------------------------------------- fused dispatch layout
// The dispatch layout of include/dispatch_layout.h computed inside the METRO
// kernel.  A METRO expert has ONE active replica, (e, choice[e]), with T[e] rows
// (routing.py:46-50, x[i, choice[i]] = T[i]), so
//   pair_row[p] = rep_off[rid(e, g)] - rep_off[slot_base[g]]   (expert's first row on rank g)
//               + occurrences of e in earlier CTAs' slices       (partial rows)
//               + occurrences of e in earlier walk-warp sub-slices of this CTA
//               + occurrences of e earlier in this warp's sub-slice (match_any)
// with e = topk_ids[p], g = choice[e] -- pairs of one replica in row-major order,
// the standalone layout kernel's convention.  The occurrence walk (walk-warp w =
// warp - 1 owns a contiguous sub-slice) runs while warp 0 runs the greedy.
struct LayoutWalk {
    const Layout *L;
    unsigned char *smem;
    int n_local, N, ws;
    int64_t *stamps;
    int dbg;
    __device__ __forceinline__ void operator()() const {
        const int wi = lay_index(static_cast<int>(threadIdx.x >> 5));
        if (wi < 0 || (dbg & 1)) return;
        if (stamps && threadIdx.x == 32 && cluster_ctarank() == 0) stamps[30] = clock64();
        walk(wi);
        if (stamps && threadIdx.x == 32 && cluster_ctarank() == 0) stamps[26] = clock64();
        // every walk warp's counts are in: exclusive prefixes over the walk warps,
        // starting at the CTA prefix (occurrences in earlier CTAs' slices) -- still
        // while warp 0 runs the greedy
        asm volatile("bar.sync 2, %0;" ::"n"(kLayWarps * 32) : "memory");
        uint32_t *s_hw = reinterpret_cast<uint32_t *>(smem + L->lhw);
        const int32_t *s_pre = reinterpret_cast<const int32_t *>(smem + L->lpre);
        for (int e = wi * 32 + static_cast<int>(threadIdx.x & 31); e < N; e += kLayWarps * 32) {
            uint32_t run = static_cast<uint32_t>(s_pre[e]);
            uint32_t c[kLayWarps];
#pragma unroll
            for (int w = 0; w < kLayWarps; ++w) c[w] = s_hw[w * N + e];
#pragma unroll
            for (int w = 0; w < kLayWarps; ++w) {
                s_hw[w * N + e] = run;
                run += c[w];
            }
        }
        if (stamps && threadIdx.x == 32 && cluster_ctarank() == 0) stamps[29] = clock64();
    }
    __device__ __forceinline__ void walk(int w) const {
        const int lane = threadIdx.x & 31;
        const int32_t *s_ids = reinterpret_cast<const int32_t *>(smem + L->ids);
        uint32_t *hw = reinterpret_cast<uint32_t *>(smem + L->lhw) + w * N;
        uint16_t *occ = reinterpret_cast<uint16_t *>(smem + L->locc);
        const int wb = min(n_local, w * ws), we = min(n_local, wb + ws);
        // blocks of four chunks of 32 pairs: the id loads and match_any of the four
        // chunks are independent (issued together); only the count updates chain
        constexpr int U = 4;
        for (int p0 = wb; p0 < we; p0 += 32 * U) {
            int e[U];
            unsigned m[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = p0 + 32 * u + lane;
                e[u] = (i < we) ? s_ids[i] : -1;  // ids already range-checked
            }
#pragma unroll
            for (int u = 0; u < U; ++u) m[u] = __match_any_sync(kFull, e[u]);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = p0 + 32 * u + lane;
                if (e[u] >= 0) occ[i] = static_cast<uint16_t>(hw[e[u]] + __popc(m[u] & lanemask_lt()));
                __syncwarp();
                if (e[u] >= 0 && lane == __ffs(m[u]) - 1) hw[e[u]] += __popc(m[u]);
                __syncwarp();
            }
        }
    }
};


// ================================================================ kernels

// ---------------------------------------------------------------- gating top-k (fused)
// Order key of an fp32 score: unsigned compare == float compare.  -0.0 is
// canonicalised to +0.0 (they compare equal, so the tie goes to the lower id, as
// the oracle's float '>' does), and every NaN maps to 0, below every number
// (-inf keys to 0x007fffff): NaN scores are taken last, ties among them to the
// lower id -- numpy's "NaN sorts last" in the reference generator's argsort(-keys)
// (core.py:322-326).  A key of 0 still beats the padding lanes (whole key 0).
__device__ __forceinline__ uint32_t okey(float f) {
    const uint32_t b = (f == 0.0f) ? 0u : __float_as_uint(f);
    const uint32_t k = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    return (f != f) ? 0u : k;
}
// Top-k of every token of this CTA's slice, fused with the histogram: one warp per
// token, two tokens in flight per warp (one for N > 256).  Lane l holds experts l + 32 j as 64-bit
// keys (score key << 32 | ~expert), sorted descending in registers (bitonic
// network), so "largest score, then lowest expert id" is the u64 max.  Round r: two
// redux.sync (max of the high words, then of the low words among the lanes holding
// that maximum) name the winner; its owner lane pops its head.  Ids are written in
// descending score order (core.py:322-326), staged in shared memory for the
// routing phases and counted into the lane-striped histogram.
__device__ __forceinline__ void cas_desc(uint64_t &a, uint64_t &b) {
    const uint64_t x = a, y = b;
    const bool sw = x < y;
    a = sw ? y : x;
    b = sw ? x : y;
}
template <int NPL>
__device__ __forceinline__ void lane_sort_desc(uint64_t (&c)[NPL]) {
    if constexpr (NPL == 8) {
        // optimal 8-input network: 19 compare-exchanges, depth 6 (bitonic: 24)
        cas_desc(c[0], c[2]); cas_desc(c[1], c[3]); cas_desc(c[4], c[6]); cas_desc(c[5], c[7]);
        cas_desc(c[0], c[4]); cas_desc(c[1], c[5]); cas_desc(c[2], c[6]); cas_desc(c[3], c[7]);
        cas_desc(c[0], c[1]); cas_desc(c[2], c[3]); cas_desc(c[4], c[5]); cas_desc(c[6], c[7]);
        cas_desc(c[2], c[4]); cas_desc(c[3], c[5]);
        cas_desc(c[1], c[4]); cas_desc(c[3], c[6]);
        cas_desc(c[1], c[2]); cas_desc(c[3], c[4]); cas_desc(c[5], c[6]);
        return;
    } else if constexpr (NPL == 4) {
        cas_desc(c[0], c[1]); cas_desc(c[2], c[3]); cas_desc(c[0], c[2]); cas_desc(c[1], c[3]);
        cas_desc(c[1], c[2]);
        return;
    }
#pragma unroll
    for (int size = 2; size <= NPL; size <<= 1)
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1)
#pragma unroll
            for (int i = 0; i < NPL; ++i) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool desc = ((i & size) == 0);
                    const uint64_t a = c[i], b = c[j];
                    const bool sw = desc ? (a < b) : (a > b);
                    c[i] = sw ? b : a;
                    c[j] = sw ? a : b;
                }
            }
}

// s_ids == nullptr: ids go to global memory only; hist[e * C + lane % C] counts.
// TPW: tokens in flight per warp (two at most for NPL <= 8: register budget).
template <int NPL, int TPW = (NPL <= 8 ? 2 : 1)>
__device__ void gate_topk(const Params &p, const Layout &L, unsigned char *smem, int64_t tok_beg, int n_tok,
                          int32_t *s_ids, int32_t *s_hist, int C) {
    static_assert(TPW == 1 || (TPW == 2 && NPL <= 8), "register budget");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int N = p.N, k = p.top_k, cm = C - 1;
    for (int t0 = TPW * warp; t0 < n_tok; t0 += TPW * kWarps) {
        const bool two = TPW == 2 && t0 + 1 < n_tok;
        uint64_t c[TPW][NPL];
#pragma unroll
        for (int q = 0; q < TPW; ++q) {
            const int tq = t0 + (q && two ? 1 : 0);
            const float *row = p.score_bytes > 0
                                   ? reinterpret_cast<const float *>(smem + L.sc) + static_cast<int64_t>(tq) * N
                                   : p.scores + (tok_beg + tq) * static_cast<int64_t>(N);
#pragma unroll
            for (int j = 0; j < NPL; ++j) {
                const int e = lane + 32 * j;
                c[q][j] = (e < N) ? ((static_cast<uint64_t>(okey(row[e])) << 32) |
                                     static_cast<uint64_t>(0xffffffffu - static_cast<uint32_t>(e)))
                                  : 0ull;
            }
            lane_sort_desc<NPL>(c[q]);
        }
        int mine[TPW];
#pragma unroll
        for (int q = 0; q < TPW; ++q) mine[q] = 0;
        for (int r = 0; r < k; ++r) {
#pragma unroll
            for (int q = 0; q < TPW; ++q) {
                const uint32_t hi = static_cast<uint32_t>(c[q][0] >> 32);
                const uint32_t mh = __reduce_max_sync(kFull, hi);
                const uint32_t lo = (hi == mh) ? static_cast<uint32_t>(c[q][0]) : 0u;
                const uint32_t ml = __reduce_max_sync(kFull, lo);
                const int e = static_cast<int>(0xffffffffu - ml);
                if ((e & 31) == lane) {
#pragma unroll
                    for (int j = 0; j + 1 < NPL; ++j) c[q][j] = c[q][j + 1];
                    c[q][NPL - 1] = 0ull;
                }
                if (lane == r) mine[q] = e;
            }
        }
        if (lane < k) {
#pragma unroll
            for (int q = 0; q < TPW; ++q) {
                if (q == 1 && !two) break;
                const int tl = t0 + q;
                const int e = mine[q];
                if (s_ids) s_ids[tl * k + lane] = e;
                p.ids_out[(tok_beg + tl) * k + lane] = e;
                atomicAdd(&s_hist[e * C + (lane & cm)], 1);
            }
        }
    }
}

// Fused dispatch layout, after the decide phase (choice final; the walk warps
// already turned their counts into exclusive prefixes during the greedy).  rep_off
// is the exclusive scan over replica ids of the rows per replica, which for METRO
// are T[e] on (e, choice[e]) and 0 elsewhere (routing.py:46-50); an expert's
// first row on its rank is rep_off[rid(e, g)] - rep_off[slot_base[g]].  Every
// step is one element per thread with a barrier between (serial per-warp chains
// measured 2-3x slower on B200): scatter rows -> block scan (two barriers) ->
// base + loads / choice -> pair_rank + pair_row of each walk warp's sub-slice.
template <int W>
__device__ void layout_tail(const Params &p, const Layout &L, unsigned char *smem, int64_t beg, int n_local,
                            int ws, bool writer, int32_t status3) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int N = p.N, G = p.G, nrep = p.nrep;
    const int32_t *s_choice = reinterpret_cast<const int32_t *>(smem + L.choice);
    const uint32_t *s_T = reinterpret_cast<const uint32_t *>(smem + L.T);
    const int32_t *s_rtab = reinterpret_cast<const int32_t *>(smem + L.lrtab);
    const int32_t *s_sb = reinterpret_cast<const int32_t *>(smem + L.lsb);
    const uint32_t *s_hw = reinterpret_cast<const uint32_t *>(smem + L.lhw);
    const uint16_t *s_occ = reinterpret_cast<const uint16_t *>(smem + L.locc);
    int32_t *s_rows = reinterpret_cast<int32_t *>(smem + L.lrows);  // zeroed in the prologue
    int32_t *s_off = reinterpret_cast<int32_t *>(smem + L.loff);
    int32_t *s_base = reinterpret_cast<int32_t *>(smem + L.lbase);
    int32_t *s_wsum = reinterpret_cast<int32_t *>(smem + L.lwsum);
    if (layout_rtab_bulk(p)) mbar_wait(reinterpret_cast<uint64_t *>(smem + L.mbar) + 2, 0);
    for (int e = tid; e < N; e += kThreads) {
        const int g = s_choice[e];
        if (g >= 0) s_rows[s_rtab[e * G + g]] = static_cast<int32_t>(s_T[e]);
    }
    cta_sync();
    if (nrep < kThreads) {
        // one replica per thread (and thread nrep writes the total, so nrep < kThreads):
        // its inclusive warp scan and the warp totals go to
        // shared memory, after ONE barrier any thread forms any offset (warp
        // totals summed in registers) -- rep_off and the experts' first rows in the
        // same pass
        int32_t *s_incl = s_off;
        const int32_t v = tid < nrep ? s_rows[tid] : 0;
        int32_t x = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int32_t y = __shfl_up_sync(kFull, x, d);
            if (lane >= d) x += y;
        }
        if (tid < nrep) s_incl[tid] = x;  // s_off holds nrep + 1 entries
        if (lane == 31) s_wsum[warp] = x;
        cta_sync();
        int32_t ws_[kWarps];
#pragma unroll
        for (int q = 0; q < kWarps / 4; ++q) {
            const int4 t4 = reinterpret_cast<const int4 *>(s_wsum)[q];
            ws_[4 * q] = t4.x; ws_[4 * q + 1] = t4.y; ws_[4 * q + 2] = t4.z; ws_[4 * q + 3] = t4.w;
        }
        auto off = [&](int i) {  // exclusive prefix at replica i (i <= nrep)
            const int wi = i >> 5;
            int32_t o = (i & 31) ? s_incl[i - 1] : 0;
#pragma unroll
            for (int q = 0; q < kWarps; ++q) o += (q < wi) ? ws_[q] : 0;
            return o;
        };
        if (writer && tid <= nrep) p.rep_off[tid] = off(tid);
        for (int e = tid; e < N; e += kThreads) {
            const int g = s_choice[e];
            if (g >= 0) s_base[e] = off(s_rtab[e * G + g]) - off(s_sb[g]);
            if (writer) {
                if (p.loads) p.loads[e] = static_cast<int32_t>(s_T[e]);
                p.choice[e] = g;
            }
        }
    } else {
        // block exclusive scan of rows[0..nrep): a contiguous chunk per thread, warp
        // shuffle scan, warp totals through shared memory
        const int per = (nrep + kThreads - 1) / kThreads;
        const int b = min(nrep, tid * per), en = min(nrep, b + per);
        int32_t sum = 0;
        for (int i = b; i < en; ++i) sum += s_rows[i];
        int32_t x = sum;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int32_t y = __shfl_up_sync(kFull, x, d);
            if (lane >= d) x += y;
        }
        if (lane == 31) s_wsum[warp] = x;
        cta_sync();
        int32_t run = x - sum;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) run += (w < warp) ? s_wsum[w] : 0;
        for (int i = b; i < en; ++i) {
            const int32_t v = s_rows[i];
            s_off[i] = run;
            if (writer) p.rep_off[i] = run;
            run += v;
        }
        if (tid == kThreads - 1) {
            s_off[nrep] = run;  // the last thread's chunk ends the array
            if (writer) p.rep_off[nrep] = run;
        }
        cta_sync();
        for (int e = tid; e < N; e += kThreads) {
            const int g = s_choice[e];
            if (g >= 0) s_base[e] = s_off[s_rtab[e * G + g]] - s_off[s_sb[g]];
            if (writer) {
                if (p.loads) p.loads[e] = static_cast<int32_t>(s_T[e]);
                p.choice[e] = g;
            }
        }
    }
    if (writer && tid == 0) {
        p.status[0] = METRO_OK;
        p.status[1] = p.status[2] = 0;
        p.status[3] = status3;
    }
    cta_sync();
    const int w = lay_index(warp);
    if (w < 0) return;
    // walk warp w writes its own sub-slice: four pairs per lane (16-byte loads of
    // the ids, 8-byte loads of the in-warp ranks, 16-byte stores), scalar tail
    const int32_t *s_ids = reinterpret_cast<const int32_t *>(smem + L.ids);
    const uint32_t *hw = s_hw + w * N;
    const int wb = min(n_local, w * ws), we = min(n_local, wb + ws);
    int32_t *pr = p.pair_rank + beg, *prow = p.pair_row + beg;
    const bool vec = ((reinterpret_cast<uintptr_t>(pr) | reinterpret_cast<uintptr_t>(prow)) & 15) == 0;
    const int we4 = vec ? wb + ((we - wb) & ~3) : wb;
    for (int i = wb + 4 * lane; i < we4; i += 128) {
        const int4 e = *reinterpret_cast<const int4 *>(s_ids + i);
        const uint2 o = *reinterpret_cast<const uint2 *>(s_occ + i);
        *reinterpret_cast<int4 *>(pr + i) = make_int4(s_choice[e.x], s_choice[e.y], s_choice[e.z], s_choice[e.w]);
        *reinterpret_cast<int4 *>(prow + i) =
            make_int4(s_base[e.x] + static_cast<int32_t>(hw[e.x]) + static_cast<int32_t>(o.x & 0xffffu),
                      s_base[e.y] + static_cast<int32_t>(hw[e.y]) + static_cast<int32_t>(o.x >> 16),
                      s_base[e.z] + static_cast<int32_t>(hw[e.z]) + static_cast<int32_t>(o.y & 0xffffu),
                      s_base[e.w] + static_cast<int32_t>(hw[e.w]) + static_cast<int32_t>(o.y >> 16));
    }
    for (int i = we4 + lane; i < we; i += 32) {
        const int e = s_ids[i];
        pr[i] = s_choice[e];
        prow[i] = s_base[e] + static_cast<int32_t>(hw[e]) + static_cast<int32_t>(s_occ[i]);
    }
}

}  // namespace metro
