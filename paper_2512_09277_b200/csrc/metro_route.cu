// metro_route.cu -- sm_100a kernels for METRO / EPLB replica routing (one MoE layer).
//
// Reference semantics (authoritative: the code, not SPEC.md):
//   aggregate_loads  /root/reference/pkg/src/eproute/core.py:236-244
//   route_metro      /root/reference/pkg/src/eproute/routing.py:105-113
//     _active_order  routing.py:75-87   order = (replica count asc, T desc, id asc)
//     _greedy_assign routing.py:90-102  argmin L over ascending replicas, strict '<'
//   route_eplb       routing.py:55-72   even split, remainder to low rank ids
//
// Kernel structure: one thread-block cluster of R CTAs routes one
// layer.  Every CTA
//   (A) stages its contiguous slice of the all-gathered top-k ids in shared memory
//       with one TMA bulk copy (cp.async.bulk + mbarrier), the rank bitmasks likewise;
//   (B) histograms the slice (lane-striped shared counters -> conflict-free);
//   (C) pushes its partial histogram into every CTA's shared memory over DSMEM and
//       passes ONE cluster barrier;
//   (D) redundantly (so no second barrier is needed) sums the partials into T,
//       applies the order-free forced prefix (experts with one replica) with
//       warp ballots, compacts + rank-sorts the replicated active experts by the
//       canonical key, and runs the serial greedy in ONE warp: lane g owns
//       counter L[g]; each step is a redux.sync min over (L << 8 | g) of the
//       candidate lanes, which is exactly "smallest L, lowest rank id on ties";
//   (E) writes pair_rank for its own slice from shared memory (ids never re-read
//       from HBM); CTA 0 writes loads / choice / rank_counts / lam / status.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <mutex>

#include "../../include/metro_route.h"

namespace metro {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxG = 128;
constexpr int kMaxN = 4096;
constexpr int kMaxCluster = 16;
constexpr int kMaxSmem = 232448;  // 227 KB opt-in on sm_100
constexpr int64_t kNoBad = INT64_MAX;

enum Kind { kMetroIds = 0, kEplbIds = 1, kMetroLoads = 2, kEplbLoads = 3, kMetroOrdered = 4 };

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
};

// ---------------------------------------------------------------- smem layout
// mbar | misc | mask | ids (staged slice) | T | choice | aux | hist | part
// The METRO decide scratch (keys, cand, sorted) aliases hist + part: both are
// dead once the partial histograms have been reduced into T.
struct Layout {
    int mbar, misc, mask, ids, T, choice, aux, hist, part, keys, cand, sorted, total;
    int NP;  // partial-row stride (words): N + 2 (bad pair lo/hi) rounded to 4
};

__host__ __device__ inline int align_up(int x, int a) { return (x + a - 1) / a * a; }

__host__ __device__ inline Layout make_layout(int kind, int N, int W, int R, int64_t slice,
                                              int C, int staged, bool warp_hist = false) {
    Layout L;
    int o = 0;
    L.mbar = o; o += 16;
    L.misc = o; o += 64 * 4;
    L.mask = o; o = align_up(o + N * W * 4, 16);
    L.NP = align_up(N + 2, 4);
    const bool ids_mode = (kind == kMetroIds || kind == kEplbIds);
    const bool metro = (kind == kMetroIds || kind == kMetroLoads || kind == kMetroOrdered);
    L.ids = o;
    if (ids_mode && staged) o = align_up(o + (int)slice * 4, 16);
    L.T = o; o = align_up(o + N * (kind == kEplbIds ? 8 : 4), 16);  // EPLB: + CTA base
    L.choice = o;
    if (metro) o = align_up(o + N * 4, 16);
    L.aux = o; o = align_up(o + kMaxG * 4, 16);  // forced counts L0 / EPLB rank counts
    L.hist = o;
    int hist_bytes = 0;
    if (ids_mode) hist_bytes = warp_hist ? kWarps * N * 4 : N * C * 4;
    L.part = align_up(o + hist_bytes, 16);
    const int end1 = ids_mode ? align_up(L.part + R * L.NP * 4, 16) : L.part;
    L.keys = o;
    L.cand = align_up(L.keys + N * 8, 16);
    L.sorted = align_up(L.cand + N * 4, 16);
    const int end2 = metro ? align_up(L.sorted + N * (W + 1) * 4, 16) : o;
    L.total = end1 > end2 ? end1 : end2;
    return L;
}

// misc word indices
enum {
    M_BAD_LO = 0, M_BAD_HI = 1,   // int64 min bad pair (local)
    M_NOREP = 2,                  // min active expert without replica
    M_M2 = 3,                     // number of replicated active experts
    M_LOADERR = 4,
    M_ANY = 5,
    M_BADALL_LO = 6, M_BADALL_HI = 7,
    M_WCNT = 16,                  // [kWarps] per-warp compaction counts
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// TMA bulk copy global -> own shared memory, completion on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_release() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Store 16 bytes into CTA `cta`'s shared memory at the address `local` has in ours.
__device__ __forceinline__ void dsmem_st_v4(const void *local, uint32_t cta, uint4 v) {
    uint32_t raddr;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(smem_u32(local)), "r"(cta));
    asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(raddr), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ void stamp(const Params &p, int i) {
    if (p.stamps && threadIdx.x == 0 && cluster_ctarank() == 0) p.stamps[i] = clock64();
}

// position of the (q+1)-th set bit of a W-word mask (q < popcount)
template <int W>
__device__ __forceinline__ int nth_set_bit(const uint32_t *mw, int q) {
#pragma unroll
    for (int j = 0; j < W; ++j) {
        int c = __popc(mw[j]);
        if (q < c) return 32 * j + (int)__fns(mw[j], 0, q + 1);
        q -= c;
    }
    return -1;
}

// ---------------------------------------------------------------- phase A
// Stage rank masks (+ this CTA's id slice) into shared memory with TMA bulk copies.
template <int W>
__device__ void stage_inputs(const Params &p, const Layout &L, unsigned char *smem,
                             int64_t beg, int n_local, bool stage_ids) {
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + L.mbar);
    uint32_t *s_mask = reinterpret_cast<uint32_t *>(smem + L.mask);
    int32_t *s_ids = reinterpret_cast<int32_t *>(smem + L.ids);
    const int mask_words = p.mask ? p.N * W : 0;  // aggregate-only launches carry no mask
    const bool mask_bulk = mask_words > 0 && ((reinterpret_cast<uintptr_t>(p.mask) & 15) == 0) &&
                           (mask_words % 4 == 0);
    const int body = stage_ids ? (n_local & ~3) : 0;
    const bool ids_bulk =
        stage_ids && body > 0 && ((reinterpret_cast<uintptr_t>(p.ids + beg) & 15) == 0);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        uint32_t bytes = (mask_bulk ? mask_words * 4u : 0u) + (ids_bulk ? body * 4u : 0u);
        mbar_arrive_expect_tx(bar, bytes);
        if (mask_bulk) bulk_g2s(s_mask, p.mask, mask_words * 4u, bar);
        if (ids_bulk) bulk_g2s(s_ids, p.ids + beg, body * 4u, bar);
    }
    if (!mask_bulk)
        for (int i = threadIdx.x; i < mask_words; i += kThreads) s_mask[i] = __ldg(p.mask + i);
    if (stage_ids) {
        const int from = ids_bulk ? body : 0;
        for (int i = from + threadIdx.x; i < n_local; i += kThreads) s_ids[i] = __ldg(p.ids + beg + i);
    }
    __syncthreads();  // mbarrier init visible before anyone waits
    mbar_wait(bar, 0);
}

// ---------------------------------------------------------------- phase D (METRO)
// Given s_T (int32 loads, all CTAs), compute choice for every expert, run the
// forced prefix + canonical sort + warp greedy.  Returns false on error
// (status written by the writer CTA).
template <int W>
__device__ bool metro_decide(const Params &p, const Layout &L, unsigned char *smem, bool writer,
                             bool from_order) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int N = p.N, G = p.G;
    int32_t *misc = reinterpret_cast<int32_t *>(smem + L.misc);
    const uint32_t *s_mask = reinterpret_cast<const uint32_t *>(smem + L.mask);
    const uint32_t *s_T = reinterpret_cast<const uint32_t *>(smem + L.T);
    int32_t *s_choice = reinterpret_cast<int32_t *>(smem + L.choice);
    uint64_t *s_keys = reinterpret_cast<uint64_t *>(smem + L.keys);
    int32_t *s_cand = reinterpret_cast<int32_t *>(smem + L.cand);
    uint32_t *s_sorted = reinterpret_cast<uint32_t *>(smem + L.sorted);
    int32_t *s_L0 = reinterpret_cast<int32_t *>(smem + L.aux);

    int m2 = 0;
    if (!from_order) {
        // ---- classify experts: inactive / forced (r == 1) / replicated (r >= 2)
        for (int base = 0; base < N; base += kThreads) {
            const int e = base + tid;
            const bool valid = e < N;
            uint32_t t = valid ? s_T[e] : 0u;
            uint32_t mw[W];
            int r = 0;
#pragma unroll
            for (int j = 0; j < W; ++j) {
                mw[j] = valid ? s_mask[e * W + j] : 0u;
                r += __popc(mw[j]);
            }
            const bool active = t > 0;
            if (active && r == 0) atomicMin(&misc[M_NOREP], e);
            const bool forced = active && r == 1;
            const bool multi = active && r >= 2;
            int g1 = -1;
            if (forced) g1 = nth_set_bit<W>(mw, 0);
            if (valid) s_choice[e] = forced ? g1 : -1;
            // forced prefix: per-rank count of single-replica active experts.  The
            // order among them is irrelevant: each lands on its
            // only replica.  One shared atomic per distinct rank per warp.
            unsigned rem = __ballot_sync(kFull, forced);
            while (rem) {
                const int leader = __ffs(rem) - 1;
                const int gg = __shfl_sync(kFull, g1, leader);
                const unsigned m = __ballot_sync(kFull, forced && g1 == gg);
                if (lane == leader) atomicAdd(&s_L0[gg], __popc(m));
                rem &= ~m;
            }
            // stream-compact replicated active experts (ascending id)
            const unsigned bm = __ballot_sync(kFull, multi);
            if (lane == 0) misc[M_WCNT + warp] = __popc(bm);
            __syncthreads();
            int off = m2, tot = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                const int c = misc[M_WCNT + w];
                off += (w < warp) ? c : 0;
                tot += c;
            }
            off += __popc(bm & lanemask_lt());
            if (multi) {
                // canonical key (routing.py:84-86): r asc, T desc, id asc
                s_keys[off] = (static_cast<uint64_t>(r) << 56) |
                              (static_cast<uint64_t>(0xffffffffu - t) << 24) |
                              static_cast<uint64_t>(e);
                s_cand[off] = e;
            }
            m2 += tot;
            __syncthreads();
        }
        if (misc[M_NOREP] != INT32_MAX) {
            if (writer && tid == 0) {
                p.status[0] = METRO_ERR_NO_REPLICA;
                p.status[1] = misc[M_NOREP];
                p.status[2] = 0;
                p.status[3] = 0;
            }
            return false;
        }
        stamp(p, 4);
        // ---- rank-by-count sort of the m2 keys (distinct: ids are unique)
        for (int c = warp; c < m2; c += kWarps) {
            const uint64_t kc = s_keys[c];
            int cnt = 0;
            for (int c2 = lane; c2 < m2; c2 += 32) cnt += (s_keys[c2] < kc) ? 1 : 0;
            cnt = __reduce_add_sync(kFull, cnt);
            const int e = s_cand[c];
            if (lane < W) s_sorted[cnt * (W + 1) + lane] = s_mask[e * W + lane];
            if (lane == W) s_sorted[cnt * (W + 1) + W] = static_cast<uint32_t>(e);
        }
    } else {
        // ---- caller-supplied order (metro-parallel): every listed expert goes
        // through the greedy, single-replica ones included (no forced prefix).
        m2 = p.order_len;
        for (int s = tid; s < m2; s += kThreads) {
            const int e = p.order[s];
            int r = 0;
            if (e >= 0 && e < N) {
#pragma unroll
                for (int j = 0; j < W; ++j) {
                    const uint32_t w = s_mask[e * W + j];
                    s_sorted[s * (W + 1) + j] = w;
                    r += __popc(w);
                }
                s_sorted[s * (W + 1) + W] = static_cast<uint32_t>(e);
            }
            if (e < 0 || e >= N || r == 0) atomicMin(&misc[M_NOREP], (e < 0 || e >= N) ? -1 : e);
        }
        for (int e = tid; e < N; e += kThreads) s_choice[e] = -1;
        __syncthreads();
        if (misc[M_NOREP] != INT32_MAX) {
            if (writer && tid == 0) {
                p.status[0] = METRO_ERR_NO_REPLICA;
                p.status[1] = misc[M_NOREP];
                p.status[2] = 0;
                p.status[3] = 0;
            }
            return false;
        }
    }
    __syncthreads();
    stamp(p, 5);

    // ---- serial greedy (routing.py:94-101) in warp 0.
    // lane owns ranks g = lane + 32 j; packed key (L << 8 | g): the warp-wide
    // min over candidate lanes is "smallest L, then smallest g" -- the
    // reference's ascending scan with strict '<'.
    if (warp == 0) {
        uint32_t Lk[W];
#pragma unroll
        for (int j = 0; j < W; ++j) {
            const int g = lane + 32 * j;
            Lk[j] = (g < G) ? ((static_cast<uint32_t>(s_L0[g]) << 8) | static_cast<uint32_t>(g))
                            : 0xffffffffu;
        }
#pragma unroll 4
        for (int s = 0; s < m2; ++s) {
            const uint32_t *ent = s_sorted + s * (W + 1);
            uint32_t v = 0xffffffffu;
#pragma unroll
            for (int j = 0; j < W; ++j) {
                const uint32_t mw = ent[j];
                v = ((mw >> lane) & 1u) ? min(v, Lk[j]) : v;
            }
            const uint32_t win = __reduce_min_sync(kFull, v);
#pragma unroll
            for (int j = 0; j < W; ++j) Lk[j] += (Lk[j] == win) ? 256u : 0u;
            if (lane == 0) s_choice[ent[W]] = static_cast<int32_t>(win & 0xffu);
        }
        uint32_t mx = 0;
#pragma unroll
        for (int j = 0; j < W; ++j) {
            const int g = lane + 32 * j;
            if (g < G) {
                const uint32_t c = Lk[j] >> 8;
                if (writer) p.rank_counts[g] = static_cast<int32_t>(c);
                mx = max(mx, c);
            }
        }
        mx = __reduce_max_sync(kFull, mx);
        if (writer && lane == 0) *p.lam = static_cast<int32_t>(mx);
    }
    __syncthreads();
    stamp(p, 6);
    return true;
}

// ---------------------------------------------------------------- histogram + exchange
// Phase B + C for the ids kernels.  On return s_T holds the global loads and
// (EPLB) s_T[N + e] holds this CTA's exclusive base (sum of earlier CTAs).
template <int W, bool PRIV, bool BASE>
__device__ bool histogram_exchange(const Params &p, const Layout &L, unsigned char *smem,
                                   int64_t beg, int n_local, uint32_t R, uint32_t rank) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int N = p.N;
    int32_t *misc = reinterpret_cast<int32_t *>(smem + L.misc);
    const int32_t *s_ids = reinterpret_cast<const int32_t *>(smem + L.ids);
    int32_t *s_hist = reinterpret_cast<int32_t *>(smem + L.hist);
    int32_t *s_part = reinterpret_cast<int32_t *>(smem + L.part);
    uint32_t *s_T = reinterpret_cast<uint32_t *>(smem + L.T);
    const int32_t *src = p.staged ? s_ids : (p.ids + beg);
    int64_t my_bad = kNoBad;

    if (!PRIV) {
        // lane-striped counters hist[e][lane % C]: within one warp instruction every
        // lane hits its own bank, so hot experts do not serialise the atomics.
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
                        my_bad = min(my_bad, beg + i + q);
                }
            }
        }
        for (int i = (vec ? n4 : 0) + tid; i < n_local; i += kThreads) {
            const int e = src[i];
            if (static_cast<unsigned>(e) < static_cast<unsigned>(N))
                atomicAdd(&s_hist[e * p.C + (lane & cm)], 1);
            else
                my_bad = min(my_bad, beg + i);
        }
    } else {
        // warp-private histograms over contiguous warp sub-slices; match_any groups
        // equal ids so one lane does a plain read-modify-write.  The same walk
        // later yields deterministic row-major occurrence ranks (EPLB pair_rank).
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
        atomicMin(reinterpret_cast<unsigned long long *>(&misc[M_BAD_LO]),
                  static_cast<unsigned long long>(my_bad));
    __syncthreads();
    stamp(p, 2);

    // local partial row -> s_part[rank]
    int32_t *row = s_part + rank * L.NP;
    if (!PRIV) {
        for (int e = warp; e < N; e += kWarps) {
            int v = (lane < p.C) ? s_hist[e * p.C + lane] : 0;
            v = __reduce_add_sync(kFull, v);
            if (lane == 0) row[e] = v;
        }
    } else {
        for (int e = tid; e < N; e += kThreads) {
            int s = 0;
#pragma unroll 4
            for (int w = 0; w < kWarps; ++w) s += s_hist[w * N + e];
            row[e] = s;
        }
    }
    if (tid == 0) {
        row[N] = misc[M_BAD_LO];
        row[N + 1] = misc[M_BAD_HI];
    }
    for (int e = N + 2 + tid; e < L.NP; e += kThreads) row[e] = 0;
    __syncthreads();
    // all CTAs of the cluster have started (arrived at kernel entry) before
    // anyone writes into a peer's shared memory
    cluster_wait();
    const int nv = L.NP / 4;
    for (int idx = tid; idx < (int)(R - 1) * nv; idx += kThreads) {
        const uint32_t d = (rank + 1 + idx / nv) % R;
        const int v = idx % nv;
        const uint4 val = reinterpret_cast<const uint4 *>(row)[v];
        dsmem_st_v4(reinterpret_cast<const uint4 *>(row) + v, d, val);
    }
    cluster_arrive_release();
    cluster_wait();
    stamp(p, 3);

    // reduce partials: T (all CTAs, redundantly); EPLB also keeps the CTA base
    for (int e = tid; e < N; e += kThreads) {
        uint32_t t = 0, b = 0;
        for (uint32_t r = 0; r < R; ++r) {
            const uint32_t v = static_cast<uint32_t>(s_part[r * L.NP + e]);
            if (r < rank) b += v;
            t += v;
        }
        s_T[e] = t;
        if (BASE) s_T[N + e] = b;
    }
    if (tid == 0) {
        unsigned long long bad = static_cast<unsigned long long>(kNoBad);
        for (uint32_t r = 0; r < R; ++r) {
            const int32_t *rw = s_part + r * L.NP;
            const unsigned long long v =
                (static_cast<unsigned long long>(static_cast<uint32_t>(rw[N + 1])) << 32) |
                static_cast<uint32_t>(rw[N]);
            bad = min(bad, v);
        }
        misc[M_BADALL_LO] = static_cast<int32_t>(bad & 0xffffffffu);
        misc[M_BADALL_HI] = static_cast<int32_t>(bad >> 32);
    }
    __syncthreads();
    const unsigned long long bad =
        (static_cast<unsigned long long>(static_cast<uint32_t>(misc[M_BADALL_HI])) << 32) |
        static_cast<uint32_t>(misc[M_BADALL_LO]);
    if (bad != static_cast<unsigned long long>(kNoBad)) {
        if (rank == 0 && tid == 0) {
            p.status[0] = METRO_ERR_ID_RANGE;
            p.status[1] = static_cast<int32_t>(bad & 0xffffffffu);
            p.status[2] = static_cast<int32_t>(bad >> 32);
            p.status[3] = p.ids[bad];
        }
        return false;
    }
    return true;
}

__device__ void zero_smem(unsigned char *smem, int from, int to) {
    for (int i = from / 16 + threadIdx.x; i < to / 16; i += kThreads)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0, 0, 0, 0);
}

__device__ void init_misc(int32_t *misc) {
    if (threadIdx.x < 64) misc[threadIdx.x] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
        misc[M_BAD_LO] = static_cast<int32_t>(0xffffffffu);
        misc[M_BAD_HI] = 0x7fffffff;
        misc[M_NOREP] = INT32_MAX;
    }
}

// ================================================================ kernels
template <int W>
__global__ void __launch_bounds__(kThreads, 1) metro_ids_kernel(const Params p) {
    extern __shared__ __align__(128) unsigned char smem[];
    cluster_arrive_relaxed();  // paired with the wait before the first DSMEM store
    stamp(p, 0);
    const uint32_t R = cluster_nctarank(), rank = cluster_ctarank();
    const Layout L = make_layout(kMetroIds, p.N, W, R, p.slice, p.C, p.staged);
    int32_t *misc = reinterpret_cast<int32_t *>(smem + L.misc);
    const int64_t beg = static_cast<int64_t>(rank) * p.slice;
    const int64_t rem_pairs = p.num_pairs - beg;
    const int n_local = rem_pairs <= 0 ? 0 : static_cast<int>(rem_pairs < p.slice ? rem_pairs : p.slice);

    init_misc(misc);
    zero_smem(smem, L.aux, L.part);  // forced counts + histogram
    stage_inputs<W>(p, L, smem, beg, n_local, p.staged != 0);
    stamp(p, 1);
    if (!histogram_exchange<W, false, false>(p, L, smem, beg, n_local, R, rank)) return;
    const bool writer = (rank == 0);
    if (!p.mask) {  // aggregate_loads only (core.py:236-244)
        if (writer) {
            const uint32_t *s_T = reinterpret_cast<const uint32_t *>(smem + L.T);
            for (int e = threadIdx.x; e < p.N; e += kThreads) p.loads[e] = static_cast<int32_t>(s_T[e]);
            if (threadIdx.x == 0) {
                p.status[0] = METRO_OK;
                p.status[1] = p.status[2] = 0;
                p.status[3] = static_cast<int32_t>(R);
            }
        }
        return;
    }
    if (!metro_decide<W>(p, L, smem, writer, false)) return;

    // ---- outputs
    const int32_t *s_choice = reinterpret_cast<const int32_t *>(smem + L.choice);
    if (p.pair_rank) {
        const int32_t *src = p.staged ? reinterpret_cast<const int32_t *>(smem + L.ids) : (p.ids + beg);
        int32_t *dst = p.pair_rank + beg;
        const int n4 = n_local & ~3;
        const bool vec = ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) &&
                         (p.staged || ((reinterpret_cast<uintptr_t>(src) & 15) == 0));
        if (vec) {
            for (int i = threadIdx.x * 4; i < n4; i += kThreads * 4) {
                const int4 v = *reinterpret_cast<const int4 *>(src + i);
                int4 o;
                o.x = s_choice[v.x];
                o.y = s_choice[v.y];
                o.z = s_choice[v.z];
                o.w = s_choice[v.w];
                *reinterpret_cast<int4 *>(dst + i) = o;
            }
        }
        for (int i = (vec ? n4 : 0) + threadIdx.x; i < n_local; i += kThreads) dst[i] = s_choice[src[i]];
    }
    if (writer) {
        const uint32_t *s_T = reinterpret_cast<const uint32_t *>(smem + L.T);
        for (int e = threadIdx.x; e < p.N; e += kThreads) {
            if (p.loads) p.loads[e] = static_cast<int32_t>(s_T[e]);
            p.choice[e] = s_choice[e];
        }
        if (threadIdx.x == 0) {
            p.status[0] = METRO_OK;
            p.status[1] = p.status[2] = 0;
            p.status[3] = static_cast<int32_t>(R);
        }
    }
    stamp(p, 7);
}

// METRO from loads (compat route_metro(T, A)) or from a caller order (metro-parallel).
template <int W>
__global__ void __launch_bounds__(kThreads, 1) metro_loads_kernel(const Params p, int ordered) {
    extern __shared__ __align__(128) unsigned char smem[];
    const Layout L = make_layout(ordered ? kMetroOrdered : kMetroLoads, p.N, W, 1, 0, 1, 0);
    int32_t *misc = reinterpret_cast<int32_t *>(smem + L.misc);
    uint32_t *s_T = reinterpret_cast<uint32_t *>(smem + L.T);
    init_misc(misc);
    zero_smem(smem, L.aux, L.hist);
    stage_inputs<W>(p, L, smem, 0, 0, false);
    if (!ordered) {
        for (int e = threadIdx.x; e < p.N; e += kThreads) {
            const int64_t t = p.loads_in[e];
            if (t < 0 || t > 0xffffffffLL) atomicMax(&misc[M_LOADERR], 1);
            s_T[e] = static_cast<uint32_t>(t);
        }
        __syncthreads();
        if (misc[M_LOADERR]) {
            if (threadIdx.x == 0) {
                p.status[0] = METRO_ERR_LOAD_RANGE;
                p.status[1] = p.status[2] = p.status[3] = 0;
            }
            return;
        }
    }
    if (!metro_decide<W>(p, L, smem, true, ordered != 0)) return;
    const int32_t *s_choice = reinterpret_cast<const int32_t *>(smem + L.choice);
    for (int e = threadIdx.x; e < p.N; e += kThreads) p.choice[e] = s_choice[e];
    if (threadIdx.x == 0) {
        p.status[0] = METRO_OK;
        p.status[1] = p.status[2] = 0;
        p.status[3] = 1;
    }
}

// ---------------------------------------------------------------- EPLB
// Shared by both EPLB kernels: per-rank activated counts (y = x > 0), lam, x.
// T64 supplies the load of expert e.
template <int W, typename LoadFn, typename XT>
__device__ void eplb_counts_and_x(const Params &p, const Layout &L, unsigned char *smem,
                                  bool writer, LoadFn T64, XT *x) {
    const int tid = threadIdx.x, lane = tid & 31;
    const int N = p.N, G = p.G;
    const uint32_t *s_mask = reinterpret_cast<const uint32_t *>(smem + L.mask);
    int32_t *s_cnt = reinterpret_cast<int32_t *>(smem + L.aux);
    int32_t *misc = reinterpret_cast<int32_t *>(smem + L.misc);
    for (int base = 0; base < N; base += kThreads) {
        const int e = base + tid;
        const bool valid = e < N;
        const int64_t t = valid ? T64(e) : 0;
        uint32_t mw[W], act[W];
        int r = 0;
#pragma unroll
        for (int j = 0; j < W; ++j) {
            mw[j] = valid ? s_mask[e * W + j] : 0u;
            r += __popc(mw[j]);
        }
        if (t > 0 && r == 0) atomicMin(&misc[M_NOREP], e);
        // x > 0 exactly on the first min(T, r) replicas in ascending rank id
        int64_t a = (t < r) ? t : r;
#pragma unroll
        for (int j = 0; j < W; ++j) {
            const int c = __popc(mw[j]);
            const int take = static_cast<int>(a < c ? a : c);
            act[j] = (take == c) ? mw[j] : (take == 0 ? 0u : (mw[j] & ((1u << __fns(mw[j], 0, take + 1)) - 1u)));
            a -= take;
        }
        if (W == 1) {
            // per-rank column sums with one ballot per rank
            int mine = 0;
            for (int g = 0; g < G && g < 32; ++g) {
                const unsigned b = __ballot_sync(kFull, (act[0] >> g) & 1u);
                if (lane == g) mine = __popc(b);
            }
            if (lane < G && mine) atomicAdd(&s_cnt[lane], mine);
        } else {
#pragma unroll
            for (int j = 0; j < W; ++j) {
                uint32_t bits = act[j];
                while (bits) {
                    const int b = __ffs(bits) - 1;
                    atomicAdd(&s_cnt[32 * j + b], 1);
                    bits &= bits - 1;
                }
            }
        }
    }
    __syncthreads();
    if (misc[M_NOREP] != INT32_MAX) return;
    if (writer) {
        if (tid < 32) {
            int mx = 0;
            for (int g = lane; g < G; g += 32) {
                p.rank_counts[g] = s_cnt[g];
                mx = max(mx, s_cnt[g]);
            }
            mx = __reduce_max_sync(kFull, mx);
            if (lane == 0) *p.lam = mx;
        }
        if (x) {
            // x[e][g] = base + (q < rem) on replicas, 0 elsewhere (routing.py:67-69)
            for (int idx = tid; idx < N * G; idx += kThreads) {
                const int e = idx / G, g = idx - e * G;
                const uint32_t w = s_mask[e * W + (g >> 5)];
                XT v = 0;
                if ((w >> (g & 31)) & 1u) {
                    const int64_t t = T64(e);
                    int r = 0, q = 0;
#pragma unroll
                    for (int j = 0; j < W; ++j) {
                        const uint32_t mj = s_mask[e * W + j];
                        r += __popc(mj);
                        if (j < (g >> 5)) q += __popc(mj);
                    }
                    q += __popc(w & ((1u << (g & 31)) - 1u));
                    const int64_t b = t / r, rem = t - b * r;
                    v = static_cast<XT>(b + (q < rem ? 1 : 0));
                }
                x[idx] = v;
            }
        }
    }
}

template <int W, bool PAIR>
__global__ void __launch_bounds__(kThreads, 1) eplb_ids_kernel(const Params p) {
    extern __shared__ __align__(128) unsigned char smem[];
    cluster_arrive_relaxed();
    const uint32_t R = cluster_nctarank(), rank = cluster_ctarank();
    const Layout L = make_layout(kEplbIds, p.N, W, R, p.slice, p.C, p.staged, PAIR);
    int32_t *misc = reinterpret_cast<int32_t *>(smem + L.misc);
    const int64_t beg = static_cast<int64_t>(rank) * p.slice;
    const int64_t rem_pairs = p.num_pairs - beg;
    const int n_local = rem_pairs <= 0 ? 0 : static_cast<int>(rem_pairs < p.slice ? rem_pairs : p.slice);
    init_misc(misc);
    zero_smem(smem, L.aux, L.part);  // rank counts + histogram
    stage_inputs<W>(p, L, smem, beg, n_local, p.staged != 0);
    if (!histogram_exchange<W, PAIR, true>(p, L, smem, beg, n_local, R, rank)) return;
    const bool writer = (rank == 0);
    const uint32_t *s_T = reinterpret_cast<const uint32_t *>(smem + L.T);
    eplb_counts_and_x<W>(p, L, smem, writer, [&](int e) { return static_cast<int64_t>(s_T[e]); }, p.x32);
    if (misc[M_NOREP] != INT32_MAX) {
        if (writer && threadIdx.x == 0) {
            p.status[0] = METRO_ERR_NO_REPLICA;
            p.status[1] = misc[M_NOREP];
            p.status[2] = p.status[3] = 0;
        }
        return;
    }
    if (PAIR && p.pair_rank) {
        // occurrence o of expert e (global row-major) -> replica (o mod r_e)
        const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, N = p.N;
        int32_t *s_hist = reinterpret_cast<int32_t *>(smem + L.hist);
        const uint32_t *s_mask = reinterpret_cast<const uint32_t *>(smem + L.mask);
        for (int e = tid; e < N; e += kThreads) {
            int run = static_cast<int>(s_T[N + e]);  // earlier CTAs
            for (int w = 0; w < kWarps; ++w) {
                const int c = s_hist[w * N + e];
                s_hist[w * N + e] = run;
                run += c;
            }
        }
        __syncthreads();
        const int32_t *src = p.staged ? reinterpret_cast<const int32_t *>(smem + L.ids) : (p.ids + beg);
        const int ws = align_up((n_local + kWarps - 1) / kWarps, 32);
        const int wb = min(n_local, warp * ws), we = min(n_local, wb + ws);
        int32_t *hw = s_hist + warp * N;
        for (int p0 = wb; p0 < we; p0 += 32) {
            const int i = p0 + lane;
            const int e = (i < we) ? src[i] : -1;
            const unsigned m = __match_any_sync(kFull, e);
            int o = 0;
            if (e >= 0) o = hw[e] + __popc(m & lanemask_lt());
            __syncwarp();
            if (e >= 0 && lane == __ffs(m) - 1) hw[e] += __popc(m);
            __syncwarp();
            if (e >= 0) {
                uint32_t mw[W];
                int r = 0;
#pragma unroll
                for (int j = 0; j < W; ++j) {
                    mw[j] = s_mask[e * W + j];
                    r += __popc(mw[j]);
                }
                p.pair_rank[beg + i] = nth_set_bit<W>(mw, o % r);
            }
        }
    }
    if (writer) {
        for (int e = threadIdx.x; e < p.N; e += kThreads)
            if (p.loads) p.loads[e] = static_cast<int32_t>(s_T[e]);
        if (threadIdx.x == 0) {
            p.status[0] = METRO_OK;
            p.status[1] = p.status[2] = 0;
            p.status[3] = static_cast<int32_t>(R);
        }
    }
}

template <int W>
__global__ void __launch_bounds__(kThreads, 1) eplb_loads_kernel(const Params p) {
    extern __shared__ __align__(128) unsigned char smem[];
    const Layout L = make_layout(kEplbLoads, p.N, W, 1, 0, 1, 0);
    int32_t *misc = reinterpret_cast<int32_t *>(smem + L.misc);
    init_misc(misc);
    zero_smem(smem, L.aux, L.hist);
    stage_inputs<W>(p, L, smem, 0, 0, false);
    eplb_counts_and_x<W>(p, L, smem, true, [&](int e) { return p.loads_in[e]; }, p.x64);
    if (threadIdx.x == 0) {
        if (misc[M_NOREP] != INT32_MAX) {
            p.status[0] = METRO_ERR_NO_REPLICA;
            p.status[1] = misc[M_NOREP];
        } else {
            p.status[0] = METRO_OK;
            p.status[1] = 0;
        }
        p.status[2] = 0;
        p.status[3] = 1;
    }
}

// ================================================================ host side
static thread_local int g_last_cuda_error = 0;
static int64_t *g_stamps = nullptr;

static int cuda_fail(cudaError_t e) {
    g_last_cuda_error = static_cast<int>(e);
    return METRO_ECUDA;
}

// One-time attribute setup per kernel (227 KB dynamic smem, 16-CTA clusters).
// Keyed by the kernel address: every instantiation has the same C++ type.
template <typename K>
static cudaError_t prepare(K kernel) {
    static std::mutex mu;
    static const void *done[256];
    static int done_dev[256];
    static int ndone = 0;
    const void *key = reinterpret_cast<const void *>(kernel);
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    for (int i = 0; i < ndone; ++i)
        if (done[i] == key && done_dev[i] == dev) return cudaSuccess;
    cudaError_t err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
    if (err == cudaSuccess)
        err = cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (err == cudaSuccess && ndone < 256) {
        done[ndone] = key;
        done_dev[ndone++] = dev;
    }
    return err;
}

template <typename K, typename... Args>
static int launch(K kernel, int R, int smem, cudaStream_t s, Args... args) {
    cudaError_t e = prepare(kernel);
    if (e != cudaSuccess) return cuda_fail(e);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(R, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = R;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kernel, args...);
    if (e != cudaSuccess) return cuda_fail(e);
    return METRO_OK;
}

static int words_for(int G) { return (G + 31) / 32; }
static int copies_for(int N) {
    int C = 32;
    while (C > 1 && N * C * 4 > 64 * 1024) C >>= 1;
    return C;
}
static int auto_cluster(int64_t num_pairs) {
    int R = 1;
    while (R < kMaxCluster && num_pairs > (int64_t)R * 1024) R <<= 1;
    return R;
}

static int check_dims(int N, int G) {
    if (N < 1 || N > kMaxN || G < 1 || G > kMaxG) return METRO_EDIMS;
    return METRO_OK;
}

// Choose cluster size R, staging and histogram copies for an ids-mode kernel so
// the layout fits 227 KB: prefer the requested / auto R, then a staged slice,
// then more histogram copies.  Returns smem bytes or an error code.
static int plan_ids(Kind kind, bool warp_hist, int64_t num_pairs, int N, int W, int requested,
                    Params &p, int &R) {
    int cands[8], nc = 0;
    if (requested > 0) {
        if (requested != 1 && requested != 2 && requested != 4 && requested != 8 && requested != 16)
            return METRO_EARG;
        cands[nc++] = requested;
    } else {
        for (int r = auto_cluster(num_pairs); r >= 1; r >>= 1) cands[nc++] = r;
    }
    for (int ci = 0; ci < nc; ++ci) {
        const int r = cands[ci];
        int64_t slice = (num_pairs + r - 1) / r;
        slice = (slice + 3) & ~int64_t(3);
        if (slice < 4) slice = 4;
        if (slice > INT32_MAX / 8) continue;
        for (int staged = 1; staged >= 0; --staged) {
            for (int C = copies_for(N); C >= 1; C >>= 1) {
                const Layout L = make_layout(kind, N, W, r, slice, C, staged, warp_hist);
                if (L.total <= kMaxSmem) {
                    p.slice = slice;
                    p.staged = staged;
                    p.C = C;
                    R = r;
                    return L.total;
                }
                if (warp_hist) break;  // C does not apply
            }
        }
    }
    return METRO_EDIMS;
}

}  // namespace metro

using namespace metro;

extern "C" {

int metro_abi_version(void) { return METRO_ABI_VERSION; }

const char *metro_strerror(int code) {
    switch (code) {
        case METRO_OK: return "ok";
        case METRO_ERR_ID_RANGE: return "expert id out of range";
        case METRO_ERR_NO_REPLICA: return "placement invariant: every expert has a replica";
        case METRO_ERR_LOAD_RANGE: return "load does not fit 32 bits on the device loads path";
        case METRO_EARG: return "invalid argument";
        case METRO_EDIMS: return "unsupported dimensions (1 <= G <= 128, 1 <= N <= 4096) or shared memory exceeded";
        case METRO_ECUDA: return "CUDA error";
        case METRO_ENOTBINARY: return "placement matrix must be binary";
        default: return "unknown error";
    }
}

int metro_last_cuda_error(void) { return g_last_cuda_error; }
int metro_mask_words(int32_t G) { return words_for(G); }
void metro_debug_set_stamps(int64_t *stamps) { g_stamps = stamps; }

int metro_pack_placement(const int8_t *A, int32_t N, int32_t G, uint32_t *mask) {
    if (!A || !mask || N < 0 || G < 0) return METRO_EARG;
    const int W = words_for(G > 0 ? G : 1);
    memset(mask, 0, sizeof(uint32_t) * (size_t)N * W);
    for (int i = 0; i < N; ++i)
        for (int g = 0; g < G; ++g) {
            const int8_t a = A[(int64_t)i * G + g];
            if (a != 0 && a != 1) return METRO_ENOTBINARY;
            if (a) mask[(int64_t)i * W + g / 32] |= 1u << (g % 32);
        }
    return METRO_OK;
}

#define METRO_DISPATCH_W(W, ...)                                  \
    switch (W) {                                                  \
        case 1: { constexpr int kW = 1; __VA_ARGS__; } break;     \
        case 2: { constexpr int kW = 2; __VA_ARGS__; } break;     \
        case 3: { constexpr int kW = 3; __VA_ARGS__; } break;     \
        case 4: { constexpr int kW = 4; __VA_ARGS__; } break;     \
        default: return METRO_EDIMS;                              \
    }

static int effective_w(int G) { return words_for(G); }

int metro_route_v1(const int32_t *ids, int64_t num_pairs, const uint32_t *mask, int32_t N,
                   int32_t G, int32_t *loads, int32_t *choice, int32_t *rank_counts, int32_t *lam,
                   int32_t *pair_rank, int32_t *status, int32_t cluster_ctas, void *stream) {
    if ((!ids && num_pairs > 0) || !mask || !choice || !rank_counts || !lam || !status || num_pairs < 0)
        return METRO_EARG;
    int rc = check_dims(N, G);
    if (rc) return rc;
    const int W = effective_w(G);
    Params p = {};
    p.ids = ids; p.num_pairs = num_pairs; p.mask = mask; p.N = N; p.G = G;
    p.loads = loads; p.choice = choice; p.rank_counts = rank_counts; p.lam = lam;
    p.pair_rank = pair_rank; p.status = status; p.stamps = g_stamps;
    int R = 1;
    const int smem = plan_ids(kMetroIds, false, num_pairs, N, W, cluster_ctas, p, R);
    if (smem < 0) return smem;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    METRO_DISPATCH_W(W, return launch(metro_ids_kernel<kW>, R, smem, s, p));
    return METRO_EDIMS;
}

int metro_aggregate_loads_v1(const int32_t *ids, int64_t num_pairs, int32_t N, int32_t *loads,
                             int32_t *status, int32_t cluster_ctas, void *stream) {
    if ((!ids && num_pairs > 0) || !loads || !status || num_pairs < 0) return METRO_EARG;
    if (N < 1 || N > kMaxN) return METRO_EDIMS;
    Params p = {};
    p.ids = ids; p.num_pairs = num_pairs; p.N = N; p.G = 1; p.loads = loads; p.status = status;
    p.stamps = g_stamps;
    int R = 1;
    const int smem = plan_ids(kMetroIds, false, num_pairs, N, 1, cluster_ctas, p, R);
    if (smem < 0) return smem;
    return launch(metro_ids_kernel<1>, R, smem, static_cast<cudaStream_t>(stream), p);
}

int metro_route_from_loads_v1(const int64_t *loads, const uint32_t *mask, int32_t N, int32_t G,
                              int32_t *choice, int32_t *rank_counts, int32_t *lam, int32_t *status,
                              void *stream) {
    if (!loads || !mask || !choice || !rank_counts || !lam || !status) return METRO_EARG;
    int rc = check_dims(N, G);
    if (rc) return rc;
    const int W = effective_w(G);
    Params p = {};
    p.loads_in = loads; p.mask = mask; p.N = N; p.G = G; p.choice = choice;
    p.rank_counts = rank_counts; p.lam = lam; p.status = status; p.C = 1;
    const int smem = make_layout(kMetroLoads, N, W, 1, 0, 1, 0).total;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    METRO_DISPATCH_W(W, return launch(metro_loads_kernel<kW>, 1, smem, s, p, 0));
    return METRO_EDIMS;
}

int metro_route_ordered_v1(const int32_t *order, int32_t m, const uint32_t *mask, int32_t N,
                           int32_t G, int32_t *choice, int32_t *rank_counts, int32_t *lam,
                           int32_t *status, void *stream) {
    if ((!order && m > 0) || m < 0 || m > N || !mask || !choice || !rank_counts || !lam || !status)
        return METRO_EARG;
    int rc = check_dims(N, G);
    if (rc) return rc;
    const int W = effective_w(G);
    Params p = {};
    p.order = order; p.order_len = m; p.mask = mask; p.N = N; p.G = G; p.choice = choice;
    p.rank_counts = rank_counts; p.lam = lam; p.status = status; p.C = 1;
    const int smem = make_layout(kMetroOrdered, N, W, 1, 0, 1, 0).total;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    METRO_DISPATCH_W(W, return launch(metro_loads_kernel<kW>, 1, smem, s, p, 1));
    return METRO_EDIMS;
}

int eplb_route_v1(const int32_t *ids, int64_t num_pairs, const uint32_t *mask, int32_t N,
                  int32_t G, int32_t *loads, int32_t *x, int32_t *rank_counts, int32_t *lam,
                  int32_t *pair_rank, int32_t *status, int32_t cluster_ctas, void *stream) {
    if ((!ids && num_pairs > 0) || !mask || !rank_counts || !lam || !status || num_pairs < 0)
        return METRO_EARG;
    int rc = check_dims(N, G);
    if (rc) return rc;
    const int W = effective_w(G);
    Params p = {};
    p.ids = ids; p.num_pairs = num_pairs; p.mask = mask; p.N = N; p.G = G; p.loads = loads;
    p.x32 = x; p.rank_counts = rank_counts; p.lam = lam; p.pair_rank = pair_rank; p.status = status;
    int R = 1;
    const int smem = plan_ids(kEplbIds, pair_rank != nullptr, num_pairs, N, W, cluster_ctas, p, R);
    if (smem < 0) return smem;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (pair_rank) {
        METRO_DISPATCH_W(W, return launch(eplb_ids_kernel<kW, true>, R, smem, s, p));
    } else {
        METRO_DISPATCH_W(W, return launch(eplb_ids_kernel<kW, false>, R, smem, s, p));
    }
    return METRO_EDIMS;
}

int eplb_route_from_loads_v1(const int64_t *loads, const uint32_t *mask, int32_t N, int32_t G,
                             int64_t *x, int32_t *rank_counts, int32_t *lam, int32_t *status,
                             void *stream) {
    if (!loads || !mask || !rank_counts || !lam || !status) return METRO_EARG;
    int rc = check_dims(N, G);
    if (rc) return rc;
    const int W = effective_w(G);
    Params p = {};
    p.loads_in = loads; p.mask = mask; p.N = N; p.G = G; p.x64 = x; p.rank_counts = rank_counts;
    p.lam = lam; p.status = status; p.C = 1;
    const int smem = make_layout(kEplbLoads, N, W, 1, 0, 1, 0).total;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    METRO_DISPATCH_W(W, return launch(eplb_loads_kernel<kW>, 1, smem, s, p));
    return METRO_EDIMS;
}

// ---- end-to-end from host buffers
// device workspace: [ids (num_pairs, 256-aligned)] [status 4 | lam 1 | pad 3 | counts G | choice N]
//                   [pair_rank num_pairs]
static size_t ws_ids_bytes(int64_t num_pairs) { return ((size_t)num_pairs * 4 + 255) & ~(size_t)255; }
static size_t ws_out_words(int N, int G) { return 8 + (size_t)G + (size_t)N; }

size_t metro_host_workspace_bytes(int64_t num_pairs, int32_t N, int32_t G) {
    return ws_ids_bytes(num_pairs) + ((ws_out_words(N, G) * 4 + 255) & ~(size_t)255) +
           (size_t)num_pairs * 4 + 256;
}

int metro_route_host_v1(const int32_t *ids_host, int64_t num_pairs, const uint32_t *mask_dev,
                        int32_t N, int32_t G, void *ws, int32_t *host_out, int32_t *pair_rank_host,
                        int32_t cluster_ctas, void *stream) {
    if (!ws || !host_out || !mask_dev || (num_pairs > 0 && !ids_host) || num_pairs < 0) return METRO_EARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    unsigned char *base = static_cast<unsigned char *>(ws);
    int32_t *d_ids = reinterpret_cast<int32_t *>(base);
    int32_t *d_out = reinterpret_cast<int32_t *>(base + ws_ids_bytes(num_pairs));
    int32_t *d_pr = reinterpret_cast<int32_t *>(reinterpret_cast<unsigned char *>(d_out) +
                                                ((ws_out_words(N, G) * 4 + 255) & ~(size_t)255));
    cudaError_t e;
    if (num_pairs > 0) {
        e = cudaMemcpyAsync(d_ids, ids_host, (size_t)num_pairs * 4, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return cuda_fail(e);
    }
    int rc = metro_route_v1(d_ids, num_pairs, mask_dev, N, G, nullptr, d_out + 8 + G, d_out + 8,
                            d_out + 4, pair_rank_host ? d_pr : nullptr, d_out, cluster_ctas, stream);
    if (rc) return rc;
    e = cudaMemcpyAsync(host_out, d_out, ws_out_words(N, G) * 4, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_fail(e);
    if (pair_rank_host && num_pairs > 0) {
        e = cudaMemcpyAsync(pair_rank_host, d_pr, (size_t)num_pairs * 4, cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) return cuda_fail(e);
    }
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e);
    return METRO_OK;
}

}  // extern "C"
