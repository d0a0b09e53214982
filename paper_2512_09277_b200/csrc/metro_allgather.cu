// metro_allgather.cu -- the global-knowledge step fused with METRO routing: one
// kernel per EP rank exchanges per-rank expert histograms (and optionally the
// top-k ids) through peer memory and routes (include/metro_exchange.h).
//
// Reference: the all-gather that gives every rank the global top-k knowledge
// (costmodel.py:102-129 ALL_GATHER, selected for the greedy
// routers at simulate.py:33, :69-70), then route_metro (routing.py:105-113) on
// the global loads T = aggregate_loads of the gathered batch (core.py:236-244).
// T is the sum of the ranks' local histograms, so the rows carry the same
// knowledge as the ids for every routing output.
//
// Exchange buffer of one rank (all offsets 16-byte aligned), LL protocol: every
// entry is an 8-byte {value, epoch of the call that wrote it} word, so readiness
// travels with the data (no flags, no fences; NCCL's LL idea):
//   [0, 128)   header: word 0 = calls completed on this rank (epoch)
//   rows[2][world][XR] u64   XR = N + 3 rounded to 2: counts, bad lo, bad hi, bad id
//   ids [2][world][max_local_pairs] u64  (only used when ids are gathered)
// [2] = call parity: a rank is at most one call ahead of its slowest peer (it
// cannot finish call t + 1 without every peer's row of t + 1, which a peer sends
// only after it finished reading call t's slot).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/metro_exchange.h"
#include "lib_internal.h"
#include "metro_core.cuh"

namespace metro {

constexpr int kMaxWorld = METRO_MAX_WORLD;
constexpr int kHdrBytes = 128;

// LL row entries per rank: N counts + bad lo / hi / id, rounded to 16 bytes
__host__ __device__ inline int xrow_words(int N) { return align_up(N + 3, 2); }
__host__ __device__ inline size_t x_rows_off() { return kHdrBytes; }
__host__ __device__ inline size_t x_ids_off(int N, int world) {
    return x_rows_off() + static_cast<size_t>(2) * world * xrow_words(N) * 8;
}
__host__ __device__ inline size_t x_bytes(int N, int world, int64_t max_local) {
    return (x_ids_off(N, world) + static_cast<size_t>(2) * world * static_cast<size_t>(max_local) * 8 + 127) &
           ~static_cast<size_t>(127);
}

struct XParams {
    Params p;  // ids = local ids, num_pairs = local pairs, slice = staged capacity
    unsigned char *peers[kMaxWorld];
    int32_t rank, world;
    int64_t max_local;
    int32_t *gathered;  // nullable [world * num_pairs]
    uint64_t timeout_ns;
    int64_t *stamps;    // debug: globaltimer ns per phase, [rank * 8 + phase]
};

// LL entries: {value (low 32), epoch (high 32)} as one 8-byte word, single-copy
// atomic at system scope (peer GPUs)
__device__ __forceinline__ uint64_t x_ld_ll(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void x_st_ll2(uint64_t *p, uint64_t a, uint64_t b) {
    asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void x_st_ll1(uint64_t *p, uint64_t a) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(a) : "memory");
}
__device__ __forceinline__ uint64_t x_now() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void xstamp(const struct XParams &x, int i);

// misc words of this kernel (beyond the routing ones, < 64)
enum { X_EPOCH = 40, X_TIMEOUT = 41, X_TAIL = 48 /* .. 55 */ };

__device__ __forceinline__ void xstamp(const XParams &x, int i) {
    if (x.stamps && threadIdx.x == 0) x.stamps[x.rank * 8 + i] = static_cast<int64_t>(x_now());
}

template <int W, bool LAYOUT = false>
__global__ void __launch_bounds__(kThreads, 1) metro_allgather_kernel(const XParams x) {
    extern __shared__ __align__(128) unsigned char smem[];
    const Params &p = x.p;
    const int tid = threadIdx.x, N = p.N, P = x.world, me = x.rank;
    const Layout L = make_layout(kMetroIds, N, W, P, p.slice, p.C, 1, false, 0, false, LAYOUT ? p.G : 0,
                                 LAYOUT ? p.nrep : 0);
    const int n_local = static_cast<int>(p.num_pairs);
    const int XR = xrow_words(N);
    unsigned char *own = x.peers[me];

    xstamp(x, 0);
    // ---- stage + count the local ids (metro_ids_kernel's phases A-B, one CTA)
    const StagePlan sp = stage_plan<W>(p, 0, n_local, true);
    // PDL: shared-memory prologue while the previous kernel finishes; no global
    // (or peer) access before griddep_wait
    int32_t *misc = reinterpret_cast<int32_t *>(smem + L.misc);
    init_misc(misc);
    zero_smem(smem, L.aux, L.part);
    if (LAYOUT) zero_smem(smem, L.lhw, L.locc);  // walk-warp counts + rows per replica
    griddep_wait();
    griddep_launch_dependents();  // only once this kernel runs: at most one dependent waits
    if (tid == 0) stage_issue(p, L, smem, 0, sp);
    // the dispatch layout's tables (as metro_ids_kernel<..., LAYOUT>): slot bases in a
    // register until after the exchange, the replica table by TMA when it can
    int32_t sb_reg = 0;
    if (LAYOUT) {
        if (!layout_rtab_bulk(p))
            for (int i = tid; i < N * p.G; i += kThreads)
                reinterpret_cast<int32_t *>(smem + L.lrtab)[i] = __ldg(p.rid_tab + i);
        if (tid <= p.G) sb_reg = __ldg(p.slot_base + tid);
    }
    stage_rest(p, L, smem, 0, n_local, true, sp);
    // (the threads that initialised these misc words: program order, no race)
    if (tid == X_EPOCH) misc[X_EPOCH] = static_cast<int32_t>(*reinterpret_cast<volatile uint32_t *>(own) + 1u);
    if (tid == X_TIMEOUT) misc[X_TIMEOUT] = INT32_MAX;
    cta_sync();
    mbar_wait(reinterpret_cast<uint64_t *>(smem + L.mbar), 0);
    histogram_push<false>(p, L, smem, 0, n_local, 1, 0);  // s_part row 0 = local counts
    cta_sync();
    const uint32_t epoch = static_cast<uint32_t>(misc[X_EPOCH]);
    const int par = epoch & 1;
    int32_t *s_part = reinterpret_cast<int32_t *>(smem + L.part);
    const int32_t *s_ids = reinterpret_cast<const int32_t *>(smem + L.ids);

    // the outgoing row: counts, then this rank's first bad pair as a GLOBAL
    // (rank-major) pair index + its id in the tail words [N, XR) (misc[X_TAIL..])
    int32_t *row0 = s_part;
    const int32_t *xtail = misc + X_TAIL;
    if (tid == 0) {
        const uint32_t lo = static_cast<uint32_t>(misc[M_BAD_LO]), hi = static_cast<uint32_t>(misc[M_BAD_HI]);
        const bool bad = lo != kBadLo || hi != kBadHi;
        const int64_t lb = join64(lo, hi);
        const int64_t gb = bad ? static_cast<int64_t>(me) * n_local + lb : kNoBad;
        misc[X_TAIL + 0] = static_cast<int32_t>(static_cast<uint64_t>(gb) & 0xffffffffu);
        misc[X_TAIL + 1] = static_cast<int32_t>(static_cast<uint64_t>(gb) >> 32);
        misc[X_TAIL + 2] = bad ? s_ids[lb] : 0;
        for (int j = 3; j < 8; ++j) misc[X_TAIL + j] = 0;
    }
    cta_sync();

    xstamp(x, 1);
    // ---- push (LL protocol: every 8-byte entry is {value, epoch}, stored single-copy
    // atomic, so a receiver that sees this call's epoch in an entry has its value:
    // no fence, no flag round trip).  Row entries: N counts + bad lo / hi / id.
    const uint64_t tag = static_cast<uint64_t>(epoch) << 32;
    const int XU = N + 3;  // entries in use per row
    if (P > 1) {
        const int nv = XR / 2;  // 16-byte pieces (two entries) per row
        for (int idx = tid; idx < (P - 1) * nv; idx += kThreads) {
            const int q = (me + 1 + idx / nv) % P;
            const int v = idx % nv, e0 = 2 * v;
            const uint32_t a0 = static_cast<uint32_t>(e0 < N ? row0[e0] : xtail[e0 - N]);
            const uint32_t a1 = static_cast<uint32_t>(e0 + 1 < N ? row0[e0 + 1] : xtail[e0 + 1 - N]);
            uint64_t *dst = reinterpret_cast<uint64_t *>(x.peers[q] + x_rows_off()) + (par * P + me) * XR;
            x_st_ll2(dst + e0, tag | a0, tag | a1);
        }
        if (x.gathered) {
            const int n2 = n_local >> 1;
            for (int idx = tid; idx < (P - 1) * n2; idx += kThreads) {
                const int q = (me + 1 + idx / n2) % P;
                const int v = idx % n2;
                uint64_t *dst = reinterpret_cast<uint64_t *>(x.peers[q] + x_ids_off(N, P)) + (par * P + me) * x.max_local;
                x_st_ll2(dst + 2 * v, tag | static_cast<uint32_t>(s_ids[2 * v]),
                         tag | static_cast<uint32_t>(s_ids[2 * v + 1]));
            }
            if ((n_local & 1) && tid < P && tid != me)
                x_st_ll1(reinterpret_cast<uint64_t *>(x.peers[tid] + x_ids_off(N, P)) + (par * P + me) * x.max_local +
                             (n_local - 1),
                         tag | static_cast<uint32_t>(s_ids[n_local - 1]));
        }
    }
    if (x.gathered) {  // own slice of the gathered batch
        for (int i = tid; i < n_local; i += kThreads) x.gathered[static_cast<int64_t>(me) * n_local + i] = s_ids[i];
    }

    xstamp(x, 2);
    // ---- receive: poll this call's P - 1 rows in the own buffer (bounded) straight
    // into s_part rows 1..P-1 (any order: only the sum matters); the bad words go to
    // the rows' tail words N, N + 1 (metro_decide's layout), the bad id stays put
    if (P > 1) {
        const uint64_t *xin = reinterpret_cast<const uint64_t *>(own + x_rows_off()) + par * P * XR;
        const uint64_t t0 = x_now();
        bool late = false;
        // U independent loads per thread in flight, then each entry is checked (and
        // re-polled only if its writer has not landed yet): one L2 round trip per
        // batch instead of one per entry
        auto poll = [&](int total, auto addr, auto consume) {
            constexpr int U = 8;
            for (int base = tid; base < total && !late; base += kThreads * U) {
                uint32_t pending = 0;
#pragma unroll
                for (int u = 0; u < U; ++u) pending |= (base + u * kThreads < total ? 1u : 0u) << u;
                uint64_t v[U];
                while (pending) {
                    // every still-pending entry's load in flight at once, then check all
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if ((pending >> u) & 1u) v[u] = x_ld_ll(addr(base + u * kThreads));
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (((pending >> u) & 1u) && (v[u] >> 32) == epoch) {
                            consume(base + u * kThreads, static_cast<int32_t>(v[u]));
                            pending &= ~(1u << u);
                        }
                    if (pending && x_now() - t0 > x.timeout_ns) {
                        const int idx = base + (__ffs(pending) - 1) * kThreads;
                        atomicMin(&misc[X_TIMEOUT], (me + 1 + idx / (total / (P - 1))) % P);
                        late = true;
                        break;
                    }
                }
            }
        };
        poll((P - 1) * XU,
             [&](int idx) {
                 const int j = idx / XU, e = idx - j * XU;
                 return xin + ((me + 1 + j) % P) * XR + e;
             },
             [&](int idx, int32_t val) {
                 const int j = idx / XU, e = idx - j * XU;
                 if (e < N + 2) s_part[(j + 1) * L.NP + e] = val;
             });
        if (x.gathered) {
            const uint64_t *xids = reinterpret_cast<const uint64_t *>(own + x_ids_off(N, P)) + par * P * x.max_local;
            poll((P - 1) * n_local,
                 [&](int idx) {
                     const int j = idx / n_local, t = idx - j * n_local;
                     return xids + ((me + 1 + j) % P) * x.max_local + t;
                 },
                 [&](int idx, int32_t val) {
                     const int j = idx / n_local, t = idx - j * n_local;
                     x.gathered[static_cast<int64_t>((me + 1 + j) % P) * n_local + t] = val;
                 });
        }
    }
    cta_sync();
    if (misc[X_TIMEOUT] != INT32_MAX) {
        if (tid == 0) {
            p.status[0] = METRO_ERR_PEER_TIMEOUT;
            p.status[1] = misc[X_TIMEOUT];
            p.status[2] = p.status[3] = 0;
        }
        return;  // the epoch is not advanced: the call did not complete
    }

    // ---- the global first bad pair over all ranks (identical on every rank)
    if (tid < 32) {
        const int lane = tid;
        uint32_t lo = kBadLo, hi = kBadHi;
        if (lane == 0) {
            lo = static_cast<uint32_t>(xtail[0]);
            hi = static_cast<uint32_t>(xtail[1]);
        } else if (lane < P) {
            lo = static_cast<uint32_t>(s_part[lane * L.NP + N]);
            hi = static_cast<uint32_t>(s_part[lane * L.NP + N + 1]);
        }
        if (__any_sync(kFull, lo != kBadLo || hi != kBadHi)) {
            const uint32_t mhi = __reduce_min_sync(kFull, hi);
            const uint32_t mlo = __reduce_min_sync(kFull, hi == mhi ? lo : 0xffffffffu);
            const unsigned who = __ballot_sync(kFull, lo == mlo && hi == mhi && lane < P);
            if (lane == 0) {
                const int j = __ffs(who) - 1;  // s_part row: 0 = own, j = rank (me + j) % P
                const int src = (me + j) % P;
                const uint64_t *xin = reinterpret_cast<const uint64_t *>(own + x_rows_off()) + par * P * XR;
                p.status[0] = METRO_ERR_ID_RANGE;
                p.status[1] = static_cast<int32_t>(mlo);
                p.status[2] = static_cast<int32_t>(mhi);
                p.status[3] = j == 0 ? xtail[2] : static_cast<int32_t>(x_ld_ll(xin + src * XR + N + 2));
                misc[M_BADALL_LO] = 0;  // any value != kBadLo: error seen
            }
        }
    }
    if (tid == 0) {
        *reinterpret_cast<volatile uint32_t *>(own) = epoch;  // this call's exchange is complete
        misc[M_BAD_LO] = static_cast<int32_t>(kBadLo);   // errors are handled above
        misc[M_BAD_HI] = static_cast<int32_t>(kBadHi);
    }
    cta_sync();
    if (misc[M_BADALL_LO] != static_cast<int32_t>(kBadLo)) return;
    for (int j = 1 + tid; j < P; j += kThreads) {  // no bad words left for metro_decide's check
        s_part[j * L.NP + N] = static_cast<int32_t>(kBadLo);
        s_part[j * L.NP + N + 1] = static_cast<int32_t>(kBadHi);
    }
    cta_sync();
    xstamp(x, 3);

    // ---- the METRO decision over T = sum of the P rows (identical on every rank)
    if (LAYOUT) {
        // this rank's pairs follow the earlier ranks' in the global (rank-major)
        // order: their occurrences come first.  s_part row j holds rank (me + j) % P.
        if (tid <= p.G) reinterpret_cast<int32_t *>(smem + L.lsb)[tid] = sb_reg;
        int32_t *s_pre = reinterpret_cast<int32_t *>(smem + L.lpre);
        for (int e = tid; e < N; e += kThreads) {
            int32_t pre = 0;
            for (int j = P - me; j < P; ++j) pre += s_part[j * L.NP + e];
            s_pre[e] = pre;
        }
        const int ws = align_up((n_local + kLayWarps - 1) / kLayWarps, 32);
        if (!metro_decide<W, kFromIds>(p, L, smem, true, static_cast<uint32_t>(P), 0,
                                       LayoutWalk{&L, smem, n_local, N, ws, nullptr, 0}))
            return;
        xstamp(x, 4);
        layout_tail<W>(p, L, smem, 0, n_local, ws, true, P);
        xstamp(x, 5);
        return;
    }
    if (!metro_decide<W, kFromIds>(p, L, smem, true, static_cast<uint32_t>(P), 0)) return;
    xstamp(x, 4);
    const int32_t *s_choice = reinterpret_cast<const int32_t *>(smem + L.choice);
    if (p.pair_rank) {
        const int n4 = n_local >> 2;
        const bool vec = (reinterpret_cast<uintptr_t>(p.pair_rank) & 15) == 0;
        if (vec)
            for (int i = tid; i < n4; i += kThreads) {
                const int4 v = reinterpret_cast<const int4 *>(s_ids)[i];
                reinterpret_cast<int4 *>(p.pair_rank)[i] =
                    make_int4(s_choice[v.x], s_choice[v.y], s_choice[v.z], s_choice[v.w]);
            }
        for (int i = (vec ? 4 * n4 : 0) + tid; i < n_local; i += kThreads) p.pair_rank[i] = s_choice[s_ids[i]];
    }
    const uint32_t *s_T = reinterpret_cast<const uint32_t *>(smem + L.T);
    for (int e = tid; e < N; e += kThreads) {
        if (p.loads) p.loads[e] = static_cast<int32_t>(s_T[e]);
        p.choice[e] = s_choice[e];
    }
    if (tid == 0) {
        p.status[0] = METRO_OK;
        p.status[1] = p.status[2] = 0;
        p.status[3] = P;
    }
    xstamp(x, 5);
}

template <int W, bool LAYOUT>
static int x_launch(const XParams &x, int smem, cudaStream_t s) {
    static bool done[kMaxWorld] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < kMaxWorld && !done[dev]) {
        cudaError_t e = cudaFuncSetAttribute(metro_allgather_kernel<W, LAYOUT>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
        if (e != cudaSuccess) return cuda_fail(e);
        done[dev] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // griddep_wait before global access
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, metro_allgather_kernel<W, LAYOUT>, x);
    return e == cudaSuccess ? METRO_OK : cuda_fail(e);
}

}  // namespace metro

using namespace metro;

static int64_t *g_x_stamps = nullptr;

extern "C" {

void metro_allgather_debug_stamps(int64_t *dev_stamps) { g_x_stamps = dev_stamps; }

size_t metro_exchange_bytes(int32_t N, int32_t world, int64_t max_local_pairs) {
    if (N < 1 || world < 1 || world > kMaxWorld || max_local_pairs < 0) return 0;
    return x_bytes(N, world, max_local_pairs);
}

}  // extern "C"

static int allgather_route(const int32_t *local_ids, int64_t local_pairs, int32_t rank, int32_t world,
                           void *const *peer_exchange, int64_t max_local_pairs, const uint32_t *mask, int32_t N,
                           int32_t G, int32_t *loads, int32_t *choice, int32_t *rank_counts, int32_t *lam,
                           int32_t *local_pair_rank, int32_t *gathered_ids, int32_t *status, void *stream,
                           const int32_t *rid_tab, const int32_t *slot_base, int32_t nrep, int32_t *pair_row,
                           int32_t *rep_off) {
    if ((!local_ids && local_pairs > 0) || local_pairs < 0 || !peer_exchange || !mask || !choice || !rank_counts ||
        !lam || !status || world < 1 || world > kMaxWorld || rank < 0 || rank >= world)
        return METRO_EARG;
    const bool layout = nrep > 0;
    if (layout && (!rid_tab || !slot_base || !rep_off || nrep > 4096 ||
                   (local_pairs > 0 && (!local_pair_rank || !pair_row))))
        return METRO_EARG;
    if (N < 1 || N > kMaxN || G < 1 || G > kMaxG) return METRO_EDIMS;
    if (gathered_ids && (local_pairs > max_local_pairs || (max_local_pairs & 3))) return METRO_EARG;
    XParams x = {};
    for (int q = 0; q < world; ++q) {
        x.peers[q] = static_cast<unsigned char *>(peer_exchange[q]);
        if (!x.peers[q] || (reinterpret_cast<uintptr_t>(x.peers[q]) & 127)) return METRO_EARG;
    }
    x.rank = rank;
    x.world = world;
    x.max_local = max_local_pairs;
    x.gathered = gathered_ids;
    x.stamps = g_x_stamps;
    {
        const char *t = getenv("METRO_PEER_TIMEOUT_MS");
        const long ms = t ? atol(t) : 5000;
        x.timeout_ns = static_cast<uint64_t>(ms > 0 ? ms : 5000) * 1000000ull;
    }
    Params &p = x.p;
    p.ids = local_ids;
    p.num_pairs = local_pairs;
    p.mask = mask;
    p.N = N;
    p.G = G;
    p.loads = loads;
    p.choice = choice;
    p.rank_counts = rank_counts;
    p.lam = lam;
    p.pair_rank = local_pair_rank;
    p.status = status;
    p.staged = 1;
    if (layout) {
        p.rid_tab = rid_tab; p.slot_base = slot_base; p.nrep = nrep; p.pair_row = pair_row; p.rep_off = rep_off;
    }
    int64_t slice = (local_pairs + 3) & ~int64_t(3);
    if (slice < 4) slice = 4;
    p.slice = slice;
    const int W = (G + 31) / 32;
    int smem = -1;
    // lane-striped histogram copies: 32 for large slices; a rank's slice is small
    // (B / P tokens), where zeroing + summing 32 copies per expert costs more than
    // the atomic conflicts 8 copies leave
    const int c0 = local_pairs > 2048 ? 32 : 8;
    for (int C = c0; C >= 1; C >>= 1) {
        if (C > 1 && N * C * 4 > 64 * 1024) continue;
        const Layout L = make_layout(kMetroIds, N, W, world, slice, C, 1, false, 0, false, layout ? G : 0,
                                     layout ? nrep : 0);
        if (L.total <= kMaxSmem && (!layout || slice <= 65535)) {
            p.C = C;
            smem = L.total;
            break;
        }
    }
    if (smem < 0) return METRO_EDIMS;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (layout) {
        switch (W) {
            case 1: return x_launch<1, true>(x, smem, s);
            case 2: return x_launch<2, true>(x, smem, s);
            case 3: return x_launch<3, true>(x, smem, s);
            case 4: return x_launch<4, true>(x, smem, s);
            default: return METRO_EDIMS;
        }
    }
    switch (W) {
        case 1: return x_launch<1, false>(x, smem, s);
        case 2: return x_launch<2, false>(x, smem, s);
        case 3: return x_launch<3, false>(x, smem, s);
        case 4: return x_launch<4, false>(x, smem, s);
        default: return METRO_EDIMS;
    }
}

extern "C" {

int metro_allgather_route_v1(const int32_t *local_ids, int64_t local_pairs, int32_t rank, int32_t world,
                             void *const *peer_exchange, int64_t max_local_pairs, const uint32_t *mask, int32_t N,
                             int32_t G, int32_t *loads, int32_t *choice, int32_t *rank_counts, int32_t *lam,
                             int32_t *local_pair_rank, int32_t *gathered_ids, int32_t *status, void *stream) {
    return allgather_route(local_ids, local_pairs, rank, world, peer_exchange, max_local_pairs, mask, N, G, loads,
                           choice, rank_counts, lam, local_pair_rank, gathered_ids, status, stream, nullptr, nullptr,
                           0, nullptr, nullptr);
}

int metro_allgather_route_layout_v1(const int32_t *local_ids, int64_t local_pairs, int32_t rank, int32_t world,
                                    void *const *peer_exchange, int64_t max_local_pairs, const uint32_t *mask,
                                    int32_t N, int32_t G, const int32_t *rid_tab, const int32_t *slot_base,
                                    int32_t nrep, int32_t *loads, int32_t *choice, int32_t *rank_counts,
                                    int32_t *lam, int32_t *local_pair_rank, int32_t *local_pair_row,
                                    int32_t *rep_off, int32_t *status, void *stream) {
    if (nrep < 1) return METRO_EDIMS;
    return allgather_route(local_ids, local_pairs, rank, world, peer_exchange, max_local_pairs, mask, N, G, loads,
                           choice, rank_counts, lam, local_pair_rank, nullptr, status, stream, rid_tab, slot_base,
                           nrep, local_pair_row, rep_off);
}

int metro_exchange_alloc(size_t bytes, void **dev_ptr_out) {
    if (!dev_ptr_out || bytes == 0) return METRO_EARG;
    *dev_ptr_out = nullptr;
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);  // its own allocation: an IPC handle maps exactly it
    if (e != cudaSuccess) return cuda_fail(e);
    // zeroed on a private stream (no device-wide synchronise: a resident router
    // CTA elsewhere in the process would hold it up)
    cudaStream_t zs = nullptr;
    e = cudaStreamCreateWithFlags(&zs, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMemsetAsync(p, 0, bytes, zs);
    if (e == cudaSuccess) e = cudaStreamSynchronize(zs);
    if (zs) cudaStreamDestroy(zs);
    if (e != cudaSuccess) {
        cudaFree(p);
        return cuda_fail(e);
    }
    *dev_ptr_out = p;
    return METRO_OK;
}

int metro_exchange_free(void *dev_ptr) {
    if (!dev_ptr) return METRO_OK;
    cudaError_t e = cudaFree(dev_ptr);
    return e == cudaSuccess ? METRO_OK : cuda_fail(e);
}

int metro_ipc_get_handle(void *dev_ptr, void *handle_out64) {
    if (!dev_ptr || !handle_out64) return METRO_EARG;
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, dev_ptr);
    if (e != cudaSuccess) return cuda_fail(e);
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    memcpy(handle_out64, &h, sizeof(h));
    return METRO_OK;
}

int metro_ipc_open_handle(const void *handle64, void **dev_ptr_out) {
    if (!handle64 || !dev_ptr_out) return METRO_EARG;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, sizeof(h));
    cudaError_t e = cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
    return e == cudaSuccess ? METRO_OK : cuda_fail(e);
}

int metro_ipc_close_handle(void *dev_ptr) {
    if (!dev_ptr) return METRO_EARG;
    cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
    return e == cudaSuccess ? METRO_OK : cuda_fail(e);
}

}  // extern "C"
