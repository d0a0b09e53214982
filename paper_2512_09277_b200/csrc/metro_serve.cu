// metro_serve.cu -- persistent end-to-end METRO router for host callers
// (include/metro_serve.h).
//
// One resident CTA per server: 16 routing warps + 1-4 doorbell warps.  Lane 0 of
// each doorbell warp keeps one system-scope acquire load of the doorbell word
// (pinned host memory) in flight, the warps staggered; the first to see a new
// request claims it and arrives on a named barrier the routing warps wait on.
// The routing warps then run the phases of one metro_ids_kernel launch with
// R = 1 (metro_core.cuh): the ids are read from host memory with system-scope
// 16-byte loads and counted into the lane-striped histogram as they arrive,
// METRO decision (routing.py:105-113: order by (r asc, T desc, id asc), greedy
// argmin with the ascending strict-'<' scan) -> per-pair ranks, results stored
// into the caller's pinned buffers, and thread 0 publishes the completion word
// with a system-scope release store (cumulative over the CTA barrier).  No
// kernel launch and no stream synchronisation on the per-call path: the launch
// + sync floor of the one-launch path (~9 us measured on the B200 box,
// tools/host_latency.cu) is replaced by two PCIe round trips.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "../../include/metro_serve.h"
#include "lib_internal.h"
#include "metro_core.cuh"

namespace metro {

// Control block in pinned, device-mapped host memory.  The host owns the first
// line (doorbell + buffer addresses) and `stop`; the device owns the second
// (completion word, state) and the third (per-phase timestamps of the last
// request).  Separate 64-byte lines so neither side's writes disturb the
// other's polling.
//
// Doorbell word (one 8-byte store / load, so a request is seen whole):
//   bits  0..23  request sequence number (mod 2^24)
//   bit  24      the buffer addresses changed (the device re-reads them)
//   bits 32..63  num_pairs
struct alignas(64) ServeCtl {
    uint64_t doorbell;
    uint64_t ids, pair_rank, out;  // device-visible addresses of the caller's buffers
    uint32_t stop;
    uint32_t pad0[7];
    alignas(64) uint32_t done;   // sequence number of the newest completed request
    uint32_t state;              // kServeLaunched / kServeIdleExit / kServeStopped
    uint32_t pad1[14];
    alignas(64) int64_t stamps[8];  // globaltimer ns at the phases of the last request, + SM clocks
};
static_assert(sizeof(ServeCtl) == 192, "control block layout");
constexpr uint32_t kSeqMask = 0xffffffu, kNewPtrs = 1u << 24;

enum : uint32_t { kServeLaunched = 1, kServeIdleExit = 2, kServeStopped = 3 };

__device__ __forceinline__ uint32_t ld_relaxed_sys(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t ld_acquire_sys64(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_sys64(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int4 ld_relaxed_sys_v4(const int4 *p) {
    int4 v;
    asm volatile("ld.relaxed.sys.global.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
__device__ __forceinline__ int ld_relaxed_sys_s32(const int32_t *p) {
    int v;
    asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// shared words of the request loop (outside the routing layout)
struct ServeReq {
    uint32_t seq, verdict;  // verdict: 0 serve, 1 stop, 2 idle exit
    uint32_t new_ptrs, go;  // go: epoch of the last request a doorbell warp claimed (CAS)
    uint32_t ready, pad;    // ready: epoch of the last request whose words are filled
    const int32_t *ids;
    int32_t *pair_rank, *out;
    int64_t num_pairs;
    uint64_t t_seen;
    int64_t c_seen;
    int64_t rtt;  // duration of the doorbell load that saw the request (ns)
};

// Thread roles.  Warps 0..15 (kThreads) route, with the named barrier 1 of
// metro_core.cuh (cta_sync).  Warps 16.. (1-4 of them, default 2) only poll: lane 0
// of each keeps one system-scope acquire load of the doorbell in flight, the
// warps started `stagger` ns apart, so a doorbell load reaches host memory every
// ~RTT / (doorbell warps).  The first to see a new request claims it and arrives
// on barrier 2 (the routing warps sync on it): the routing warps never wait for
// the other pollers' loads still in flight.  Barrier 3 (everyone) closes a
// request.  Acquire loads + barrier give the formal order: the routing warps'
// id loads happen after the doorbell load that saw the request.
constexpr int kMaxDoorbellWarps = 4;
constexpr int kServeThreads = kThreads + 32 * kMaxDoorbellWarps;  // launch bound; the launch may use fewer
enum FenceMode { kFenceRelease = 0, kFenceOne = 1, kFenceAll = 2 };

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int W>
__global__ void __launch_bounds__(kServeThreads, 1)
    metro_serve_kernel(const Params base, ServeCtl *ctl, uint32_t seq, uint64_t idle_ns, int fence_mode,
                       uint32_t stagger, int32_t *scratch) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31;
    const Layout L = make_layout(kMetroIds, base.N, W, 1, base.slice, base.C, base.staged, false, 0,
                                 base.private_scratch != 0);
    const bool staged = base.staged != 0;
    ServeReq &rq = *reinterpret_cast<ServeReq *>(smem + align_up(L.total, 16));

    const int nthreads = static_cast<int>(blockDim.x);  // kThreads + 32 x doorbell warps
    if (tid >= kThreads) {
        // ================= doorbell warps
        const int d = (tid - kThreads) >> 5;
        volatile ServeReq &vrq = rq;
        uint64_t t_wait = globaltimer_ns();
        for (uint32_t epoch = 1;; ++epoch) {
            bar_sync(3, nthreads);  // the previous request is closed
            int won = 0;
            if (lane == 0) {
                if (d) __nanosleep(d * stagger);
                uint32_t it = 0;
                for (;;) {
                    const uint64_t t0 = globaltimer_ns();
                    const uint64_t v = ld_acquire_sys64(&ctl->doorbell);
                    if (vrq.go == epoch) break;
                    uint32_t verdict = 0;
                    if ((static_cast<uint32_t>(v) & kSeqMask) == seq) {
                        if (d != 0 || (++it & 15) != 0) continue;
                        verdict = ld_relaxed_sys(&ctl->stop) ? 1u : (t0 - t_wait > idle_ns ? 2u : 0u);
                        if (!verdict) continue;
                    }
                    if (atomicCAS(&rq.go, epoch - 1, epoch) != epoch - 1) break;
                    won = 1;
                    const uint64_t t1 = globaltimer_ns();
                    rq.verdict = verdict;
                    rq.t_seen = t1;
                    rq.c_seen = clock64();
                    rq.rtt = static_cast<int64_t>(t1 - t0);
                    if (!verdict) {
                        rq.seq = static_cast<uint32_t>(v) & kSeqMask;
                        rq.num_pairs = static_cast<int64_t>(v >> 32);
                        rq.new_ptrs = (static_cast<uint32_t>(v) & kNewPtrs) ? 1u : 0u;
                        if (rq.new_ptrs) {
                            rq.ids = reinterpret_cast<const int32_t *>(ld_relaxed_sys64(&ctl->ids));
                            rq.pair_rank = reinterpret_cast<int32_t *>(ld_relaxed_sys64(&ctl->pair_rank));
                            rq.out = reinterpret_cast<int32_t *>(ld_relaxed_sys64(&ctl->out));
                        }
                    }
                    __threadfence_block();
                    vrq.ready = epoch;
                    break;
                }
            }
            won = __shfl_sync(kFull, won, 0);
            if (won) bar_arrive(2, kThreads + 32);
            // every doorbell warp learns the outcome from the claimer
            if (lane == 0)
                while (vrq.ready != epoch) {
                }
            __syncwarp();
            if (vrq.verdict) return;
            seq = vrq.seq;
            t_wait = globaltimer_ns();
        }
    }

    // ================= routing warps
    // the rank masks stay in shared memory for the life of this launch (the layout
    // never overlays L.mask)
    uint32_t *s_mask = reinterpret_cast<uint32_t *>(smem + L.mask);
    for (int i = tid; i < base.N * W; i += kThreads) s_mask[i] = __ldg(base.mask + i);
    // buffer addresses of the last request (a relaunch after an idle exit picks
    // them up here: the host wrote them before any doorbell that used them)
    if (tid == 0) {
        rq.ids = reinterpret_cast<const int32_t *>(ld_relaxed_sys64(&ctl->ids));
        rq.pair_rank = reinterpret_cast<int32_t *>(ld_relaxed_sys64(&ctl->pair_rank));
        rq.out = reinterpret_cast<int32_t *>(ld_relaxed_sys64(&ctl->out));
        rq.go = rq.ready = 0;
    }
    cta_sync();
    const int32_t *ids = rq.ids;
    int32_t *pair_rank = rq.pair_rank, *out = rq.out;
    int32_t *misc = reinterpret_cast<int32_t *>(smem + L.misc);
    int32_t *s_ids = reinterpret_cast<int32_t *>(smem + L.ids);
    int32_t *s_hist = reinterpret_cast<int32_t *>(smem + L.hist);
    const int cm = base.C - 1;

    for (;;) {
        // ---- per-request state, cleared before the doorbell warps are released
        init_misc(misc);
        zero_smem(smem, L.aux, L.part);  // forced counts + histogram
        bar_sync(3, nthreads);
        bar_sync(2, kThreads + 32);  // a doorbell warp claimed a request (or stop / idle)
        if (rq.verdict) {
            if (tid == 0) st_release_sys(&ctl->state, rq.verdict == 1 ? kServeStopped : kServeIdleExit);
            return;
        }
        if (rq.new_ptrs) {
            ids = rq.ids;
            pair_rank = rq.pair_rank;
            out = rq.out;
        }
        const uint32_t rseq = rq.seq;
        Params p = base;
        p.ids = ids;
        p.num_pairs = rq.num_pairs;
        p.pair_rank = pair_rank;
        p.status = out;
        p.lam = out + 4;
        p.rank_counts = out + 8;
        p.choice = out + 8 + p.G;
        p.loads = nullptr;
        const int n = static_cast<int>(p.num_pairs);

        // ---- stage the ids from host memory (zero-copy, system scope: never a
        // stale line from an earlier request in the same buffer), counting each
        // 16-byte group into the lane-striped histogram as it arrives
        {
            int64_t my_bad = kNoBad;
            const int n4 = n >> 2;
            const int4 *src4 = reinterpret_cast<const int4 *>(p.ids);
            constexpr int U = 4;  // four 16-byte loads in flight per thread
            for (int i0 = tid; i0 < n4; i0 += kThreads * U) {
                int4 v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = i0 + u * kThreads;
                    v[u] = i < n4 ? ld_relaxed_sys_v4(src4 + i) : make_int4(0, 0, 0, 0);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = i0 + u * kThreads;
                    if (i < n4) {
                        if (staged) reinterpret_cast<int4 *>(s_ids)[i] = v[u];
                        else reinterpret_cast<int4 *>(scratch)[i] = v[u];  // HBM copy for the second pass
                        const int ev[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            if (static_cast<unsigned>(ev[q]) < static_cast<unsigned>(p.N))
                                atomicAdd(&s_hist[ev[q] * p.C + (lane & cm)], 1);
                            else
                                my_bad = min(my_bad, static_cast<int64_t>(4 * i + q));
                        }
                    }
                }
            }
            for (int i = n4 * 4 + tid; i < n; i += kThreads) {
                const int e = ld_relaxed_sys_s32(p.ids + i);
                if (staged) s_ids[i] = e;
                else scratch[i] = e;
                if (static_cast<unsigned>(e) < static_cast<unsigned>(p.N))
                    atomicAdd(&s_hist[e * p.C + (lane & cm)], 1);
                else
                    my_bad = min(my_bad, static_cast<int64_t>(i));
            }
            if (my_bad != kNoBad)
                atomicMin(reinterpret_cast<unsigned long long *>(&misc[M_BAD_LO]),
                          static_cast<unsigned long long>(my_bad));
        }
        const uint64_t t_staged = globaltimer_ns();

        // ---- route: the phases of metro_ids_kernel with one CTA (the histogram is
        // already counted: row sums, then the METRO decision)
        histogram_push<false, false>(p, L, smem, 0, n, 1, 0);
        const bool ok = metro_decide<W, kFromIds>(p, L, smem, true, 1, 0);
        const uint64_t t_routed = globaltimer_ns();
        if (ok) {
            const int32_t *s_choice = reinterpret_cast<const int32_t *>(smem + L.choice);
            if (p.pair_rank) {
                const int n4 = n >> 2;
                const int4 *src4 = reinterpret_cast<const int4 *>(p.ids);
                for (int i = tid; i < n4; i += kThreads) {
                    const int4 v = staged ? reinterpret_cast<const int4 *>(s_ids)[i]
                                          : reinterpret_cast<const int4 *>(scratch)[i];
                    reinterpret_cast<int4 *>(p.pair_rank)[i] =
                        make_int4(s_choice[v.x], s_choice[v.y], s_choice[v.z], s_choice[v.w]);
                }
                for (int i = n4 * 4 + tid; i < n; i += kThreads)
                    p.pair_rank[i] = s_choice[staged ? s_ids[i] : scratch[i]];
            }
            for (int e = tid; e < p.N; e += kThreads) p.choice[e] = s_choice[e];
            if (tid == 0) {
                p.status[0] = METRO_OK;
                p.status[1] = p.status[2] = 0;
                p.status[3] = 1;
            }
        }
        // ---- publish.  The barrier orders every routing thread's host stores before
        // thread 0's system-scope release of the completion word (release is
        // cumulative in the PTX memory model); kFenceOne / kFenceAll add explicit
        // fence.sc.sys (tuning / verification: METRO_SERVE_FENCE=one|all).
        const uint64_t t_written = globaltimer_ns();
        if (fence_mode == kFenceAll) __threadfence_system();
        cta_sync();
        if (tid == 0) {
            if (fence_mode == kFenceOne) __threadfence_system();
            const uint64_t t_fenced = globaltimer_ns();
            const int64_t c_end = clock64();
            int64_t *st = ctl->stamps;  // phase times of this request (debug; posted writes)
            st[0] = static_cast<int64_t>(rq.t_seen);
            st[1] = static_cast<int64_t>(t_staged - rq.t_seen);
            st[2] = static_cast<int64_t>(t_routed - t_staged);
            st[3] = static_cast<int64_t>(t_written - t_routed);
            st[4] = static_cast<int64_t>(t_fenced - t_written);
            st[5] = c_end - rq.c_seen;  // SM cycles over the same span (clock rate check)
            st[6] = static_cast<int64_t>(t_fenced - rq.t_seen);
            st[7] = rq.rtt;
            st_release_sys(&ctl->done, rseq);
        }
    }
}

// shared-memory plan of the resident CTA: the routing layout with the whole
// batch staged (one CTA), lane-striped histogram copies as metro_route_v1
// (32, fewer when N * C words exceed 64 KB), + the request words
static int serve_plan(int N, int W, int64_t max_pairs, Params &p) {
    int64_t slice = (max_pairs + 3) & ~int64_t(3);
    if (slice < 4) slice = 4;
    int C0 = 32;
    while (C0 > 1 && N * C0 * 4 > 64 * 1024) C0 >>= 1;
    // staged: the whole batch in shared memory; otherwise (batches beyond ~40k
    // pairs) the first pass also copies the ids to a device scratch buffer that
    // the pair-rank pass reads (HBM instead of a second PCIe read)
    for (int staged = 1; staged >= 0; --staged)
        for (int C = C0; C >= 1; C >>= 1)
            for (int priv = 1; priv >= 0; --priv) {  // own sort scratch when it fits (no barrier)
                const Layout L = make_layout(kMetroIds, N, W, 1, slice, C, staged, false, 0, priv != 0);
                const int total = align_up(L.total, 16) + static_cast<int>(sizeof(ServeReq));
                if (total <= kMaxSmem) {
                    p.slice = slice;
                    p.staged = staged;
                    p.C = C;
                    p.private_scratch = priv;
                    return total;
                }
            }
    return METRO_EDIMS;
}

}  // namespace metro

using namespace metro;

struct metro_server {
    ServeCtl *ctl = nullptr;  // pinned, device-mapped
    cudaStream_t stream = nullptr;
    int device = 0;
    Params base = {};
    int W = 1, smem = 0;
    uint64_t idle_ns = 0;
    uint32_t seq = 0;
    int fence_mode = 0, doorbell_warps = 2;
    int32_t *scratch = nullptr;  // unstaged mode: device copy of the ids
    uint32_t stagger = 1000;
    bool sent_ptrs = false;
    int64_t max_pairs = 0, launches = 0;
    const void *ok_ids = nullptr, *ok_out = nullptr, *ok_pr = nullptr;
};

static bool host_mapped(const void *p) {
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return (attr.type == cudaMemoryTypeHost || attr.type == cudaMemoryTypeManaged) && attr.devicePointer == p;
}

template <typename T>
static T host_load_acquire(const T *p) {
    return __atomic_load_n(p, __ATOMIC_ACQUIRE);
}

static int serve_launch(metro_server *s) {
    cudaError_t e = cudaSuccess;
    __atomic_store_n(&s->ctl->state, kServeLaunched, __ATOMIC_RELEASE);
    const uint32_t seq0 = s->seq;  // the last request this server completed
    switch (s->W) {
        case 1: metro_serve_kernel<1><<<1, kThreads + 32 * s->doorbell_warps, s->smem, s->stream>>>(s->base, s->ctl, seq0, s->idle_ns, s->fence_mode, s->stagger, s->scratch); break;
        case 2: metro_serve_kernel<2><<<1, kThreads + 32 * s->doorbell_warps, s->smem, s->stream>>>(s->base, s->ctl, seq0, s->idle_ns, s->fence_mode, s->stagger, s->scratch); break;
        case 3: metro_serve_kernel<3><<<1, kThreads + 32 * s->doorbell_warps, s->smem, s->stream>>>(s->base, s->ctl, seq0, s->idle_ns, s->fence_mode, s->stagger, s->scratch); break;
        case 4: metro_serve_kernel<4><<<1, kThreads + 32 * s->doorbell_warps, s->smem, s->stream>>>(s->base, s->ctl, seq0, s->idle_ns, s->fence_mode, s->stagger, s->scratch); break;
        default: return METRO_EDIMS;
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e);
    ++s->launches;
    return METRO_OK;
}

template <int W>
static cudaError_t serve_attr() {
    return cudaFuncSetAttribute(metro_serve_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
}

extern "C" {

int metro_server_create_v1(const uint32_t *mask, int32_t N, int32_t G, int64_t max_pairs, int32_t idle_timeout_us,
                           metro_server **out) {
    if (!out || !mask || max_pairs < 0 || max_pairs > INT32_MAX / 8 || idle_timeout_us <= 0) return METRO_EARG;
    *out = nullptr;
    if (N < 1 || N > kMaxN || G < 1 || G > kMaxG) return METRO_EDIMS;
    metro_server *s = new metro_server();
    s->W = (G + 31) / 32;
    s->max_pairs = max_pairs;
    s->idle_ns = static_cast<uint64_t>(idle_timeout_us) * 1000ull;
    s->base.mask = mask;
    s->base.N = N;
    s->base.G = G;
    {
        const char *f = getenv("METRO_SERVE_FENCE");  // tuning: "one" | "all" add fence.sc.sys
        const char *dw = getenv("METRO_SERVE_DOORBELL_WARPS");  // tuning: 1..4 polling warps
        if (dw) s->doorbell_warps = atoi(dw) < 1 ? 1 : (atoi(dw) > kMaxDoorbellWarps ? kMaxDoorbellWarps : atoi(dw));
        const char *st = getenv("METRO_SERVE_STAGGER_NS");  // tuning: doorbell load spacing
        if (st) s->stagger = static_cast<uint32_t>(atoi(st));
        s->fence_mode = !f ? kFenceRelease : strcmp(f, "all") == 0 ? kFenceAll : strcmp(f, "one") == 0 ? kFenceOne
                                                                                                          : kFenceRelease;
    }
    s->smem = serve_plan(N, s->W, max_pairs, s->base);
    cudaError_t e = cudaGetDevice(&s->device);
    int rc = s->smem < 0 ? s->smem : METRO_OK;
    if (rc == METRO_OK && e != cudaSuccess) rc = cuda_fail(e);
    if (rc == METRO_OK) {
        switch (s->W) {
            case 1: e = serve_attr<1>(); break;
            case 2: e = serve_attr<2>(); break;
            case 3: e = serve_attr<3>(); break;
            default: e = serve_attr<4>(); break;
        }
        if (e != cudaSuccess) rc = cuda_fail(e);
    }
    if (rc == METRO_OK) {
        e = cudaHostAlloc(reinterpret_cast<void **>(&s->ctl), sizeof(ServeCtl), cudaHostAllocMapped | cudaHostAllocPortable);
        if (e != cudaSuccess) rc = cuda_fail(e);
        else memset(s->ctl, 0, sizeof(ServeCtl));
    }
    if (rc == METRO_OK && !host_mapped(s->ctl)) rc = METRO_EARG;  // UVA identity mapping required
    if (rc == METRO_OK && !s->base.staged) {
        e = cudaMalloc(reinterpret_cast<void **>(&s->scratch), static_cast<size_t>(s->base.slice) * 4);
        if (e != cudaSuccess) rc = cuda_fail(e);
    }
    if (rc == METRO_OK) {
        // non-blocking: the resident CTA never serialises the legacy default stream
        e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) rc = cuda_fail(e);
    }
    if (rc == METRO_OK) rc = serve_launch(s);
    if (rc != METRO_OK) {
        metro_server_destroy_v1(s);
        return rc;
    }
    *out = s;
    return METRO_OK;
}

int metro_server_route_v1(metro_server *s, const int32_t *ids, int64_t num_pairs, int32_t *host_out,
                          int32_t *pair_rank) {
    if (!s || !host_out || num_pairs < 0 || num_pairs > s->max_pairs || (num_pairs > 0 && !ids)) return METRO_EARG;
    if ((reinterpret_cast<uintptr_t>(ids) | reinterpret_cast<uintptr_t>(pair_rank) |
         reinterpret_cast<uintptr_t>(host_out)) & 15)
        return METRO_EARG;
    if (ids != s->ok_ids || host_out != s->ok_out || pair_rank != s->ok_pr) {
        // pointer validation once per buffer triple (cached like METRO_HOST_STABLE_BUFFERS)
        if ((ids && !host_mapped(ids)) || !host_mapped(host_out) || (pair_rank && !host_mapped(pair_rank)))
            return METRO_EARG;
        s->ok_ids = ids;
        s->ok_out = host_out;
        s->ok_pr = pair_rank;
    }
    ServeCtl *c = s->ctl;
    if (host_load_acquire(&c->state) != kServeLaunched) {
        // the resident CTA left after its idle timeout: reap it and start another
        cudaError_t e = cudaStreamSynchronize(s->stream);
        if (e != cudaSuccess) return cuda_fail(e);
        int rc = serve_launch(s);
        if (rc) return rc;
    }
    uint32_t flags = 0;
    if (!s->sent_ptrs || ids != reinterpret_cast<const int32_t *>(c->ids) ||
        pair_rank != reinterpret_cast<int32_t *>(c->pair_rank) || host_out != reinterpret_cast<int32_t *>(c->out)) {
        c->ids = reinterpret_cast<uint64_t>(ids);
        c->pair_rank = reinterpret_cast<uint64_t>(pair_rank);
        c->out = reinterpret_cast<uint64_t>(host_out);
        flags = kNewPtrs;
    }
    const uint32_t seq = (s->seq + 1) & kSeqMask;
    // doorbell (x86: ordered after the address stores); one 8-byte store
    __atomic_store_n(&c->doorbell, (static_cast<uint64_t>(num_pairs) << 32) | flags | seq, __ATOMIC_RELEASE);
    uint64_t spins = 0;
    timespec t0 = {0, 0};
    for (;;) {
        if (host_load_acquire(&c->done) == seq) break;
        if ((++spins & 4095) == 0) {
            if (host_load_acquire(&c->state) != kServeLaunched) {
                // the CTA exited (idle timeout) before it saw this doorbell: relaunch;
                // the new launch starts from the last completed sequence number and
                // serves the pending request
                if (host_load_acquire(&c->done) == seq) break;
                cudaError_t e = cudaStreamSynchronize(s->stream);
                if (e != cudaSuccess) return cuda_fail(e);
                if (host_load_acquire(&c->done) == seq) break;
                int rc = serve_launch(s);
                if (rc) return rc;
                continue;
            }
            timespec t;
            clock_gettime(CLOCK_MONOTONIC, &t);
            if (t0.tv_sec == 0 && t0.tv_nsec == 0) {
                t0 = t;
            } else if ((t.tv_sec - t0.tv_sec) * 1000000000ll + (t.tv_nsec - t0.tv_nsec) > 2000000000ll) {
                cudaError_t e = cudaStreamQuery(s->stream);
                return cuda_fail(e == cudaSuccess || e == cudaErrorNotReady ? cudaErrorLaunchTimeout : e);
            }
        }
#if defined(__x86_64__)
        __builtin_ia32_pause();
#endif
    }
    s->seq = seq;
    s->sent_ptrs = true;
    return METRO_OK;
}

int metro_server_debug_stamps(const metro_server *s, int64_t *out8) {
    if (!s || !out8) return METRO_EARG;
    for (int i = 0; i < 8; ++i) out8[i] = __atomic_load_n(&s->ctl->stamps[i], __ATOMIC_ACQUIRE);
    return METRO_OK;
}

int64_t metro_server_launches(const metro_server *s) { return s ? s->launches : 0; }

int metro_server_destroy_v1(metro_server *s) {
    if (!s) return METRO_OK;
    int rc = METRO_OK;
    if (s->ctl) {
        __atomic_store_n(&s->ctl->stop, 1u, __ATOMIC_RELEASE);
        if (s->stream) {
            cudaError_t e = cudaStreamSynchronize(s->stream);
            if (e != cudaSuccess) rc = cuda_fail(e);
        }
        cudaFreeHost(s->ctl);
    }
    if (s->stream) cudaStreamDestroy(s->stream);
    if (s->scratch) cudaFree(s->scratch);
    delete s;
    return rc;
}

}  // extern "C"
