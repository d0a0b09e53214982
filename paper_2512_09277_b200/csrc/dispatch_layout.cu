// dispatch_layout.cu -- sm_100a dispatch layout after routing (include/dispatch_layout.h).
//
// Given every pair's expert (topk_ids) and serving rank (pair_rank, from the
// routing kernels), compute each pair's row in its rank's receive buffer, rows
// grouped by replica (rank-major, local slot ascending) and, inside a replica,
// by pair index ascending.  Row counts per replica equal the reference's
// assignment entries x[i, g] (routing.py:41-52 METRO, routing.py:64-69 EPLB);
// the row order is this library's convention (the reference stops at x).
//
// One thread-block cluster of R CTAs; CTA c owns the contiguous pair slice
// [c * slice, (c + 1) * slice), and inside it warp w owns a contiguous
// sub-slice, so "pair index ascending" is the lexicographic order
// (CTA, warp, chunk of 32, lane):
//   (1) each warp walks its sub-slice 32 pairs at a time; __match_any_sync groups
//       equal replica ids, giving every pair its rank among the warp's earlier
//       pairs of the same replica, and one lane bumps the warp-private count;
//   (2) per replica, a scan over the 16 warp counts -> warp prefixes + CTA total;
//   (3) one cluster barrier, then every CTA reads the R CTA totals of each
//       replica from its peers' shared memory (DSMEM): prefix over earlier
//       CTAs and the global total; a block scan of the totals gives rep_off;
//   (4) row = rep_off[rid] - rep_off[first rid of the rank] + CTA prefix +
//       warp prefix + in-warp rank.
// The work is a few passes over 8 bytes per pair: latency-bound at every
// BASELINE shape (8192 pairs at DeepSeek-V3 B=1024).
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <mutex>

#include "../../include/dispatch_layout.h"
#include "lib_internal.h"
#include "sm100_ptx.cuh"

namespace metro {
namespace dl {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxRep = 4096;
constexpr int kMaxSlice = 8192;
static_assert(kMaxSlice < 65536, "per-warp replica counts and prefixes are uint16");
constexpr int kMaxCluster = 16;
constexpr uint64_t kNoBad = ~0ull;

struct Params {
    const int32_t *ids;
    const int32_t *pair_rank;
    int64_t num_pairs;
    int32_t slice;
    const int32_t *rid_tab;
    const int32_t *slot_base;
    int32_t N, G, nrep;
    int32_t *pair_row;
    int32_t *rep_off;
    int32_t *status;
    int32_t rtab_smem;  // 1: the replica table is staged in shared memory
};

// smem: bad (8) | cta_tot [nrep + 1] | pre [nrep] | loc [nrep + 1] | off [nrep + 1] | sb [G + 1] | wsum [32] |
//       hw [kWarps][nrep] (uint16) | pk [slice] | rtab [N * G] (optional) | base [nrep] | e [slice] | g [slice]
//       (pk = rid << 16 | in-warp rank; rtab = the replica table staged once;
//        base[rid] = first row offset of rid's rank)
struct Layout {
    int bad, tot, pre, loc, off, sb, wsum, hw, pk, rtab, base, se, sg, total;
};
__host__ __device__ inline int al16(int x) { return (x + 15) & ~15; }
__host__ __device__ inline Layout make_layout(int nrep, int slice, int G, int rtab_words) {
    Layout L;
    int o = 0;
    L.bad = o;  o += 16;
    L.tot = o;  o = al16(o + (nrep + 1) * 4);
    L.pre = o;  o = al16(o + nrep * 4);
    L.loc = o;  o = al16(o + (nrep + 1) * 4);
    L.off = o;  o = al16(o + (nrep + 1) * 4);
    L.sb = o;   o = al16(o + (G + 1) * 4);
    L.wsum = o; o = al16(o + 32 * 4);
    L.hw = o;   o = al16(o + kWarps * nrep * 2);  // uint16: counts and prefixes <= kMaxSlice
    L.pk = o;   o = al16(o + slice * 4);
    L.rtab = o; o = al16(o + rtab_words * 4);
    L.base = o; o = al16(o + nrep * 4);
    L.se = o;   o = al16(o + slice * 4);
    L.sg = o;   o = al16(o + slice * 4);
    L.total = o;
    return L;
}

__device__ __forceinline__ unsigned lane_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// exclusive block scan of v[0..n) into out[0..n], out[n] = total (512 threads)
__device__ void block_exscan(const int32_t *v, int32_t *out, int n, int32_t *wsum) {
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
    __syncthreads();
    if (warp == 0) {
        int32_t w = lane < kWarps ? wsum[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int32_t y = __shfl_up_sync(kFull, w, d);
            if (lane >= d) w += y;
        }
        if (lane < kWarps) wsum[lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    int32_t run = x - s + (warp > 0 ? wsum[warp - 1] : 0);
    for (int i = b; i < e; ++i) {
        out[i] = run;
        run += v[i];
    }
    if (tid == kThreads - 1) out[n] = wsum[kWarps - 1];
    __syncthreads();
}

__global__ void __launch_bounds__(kThreads, 1) layout_kernel(const Params p) {
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t R = cluster_nctarank(), cta = cluster_ctarank();
    const Layout L = make_layout(p.nrep, p.slice, p.G, p.rtab_smem ? p.N * p.G : 0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nrep = p.nrep;
    unsigned long long *s_bad = reinterpret_cast<unsigned long long *>(smem + L.bad);
    int32_t *s_tot = reinterpret_cast<int32_t *>(smem + L.tot);
    int32_t *s_pre = reinterpret_cast<int32_t *>(smem + L.pre);
    int32_t *s_loc = reinterpret_cast<int32_t *>(smem + L.loc);
    int32_t *s_off = reinterpret_cast<int32_t *>(smem + L.off);
    int32_t *s_sb = reinterpret_cast<int32_t *>(smem + L.sb);
    int32_t *s_wsum = reinterpret_cast<int32_t *>(smem + L.wsum);
    uint16_t *s_hw = reinterpret_cast<uint16_t *>(smem + L.hw);  // per-warp replica counts
    uint32_t *s_pk = reinterpret_cast<uint32_t *>(smem + L.pk);
    int32_t *s_rtab = reinterpret_cast<int32_t *>(smem + L.rtab);
    int32_t *s_base = reinterpret_cast<int32_t *>(smem + L.base);
    int32_t *s_e = reinterpret_cast<int32_t *>(smem + L.se);
    int32_t *s_g = reinterpret_cast<int32_t *>(smem + L.sg);

    const int64_t beg = static_cast<int64_t>(cta) * p.slice;
    const int64_t rem = p.num_pairs - beg;
    const int n_local = rem <= 0 ? 0 : static_cast<int>(rem < p.slice ? rem : p.slice);
    // PDL: shared-memory prologue, then wait for the routing kernel's outputs
    if (tid == 0) *s_bad = kNoBad;
    for (int i = tid; i < kWarps * nrep; i += kThreads) s_hw[i] = 0;
    griddep_wait();
    griddep_launch_dependents();  // only once this kernel runs: at most one dependent waits
    for (int i = tid; i <= p.G; i += kThreads) s_sb[i] = __ldg(p.slot_base + i);
    if (p.rtab_smem)  // the replica table (N * G words) once into shared memory: the
        for (int i = tid; i < p.N * p.G; i += kThreads) s_rtab[i] = __ldg(p.rid_tab + i);  // lookups are LDS
    // the CTA's pairs (expert, serving rank) into shared memory with independent
    // 16-byte loads, all in flight at once: the rank loop below then never waits
    // on global memory
    {
        const int32_t *ge = p.ids + beg, *gg = p.pair_rank + beg;
        const bool vec = ((reinterpret_cast<uintptr_t>(ge) | reinterpret_cast<uintptr_t>(gg)) & 15) == 0;
        const int n4 = vec ? (n_local >> 2) : 0;
        for (int i = tid; i < n4; i += kThreads) {
            reinterpret_cast<int4 *>(s_e)[i] = __ldg(reinterpret_cast<const int4 *>(ge) + i);
            reinterpret_cast<int4 *>(s_g)[i] = __ldg(reinterpret_cast<const int4 *>(gg) + i);
        }
        for (int i = 4 * n4 + tid; i < n_local; i += kThreads) {
            s_e[i] = __ldg(ge + i);
            s_g[i] = __ldg(gg + i);
        }
    }
    __syncthreads();
    const int32_t *rtab = p.rtab_smem ? s_rtab : p.rid_tab;

    // (1) warp sub-slices, match_any ranks
    const int ws = (((n_local + kWarps - 1) / kWarps) + 31) & ~31;
    const int wb = min(n_local, warp * ws), we = min(n_local, wb + ws);
    uint16_t *hw = s_hw + warp * nrep;
    unsigned long long my_bad = kNoBad;
    for (int p0 = wb; p0 < we; p0 += 32) {
        const int i = p0 + lane;
        int rid = -1;
        if (i < we) {
            const int e = s_e[i];
            const int g = s_g[i];
            const unsigned long long gi = static_cast<unsigned long long>(beg + i);
            if (static_cast<unsigned>(e) >= static_cast<unsigned>(p.N)) {
                my_bad = min(my_bad, gi << 1);
            } else if (static_cast<unsigned>(g) >= static_cast<unsigned>(p.G) ||
                       (rid = rtab[static_cast<int64_t>(e) * p.G + g]) < 0) {
                rid = -1;
                my_bad = min(my_bad, (gi << 1) | 1ull);
            }
        }
        const unsigned m = __match_any_sync(kFull, rid);
        if (rid >= 0) {
            const int r = hw[rid] + __popc(m & lane_lt());
            s_pk[i] = (static_cast<uint32_t>(rid) << 16) | static_cast<uint32_t>(r);
        }
        __syncwarp();
        if (rid >= 0 && lane == __ffs(m) - 1) hw[rid] = static_cast<uint16_t>(hw[rid] + __popc(m));
        __syncwarp();
    }
    if (my_bad != kNoBad) atomicMin(s_bad, my_bad);
    __syncthreads();

    // (2) warp prefixes per replica, CTA totals
    for (int rid = tid; rid < nrep; rid += kThreads) {
        int32_t run = 0;
#pragma unroll 4
        for (int w = 0; w < kWarps; ++w) {
            const int32_t c = s_hw[w * nrep + rid];
            s_hw[w * nrep + rid] = static_cast<uint16_t>(run);
            run += c;
        }
        s_tot[rid] = run;
    }
    // (3) exchange: every CTA's totals and bad word become visible cluster-wide
    __syncthreads();
    if (R > 1) {
        cluster_arrive_release();
        cluster_wait();
    }
    unsigned long long bad = *s_bad;
    if (R > 1) {
        for (uint32_t q = 0; q < R; ++q) {
            if (q == cta) continue;
            const uint32_t lo = dsmem_ld(reinterpret_cast<const uint32_t *>(s_bad), q);
            const uint32_t hi = dsmem_ld(reinterpret_cast<const uint32_t *>(s_bad) + 1, q);
            bad = min(bad, (static_cast<unsigned long long>(hi) << 32) | lo);
        }
        for (int rid = tid; rid < nrep; rid += kThreads) {
            // every peer's load in flight before the first use (R <= 16)
            int32_t v[kMaxCluster];
#pragma unroll
            for (int q = 0; q < kMaxCluster; ++q)
                v[q] = (q < static_cast<int>(R) && q != static_cast<int>(cta))
                           ? static_cast<int32_t>(dsmem_ld(s_tot + rid, q)) : 0;
            int32_t pre = 0, all = s_tot[rid];
#pragma unroll
            for (int q = 0; q < kMaxCluster; ++q) {
                pre += (q < static_cast<int>(cta)) ? v[q] : 0;
                all += v[q];
            }
            s_pre[rid] = pre;
            s_loc[rid] = all;  // global totals (scanned below)
        }
        // peers may exit / reuse their smem once everyone has read it
        cluster_arrive_relaxed();
    } else {
        for (int rid = tid; rid < nrep; rid += kThreads) {
            s_pre[rid] = 0;
            s_loc[rid] = s_tot[rid];
        }
    }
    __syncthreads();
    if (bad != kNoBad) {
        if (cta == 0 && tid == 0) {
            const int64_t idx = static_cast<int64_t>(bad >> 1);
            p.status[0] = (bad & 1ull) ? METRO_ERR_PAIR_RANK : METRO_ERR_ID_RANGE;
            p.status[1] = static_cast<int32_t>(idx & 0xffffffff);
            p.status[2] = static_cast<int32_t>(idx >> 32);
            p.status[3] = (bad & 1ull) ? p.pair_rank[idx] : p.ids[idx];
        }
        if (R > 1) cluster_wait();
        return;
    }
    // global exclusive offsets in rid order (s_tot and s_bad stay untouched: peers
    // may still be reading them until the final cluster barrier)
    block_exscan(s_loc, s_off, nrep, s_wsum);
    if (cta == 0)
        for (int i = tid; i <= nrep; i += kThreads) p.rep_off[i] = s_off[i];
    // per replica: global offset + this CTA's prefix - the first row of its rank
    // (replicas are numbered rank-major: rank g owns [sb[g], sb[g + 1]))
    for (int g = 0; g < p.G; ++g)
        for (int rid = s_sb[g] + tid; rid < s_sb[g + 1]; rid += kThreads)
            s_base[rid] = s_off[rid] + s_pre[rid] - s_off[s_sb[g]];
    __syncthreads();

    // (4) rows, relative to the first row of the serving rank
    for (int i = tid; i < n_local; i += kThreads) {
        const uint32_t pk = s_pk[i];
        const int rid = static_cast<int>(pk >> 16);
        const int w = i / ws;
        p.pair_row[beg + i] = s_base[rid] + s_hw[w * nrep + rid] + static_cast<int>(pk & 0xffffu);
    }
    if (cta == 0 && tid == 0) {
        p.status[0] = METRO_OK;
        p.status[1] = p.status[2] = 0;
        p.status[3] = static_cast<int32_t>(R);
    }
    if (R > 1) cluster_wait();
}

}  // namespace dl
}  // namespace metro

// ---------------------------------------------------------------- host
namespace {
using namespace metro::dl;

cudaError_t prepare_layout() {
    static std::mutex mu;
    static int done_dev[64];
    static int ndone = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    for (int i = 0; i < ndone; ++i)
        if (done_dev[i] == dev) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(layout_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(layout_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e == cudaSuccess && ndone < 64) done_dev[ndone++] = dev;
    return e;
}
}  // namespace

extern "C" {

int metro_replica_table(const int8_t *A, int32_t N, int32_t G, int32_t *rid_tab, int32_t *slot_base) {
    if (!A || !rid_tab || !slot_base || N < 0 || G < 0) return METRO_EARG;
    int32_t rid = 0;
    for (int g = 0; g < G; ++g) {
        slot_base[g] = rid;
        for (int i = 0; i < N; ++i) {
            const int8_t a = A[(int64_t)i * G + g];
            if (a != 0 && a != 1) return METRO_ENOTBINARY;
            rid_tab[(int64_t)i * G + g] = a ? rid++ : -1;
        }
    }
    slot_base[G] = rid;
    return METRO_OK;
}

int metro_dispatch_layout_v1(const int32_t *ids, const int32_t *pair_rank, int64_t num_pairs,
                             const int32_t *rid_tab, const int32_t *slot_base, int32_t N, int32_t G,
                             int32_t nrep, int32_t *pair_row, int32_t *rep_off, int32_t *status,
                             int32_t cluster_ctas, void *stream) {
    if (num_pairs < 0 || !rid_tab || !slot_base || !rep_off || !status ||
        (num_pairs > 0 && (!ids || !pair_rank || !pair_row)))
        return METRO_EARG;
    if (N < 1 || N > 4096 || G < 1 || G > 128 || nrep < 1 || nrep > kMaxRep) return METRO_EDIMS;
    int R = cluster_ctas;
    if (R == 0) {
        R = 1;
        while (R < kMaxCluster && (num_pairs > static_cast<int64_t>(R) * 1024 ||
                                   num_pairs > static_cast<int64_t>(R) * kMaxSlice))
            R *= 2;
    }
    if (R != 1 && R != 2 && R != 4 && R != 8 && R != 16) return METRO_EARG;
    const int64_t slice64 = (num_pairs + R - 1) / R;
    if (slice64 > kMaxSlice) return METRO_EDIMS;
    const int slice = static_cast<int>(slice64 < 32 ? 32 : slice64);
    // stage the replica table in shared memory when it fits (N * G words)
    int rtab_smem = 1;
    Layout L = make_layout(nrep, slice, G, N * G);
    if (L.total > 232448) {
        rtab_smem = 0;
        L = make_layout(nrep, slice, G, 0);
    }
    if (L.total > 232448) return METRO_EDIMS;
    cudaError_t e = prepare_layout();
    if (e != cudaSuccess) return metro::cuda_fail(e);
    Params p;
    p.ids = ids; p.pair_rank = pair_rank; p.num_pairs = num_pairs; p.slice = slice;
    p.rid_tab = rid_tab; p.slot_base = slot_base; p.N = N; p.G = G; p.nrep = nrep;
    p.pair_row = pair_row; p.rep_off = rep_off; p.status = status; p.rtab_smem = rtab_smem;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(R, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = L.total;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = R;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // griddep_wait before global reads
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    e = cudaLaunchKernelEx(&cfg, layout_kernel, p);
    if (e != cudaSuccess) return metro::cuda_fail(e);
    return METRO_OK;
}

}  // extern "C"
