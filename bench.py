#!/usr/bin/env python
"""METRO routing benchmark (BASELINE.json metric): µs per MoE layer incl. the
all-gather, and max activated replicas per EP rank, METRO vs EPLB.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config ds] [--impl b200|reference]

N > 1 is launched by the driver with torch.distributed.run (one rank per GPU,
NCCL).  A step = one MoE layer: [NCCL all-gather of every rank's top-k ids] +
the sm_100a METRO routing kernel over the global batch.  The global decode
batch (B tokens) is fixed as N grows ("strong" scaling); every rank routes the
whole batch (replicated, deterministic).  N = 1: CUDA-graph replays over a
256 MiB pool of distinct batches (> L2).  N > 1: 256 MiB L2 flush per step,
flush-only loop subtracted.  Also reported: e2e from pinned host buffers, the
CPU oracle port, and K3 (the bottleneck rank's expert FFN, METRO vs EPLB).

Rank 0 prints ONE JSON line.  --impl reference times the reference algorithm's
CPU path (the oracle port, oracle/metro_oracle.c: aggregate_loads + route_metro +
per-pair replica) on the host on the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "METRO routing µs/MoE layer (incl. allGather); max activated replicas/GPU vs EPLB"

CONFIGS = {
    "ds": dict(workload="DeepSeek-V3 shape: 256 routed experts top-8, 8 EP ranks, 50% replication "
                        "(EPLB placement), 1024 decode tokens", N=256, k=8, G=8, ratio=1.5, B=1024),
    "q30": dict(workload="Qwen3-30B-A3B shape: 128 experts top-8, 8 EP ranks, 50% replication, "
                         "256 decode tokens", N=128, k=8, G=8, ratio=1.5, B=256),
    "q235_125": dict(workload="Qwen3-235B-A22B shape: 128 experts top-8, 16 logical EP ranks, 25% "
                              "replication, 1024 decode tokens", N=128, k=8, G=16, ratio=1.25, B=1024),
    "q235_150": dict(workload="Qwen3-235B-A22B shape, 50% replication", N=128, k=8, G=16, ratio=1.5, B=1024),
    "q235_200": dict(workload="Qwen3-235B-A22B shape, 100% replication", N=128, k=8, G=16, ratio=2.0, B=1024),
}
for _b in (64, 128, 256, 512, 2048, 4096, 8192):
    CONFIGS[f"ds_b{_b}"] = dict(workload=f"DeepSeek-V3 shape, decode batch {_b}", N=256, k=8, G=8,
                                ratio=1.5, B=_b)
# Zipf skew of the decode batch's expert popularity (BASELINE configs[2]; the
# placement is always built from a Zipf(1.2) history, as the reference's fixtures)
for _s in (0.5, 2.0):
    for _b in (64, 1024, 8192):
        CONFIGS[f"ds_b{_b}_skew{_s}"] = dict(workload=f"DeepSeek-V3 shape, decode batch {_b}, Zipf({_s}) "
                                                     f"expert popularity", N=256, k=8, G=8, ratio=1.5, B=_b,
                                             skew=_s)

POOL = 32          # distinct batches resident in HBM, cycled through the steps
LAMBDA_SEEDS = 128  # fresh batches for the lambda statistics (>= 100 seeds)
VIRTUAL = int(os.environ.get("METRO_VIRTUAL_RANKS", "0"))  # set in the --virtual-ranks children
FLUSH_BYTES = 256 << 20
POOL_BYTES = 256 << 20   # N=1 input pool (> 126 MB L2)
SKEW = 1.2
POP_SEED = 7


def parse_args():
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--config", default="ds", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cluster", type=int, default=0, help="CTAs per routing cluster (0 = auto)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="CPU-baseline sample length")
    ap.add_argument("--e2e-steps", type=int, default=1000)
    ap.add_argument("--detail", default=None, help="write extra per-run detail JSON here")
    ap.add_argument("--no-moe", action="store_true", help="skip the K3 expert-FFN measurement")
    ap.add_argument("--virtual-ranks", type=int, default=0,
                    help="run the N > 1 code path as P processes sharing ONE GPU (gloo plumbing, the fused "
                         "exchange over CUDA IPC on one device): a dry run of the multi-GPU branch, not a "
                         "scaling number")
    return ap.parse_args()


def workload(cfg, world: int):
    from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement

    A = make_placement(cfg["N"], cfg["G"], cfg["ratio"], POP_SEED).matrix
    batches = [gen_zipf_topk(cfg["N"], cfg["k"], cfg["B"], cfg.get("skew", SKEW), 1000 + s, popularity_seed=POP_SEED)
               for s in range(POOL)]
    return A, batches


def algorithmic_bytes(cfg) -> int:
    """Per routing launch: read ids + rank masks; write loads,
    choice, rank_counts, lam, status, pair_rank."""
    pairs = cfg["B"] * cfg["k"]
    w = (cfg["G"] + 31) // 32
    return pairs * 4 + cfg["N"] * w * 4 + cfg["N"] * 4 * 2 + cfg["G"] * 4 + 4 + 16 + pairs * 4


def load_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)", pk
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)", {}


def load_traffic(cfg_name: str):
    path = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(cfg_name)
    except Exception:
        return None


class ClockSampler:
    """NVML SM clock + throttle reasons sampled from a thread during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period: float = 0.005):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period = period
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


# ------------------------------------------------------------------ CPU (oracle port)
class OneCore:
    """Pin the calling thread to one host core (the last of its affinity set) for
    a single-thread CPU timing, restoring the affinity afterwards."""

    def __enter__(self):
        self.saved = os.sched_getaffinity(0)
        self.core = max(self.saved)
        os.sched_setaffinity(0, {self.core})
        return self

    def __exit__(self, *a):
        os.sched_setaffinity(0, self.saved)


def cpu_layer_sample(A, batches, seconds: float, min_layers: int = 200):
    """The oracle port's layer (aggregate_loads + route_metro + pair_rank) timed
    one layer at a time (perf_counter around each call) on ONE pinned host core,
    cycling through the batches, for at least `seconds` and `min_layers` layers.
    Returns (per-layer µs list, outputs of the batches for the parity check).
    Both arms use this one function: the reference arm and the b200 arm's
    cpu_baseline leg measure the same thing the same way."""
    import oracle

    outs = [oracle.metro_layer(b, A) for b in batches]  # warm + results for the parity check
    scratch = [tuple(np.copy(x) for x in o) for o in outs]
    per = []
    t_end = time.perf_counter() + seconds
    i = 0
    with OneCore():
        while True:
            b = batches[i % len(batches)]
            t0 = time.perf_counter()
            oracle.metro_layer(b, A, scratch[i % len(batches)])
            per.append(time.perf_counter() - t0)
            i += 1
            if len(per) >= min_layers and (i % len(batches) == 0) and time.perf_counter() >= t_end:
                break
    return [x * 1e6 for x in per], outs


def stats_us(per):
    s = sorted(per)
    return {"mean": statistics.mean(s), "median": s[len(s) // 2], "p99": s[int(len(s) * 0.99)], "layers": len(s)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_per_layer_stats(A, batches, reps: int = 400):
    """Median / p99 µs of single layers (perf_counter around each call) for the
    oracle port's METRO layer and its EPLB counterpart (aggregate_loads +
    route_eplb + EPLB pair ranks), one host thread."""
    import oracle

    def one(fn):
        ts = []
        for i in range(reps):
            b = batches[i % len(batches)]
            t0 = time.perf_counter()
            fn(b)
            ts.append((time.perf_counter() - t0) * 1e6)
        ts.sort()
        return {"median": ts[len(ts) // 2], "p99": ts[int(len(ts) * 0.99)], "reps": reps}

    def eplb_layer(b):
        T = oracle.aggregate_loads(b, A.shape[0])
        oracle.route_eplb(T, A)
        oracle.pair_rank_eplb(b, A)

    for b in batches[:4]:
        oracle.metro_layer(b, A)
        eplb_layer(b)
    return {"metro_layer_us": one(lambda b: oracle.metro_layer(b, A)), "eplb_layer_us": one(eplb_layer)}


def python_reference_layer(cfg, A, batches, seconds: float = 1.0, min_reps: int = 200):
    """Context only: the UNMODIFIED Python reference's layer --
    eproute.aggregate_loads(TokenBatch) + eproute.routing.route_metro(T, A)
    (core.py:236-244, routing.py:105-113) -- imported from baseline/_ref (the
    offline install of /root/reference), on the same pinned core,
    median over >= min_reps layers and >= `seconds`.  None when not installed."""
    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "eproute")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        from eproute.core import ModelSpec, PlacementMap, Token, TokenBatch, aggregate_loads
        from eproute.routing import route_metro
    except Exception as ex:  # noqa: BLE001
        return {"unavailable": f"{type(ex).__name__}: {ex}"}
    G = cfg["G"]
    model = ModelSpec(num_experts=cfg["N"], top_k=cfg["k"], hidden_dim=7168, dtype_bytes=2,
                      expert_weight_bytes=1.0, dense_weight_bytes=1.0, flops_per_token_per_expert=1.0,
                      num_moe_layers=1)
    place = PlacementMap(matrix=np.asarray(A, np.int8), slots_per_gpu=int(np.asarray(A).sum(axis=0).max()))
    tbs = [TokenBatch([Token(source_gpu=j % G, expert_ids=tuple(int(e) for e in row)) for j, row in enumerate(b)])
           for b in batches[:8]]
    per = []
    with OneCore() as pin:
        route_metro(aggregate_loads(tbs[0], model), place)
        t_end = time.perf_counter() + seconds
        i = 0
        while time.perf_counter() < t_end or len(per) < min_reps:
            t0 = time.perf_counter()
            route_metro(aggregate_loads(tbs[i % len(tbs)], model), place)
            per.append((time.perf_counter() - t0) * 1e6)
            i += 1
        core = pin.core
    per.sort()
    return {"what": "unmodified reference (baseline/_ref eproute 0.1.0): aggregate_loads + route_metro, CPython",
            "median_us": per[len(per) // 2], "mean_us": statistics.mean(per), "p99_us": per[int(len(per) * 0.99)],
            "reps": len(per), "cores": 1, "pinned_core": core}


def cpu_allcores_throughput(A, batches, seconds: float = 2.0):
    """Independent layers on every host core (context only; one layer is serial)."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle

    cores = len(os.sched_getaffinity(0))
    oracle.lib()

    def worker(_):
        scratch = [oracle.metro_layer(b, A) for b in batches]
        n, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < seconds:
            for i, b in enumerate(batches):
                oracle.metro_layer(b, A, scratch[i])
            n += len(batches)
        return n

    t0 = time.perf_counter()
    with ThreadPoolExecutor(cores) as ex:  # ctypes releases the GIL during the C call
        total = sum(ex.map(worker, range(cores)))
    return total / (time.perf_counter() - t0), cores


def run_reference(args, cfg, rank: int, world: int):
    """The reference algorithm's CPU path (the oracle port) on one pinned host
    core, on this arm's workload.  A step is a bounded sample of layers sized so
    the whole timed run covers >= 1 s and >= 200 layers whatever --steps is;
    value = mean µs per layer over every timed layer (median / p99 beside it)."""
    if rank != 0:
        return None
    A, batches = workload(cfg, world)
    import oracle

    oracle.build()
    steps = max(1, args.steps)
    # calibrate: layers per step so that steps x per_step >= max(200 layers, 1 s)
    cal, _ = cpu_layer_sample(A, batches, 0.2, 64)
    target = max(200, int(1.0 / (statistics.mean(cal) * 1e-6)) + 1)
    per_step = -(-max(1, -(-target // steps)) // len(batches)) * len(batches)  # whole passes over the pool
    for _ in range(args.warmup):
        cpu_layer_sample(A, batches, 0.0, min(per_step, 64))
    per = []
    for _ in range(steps):
        p, _ = cpu_layer_sample(A, batches, 0.0, per_step)
        per.extend(p)
    st = stats_us(per)
    us = st["mean"]
    thr, cores = cpu_allcores_throughput(A, batches, 1.0)
    sample = (f"{st['layers']} layers of the {args.config} workload (B={cfg['B']}, N={cfg['N']}, G={cfg['G']}): "
              f"{steps} steps of {per_step} layers, each layer timed alone, one pinned host core")
    return {
        "impl": "reference", "metric": METRIC, "value": us, "unit": "us/layer", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": us * per_step / 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": data_str(cfg),
        "config": config_dict(args, cfg, world),
        "arm": "reference algorithm's CPU path: the oracle port (oracle/metro_oracle.c), single thread, pinned",
        "cpu_baseline": {"value": us, "unit": "us/layer", "cores": 1, "kind": "port", "sample": sample,
                         "per_layer_us": st, "all_cores_layers_per_s": thr, "host_cores": cores,
                         "cpu_model": cpu_model(), "python_reference": python_reference_layer(cfg, A, batches)},
        "e2e": {"value": us, "unit": "us/layer", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def data_str(cfg=None):
    skew = (cfg or {}).get("skew", SKEW)
    return (f"synthetic: Zipf({skew}) expert popularity, top-8 distinct ids per token by Gumbel top-k; "
            "EPLB placement from a Zipf(1.2) history (reference generators, popularity seed 7)")


def config_dict(args, cfg, world):
    """The workload, identical in both arms (the driver compares the two lines'
    config); how each arm runs it is under the line's "arm" / "timing" keys."""
    return {"workload": cfg["workload"], "name": args.config, "num_experts": cfg["N"], "top_k": cfg["k"],
            "ep_ranks": cfg["G"], "replication": cfg["ratio"], "global_batch": cfg["B"],
            "parallelism": f"ep all-gather over {world} GPU(s), routing replicated per rank",
            "l2": ("inputs larger than L2 (256 MiB pool cycled, no flush)" if world == 1 else
                   "flushed between steps (256 MiB memset, subtracted)"),
            "pool_batches": POOL}


# ------------------------------------------------------------------ GPU
def run_b200(args, cfg, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist

    from paper_2512_09277_b200 import DevicePlacement, HostRouter, Router
    from paper_2512_09277_b200.dist import DistributedRouter, FusedAllGatherRouter, allgather_topk

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    A, batches = workload(cfg, world)
    B, k = cfg["B"], cfg["k"]
    if B % world:
        raise SystemExit(f"global batch {B} not divisible by {world} GPUs")
    lt = B // world
    pl = DevicePlacement(A, dev)
    router = Router(pl, "metro", args.cluster)
    base = torch.from_numpy(np.stack(batches)).to(dev)  # [POOL, B, k] exact Zipf batches
    out = router.alloc(B * k, top_k=k)
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device=dev)
    K = args.steps

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    virtual = VIRTUAL > 1  # P ranks sharing one GPU over gloo (--virtual-ranks)
    cdev = torch.device("cpu") if virtual else dev  # device of the plumbing collectives' tensors

    def max_over_ranks(vals):
        if world == 1:
            return vals
        t = torch.tensor(vals, dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    def loop_ms(n, body, with_flush):
        """One CUDA-event pair around n iterations of [L2 flush] + body(i)."""
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sync_all()
        e0.record()
        for i in range(n):
            if with_flush:
                flush.zero_()
            body(i)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    gathered = torch.empty((B, k), dtype=torch.int32, device=dev)
    local_pool = [base[s, rank * lt:(rank + 1) * lt].contiguous() for s in range(POOL)]

    def ag(i):
        allgather_topk(local_pool[i % POOL], gathered)

    def ag_route(i):
        ag(i)
        router.route(gathered, out=out)

    def route_base(i):
        router.route(base[i % POOL], out=out)

    for i in range(max(args.warmup, 3)):  # warm-up (the .so is prebuilt; no JIT)
        (ag_route if world > 1 else route_base)(i)
        flush.zero_()
    sync_all()

    method = {}
    with ClockSampler(local_rank) as clk:
        if world == 1:
            # (a) primary: EXACTLY K launches, back to back from CUDA graphs, launch j on
            # slot j % P of a pool of distinct batches larger than L2 (rows resampled
            # from the exact Zipf batches).  Every graph is replayed once untimed (graph
            # upload), then a 256 MiB flush empties L2, so every timed launch reads
            # its ids from HBM (a slot recurs only P launches = 256 MiB later).
            from paper_2512_09277_b200 import _native

            per_batch = B * k * 4
            P = max(256, -(-POOL_BYTES // per_batch))
            gen = torch.Generator(device=dev).manual_seed(1234)
            rows = torch.randint(0, POOL * B, (P, B), device=dev, generator=gen)
            big = base.reshape(POOL * B, k)[rows].contiguous()  # [P, B, k]
            chunk = 256
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

            def build(n):
                graphs = []
                for c0 in range(0, n, chunk):
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g):
                        for j in range(c0, min(n, c0 + chunk)):
                            router.route(big[j % P], out=out)
                    graphs.append(g)
                return graphs

            def timed(graphs, n):
                for g in graphs:  # untimed: graph upload
                    g.replay()
                flush.zero_()
                sync_all()
                w0 = time.perf_counter()
                e0.record()
                for g in graphs:
                    g.replay()
                e1.record()
                torch.cuda.synchronize()
                return e0.elapsed_time(e1) / n, time.perf_counter() - w0

            graphs = build(K)
            step_ms, wall = timed(graphs, K)
            del graphs
            K_eff = K
            kern_ms = step_ms
            ag_ms = 0.0
            method = {"method": "exactly K launches replayed back-to-back from CUDA graphs, launch j on slot j % {} "
                                "of a {:.0f} MiB pool of distinct batches (> L2), L2 flushed before the timed "
                                "replay".format(P, P * per_batch / 2 ** 20),
                      "pdl": "programmatic dependent launch: each routing kernel's shared-memory prologue "
                             "overlaps the previous kernel; it waits for that kernel's completion before "
                             "reading its ids (as behind the gating kernel in a decode step)"}
            # the same measurement with PDL off (every launch fully serialised)
            _native.lib().metro_set_pdl(0)
            try:
                n_np = min(K, 2048)
                graphs = build(n_np)
                method["no_pdl_us"] = timed(graphs, n_np)[0] * 1e3
                del graphs
            finally:
                _native.lib().metro_set_pdl(1)
            # routing + dispatch layout in ONE launch (metro_route_layout_v1) over the
            # same pool, and the two-launch chain it replaces
            from paper_2512_09277_b200 import DispatchLayout

            dl = DispatchLayout(pl, args.cluster)
            lo = dl.alloc(B * k, k)
            n_l = min(max(K, 256), 2048)
            fgraphs = []
            for c0 in range(0, n_l, chunk):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for j in range(c0, min(n_l, c0 + chunk)):
                        dl.route_metro(big[j % P], out=out, layout_out=lo)
                fgraphs.append(g)
            method["route_layout_fused_us"] = timed(fgraphs, n_l)[0] * 1e3
            del fgraphs
            sgraphs = []
            for c0 in range(0, n_l, chunk):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for j in range(c0, min(n_l, c0 + chunk)):
                        router.route(big[j % P], out=out)
                        dl(big[j % P], out.pair_rank, out=lo)
                sgraphs.append(g)
            method["route_then_layout_us"] = timed(sgraphs, n_l)[0] * 1e3
            del sgraphs
            del big
            # (b) context: eager launch after a 256 MiB L2 flush, flush time subtracted
            Kb = min(K, 2000)
            tf = loop_ms(Kb, lambda i: None, True)
            tr = loop_ms(Kb, route_base, True)
            method["after_flush_eager_us"] = (tr - tf) / Kb * 1e3
            # single launches one at a time (events around each, stream idle before):
            # the latency distribution of one layer's routing, launch included
            single = []
            for i in range(500):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                route_base(i)
                e1.record()
                torch.cuda.synchronize()
                single.append(e0.elapsed_time(e1) * 1e3)
            single.sort()
            method["single_launch_us"] = {"mean": statistics.mean(single), "p50": single[len(single) // 2],
                                          "p99": single[int(len(single) * 0.99)], "samples": len(single),
                                          "note": "events around one eager Router.route launch on an idle "
                                                  "stream: includes the host launch path (Python, ctypes, "
                                                  "driver)"}
            # the lean eager path: a launch plan bound to fixed buffers (Router.bind,
            # metro_route_plan_launch_v1), the ids refilled in place each layer
            slot = base[0].clone()
            plan = router.bind(slot, out=out)
            single = []
            for i in range(500):
                slot.copy_(base[i % POOL])
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                plan()
                e1.record()
                torch.cuda.synchronize()
                single.append(e0.elapsed_time(e1) * 1e3)
            single.sort()
            method["single_launch_bound_us"] = {"mean": statistics.mean(single), "p50": single[len(single) // 2],
                                                "p99": single[int(len(single) * 0.99)], "samples": len(single),
                                                "api": "Router.bind(...)() (metro_route_plan_launch_v1)"}
            plan.close()
            # the floor of ANY eager launch measured this way on this box: a one-element
            # torch kernel between the same two events
            tiny = torch.zeros(1, device=dev)
            single = []
            for i in range(300):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                tiny.add_(1)
                e1.record()
                torch.cuda.synchronize()
                single.append(e0.elapsed_time(e1) * 1e3)
            method["single_launch_floor_us"] = {"p50": statistics.median(single),
                                                "what": "torch one-element add between the same two events: "
                                                        "the host launch path + launch latency of any kernel"}
        else:
            # every step: 256 MiB L2 flush, NCCL all-gather of the local top-k ids,
            # routing kernel on the gathered batch; the flush-only loop is
            # subtracted (one event pair per loop, per-rank max)
            wall0 = time.perf_counter()
            tf = loop_ms(K, lambda i: None, True)
            ts = loop_ms(K, ag_route, True)
            ta = loop_ms(K, ag, True)
            tr = loop_ms(K, lambda i: router.route(gathered, out=out), True)
            wall = time.perf_counter() - wall0
            step_ms, ag_ms, kern_ms = max_over_ranks([(ts - tf) / K, (ta - tf) / K, (tr - tf) / K])
            K_eff = K
            method = {"method": "per step: 256 MiB L2 flush + all-gather + route; flush-only loop "
                                "subtracted; one event pair per K-step loop; max over ranks"}
            # the product path: exchange + route fused in ONE kernel per rank over NVLink
            # peer memory (metro_exchange.h); the NCCL all-gather + route above is the
            # baseline it replaces.  Any rank failing to set it up or to complete the
            # warm-up exchange disables it on every rank (no hang, no partial run).
            fused_ms, fused_err = None, None
            fz = None
            try:
                fz = FusedAllGatherRouter(pl, lt, k)
                for i in range(3):
                    fz.step(local_pool[i % POOL])
                torch.cuda.synchronize()
                st = int(fz.out.status[0].item())
                if st != 0:
                    raise RuntimeError(f"fused exchange status {st}")
                ag_route(2)  # same batch through the NCCL path: identical routing required
                torch.cuda.synchronize()
                if not (torch.equal(fz.out.choice, out.choice) and int(fz.out.lam.item()) == int(out.lam.item())):
                    raise RuntimeError("fused routing differs from the NCCL path")
                bad = 0
            except Exception as ex:  # noqa: BLE001 -- reported in the JSON line
                fused_err, bad = repr(ex)[:200], 1
            flag = torch.tensor([bad], dtype=torch.int32, device=cdev)
            dist.all_reduce(flag, op=dist.ReduceOp.MAX)
            if int(flag.item()) == 0:
                tfz = loop_ms(K, lambda i: fz.step(local_pool[i % POOL]), True)
                fused_ms = max_over_ranks([(tfz - tf) / K])[0]
                nccl_ms = step_ms
                step_ms = fused_ms
                method["method"] = ("per step: 256 MiB L2 flush + fused exchange+route kernel (metro_exchange.h, "
                                    "NVLink peer stores); flush-only loop subtracted; one event pair per K-step "
                                    "loop; max over ranks")
                method["nccl_allgather_plus_route_us"] = nccl_ms * 1e3
                # the same exchange + route fused with the GLOBAL dispatch layout (rows of
                # this rank's pairs in their serving ranks' receive buffers, no ids gather)
                from paper_2512_09277_b200 import DispatchLayout

                fzl = FusedAllGatherRouter(pl, lt, k, layout=DispatchLayout(pl))
                for i in range(3):
                    fzl.step(local_pool[i % POOL])
                torch.cuda.synchronize()
                tfl = loop_ms(K, lambda i: fzl.step(local_pool[i % POOL]), True)
                method["fused_exchange_route_layout_us"] = max_over_ranks([(tfl - tf) / K])[0] * 1e3
                sync_all()
                fzl.close()
            else:
                method["fused_unavailable"] = fused_err or "another rank failed"
            method["fused_exchange_route_us"] = None if fused_ms is None else fused_ms * 1e3
        sync_all()

    # lambda METRO vs EPLB through the device routers over >= 100 fresh Zipf batches
    # (SURVEY.md §8(d)); Qwen3-235B: per physical GPU beside the per-column value
    sys.path.insert(0, os.path.join(REPO, "tools"))
    import lambda_stats

    lam = lambda_stats.run(cfg, LAMBDA_SEEDS, dev, physical_group=2 if cfg["G"] == 16 else 0)
    lam_m = lam.pop("metro_per_seed")  # seeds 1000 + s: the first POOL are this bench's exact batches

    # end to end from host buffers: H2D ids, route, D2H results, sync
    E = min(args.e2e_steps, K)
    if world == 1:
        # the reference-facing host call (ServedRouter, include/metro_serve.h): the
        # caller's batch is in pinned host memory; a resident CTA reads it over PCIe,
        # routes it and writes choice / counts / lam / status + pair_rank back into
        # host memory; the call returns when the results are there.  (No
        # device-wide synchronise while it runs: it would wait for the resident CTA.)
        from paper_2512_09277_b200 import ServedRouter

        cur = torch.cuda.current_stream()
        hosts = [b.reshape(-1).copy() for b in batches]
        with ServedRouter(pl, B * k) as sr:
            ids_np = sr.ids.numpy()
            for i in range(10):
                ids_np[:] = hosts[i % POOL]
                sr.run(B * k)
            per = []
            for i in range(E):
                ids_np[:] = hosts[i % POOL]  # the caller's batch arrives in host memory
                flush.zero_()
                cur.synchronize()
                t0 = time.perf_counter()
                out_np = sr.run(B * k)
                per.append(time.perf_counter() - t0)
                if i < POOL and int(out_np[0]) != 0:
                    raise RuntimeError("e2e routing reported an error status")
            e2e_launches = sr.launches
        e2e_us = statistics.mean(per) * 1e6
        h2d = B * k * 4
        d2h = (8 + cfg["G"] + cfg["N"]) * 4 + B * k * 4
        # the one-launch host call (metro_route_host_v1, zero-copy) for context
        hr = HostRouter(pl, B * k, args.cluster, zero_copy=True)
        ids_np = hr.ids.numpy()
        per1 = []
        for i in range(min(E, 300) + 10):
            ids_np[:] = hosts[i % POOL]
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            hr.run(B * k)
            if i >= 10:
                per1.append(time.perf_counter() - t0)
        e2e_extra = {"api": "ServedRouter.run (persistent router, include/metro_serve.h)",
                     "p50_us": statistics.median(per) * 1e6, "resident_cta_launches": e2e_launches,
                     "launch_per_call_us": statistics.mean(per1) * 1e6,
                     "launch_per_call_api": "HostRouter.run (metro_route_host_v1, zero-copy, one launch + sync)"}
    else:
        use_fused = method.get("fused_exchange_route_us") is not None
        dr = None if use_fused else DistributedRouter(pl, lt, k, "metro", args.cluster)
        local_d = torch.empty((lt, k), dtype=torch.int32, device=dev)
        hosts = [torch.from_numpy(b[rank * lt:(rank + 1) * lt].copy()).pin_memory() for b in batches]
        small_h = torch.empty(8 + cfg["G"] + cfg["N"], dtype=torch.int32).pin_memory()
        own_h = torch.empty(lt * k, dtype=torch.int32).pin_memory()
        small_d = torch.empty_like(small_h, device=dev)
        per = []
        for i in range(E + 10):
            flush.zero_()
            sync_all()
            t0 = time.perf_counter()
            if use_fused:  # the product path: fused exchange + route (metro_exchange.h)
                local_d.copy_(hosts[i % POOL].view(lt, k), non_blocking=True)
                o = fz.step(local_d)
                own = o.pair_rank
            else:
                dr.local.copy_(hosts[i % POOL].view(lt, k), non_blocking=True)
                o = dr.step()
                own = dr.own_pair_rank()
            small_d[0:4].copy_(o.status)
            small_d[4:5].copy_(o.lam)
            small_d[8:8 + cfg["G"]].copy_(o.rank_counts)
            small_d[8 + cfg["G"]:].copy_(o.choice)
            small_h.copy_(small_d, non_blocking=True)
            own_h.copy_(own, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            if i >= 10:
                per.append(time.perf_counter() - t0)
        e2e_us = max_over_ranks([statistics.mean(per)])[0] * 1e6
        e2e_extra = {"api": ("FusedAllGatherRouter.step (fused exchange + route)" if use_fused else
                             "DistributedRouter (NCCL all-gather + route)") + " from pinned host buffers"}
        h2d = lt * k * 4
        d2h = small_h.numel() * 4 + lt * k * 4

    if rank != 0:
        return None

    peak, peak_src, _ = load_peaks()
    alg = algorithmic_bytes(cfg)
    achieved = alg / (kern_ms * 1e-3) / 1e9
    res = {
        "metric": METRIC, "value": step_ms * 1e3, "unit": "us/layer", "n_gpus": world, "steps": K_eff,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "int32", "data": data_str(cfg),
        "config": config_dict(args, cfg, world),
        "arm": "b200: sm_100a routing kernels (libmetro_b200.so) through the C ABI",
        "e2e": dict({"value": e2e_us, "unit": "us/layer", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
                    **e2e_extra),
        "gpu_launches": K_eff,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": load_traffic(args.config),
                     "peak_source": peak_src, "algorithmic_bytes_per_launch": alg,
                     "kernel": "metro_ids_kernel", "kernel_us": kern_ms * 1e3,
                     "note": "latency-bound serial greedy; HBM fraction is low by construction"},
        "timing": dict(method, allgather_us=ag_ms * 1e3, route_kernel_us=kern_ms * 1e3, timed_wall_s=wall),
        "lambda": dict({"metro_mean": lam["metro"]["mean"], "eplb_mean": lam["eplb"]["mean"],
                        "metro_max": lam["metro"]["max"], "eplb_max": lam["eplb"]["max"],
                        "metro_le_eplb_all": lam["metro_le_eplb_all"], "batches": lam["seeds"]}, detail=lam),
        "clocks": clk.summary(),
    }
    if world > 1:
        recv = (world - 1) * lt * k * 4
        res["nvlink"] = {"allgather_recv_bytes_per_rank": recv,
                         "fused_exchange_recv_bytes_per_rank": (world - 1) * (cfg["N"] + 3) * 8,
                         "achieved_gbs": recv / (ag_ms * 1e-3) / 1e9, "peak_gbs": 770.0,
                         "frac": recv / (ag_ms * 1e-3) / 1e9 / 770.0,
                         "peak_source": "measured peer copy, B200_PROFILING.md"}
    if world == 1 and not args.no_moe and cfg["N"] == 256 and cfg["G"] == 8:
        # BASELINE configs[4]: the bottleneck rank's expert FFN (K3, tcgen05) under the
        # METRO vs EPLB routing of the same batches -> weight bytes vs activated replicas
        sys.path.insert(0, os.path.join(REPO, "tools"))
        import moe_layer_bench

        m = moe_layer_bench.run(batches=2, reps=3, B=cfg["B"], ratio=cfg["ratio"])
        res["moe_layer_k3"] = {
            "what": "expert FFN (gate_up + silu*mul + down, bf16, D=7168 I=2048) on the rank with the most "
                    "activated replicas; tcgen05 grouped GEMM streaming the activated experts' weights",
            "metro": m["metro"], "eplb": m["eplb"],
            "ffn_speedup_metro_vs_eplb": m["ffn_speedup_metro_vs_eplb"],
            "weight_byte_ratio_eplb_over_metro": m["weight_byte_ratio_eplb_over_metro"],
            "device_layer_speedup_metro_vs_eplb": m["device_layer_speedup_metro_vs_eplb"],
            "device_layer_what": "the same rank's whole layer in one CUDA graph: route -> dispatch layout -> "
                                 "K3 work items -> row gather -> FFN, no host round trip",
            "roofline": {"bound": "hbm", "achieved": m["metro"]["achieved_gbs"], "peak": m["peak_gbs"],
                         "unit": "GB/s", "frac": m["metro"]["frac"], "kernel": "moe_gemm_kernel"},
        }
        # the same with FP8 (E4M3) experts, as DeepSeek-V3 ships them: half the bytes
        m8 = moe_layer_bench.run(batches=2, reps=3, B=cfg["B"], ratio=cfg["ratio"], dtype="fp8")
        res["moe_layer_k3_fp8"] = {
            "what": "as moe_layer_k3 with E4M3 expert weights (scale per 128-row block) and E4M3 activations "
                    "(scale per token), tcgen05 kind::f8f6f4",
            "metro": m8["metro"], "eplb": m8["eplb"],
            "ffn_speedup_metro_vs_eplb": m8["ffn_speedup_metro_vs_eplb"],
            "device_layer_speedup_metro_vs_eplb": m8["device_layer_speedup_metro_vs_eplb"],
            "routing_share_of_metro_layer": step_ms * 1e3 / m8["metro"]["device_layer_us"],
        }
    if world == 1:
        per, outs = cpu_layer_sample(A, batches, args.cpu_seconds)
        st = stats_us(per)
        lam_cpu = [int(o[3][0]) for o in outs]
        parity = lam_cpu == lam_m[:len(lam_cpu)]
        # full-output parity of the last exact batch (choice / pair_rank)
        router.route(base[-1], out=out)
        torch.cuda.synchronize()
        o = outs[-1]
        parity = parity and np.array_equal(out.choice.cpu().numpy(), o[1]) and \
            np.array_equal(out.pair_rank.cpu().numpy(), o[4].reshape(-1))
        thr, cores = cpu_allcores_throughput(A, batches, 1.0)
        res["cpu_baseline"] = {
            "value": st["mean"], "unit": "us/layer", "cores": 1, "kind": "port",
            "sample": f"{st['layers']} layers ({args.cpu_seconds:.0f} s) of this workload through the oracle "
                      "port (aggregate_loads + route_metro + pair_rank), each layer timed alone, one pinned "
                      "host core (the same function as --impl reference)",
            "per_layer_us": st, "all_cores_layers_per_s": thr, "host_cores": cores, "cpu_model": cpu_model(),
            "eplb_layer_us": cpu_per_layer_stats(A, batches)["eplb_layer_us"], "parity_vs_gpu": bool(parity),
            "python_reference": python_reference_layer(cfg, A, batches),
        }
    return res


def run_virtual(args) -> int:
    """--virtual-ranks P: launch P copies of this bench as ranks 0..P-1 of a gloo
    process group, all on cuda:0 (torchrun's environment contract), and relay
    rank 0's JSON line.  Exercises the N > 1 branch end to end on one GPU."""
    import socket
    import subprocess

    P = args.virtual_ranks
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    argv = [a for a in sys.argv[1:]]
    i = argv.index("--virtual-ranks") if "--virtual-ranks" in argv else -1
    if i >= 0:
        del argv[i:i + 2]
    argv = [x for x in argv if not x.startswith("--virtual-ranks=")]
    if "--gpus" in argv:
        j = argv.index("--gpus")
        del argv[j:j + 2]
    procs = []
    for r in range(P):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(P), LOCAL_RANK="0", LOCAL_WORLD_SIZE=str(P),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), METRO_VIRTUAL_RANKS=str(P))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__), "--gpus", str(P)] + argv, env=env,
                                      stdout=subprocess.PIPE if r == 0 else subprocess.DEVNULL, text=True))
    out, _ = procs[0].communicate()
    rcs = [procs[0].returncode] + [p.wait() for p in procs[1:]]
    lines = [ln for ln in (out or "").splitlines() if ln.startswith("{")]
    if any(rcs) or not lines:
        print(json.dumps({"virtual_ranks": P, "error": f"rank exit codes {rcs}"}))
        return 1
    print(lines[-1])
    return 0


def main():
    args = parse_args()
    if args.virtual_ranks > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(run_virtual(args))
    # a peer that never joins the fused exchange is reported after 2 s, never a hang
    os.environ.setdefault("METRO_PEER_TIMEOUT_MS", "2000")
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank != 0:
            return
        res = run_reference(args, cfg, rank, world)
    else:
        if world > 1:
            import torch
            import torch.distributed as dist

            torch.cuda.set_device(local_rank)
            if VIRTUAL > 1:  # ranks sharing one GPU: NCCL refuses that, gloo carries the plumbing
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        res = run_b200(args, cfg, rank, world, local_rank)
        if res is not None and VIRTUAL > 1:
            res["virtual_ranks"] = {"ranks": VIRTUAL, "note": "N > 1 code path on ONE GPU (P processes, gloo "
                                    "plumbing, exchange over CUDA IPC on one device): a dry run, not a scaling "
                                    "measurement"}
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
    if res is not None:
        print(json.dumps(res))
        if args.detail:
            with open(args.detail, "w") as f:
                json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
