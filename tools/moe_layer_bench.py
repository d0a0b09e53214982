"""DeepSeek-V3 MoE layer on one EP rank: routing -> the rank's activated replicas
-> K3 grouped expert FFN (tcgen05), METRO vs EPLB on the same batches.

Measures what routing buys (BASELINE.json configs[4]): weight bytes streamed from
HBM and FFN time on the bottleneck rank (the rank with the most activated
replicas, which sets the layer time in EP decode).

    python tools/moe_layer_bench.py [--batches 4] [--reps 5] [--json out.json]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_09277_b200 import DevicePlacement, Router, moe  # noqa: E402
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement  # noqa: E402

HIDDEN, INTER = 7168, 2048  # DeepSeek-V3 routed expert


def peak_gbs():
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def time_ffn(ffn, X, i1, i2, bufs, reps):
    """Device time of the rank's expert FFN (all its kernels captured in one CUDA
    graph, so host launch gaps between them are not counted)."""
    return time_graph(lambda st: ffn.forward(X, i1, i2, bufs), reps)


def time_graph(fn, reps, inner=1):
    """Median per-call device time of ``fn`` captured ``inner`` times in one CUDA graph."""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(inner):
                fn(s)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / inner)
    return statistics.median(ts)


def run(batches=4, reps=5, B=1024, ratio=1.5, seed0=1000, dtype="bf16"):
    dev = torch.device("cuda", 0)
    N, k, G = 256, 8, 8
    A = make_placement(N, G, ratio, 7).matrix
    slots = int(A.sum(axis=0).max())
    pl = DevicePlacement(A, dev)
    rm, re_ = Router(pl, "metro"), Router(pl, "eplb")
    ffn = moe.ExpertFFN(slots, HIDDEN, INTER, dev, seed=0, dtype=dtype)
    eb = 1 if dtype == "fp8" else 2  # bytes per GEMM input element
    pk, pk_src = peak_gbs()
    rows = []
    for b in range(batches):
        ids = torch.from_numpy(gen_zipf_topk(N, k, B, 1.2, seed0 + b, popularity_seed=7)).to(dev)
        om = rm.route(ids).check()
        oe = re_.route(ids, with_x=True).check()
        loads = om.loads.cpu().numpy()
        choice = om.choice.cpu().numpy()
        x = oe.x.cpu().numpy()
        res = {}
        for kind, counts in (("metro", om.rank_counts.cpu().numpy()), ("eplb", oe.rank_counts.cpu().numpy())):
            g = int(np.argmax(counts))
            wl = (moe.rank_workload_metro(choice, loads, A, g) if kind == "metro"
                  else moe.rank_workload_eplb(x, A, g))
            i1, i2 = ffn.plan(wl, dev)
            X = torch.randn((max(wl.tokens, 1), HIDDEN), device=dev).to(torch.bfloat16)
            bufs = (torch.empty((X.shape[0], 2 * INTER), dtype=torch.bfloat16, device=dev),
                    torch.empty((X.shape[0], INTER), dtype=torch.bfloat16, device=dev),
                    torch.empty((X.shape[0], HIDDEN), dtype=torch.bfloat16, device=dev))
            us = time_ffn(ffn, X, i1, i2, bufs, reps)
            wbytes = ffn.weight_bytes(wl.activated)
            # activations: X in, GU out + in (bf16), H in, Y out (bf16)
            abytes = wl.tokens * (HIDDEN * eb + 2 * INTER * 2 * 2 + INTER * eb + HIDDEN * 2)
            res[kind] = {"rank": g, "activated": wl.activated, "tokens": wl.tokens, "ffn_us": us,
                         "weight_bytes": wbytes, "achieved_gbs": (wbytes + abytes) / (us * 1e-6) / 1e9}
            res[kind]["frac"] = res[kind]["achieved_gbs"] / pk
            # the same rank's whole layer on device, one CUDA graph: route -> dispatch
            # layout -> work items -> row gather -> FFN (no host round trip)
            pipe = moe.RankMoE(pl, kind, g, ffn, max_pairs=B * k, top_k=k)
            hidden = torch.randn((B, HIDDEN), device=dev).to(torch.bfloat16)
            res[kind]["device_layer_us"] = time_graph(lambda st: pipe(ids, hidden, stream=st), reps)
            if int(pipe.counts[2].item()) != wl.tokens:
                raise RuntimeError("device layout rows differ from the host workload")
            lay = pipe.layout
            pr = pipe.route_out.pair_rank[: ids.numel()]
            lout = pipe.layout_out
            res[kind]["dispatch_layout_us"] = time_graph(
                lambda st: lay(ids, pr, out=lout, stream=st), reps, inner=200)
            # routing + dispatch layout as the layer runs them (METRO: one fused launch)
            rt, rout = pipe.router, pipe.route_out
            if kind == "metro":
                res[kind]["route_layout_us"] = time_graph(
                    lambda st: lay.route_metro(ids, out=rout, layout_out=lout, stream=st), reps, inner=200)
            else:
                res[kind]["route_layout_us"] = time_graph(
                    lambda st: (rt.route(ids, out=rout, stream=st), lay(ids, pr, out=lout, stream=st)), reps,
                    inner=200)
            del pipe
        rows.append(res)
        print(json.dumps(res), file=sys.stderr, flush=True)
    summ = {}
    for kind in ("metro", "eplb"):
        summ[kind] = {key: statistics.mean(r[kind][key] for r in rows)
                      for key in ("activated", "tokens", "ffn_us", "weight_bytes", "achieved_gbs", "frac",
                                  "device_layer_us", "dispatch_layout_us", "route_layout_us")}
    summ["dtype"] = dtype
    summ["ffn_speedup_metro_vs_eplb"] = summ["eplb"]["ffn_us"] / summ["metro"]["ffn_us"]
    summ["device_layer_speedup_metro_vs_eplb"] = summ["eplb"]["device_layer_us"] / summ["metro"]["device_layer_us"]
    summ["weight_byte_ratio_eplb_over_metro"] = summ["eplb"]["weight_bytes"] / summ["metro"]["weight_bytes"]
    summ["peak_gbs"] = pk
    summ["peak_source"] = pk_src
    summ["shape"] = {"experts": N, "top_k": k, "ep_ranks": G, "replication": ratio, "batch": B,
                     "hidden": HIDDEN, "intermediate": INTER, "dtype": dtype, "slots_per_rank": slots}
    return summ


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=4)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--json", default=None)
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp8"])
    a = ap.parse_args()
    s = run(a.batches, a.reps, a.batch, dtype=a.dtype)
    print(json.dumps(s))
    if a.json:
        with open(a.json, "w") as f:
            json.dump(s, f, indent=1)


if __name__ == "__main__":
    main()
