"""Fused gating top-k + METRO (metro_route_scores_v1) vs the unfused pair
(torch.topk on the scores, then metro_route_v1 on the ids), DeepSeek-V3 shape.

Device time per layer, CUDA graphs replayed back-to-back over a pool of distinct
score batches larger than L2 (1 MiB of fp32 scores per batch at B=1024, N=256).

    python tools/gate_bench.py [--batch 1024] [--pool-mib 256]
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_09277_b200 import DevicePlacement, Router  # noqa: E402
from paper_2512_09277_b200.placement import make_placement  # noqa: E402


def graph_time(step, P, chunk=128, reps=2):
    graphs = []
    for c0 in range(0, P, chunk):
        for j in range(c0, min(P, c0 + chunk)):
            step(j)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for j in range(c0, min(P, c0 + chunk)):
                step(j)
        graphs.append(g)
    graphs[0].replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        for g in graphs:
            g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * P)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--experts", type=int, default=256)
    ap.add_argument("--pool-mib", type=int, default=256)
    ap.add_argument("--clusters", default="0")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    N, k, G, B = a.experts, 8, 8, a.batch
    pl = DevicePlacement(make_placement(N, G, 1.5, 7).matrix, dev)
    r = Router(pl, "metro")
    P = max(16, a.pool_mib * 2 ** 20 // (B * N * 4))
    gen = torch.Generator(device=dev).manual_seed(0)
    scores = torch.randn((P, B, N), device=dev, generator=gen)
    ids = torch.empty((B, k), dtype=torch.int32, device=dev)
    out = r.alloc(B * k, top_k=k)

    def fused(j):
        r.route_scores(scores[j], k, out=out, topk_ids=ids)

    def unfused(j):
        top = torch.topk(scores[j], k, dim=1).indices
        ids.copy_(top)
        r.route(ids, out=out)

    def topk_only(j):
        ids.copy_(torch.topk(scores[j], k, dim=1).indices)

    res = {"batch": B, "experts": N, "top_k": k, "pool_batches": P,
           "unfused_topk_then_route_us": graph_time(unfused, P), "torch_topk_only_us": graph_time(topk_only, P)}
    res["fused_auto_us"] = graph_time(lambda j: r.route_scores(scores[j], k, out=out, topk_ids=ids), P)
    res["fused_whole_gpu_us"] = graph_time(
        lambda j: r.route_scores(scores[j], k, out=out, topk_ids=ids, whole_gpu=True), P)
    for c in (int(x) for x in a.clusters.split(",")):
        rc = Router(pl, "metro", c)
        res[f"fused_us_cluster{c}"] = graph_time(
            lambda j: rc.route_scores(scores[j], k, out=out, topk_ids=ids, whole_gpu=False), P)
    res["route_ids_us"] = graph_time(lambda j: r.route(ids, out=out), P)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
