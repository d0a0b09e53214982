"""Fused all-gather + METRO (metro_allgather_route_v1) with P virtual EP ranks on
ONE B200: per-layer latency, max over ranks, DeepSeek-V3 shape.

Each rank's K layers are captured in its own CUDA graph and the P graphs are
replayed concurrently on P streams; the ranks pace each other through the
exchange flags, so (end - start) / K on the slowest rank is the per-layer time
of the exchange + route.  Peer stores land in this GPU's own HBM here; across
NVLink they add the fabric latency (~1-2 us per direction).

    python tools/allgather_bench.py [--steps 2000] [--batch 1024]
"""

import argparse
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_09277_b200 import DevicePlacement, Router, _native  # noqa: E402
from paper_2512_09277_b200.dist import virtual_ranks  # noqa: E402
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--gather", action="store_true", help="also all-gather the ids")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    N, k, G, B = 256, 8, 8, a.batch
    pl = DevicePlacement(make_placement(N, G, 1.5, 7).matrix, dev)
    ids = torch.from_numpy(gen_zipf_topk(N, k, B, 1.2, 1000, popularity_seed=7)).to(dev)
    res = {"batch": B, "experts": N, "top_k": k, "ep_ranks": G, "steps": a.steps, "gather_ids": a.gather}
    # reference point: the single-launch router on the whole batch, same graph method
    r = Router(pl, "metro")
    out = r.alloc(B * k, top_k=k)
    g = torch.cuda.CUDAGraph()
    r.route(ids, out=out)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for _ in range(200):
            r.route(ids, out=out)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(a.steps // 200):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    res["route_only_us"] = e0.elapsed_time(e1) * 1e3 / (a.steps // 200 * 200)
    for P in (1, 2, 4, 8):
        lt = B // P
        routers, bufs = virtual_ranks(pl, P, lt, k, gather_ids=a.gather)
        shards = [ids[q * lt:(q + 1) * lt].contiguous() for q in range(P)]
        streams = [torch.cuda.Stream(dev) for _ in range(P)]
        stamps = torch.zeros(P * 8, dtype=torch.int64, device=dev)
        _native.lib().metro_allgather_debug_stamps(ctypes.c_void_p(stamps.data_ptr()))
        for _ in range(3):  # warm-up calls (concurrent)
            for q in range(P):
                routers[q].step(shards[q], stream=streams[q])
        torch.cuda.synchronize()
        graphs = []
        for q in range(P):
            gq = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gq, stream=streams[q]):
                for _ in range(a.steps):
                    routers[q].step(shards[q], stream=streams[q])
            graphs.append(gq)
        torch.cuda.synchronize()
        for q in range(P):  # first replay uploads the graphs (ms of skew between ranks)
            with torch.cuda.stream(streams[q]):
                graphs[q].replay()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(P)]
        for q in range(P):  # CUDAGraph.replay() launches on the current stream
            with torch.cuda.stream(streams[q]):
                ev[q][0].record(streams[q])
                graphs[q].replay()
                ev[q][1].record(streams[q])
        torch.cuda.synchronize()
        per = [ev[q][0].elapsed_time(ev[q][1]) * 1e3 / a.steps for q in range(P)]
        st = [int(routers[q].out.status[0].item()) for q in range(P)]
        lam = {int(routers[q].out.lam.item()) for q in range(P)}
        res[f"P{P}"] = {"us_per_layer_max_over_ranks": max(per), "us_min": min(per), "status": st,
                        "lambda": sorted(lam)}
        # per-phase globaltimer stamps of the LAST graph-replayed step (captured
        # into the graphs: no host launch skew between the ranks)
        st_ns = stamps.view(P, 8).cpu().numpy()
        t0 = st_ns[:, 0].min()
        res[f"P{P}"]["phases_ns_last_step"] = {
            "start_skew": int(st_ns[:, 0].max() - t0),
            "count": int((st_ns[:, 1] - st_ns[:, 0]).max()), "push": int((st_ns[:, 2] - st_ns[:, 1]).max()),
            "receive": int((st_ns[:, 3] - st_ns[:, 2]).max()), "route": int((st_ns[:, 4] - st_ns[:, 3]).max()),
            "outputs": int((st_ns[:, 5] - st_ns[:, 4]).max()), "kernel": int((st_ns[:, 5] - st_ns[:, 0]).max())}
        _native.lib().metro_allgather_debug_stamps(None)
        print(P, json.dumps(res[f"P{P}"]), flush=True)
        del graphs
        for b in bufs:
            b.close()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
