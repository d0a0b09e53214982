"""Eager launch-path probe: device time between an event recorded on an idle
stream and the end of one routing launch (host launch path + launch latency +
kernel), and the host time of the call itself, for each API layer.

    python tools/launch_probe.py [--config ds]
"""
import argparse
import json
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_09277_b200 import DevicePlacement, Router  # noqa: E402
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement  # noqa: E402


def probe(fn, n=400):
    dev, host = [], []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        t0 = time.perf_counter()
        fn()
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        dev.append(e0.elapsed_time(e1) * 1e3)
        host.append((t1 - t0) * 1e6)
    return {"dev_p50": statistics.median(dev), "host_p50": statistics.median(host)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=1024)
    ap.add_argument("--N", type=int, default=256)
    a = ap.parse_args()
    A = make_placement(a.N, 8, 1.5, 7).matrix
    ids = torch.from_numpy(gen_zipf_topk(a.N, 8, a.B, 1.2, 1000, popularity_seed=7)).cuda()
    pl = DevicePlacement(A)
    r = Router(pl, "metro")
    out = r.alloc(ids.numel(), top_k=8)
    plan = r.bind(ids, out=out)
    tiny = torch.zeros(1, device="cuda")
    res = {"torch_tiny_add": probe(lambda: tiny.add_(1)),
           "route": probe(lambda: r.route(ids, out=out)),
           "bound_plan": probe(plan)}
    # kernel time alone (graph, back to back)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(100):
            plan()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    res["graph_per_launch_us"] = e0.elapsed_time(e1) * 10
    res["env"] = {k: v for k, v in os.environ.items() if k.startswith("METRO_")}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
