"""Route + dispatch layout per MoE layer: the fused launch (metro_route_layout_v1)
against routing followed by the standalone layout kernel (metro_route_v1 +
metro_dispatch_layout_v1, two launches with PDL).  CUDA-graph replays over a
pool of distinct batches larger than L2, every launch reading its ids from HBM.

    python tools/fused_layout_bench.py [--out gpurun_out/fused_layout.json]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_09277_b200 import DevicePlacement, DispatchLayout, Router  # noqa: E402
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement  # noqa: E402

SHAPES = {"q30": (128, 8, 1.5, 256), "ds_b64": (256, 8, 1.5, 64), "ds_b256": (256, 8, 1.5, 256),
          "ds": (256, 8, 1.5, 1024), "ds_b4096": (256, 8, 1.5, 4096), "ds_b8192": (256, 8, 1.5, 8192),
          "q235_200": (128, 16, 2.0, 1024)}


def timed(fn, n, e0, e1):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for j in range(n):
            fn(j)
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/fused_layout.json")
    ap.add_argument("--launches", type=int, default=512)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    res = {}
    for name, (n, g, ratio, B) in SHAPES.items():
        pl = DevicePlacement(make_placement(n, g, ratio, 7).matrix, dev)
        base = torch.stack([torch.from_numpy(gen_zipf_topk(n, 8, B, 1.2, 1000 + s, popularity_seed=7))
                            for s in range(16)]).to(dev)
        P = max(64, (192 << 20) // (B * 8 * 4))
        rows = torch.randint(0, 16 * B, (P, B), device=dev, generator=torch.Generator(device=dev).manual_seed(1))
        pool = base.reshape(16 * B, 8)[rows].contiguous()
        r = Router(pl, "metro")
        dl = DispatchLayout(pl)
        out = r.alloc(B * 8, top_k=8)
        lo = dl.alloc(B * 8, 8)
        sep = timed(lambda j: (r.route(pool[j % P], out=out), dl(pool[j % P], out.pair_rank, out=lo)),
                    a.launches, e0, e1)
        fused = timed(lambda j: dl.route_metro(pool[j % P], out=out, layout_out=lo), a.launches, e0, e1)
        route = timed(lambda j: r.route(pool[j % P], out=out), a.launches, e0, e1)
        res[name] = {"route_us": route, "route_plus_layout_us": sep, "fused_us": fused}
        print(name, {k: round(v, 2) for k, v in res[name].items()}, flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
