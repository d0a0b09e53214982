"""Routing µs per layer by cluster size R and batch, graph-replayed over a >L2 pool
with PDL (the auto policy's data).  python tools/cluster_sweep.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_09277_b200 import DevicePlacement, Router  # noqa: E402
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement  # noqa: E402


def pool_us(r, pool, out, n=1024):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for j in range(n):
            r.route(pool[j % pool.shape[0]], out=out)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


def main():
    dev = torch.device("cuda", 0)
    res = {}
    for name, (N, G, ratio) in {"ds": (256, 8, 1.5), "q30": (128, 8, 1.5), "q235": (128, 16, 2.0)}.items():
        pl = DevicePlacement(make_placement(N, G, ratio, 7).matrix, dev)
        for B in (64, 128, 256, 512, 1024, 2048, 4096, 8192):
            base = torch.from_numpy(gen_zipf_topk(N, 8, B, 1.2, 1000, popularity_seed=7)).to(dev)
            P = max(64, (256 << 20) // (B * 32))
            rows = torch.randint(0, B, (P, B), device=dev, generator=torch.Generator(device=dev).manual_seed(1))
            pool = base[rows].contiguous()
            row = {}
            for R in (1, 2, 4, 8, 16):
                if B * 8 > R * 65536:  # staged slice must fit
                    continue
                r = Router(pl, "metro", R)
                out = r.alloc(B * 8, top_k=8)
                row[R] = round(pool_us(r, pool, out), 3)
            r = Router(pl, "metro", 0)
            row["auto"] = round(pool_us(r, pool, r.alloc(B * 8, top_k=8)), 3)
            res[f"{name}/B{B}"] = row
            print(name, B, json.dumps(row), flush=True)
            del pool
    with open("gpurun_out/cluster_sweep.json", "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
