"""Dispatch layout (metro_dispatch_layout_v1) per-launch time by cluster size,
DS shape, CUDA-graph replays (L2-warm: the same batch).  python tools/layout_bench.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_09277_b200 import DevicePlacement, DispatchLayout, Router  # noqa: E402
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    pl = DevicePlacement(make_placement(256, 8, 1.5, 7).matrix, dev)
    res = {}
    for B in (64, 1024, 8192):
        ids = torch.from_numpy(gen_zipf_topk(256, 8, B, 1.2, 1000, popularity_seed=7)).to(dev)
        r = Router(pl, "metro")
        out = r.route(ids)
        torch.cuda.synchronize()
        for R in (1, 2, 4, 8, 16, 0):
            if B * 8 > R * 8192 and R:
                continue
            lay = DispatchLayout(pl, R)
            lo = lay(ids.reshape(-1), out.pair_rank)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(200):
                    lay(ids.reshape(-1), out.pair_rank, out=lo)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(5):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            res[f"B{B}/R{R}"] = e0.elapsed_time(e1) * 1e3 / 1000
            print(f"B{B}/R{R}", round(res[f"B{B}/R{R}"], 3), flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
