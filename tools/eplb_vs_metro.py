"""Routing cost of the two routers on the device, same batches (DeepSeek-V3 shape,
B = 64 / 1024 / 8192): METRO (replica choice + pair ranks) vs EPLB (even split,
dense x + pair ranks).  CUDA graphs over a > L2 pool.  python tools/eplb_vs_metro.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_09277_b200 import DevicePlacement, Router  # noqa: E402
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement  # noqa: E402
from gate_bench import graph_time  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    pl = DevicePlacement(make_placement(256, 8, 1.5, 7).matrix, dev)
    res = {}
    for B in (64, 1024, 8192):
        P = max(16, (256 << 20) // (B * 8 * 4))
        base = torch.stack([torch.from_numpy(gen_zipf_topk(256, 8, B, 1.2, 1000 + j, popularity_seed=7))
                            for j in range(8)]).to(dev)
        rows = torch.randint(0, B, (P, B), device=dev, generator=torch.Generator(device=dev).manual_seed(1))
        pool = base[torch.arange(P, device=dev) % 8][torch.arange(P, device=dev)[:, None], rows].contiguous()
        for kind in ("metro", "eplb"):
            r = Router(pl, kind)
            out = r.alloc(B * 8, top_k=8, with_x=(kind == "eplb"))
            res[f"B{B}/{kind}_us"] = graph_time(lambda j: r.route(pool[j], out=out), P)
        del pool
    print(json.dumps(res))


if __name__ == "__main__":
    main()
