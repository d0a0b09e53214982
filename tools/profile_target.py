"""Minimal launch sequences for ncu captures (no graphs, few launches).

    python tools/profile_target.py metro [B]     # 8 routing launches, DeepSeek-V3 shape
    python tools/profile_target.py q30 [B]       # 8 routing launches, Qwen3-30B shape (128 experts: the
                                                 # single-step r = 2 path), one CTA and a 4-CTA cluster
    python tools/profile_target.py eplb [B]      # 8 EPLB launches, same inputs
    python tools/profile_target.py gate [B]      # 8 fused gating top-k + METRO launches (fp32 scores)
    python tools/profile_target.py dispatch [B]  # 8 dispatch-layout launches behind METRO routing
    python tools/profile_target.py fused [B]     # 8 fused METRO + dispatch-layout launches
    python tools/profile_target.py exchange [B]  # 8 fused exchange + route launches, world 1
    python tools/profile_target.py regress [R]   # fused METRO + layout on the two large-table soak
                                                 # instances (N > 512 x 65 ranks), cluster R (default 8)
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_09277_b200 import DevicePlacement, DispatchLayout, Router  # noqa: E402
from paper_2512_09277_b200.dist import virtual_ranks  # noqa: E402
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement  # noqa: E402


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "metro"
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    dev = torch.device("cuda", 0)
    A = make_placement(256, 8, 1.5, 7).matrix
    pl = DevicePlacement(A, dev)
    batches = [torch.from_numpy(gen_zipf_topk(256, 8, B, 1.2, 1000 + s, popularity_seed=7)).to(dev)
               for s in range(8)]
    if what == "q30":
        A30 = make_placement(128, 8, 1.5, 7).matrix
        pl30 = DevicePlacement(A30, dev)
        for cl in (1, 4):
            r = Router(pl30, "metro", cl)
            out = r.alloc(B * 8, top_k=8)
            for s in range(8):
                ids = torch.from_numpy(gen_zipf_topk(128, 8, B, 1.2, 1000 + s, popularity_seed=7)).to(dev)
                r.route(ids, out=out)
            out.check()
    elif what in ("metro", "eplb"):
        r = Router(pl, what)
        out = r.alloc(B * 8, top_k=8)
        for b in batches:
            r.route(b, out=out)
    elif what == "gate":
        r = Router(pl, "metro")
        g = torch.Generator(device=dev).manual_seed(3)
        scores = [torch.randn((B, 256), generator=g, device=dev) for _ in range(8)]
        for sc in scores:
            r.route_scores(sc, 8)
    elif what == "dispatch":
        r = Router(pl, "metro")
        lay = DispatchLayout(pl)
        out = r.alloc(B * 8, top_k=8)
        for b in batches:
            r.route(b, out=out)
            lay(b.reshape(-1), out.pair_rank)
    elif what == "fused":
        lay = DispatchLayout(pl)
        out, lo = Router(pl, "metro").alloc(B * 8, top_k=8), lay.alloc(B * 8, 8)
        for b in batches:
            lay.route_metro(b, out=out, layout_out=lo)
    elif what == "regress":
        import numpy as np

        z = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                                 "fused_regress.npz"))
        cl = int(sys.argv[2]) if len(sys.argv) > 2 else 8
        for i in (0, 1):
            ids, A2 = torch.from_numpy(z[f"ids{i}"]).to(dev), z[f"A{i}"]
            pl2 = DevicePlacement(A2, dev)
            lay = DispatchLayout(pl2, cl)
            lay.route_metro(ids)[0].check()
            Router(pl2, "metro", cl).route(ids).check()
    elif what == "exchange":
        routers, bufs = virtual_ranks(pl, 1, B, 8)
        for b in batches:
            routers[0].step(b)
        torch.cuda.synchronize()
        for x in bufs:
            x.close()
    torch.cuda.synchronize()
    print("ok", what, B)


if __name__ == "__main__":
    main()
