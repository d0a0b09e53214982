"""Minimal launch sequences for ncu captures (no graphs, few launches).

    python tools/profile_target.py metro   # 8 routing launches, DeepSeek-V3 shape (B=1024)
    python tools/profile_target.py eplb    # 8 EPLB launches, same inputs
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_09277_b200 import DevicePlacement, Router  # noqa: E402
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement  # noqa: E402


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "metro"
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    dev = torch.device("cuda", 0)
    A = make_placement(256, 8, 1.5, 7).matrix
    pl = DevicePlacement(A, dev)
    r = Router(pl, "metro" if what == "metro" else "eplb")
    batches = [torch.from_numpy(gen_zipf_topk(256, 8, B, 1.2, 1000 + s, popularity_seed=7)).to(dev)
               for s in range(8)]
    out = r.alloc(B * 8, top_k=8)
    for b in batches:
        r.route(b, out=out)
    torch.cuda.synchronize()
    print("ok", what, B)


if __name__ == "__main__":
    main()
