"""One call of the METRO bottleneck rank's whole MoE layer (moe.RankMoE) for an ncu
launch list: python tools/rank_layer_target.py [bf16|fp8]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_09277_b200 import DevicePlacement, Router, moe  # noqa: E402
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement  # noqa: E402


def main():
    dtype = sys.argv[1] if len(sys.argv) > 1 else "bf16"
    dev = torch.device("cuda", 0)
    N, k, G, B = 256, 8, 8, 1024
    A = make_placement(N, G, 1.5, 7).matrix
    pl = DevicePlacement(A, dev)
    ids = torch.from_numpy(gen_zipf_topk(N, k, B, 1.2, 1000, popularity_seed=7)).to(dev)
    hidden = torch.randn((B, 7168), device=dev).to(torch.bfloat16)
    o = Router(pl, "metro").route(ids).check()
    g = int(np.argmax(o.rank_counts.cpu().numpy()))
    ffn = moe.ExpertFFN(int(A.sum(axis=0).max()), 7168, 2048, dev, seed=0, dtype=dtype)
    pipe = moe.RankMoE(pl, "metro", g, ffn, max_pairs=B * k, top_k=k)
    torch.cuda.synchronize()
    pipe(ids, hidden)
    torch.cuda.synchronize()
    print("ok", dtype, g, int(pipe.counts[2].item()))


if __name__ == "__main__":
    main()
