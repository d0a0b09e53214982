"""One METRO-rank down-projection GEMM launch (DeepSeek-V3 shape) for ncu:
    python tools/k3_profile_target.py [bf16|fp8] [gate_up|down]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_09277_b200 import DevicePlacement, Router, moe  # noqa: E402
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement  # noqa: E402

D, I = 7168, 2048


def main():
    dtype = sys.argv[1] if len(sys.argv) > 1 else "bf16"
    proj = sys.argv[2] if len(sys.argv) > 2 else "down"
    dev = torch.device("cuda", 0)
    A = make_placement(256, 8, 1.5, 7).matrix
    slots = int(A.sum(axis=0).max())
    pl = DevicePlacement(A, dev)
    ids = torch.from_numpy(gen_zipf_topk(256, 8, 1024, 1.2, 1000, popularity_seed=7)).to(dev)
    o = Router(pl, "metro").route(ids).check()
    g = int(np.argmax(o.rank_counts.cpu().numpy()))
    wl = moe.rank_workload_metro(o.choice.cpu().numpy(), o.loads.cpu().numpy(), A, g)
    M, K = (2 * I, D) if proj == "gate_up" else (D, I)
    items = torch.from_numpy(moe.build_items(wl.groups, M)).to(dev)
    ffn = moe.ExpertFFN(slots, D, I, dev, seed=0, dtype=dtype)
    X = torch.randn((wl.tokens, K), device=dev).to(torch.bfloat16)
    Y = torch.empty((wl.tokens, M), dtype=torch.bfloat16, device=dev)
    nt = moe.item_tokens()
    if dtype == "fp8":
        X8, xs = moe.quantize_rows_fp8(X)
        W8, ws = (ffn.W1q, ffn.W1s) if proj == "gate_up" else (ffn.W2q, ffn.W2s)
        moe.grouped_gemm_fp8(W8, ws, X8, xs, items, Y, max_item_tokens=nt)
    else:
        W = ffn.W1 if proj == "gate_up" else ffn.W2
        moe.grouped_gemm(W, X, items, Y, max_item_tokens=nt)
    torch.cuda.synchronize()
    print("ok", dtype, proj, wl.tokens, len(items))


if __name__ == "__main__":
    main()
