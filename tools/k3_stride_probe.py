"""K3 weight-stream rate vs the weight row stride (is a power-of-two K slower?).
METRO bottleneck rank, DeepSeek-V3 shape, M = 7168 rows, K swept around 2048.
    python tools/k3_stride_probe.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_09277_b200 import DevicePlacement, Router, moe  # noqa: E402
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement  # noqa: E402


def graph_us(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def main():
    dev = torch.device("cuda", 0)
    A = make_placement(256, 8, 1.5, 7).matrix
    pl = DevicePlacement(A, dev)
    ids = torch.from_numpy(gen_zipf_topk(256, 8, 1024, 1.2, 1000, popularity_seed=7)).to(dev)
    o = Router(pl, "metro").route(ids).check()
    g = int(np.argmax(o.rank_counts.cpu().numpy()))
    wl = moe.rank_workload_metro(o.choice.cpu().numpy(), o.loads.cpu().numpy(), A, g)
    E = len(wl.groups)
    nt = moe.item_tokens()
    for M in tuple(int(m) for m in os.environ.get('PROBE_M', '7168,4096').split(',')):
        items = torch.from_numpy(moe.build_items(wl.groups, M)).to(dev)
        for K in tuple(int(k) for k in os.environ.get('PROBE_K', '2048,2176,1920,4096,4224,7168').split(',')):
            W = (torch.randn((E, M, K), device=dev) * 0.02).to(torch.bfloat16)
            X = torch.randn((wl.tokens, K), device=dev).to(torch.bfloat16)
            Y = torch.empty((wl.tokens, M), dtype=torch.bfloat16, device=dev)
            t16 = graph_us(lambda: moe.grouped_gemm(W, X, items, Y, max_item_tokens=nt))
            W8, ws = moe.quantize_weights_fp8(W)
            del W
            X8, xs = moe.quantize_rows_fp8(X)
            t8 = graph_us(lambda: moe.grouped_gemm_fp8(W8, ws, X8, xs, items, Y, max_item_tokens=nt))
            b16, b8 = E * M * K * 2, E * M * K
            print(f"M {M} K {K}: bf16 {t16:7.1f} us {b16 / t16 / 1e6:5.2f} TB/s | fp8 {t8:7.1f} us "
                  f"{b8 / t8 / 1e6:5.2f} TB/s", flush=True)
            del W8, X, X8, Y
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
