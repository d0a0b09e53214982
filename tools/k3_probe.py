"""K3 per-projection timing on the METRO bottleneck rank (DeepSeek-V3 shape):
gate_up and down GEMMs separately, bf16 and FP8, achieved weight GB/s.
    python tools/k3_probe.py"""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_09277_b200 import DevicePlacement, Router, moe  # noqa: E402
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement  # noqa: E402

D, I = 7168, 2048


def t_us(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


def main():
    dev = torch.device("cuda", 0)
    A = make_placement(256, 8, 1.5, 7).matrix
    slots = int(A.sum(axis=0).max())
    pl = DevicePlacement(A, dev)
    ids = torch.from_numpy(gen_zipf_topk(256, 8, 1024, 1.2, 1000, popularity_seed=7)).to(dev)
    o = Router(pl, "metro").route(ids).check()
    g = int(np.argmax(o.rank_counts.cpu().numpy()))
    wl = moe.rank_workload_metro(o.choice.cpu().numpy(), o.loads.cpu().numpy(), A, g)
    i1 = moe.build_items(wl.groups, 2 * I)
    i2 = moe.build_items(wl.groups, D)
    T = wl.tokens
    res = {"tokens": T, "activated": wl.activated, "items": [len(i1), len(i2)]}
    for dtype in ("bf16", "fp8"):
        ffn = moe.ExpertFFN(slots, D, I, dev, seed=0, dtype=dtype)
        X = torch.randn((T, D), device=dev).to(torch.bfloat16)
        GU = torch.empty((T, 2 * I), dtype=torch.bfloat16, device=dev)
        Y = torch.empty((T, D), dtype=torch.bfloat16, device=dev)
        j1 = torch.from_numpy(i1).to(dev)
        j2 = torch.from_numpy(i2).to(dev)
        nt = moe.item_tokens()
        eb = 1 if dtype == "fp8" else 2
        if dtype == "fp8":
            X8, xs = moe.quantize_rows_fp8(X)
            H8, hs = moe.silu_mul_fp8(GU)
            r1 = t_us(lambda: moe.grouped_gemm_fp8(ffn.W1q, ffn.W1s, X8, xs, j1, GU, max_item_tokens=nt))
            r2 = t_us(lambda: moe.grouped_gemm_fp8(ffn.W2q, ffn.W2s, H8, hs, j2, Y, max_item_tokens=nt))
            rq = t_us(lambda: moe.quantize_rows_fp8(X, X8, xs))
            rs = t_us(lambda: moe.silu_mul_fp8(GU, H8, hs))
        else:
            H = torch.empty((T, I), dtype=torch.bfloat16, device=dev)
            r1 = t_us(lambda: moe.grouped_gemm(ffn.W1, X, j1, GU, max_item_tokens=nt))
            r2 = t_us(lambda: moe.grouped_gemm(ffn.W2, H, j2, Y, max_item_tokens=nt))
            rq = 0.0
            rs = t_us(lambda: moe.silu_mul(GU, H))
        w1 = wl.activated * 2 * I * D * eb
        w2 = wl.activated * D * I * eb
        res[dtype] = {"gate_up_us": r1, "gate_up_tbs": w1 / r1 / 1e6, "down_us": r2, "down_tbs": w2 / r2 / 1e6,
                      "quantize_x_us": rq, "silu_us": rs}
        print(dtype, json.dumps(res[dtype]), flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
