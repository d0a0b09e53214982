"""Routing quality through the DEVICE routers at the survey's statistical scale
(>= 100 seeds per config): max activated replicas per EP rank
(lambda) of METRO vs EPLB over fresh Zipf batches (seeds 1000 + s, popularity
seed 7, placement make_placement(N, G, ratio, 7) -- the reference fixtures'
generators, pinned by tests/golden).  For the Qwen3-235B shape (16 logical EP
ranks on 8 GPUs) the per-physical-GPU lambda is reported beside the per-column
one: GPU g hosts logical ranks 2g and 2g + 1, so its activated replicas are
the sum of those two columns of rank_counts.

    python tools/lambda_stats.py [--seeds 128] [--out gpurun_out/lambda_stats.json]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2512_09277_b200 import DevicePlacement, Router  # noqa: E402
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement  # noqa: E402


def _summ(v):
    v = list(v)
    return {"mean": statistics.mean(v), "median": statistics.median(v), "min": min(v), "max": max(v)}


def run(cfg: dict, seeds: int = 128, device=None, physical_group: int = 0) -> dict:
    """cfg: N, k, G, ratio, B (+ skew).  physical_group > 1: logical ranks per GPU."""
    dev = device or torch.device("cuda", 0)
    N, k, G, B = cfg["N"], cfg["k"], cfg["G"], cfg["B"]
    A = make_placement(N, G, cfg["ratio"], 7).matrix
    pl = DevicePlacement(A, dev)
    rm, re = Router(pl, "metro"), Router(pl, "eplb")
    om = rm.alloc(B * k, top_k=k)
    oe = re.alloc(B * k, pair_rank=False, top_k=k)
    lm, le, pm, pe = [], [], [], []
    for s in range(seeds):
        ids = torch.from_numpy(gen_zipf_topk(N, k, B, cfg.get("skew", 1.2), 1000 + s, popularity_seed=7)).to(dev)
        rm.route(ids, out=om).check()
        re.route(ids, out=oe, pair_rank=False).check()
        lm.append(int(om.lam.item()))
        le.append(int(oe.lam.item()))
        if physical_group > 1:
            cm = om.rank_counts.cpu().numpy().reshape(-1, physical_group).sum(axis=1)
            ce = oe.rank_counts.cpu().numpy().reshape(-1, physical_group).sum(axis=1)
            pm.append(int(cm.max()))
            pe.append(int(ce.max()))
    res = {"seeds": seeds, "metro": _summ(lm), "eplb": _summ(le), "metro_per_seed": lm,
           "eplb_over_metro_mean": statistics.mean(e / m for e, m in zip(le, lm) if m > 0) if any(lm) else None,
           "metro_le_eplb_all": all(a <= b for a, b in zip(lm, le)),
           "metro_lt_eplb_batches": sum(a < b for a, b in zip(lm, le))}
    if physical_group > 1:
        res["per_physical_gpu"] = {
            "logical_ranks_per_gpu": physical_group, "gpus": G // physical_group,
            "metro": _summ(pm), "eplb": _summ(pe),
            "metro_le_eplb_all": all(a <= b for a, b in zip(pm, pe)),
            "note": "GPU g hosts logical ranks 2g and 2g+1: activated replicas per GPU = sum of the two columns"}
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=128)
    ap.add_argument("--out", default="gpurun_out/lambda_stats.json")
    a = ap.parse_args()
    sys.path.insert(0, REPO)
    import bench

    out = {}
    for name, cfg in bench.CONFIGS.items():
        r = run(cfg, a.seeds, physical_group=2 if cfg["G"] == 16 else 0)
        r.pop("metro_per_seed")
        out[name] = dict(r, workload=cfg["workload"])
        line = f"{name}: METRO {r['metro']['mean']:.2f} vs EPLB {r['eplb']['mean']:.2f} ({a.seeds} seeds)"
        if "per_physical_gpu" in r:
            line += f"; per GPU {r['per_physical_gpu']['metro']['mean']:.2f} vs {r['per_physical_gpu']['eplb']['mean']:.2f}"
        print(line, flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
