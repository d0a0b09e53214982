"""Per-phase cycle breakdown of the METRO routing kernel (CTA 0 clock64 stamps)
and event timings across cluster sizes.  Usage: python tools/phase_profile.py"""

import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_09277_b200 import DevicePlacement, Router, _native  # noqa: E402
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement  # noqa: E402

CLUSTERS = tuple(int(c) for c in os.environ.get("PROFILE_CLUSTERS", "1,2,4,8,16").split(","))
PHASES = ["stage", "histogram", "exchange", "classify", "sort", "greedy", "outputs"]


def main():
    dev = torch.device("cuda", 0)
    L = _native.lib()
    stamps = torch.zeros(32, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    res = {}
    # floor: a trivial torch kernel right after the L2 flush (launch + reconfig cost)
    tiny = torch.zeros(1, device=dev)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    tt = []
    for _ in range(50):
        flush.zero_()
        e0.record()
        tiny.add_(1)
        e1.record()
        torch.cuda.synchronize()
        tt.append(e0.elapsed_time(e1) * 1e3)
    res["tiny_kernel_after_flush_us"] = float(np.median(tt))
    print("tiny kernel after flush us", res["tiny_kernel_after_flush_us"], flush=True)
    for name, (n, g, ratio, b) in {"ds": (256, 8, 1.5, 1024), "q30": (128, 8, 1.5, 256),
                                   "ds_b64": (256, 8, 1.5, 64), "ds_b8192": (256, 8, 1.5, 8192),
                                   "q235_200": (128, 16, 2.0, 1024)}.items():
        A = make_placement(n, g, ratio, 7).matrix
        ids = torch.from_numpy(gen_zipf_topk(n, 8, b, 1.2, 1000, popularity_seed=7)).to(dev)
        pl = DevicePlacement(A, dev)
        for cl in CLUSTERS:
            r = Router(pl, "metro", cl)
            out = r.alloc(ids.numel(), top_k=8)
            for _ in range(5):
                r.route(ids, out=out)
            L.metro_debug_set_stamps(ctypes.c_void_p(stamps.data_ptr()))
            flush.zero_()
            r.route(ids, out=out)
            torch.cuda.synchronize()
            L.metro_debug_set_stamps(None)
            s = stamps.cpu().numpy()
            cyc = {PHASES[i]: int(s[i + 1] - s[i]) for i in range(7)}
            cyc["total"] = int(s[7] - s[0])
            cyc["sub"] = {"classify_loop": int(s[11] - s[3]), "sync1": int(s[12] - s[11]),
                          "to_sort": int(s[4] - s[12]), "rank_loop_t0": int(s[13] - s[4]),
                          "r2": int(s[8] - s[5]), "r3": int(s[9] - s[8]), "rgen": int(s[10] - s[9]),
                          "greedy_tail": int(s[6] - s[10]),
                          "c_head": int(s[14] - s[3]), "c_body": int(s[17] - s[14]),
                          "c_tail": int(s[11] - s[17]),
                          "x_entrywait": int(s[20] - s[2]), "x_sums_push": int(s[18] - s[20]),
                          "x_arrive": int(s[19] - s[18]), "x_wait": int(s[3] - s[19])}
            # back-to-back graph replay over a pool of distinct batches > L2
            per = ids.numel() * 4
            P = max(64, (256 << 20) // per)
            rows = torch.randint(0, ids.shape[0], (P, ids.shape[0]), device=dev,
                                 generator=torch.Generator(device=dev).manual_seed(1))
            big = ids[rows].contiguous()
            outs = r.alloc(ids.numel(), top_k=8)
            gs = []
            for c0 in range(0, P, 256):
                for j in range(c0, min(P, c0 + 256)):
                    r.route(big[j], out=outs)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for j in range(c0, min(P, c0 + 256)):
                        r.route(big[j], out=outs)
                gs.append(g)
            gs[0].replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for g in gs:
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts = [e0.elapsed_time(e1) * 1e3 / P]
            del gs, big
            # warm: same batch every launch
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(100):
                    r.route(ids, out=outs)
            g.replay()
            torch.cuda.synchronize()
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / 100)
            res[f"{name}/R{cl}"] = {"cycles": cyc, "us_pool": ts[0], "us_l2warm": ts[1]}
            print(name, cl, json.dumps(res[f"{name}/R{cl}"]), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/phase_profile.json", "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
