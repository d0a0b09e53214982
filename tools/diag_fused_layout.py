"""Diagnose route_layout_fused mismatches: random soak-style instances through
DispatchLayout.route_metro at every cluster size, compared field by field with
the two-launch chain and the oracle.  python tools/diag_fused_layout.py [seconds]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import oracle  # noqa: E402
from paper_2512_09277_b200 import DevicePlacement, Router, ValidationError  # noqa: E402
from paper_2512_09277_b200.dispatch import DispatchLayout  # noqa: E402
from soak_parity import instance  # noqa: E402


def main():
    seconds = float(sys.argv[1]) if len(sys.argv) > 1 else 60
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
    t_end = time.time() + seconds
    stats, fails = {}, []
    while time.time() < t_end:
        ids, A = instance(rng)
        if ids.size == 0:
            continue
        pl = DevicePlacement(A)
        t = torch.from_numpy(np.ascontiguousarray(ids)).cuda()
        T = oracle.aggregate_loads(ids, A.shape[0])
        choice, counts, lam = oracle.route_metro(T, A)
        prk = oracle.pair_rank_metro(ids, choice)
        row, off = oracle.dispatch_layout(ids, prk, A)
        row = np.asarray(row).reshape(-1)
        for cl in (0, 1, 2, 4, 8, 16):
            try:
                fo, fl = DispatchLayout(pl, cl).route_metro(t)
                fo.check()
            except ValidationError as ex:
                stats.setdefault("skip", 0)
                stats["skip"] += 1
                continue
            torch.cuda.synchronize()
            bad = []
            if not np.array_equal(fo.choice.cpu().numpy(), choice):
                bad.append("choice")
            if int(fo.lam.item()) != lam:
                bad.append("lam")
            fpr = fo.pair_rank.cpu().numpy()[:ids.size]
            if not np.array_equal(fpr, prk.reshape(-1)):
                bad.append("pair_rank")
            frow = fl.pair_row.cpu().numpy()[:ids.size]
            if not np.array_equal(frow, row):
                bad.append("pair_row")
            foff = fl.rep_off.cpu().numpy()[:len(off)]
            if not np.array_equal(foff, off):
                bad.append("rep_off")
            key = f"cl{cl}"
            s = stats.setdefault(key, [0, 0])
            s[0] += 1
            if bad:
                s[1] += 1
                d = {"cl": cl, "N": A.shape[0], "G": A.shape[1], "B": ids.shape[0], "k": ids.shape[1],
                     "nrep": int(A.sum()), "bad": bad, "status": fo.status.cpu().tolist()}
                if "pair_row" in bad:
                    w = np.flatnonzero(frow != row)
                    d["row_ndiff"] = int(w.size)
                    d["row_first"] = int(w[0])
                    d["row_vals"] = [frow[w[:4]].tolist(), row[w[:4]].tolist()]
                if "rep_off" in bad:
                    w = np.flatnonzero(foff != off)
                    d["off_ndiff"] = int(w.size)
                    d["off_first"] = int(w[0])
                if "pair_rank" in bad:
                    w = np.flatnonzero(fpr != prk.reshape(-1))
                    d["pr_ndiff"] = int(w.size)
                    d["pr_first"] = int(w[0])
                if len(fails) < 60:
                    fails.append(d)
    out = {"stats": stats, "fails": fails}
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/diag_fused.json", "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(stats))
    for d in fails[:40]:
        print(json.dumps(d))


if __name__ == "__main__":
    main()
