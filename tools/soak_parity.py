"""Soak parity: many random instances through every device entry point, each
compared bit-exactly with the oracle (test infrastructure).  The pytest suite
samples the same spaces; this runs them for minutes on the GPU box and writes a
tally (the evidence under profiles/<round>_soak.json).

    python tools/soak_parity.py [--seconds 600] [--seed 1] [--out gpurun_out/soak.json]

Entry points: METRO / EPLB routing from ids (every cluster size; a quarter of the
METRO calls through the eager launch plan, Router.bind), METRO from
loads and from an order (metro-parallel), fused gating (cluster + whole GPU),
dispatch layout (standalone and fused with METRO routing), the persistent host router, and the fused exchange with
virtual ranks.  Instances: N 1..700 experts, G 1..128 ranks (multi-word masks),
k 1..10, batches 0..3000 tokens (Zipf or uniform ids, duplicates allowed),
placements from the reference generator or random binary matrices.
"""

import argparse
import json
import os
import re
import sys
import time
import traceback

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2512_09277_b200 import DevicePlacement, Router, ServedRouter, ValidationError  # noqa: E402
from paper_2512_09277_b200.dispatch import DispatchLayout  # noqa: E402
from paper_2512_09277_b200.dist import virtual_ranks  # noqa: E402
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement  # noqa: E402

CLUSTERS = (0, 1, 2, 4, 8, 16)


def instance(rng):
    if rng.random() < 0.3:
        n = int(rng.choice([64, 128, 256]))
        g = int(rng.choice([4, 8, 16]))
        A = make_placement(n, g, float(rng.choice([1.25, 1.5, 2.0])), int(rng.integers(1 << 20))).matrix
    else:
        n = int(rng.integers(1, 700))
        g = int(rng.choice([1, 2, 3, 8, 16, 31, 32, 33, 64, 65, 100, 128]))
        A = (rng.random((n, g)) < rng.uniform(0.0, 0.6)).astype(np.int8)
        empty = np.flatnonzero(A.sum(axis=1) == 0)
        A[empty, rng.integers(0, g, size=empty.size)] = 1
    n = A.shape[0]
    k = int(rng.integers(1, min(10, n) + 1))
    b = int(rng.choice([0, 1, 3, 17, 64, 255, 256, 1000, 1024, 3000]))
    if rng.random() < 0.5 and k <= n:
        ids = gen_zipf_topk(n, k, b, float(rng.uniform(0.3, 2.0)), int(rng.integers(1 << 30)))
    else:
        ids = rng.integers(0, n, size=(b, k)).astype(np.int32)
    return ids, A


def eq(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


def check_route(rng, ids, A):
    pl = DevicePlacement(A)
    cl = int(rng.choice(CLUSTERS))
    t = torch.from_numpy(np.ascontiguousarray(ids)).cuda()
    T = oracle.aggregate_loads(ids, A.shape[0])
    choice, counts, lam = oracle.route_metro(T, A)
    rm = Router(pl, "metro", cl)
    if rng.random() < 0.25 and ids.size > 0:
        # the eager launch plan (metro_route_plan_create/launch_v1) instead of route()
        o = rm.bind(t.reshape(-1))().check()
    else:
        o = rm.route(t).check()
    ok = (eq(o.loads.cpu(), T) and eq(o.choice.cpu(), choice) and eq(o.rank_counts.cpu(), counts)
          and int(o.lam.item()) == lam and eq(o.pair_rank.cpu().numpy().reshape(ids.shape),
                                              oracle.pair_rank_metro(ids, choice)))
    x, ec, el = oracle.route_eplb(T, A)
    e = Router(pl, "eplb", cl).route(t, with_x=True).check()
    ok_e = (eq(e.x.cpu(), x) and eq(e.rank_counts.cpu(), ec) and int(e.lam.item()) == el
            and eq(e.pair_rank.cpu().numpy().reshape(ids.shape), oracle.pair_rank_eplb(ids, A)))
    return {"metro_ids": ok, "eplb_ids": ok_e}, pl, t, choice, o


def check_loads_order(rng, ids, A):
    """The reference-compatible numpy API: route_metro(T, A) (metro_route_from_loads_v1)
    and route_metro_parallel(T, A, seed) (metro_route_ordered_v1, seeded shuffle)."""
    import paper_2512_09277_b200 as pkg

    n, g = A.shape
    T = oracle.aggregate_loads(ids, n).astype(np.int64)
    if rng.random() < 0.2:  # loads far above any batch (compat path rank-compresses them)
        T = T * int(rng.integers(1, 1 << 30))
    choice, counts, lam = oracle.route_metro(T, A)
    m = pkg.route_metro(T, A)
    y = np.zeros((n, g), np.int8)
    act = np.flatnonzero(choice >= 0)
    y[act, choice[act]] = 1
    res = {"metro_loads": eq(m.y, y) and m.lam == lam}
    seed = int(rng.integers(1 << 30))
    order = [int(i) for i in np.flatnonzero(T)]
    np.random.default_rng(seed).shuffle(order)
    oc, ocnt, olam = oracle.route_metro_order(T, A, np.asarray(order, np.int32))
    mp = pkg.route_metro_parallel(T, A, seed)
    yp = np.zeros((n, g), np.int8)
    act = np.flatnonzero(oc >= 0)
    yp[act, oc[act]] = 1
    res["metro_parallel"] = eq(mp.y, yp) and mp.lam == olam
    return res


def check_gate(rng, A):
    n, g = A.shape
    if n > 512 or g > 32:
        return {}
    k = int(rng.integers(1, min(32, n) + 1))
    B = int(rng.choice([1, 31, 256, 513, 1024, 2049]))
    u = rng.random()
    if u < 0.25:  # heavy ties: small integers
        sc = rng.integers(-3, 4, size=(B, n)).astype(np.float32)
    elif u < 0.45:  # signed zeros, NaN, +-inf among a few values (key-order edge cases)
        vals = np.array([-0.0, 0.0, -0.0, 0.0, 1.0, -1.0, np.inf, -np.inf, np.nan, 0.5], np.float32)
        sc = vals[rng.integers(0, len(vals), size=(B, n))]
    else:
        sc = rng.standard_normal((B, n)).astype(np.float32)
    r = Router(DevicePlacement(A), "metro", int(rng.choice([0, 1, 4, 16])))
    whole = [None, True, False][int(rng.integers(3))]
    ids, o = r.route_scores(torch.from_numpy(sc).cuda(), k, whole_gpu=whole)
    o.check()
    ref = oracle.gate_topk(sc, k)
    T = oracle.aggregate_loads(ref, n)
    choice, counts, lam = oracle.route_metro(T, A)
    return {"gate": eq(ids.cpu(), ref) and eq(o.choice.cpu(), choice) and int(o.lam.item()) == lam
            and eq(o.pair_rank.cpu().numpy().reshape(ref.shape), oracle.pair_rank_metro(ref, choice))}


def check_dispatch(ids, A, pl, t, o):
    if ids.size == 0:
        return {}
    lay = DispatchLayout(pl)
    res = lay(t, o.pair_rank.view(t.shape)).check()
    row, off = oracle.dispatch_layout(ids, o.pair_rank.cpu().numpy().reshape(ids.shape), A)
    ok = (eq(res.pair_row.cpu().numpy().reshape(-1), np.asarray(row).reshape(-1))
          and eq(res.rep_off.cpu().numpy()[:len(off)], off))
    # routing + layout fused in one launch (metro_route_layout_v1): must equal the chain
    fo, fl = DispatchLayout(pl, int(np.random.default_rng(ids.size).choice(CLUSTERS))).route_metro(t)
    fo.check()
    okf = (eq(fo.choice.cpu(), o.choice.cpu()) and eq(fo.pair_rank.cpu(), o.pair_rank.cpu())
           and int(fo.lam.item()) == int(o.lam.item())
           and eq(fl.pair_row.cpu().numpy()[:ids.size], np.asarray(row).reshape(-1))
           and eq(fl.rep_off.cpu().numpy()[:len(off)], off))
    return {"dispatch": ok, "route_layout_fused": okf}


def check_served(ids, A, pl):
    # one server per check, closed right after: its resident CTA would otherwise
    # hold every device-wide synchronise of the other checks for its idle timeout
    with ServedRouter(pl, max(ids.size, 4)) as sr:
        out = sr.route(ids).copy()
        pr = sr.pair_rank.numpy()[:ids.size].copy()
    n, g = A.shape
    T = oracle.aggregate_loads(ids, n)
    ch, counts, lam = oracle.route_metro(T, A)
    return {"served": int(out[4]) == lam and eq(out[8:8 + g], counts) and eq(out[8 + g:8 + g + n], ch)
            and eq(pr, oracle.pair_rank_metro(ids, ch).reshape(-1))}


def check_exchange(rng, ids, A, pl):
    world = int(rng.choice([2, 4, 8]))
    B, k = ids.shape
    if B % world or B == 0 or A.shape[1] > 32 or A.shape[0] > 512:
        return {}
    lt = B // world
    # every other call: the fused exchange + global dispatch layout variant
    # (metro_allgather_route_layout_v1: histograms only, no ids gather)
    with_layout = bool(rng.integers(2)) and int(A.sum()) <= 4096
    lay = DispatchLayout(pl) if with_layout else None
    routers, bufs = virtual_ranks(pl, world, lt, k, gather_ids=not with_layout, layout=lay)
    streams = [torch.cuda.Stream() for _ in range(world)]
    try:
        shards = [torch.from_numpy(np.ascontiguousarray(ids[r * lt:(r + 1) * lt])).cuda() for r in range(world)]
        for r, (rt, sh) in enumerate(zip(routers, shards)):
            with torch.cuda.stream(streams[r]):
                rt.step(sh, stream=streams[r])
        torch.cuda.synchronize()
        T = oracle.aggregate_loads(ids, A.shape[0])
        choice, counts, lam = oracle.route_metro(T, A)
        if with_layout:
            row, off = oracle.dispatch_layout(ids, oracle.pair_rank_metro(ids, choice), A)
            row = np.asarray(row).reshape(-1)
        ok = True
        for rt in routers:
            rt.out.check()
            own = ids[rt.rank * lt:(rt.rank + 1) * lt]
            ok = ok and eq(rt.out.choice.cpu(), choice) and int(rt.out.lam.item()) == lam and \
                eq(rt.out.pair_rank.cpu().numpy().reshape(own.shape), oracle.pair_rank_metro(own, choice))
            if with_layout:
                ok = ok and eq(rt.layout_out.pair_row.cpu().numpy()[:lt * k], row[rt.rank * lt * k:(rt.rank + 1) * lt * k]) \
                    and eq(rt.layout_out.rep_off.cpu().numpy()[:len(off)], off)
            else:
                ok = ok and eq(rt.gathered.cpu(), ids)
        return {"exchange_layout" if with_layout else "exchange": ok}
    finally:
        for b in bufs:
            b.close()


def run(seconds: float, seed: int = 1) -> dict:
    """Random instances through every device entry point for `seconds`; returns
    the tally (instances, per-check run / mismatch counts, failures)."""
    rng = np.random.default_rng(seed)
    tally, fails, skipped = {}, [], {}
    t_end = time.time() + seconds
    it = 0
    while time.time() < t_end:
        it += 1
        ids, A = instance(rng)
        res = {}
        try:
            r0, pl, t, choice, o = check_route(rng, ids, A)
            res.update(r0)
            steps = [lambda: check_loads_order(rng, ids, A)]
            if it % 3 == 0:
                steps.append(lambda: check_gate(rng, A))
            if it % 2 == 0:
                steps.append(lambda: check_dispatch(ids, A, pl, t, o))
            if it % 5 == 0 and ids.size <= 30000:
                steps.append(lambda: check_served(ids, A, pl))
            if it % 7 == 0:
                steps.append(lambda: check_exchange(rng, ids, A, pl))
            for f in steps:
                try:
                    res.update(f())
                except ValidationError as ex:  # a documented host-side limit, not a parity result
                    if "limit" in str(ex) or "unsupported dimensions" in str(ex):
                        key = re.sub(r"\d+", "#", str(ex).split(":")[0])[:80]
                        skipped[key] = skipped.get(key, 0) + 1
                    else:
                        raise
        except Exception:  # noqa: BLE001 -- a crash is a failure, recorded with its instance
            res["exception"] = False
            fails.append({"iter": it, "N": A.shape[0], "G": A.shape[1], "shape": list(ids.shape),
                          "trace": traceback.format_exc()[-600:]})
        for key, ok in res.items():
            c = tally.setdefault(key, [0, 0])
            c[0] += 1
            c[1] += 0 if ok else 1
            if not ok and len(fails) < 20 and key != "exception":
                fails.append({"iter": it, "check": key, "N": A.shape[0], "G": A.shape[1], "shape": list(ids.shape)})
    return {"seconds": seconds, "seed": seed, "instances": it,
            "checks": {k: {"run": v[0], "mismatches": v[1]} for k, v in sorted(tally.items())},
            "skipped_outside_documented_limits": skipped,
            "failures": fails}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=600)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--out", default="gpurun_out/soak.json")
    a = ap.parse_args()
    summary = run(a.seconds, a.seed)
    fails = summary["failures"]
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps({k: summary[k] for k in ("instances", "checks")}))
    print("failures:", len(fails))


if __name__ == "__main__":
    main()
