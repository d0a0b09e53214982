"""Bit-exact parity of the sm_100a kernels against the CPU oracle (-m gpu).

The oracle (oracle/metro_oracle.c) is itself pinned to the unmodified reference by
tests/test_oracle_golden.py; here the CUDA path is compared with it on the
reference's golden fixtures, the BASELINE shapes at every cluster size, random
fuzz over N/G/k/B (incl. multi-word rank masks, duplicates, ragged sizes) and
the reference's error cases.  Integer work: equality, no tolerance.
"""

import numpy as np
import pytest
import torch

import oracle
import paper_2512_09277_b200 as pkg
from paper_2512_09277_b200 import DevicePlacement, HostRouter, Router
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement

pytestmark = pytest.mark.gpu

CLUSTERS = (0, 1, 2, 4, 8, 16)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.init()


def metro_dev(ids, A, cluster=0, pair=True):
    pl = DevicePlacement(A)
    ids_t = torch.as_tensor(np.ascontiguousarray(ids, dtype=np.int32)).cuda()
    out = Router(pl, "metro", cluster).route(ids_t, pair_rank=pair).check()
    return dict(
        loads=out.loads.cpu().numpy(), choice=out.choice.cpu().numpy(),
        counts=out.rank_counts.cpu().numpy(), lam=int(out.lam.item()),
        pair=None if out.pair_rank is None else out.pair_rank.cpu().numpy().reshape(np.shape(ids)),
        status=out.status.cpu().numpy(),
    )


def eplb_dev(ids, A, cluster=0, pair=True):
    pl = DevicePlacement(A)
    ids_t = torch.as_tensor(np.ascontiguousarray(ids, dtype=np.int32)).cuda()
    out = Router(pl, "eplb", cluster).route(ids_t, pair_rank=pair, with_x=True).check()
    return dict(
        loads=out.loads.cpu().numpy(), x=out.x.cpu().numpy(), counts=out.rank_counts.cpu().numpy(),
        lam=int(out.lam.item()),
        pair=None if out.pair_rank is None else out.pair_rank.cpu().numpy().reshape(np.shape(ids)),
    )


def check_metro(ids, A, cluster=0):
    A = np.asarray(A, dtype=np.int8)
    T = oracle.aggregate_loads(ids, A.shape[0])
    choice, counts, lam = oracle.route_metro(T, A)
    d = metro_dev(ids, A, cluster)
    assert np.array_equal(d["loads"], T)
    assert np.array_equal(d["choice"], choice)
    assert np.array_equal(d["counts"], counts)
    assert d["lam"] == lam
    assert np.array_equal(d["pair"], oracle.pair_rank_metro(ids, choice))
    return d


def check_eplb(ids, A, cluster=0):
    A = np.asarray(A, dtype=np.int8)
    T = oracle.aggregate_loads(ids, A.shape[0])
    x, counts, lam = oracle.route_eplb(T, A)
    d = eplb_dev(ids, A, cluster)
    assert np.array_equal(d["loads"], T)
    assert np.array_equal(d["x"], x)
    assert np.array_equal(d["counts"], counts)
    assert d["lam"] == lam
    assert np.array_equal(d["pair"], oracle.pair_rank_eplb(ids, A))
    return d


# ------------------------------------------------------------------ golden shapes
def test_golden_shapes_all_clusters(shapes):
    for c in shapes:
        for cl in CLUSTERS:
            d = check_metro(c["ids"], c["A"], cl)
            # and against the reference's own outputs directly
            assert np.array_equal(d["choice"], c["metro_choice"]), (c["name"], cl)
            assert d["lam"] == c["metro_lam"]
            e = check_eplb(c["ids"], c["A"], cl)
            assert np.array_equal(e["x"], c["eplb_x"])
            assert e["lam"] == c["eplb_lam"]
            assert d["lam"] <= e["lam"]  # METRO <= EPLB on every golden batch


def test_golden_small_families_compat(small):
    """Reference test families through the drop-in numpy API (loads path)."""
    for c in small:
        T = pkg.ExpertLoadVector(c["T"])
        A = pkg.PlacementMap(c["A"], 1)
        m = pkg.route_metro(T, A)
        y = np.zeros_like(c["A"])
        act = c["metro_choice"] >= 0
        y[np.flatnonzero(act), c["metro_choice"][act]] = 1
        assert np.array_equal(m.y, y) and m.lam == c["metro_lam"]
        assert np.array_equal(m.x, y.astype(np.int64) * c["T"][:, None])
        e = pkg.route_eplb(T, A)
        assert np.array_equal(e.x, c["eplb_x"]) and e.lam == c["eplb_lam"]
        assert pkg.validate_assignment(m, A, T, require_single_replica=True).ok


# ------------------------------------------------------------------ fuzz
def _random_instance(rng):
    n = int(rng.integers(1, 700))
    g = int(rng.choice([1, 2, 3, 8, 16, 31, 32, 33, 64, 65, 100, 128]))
    dens = rng.uniform(0.0, 0.6)
    A = (rng.random((n, g)) < dens).astype(np.int8)
    empty = np.flatnonzero(A.sum(axis=1) == 0)
    A[empty, rng.integers(0, g, size=empty.size)] = 1
    k = int(rng.integers(1, min(10, n) + 1))
    b = int(rng.choice([0, 1, 3, 17, 64, 255, 1024, 3000]))
    if rng.random() < 0.5:
        ids = gen_zipf_topk(n, k, b, float(rng.uniform(0.3, 2.0)), int(rng.integers(1 << 30)))
    else:  # duplicates within a token allowed (aggregate_loads counts them twice)
        ids = rng.integers(0, n, size=(b, k)).astype(np.int32)
    return ids, A


def test_fuzz_metro_eplb():
    rng = np.random.default_rng(2024)
    for it in range(250):
        ids, A = _random_instance(rng)
        cl = int(rng.choice(CLUSTERS))
        check_metro(ids, A, cl)
        if A.shape[0] <= 2048:
            check_eplb(ids, A, cl)


def test_baseline_shapes_many_seeds():
    for (n, g, ratio, b) in [(128, 8, 1.5, 256), (256, 8, 1.5, 1024), (128, 16, 1.25, 1024),
                             (128, 16, 1.5, 1024), (128, 16, 2.0, 1024), (256, 8, 1.5, 64),
                             (256, 8, 1.5, 8192)]:
        A = make_placement(n, g, ratio, 7).matrix
        for seed in range(3000, 3000 + (4 if b >= 8192 else 25)):
            ids = gen_zipf_topk(n, 8, b, 1.2, seed, popularity_seed=7)
            d = check_metro(ids, A)
            e = eplb_dev(ids, A, pair=False)
            assert d["lam"] <= e["lam"]


# ------------------------------------------------------------------ edges
def test_empty_and_tiny():
    A = np.array([[1, 1], [1, 0], [0, 1]], dtype=np.int8)
    d = check_metro(np.zeros((0, 2), np.int32), A)
    assert d["lam"] == 0 and (d["choice"] == -1).all() and (d["counts"] == 0).all()
    check_metro(np.array([[2]], np.int32), A)
    check_metro(np.array([[0, 1], [1, 2], [2, 0]], np.int32), A, 16)
    check_eplb(np.zeros((0, 2), np.int32), A)
    check_eplb(np.array([[0, 0], [0, 0], [0, 0]], np.int32), A, 2)


def test_unaligned_ids_view():
    A = make_placement(256, 8, 1.5, 7).matrix
    ids = gen_zipf_topk(256, 8, 513, 1.2, 5).reshape(-1)
    t = torch.from_numpy(ids).cuda()
    for off in (1, 2, 3):
        view = t[off:off + 4097]  # not 16-byte aligned: scalar staging path
        T = oracle.aggregate_loads(view.cpu().numpy(), 256)
        choice, counts, lam = oracle.route_metro(T, A)
        for cl in (1, 4, 16):
            out = Router(DevicePlacement(A), "metro", cl).route(view).check()
            assert np.array_equal(out.choice.cpu().numpy(), choice)
            assert np.array_equal(out.pair_rank.cpu().numpy(), oracle.pair_rank_metro(view.cpu().numpy(), choice))


def test_max_sizes():
    rng = np.random.default_rng(9)
    n, g = 4096, 128
    A = (rng.random((n, g)) < 0.02).astype(np.int8)
    A[np.flatnonzero(A.sum(1) == 0), 0] = 1
    ids = rng.integers(0, n, size=(4096, 8)).astype(np.int32)
    check_metro(ids, A, 0)  # auto plan shrinks the cluster until the layout fits
    check_metro(ids, A, 2)
    with pytest.raises(pkg.ValidationError, match="shared memory"):
        metro_dev(ids, A, 16)  # 16 partial rows of 4096 experts cannot fit 227 KB
    ids = gen_zipf_topk(256, 8, 32768, 1.2, 3)  # 262144 pairs
    check_metro(ids, make_placement(256, 8, 1.5, 7).matrix, 16)


def test_packed_greedy_fallback():
    """Ranks hosting > 126 active experts leave the byte-packed greedy's range; the
    kernel must detect it and fall back to the warp greedy (still bit-exact)."""
    rng = np.random.default_rng(31)
    for n, g in [(300, 2), (256, 2), (400, 4), (256, 8)]:
        A = np.ones((n, g), dtype=np.int8)
        ids = rng.integers(0, n, size=(2048, 8)).astype(np.int32)
        for cl in (0, 1, 4):
            check_metro(ids, A, cl)
    # one rank hosting every expert (a counter could pass 255 without the guard)
    A = np.zeros((256, 4), dtype=np.int8)
    A[:, 0] = 1
    A[::3, 1] = 1
    ids = np.arange(256 * 8, dtype=np.int32).reshape(-1, 8) % 256
    check_metro(ids, A, 0)


def test_r2_single_step_threshold():
    """The packed greedy steps the r = 2 segment one at a time below
    METRO_R2_BLOCK_MIN (48) replicated active experts and in blocks of four
    (with the delta table) from 48 up: replicated-expert counts straddling the
    threshold, every r = 2 segment length mod 4, mixes of r = 2 / 3 / >= 4."""
    rng = np.random.default_rng(48)
    n, g = 256, 8
    for m in (0, 1, 2, 3, 4, 5, 31, 46, 47, 48, 49, 50, 51, 63, 64, 85, 120):
        for trial in range(2):
            A = np.zeros((n, g), dtype=np.int8)
            A[np.arange(n), rng.integers(0, g, size=n)] = 1
            multi = rng.choice(n, size=m, replace=False)
            for e in multi:
                r = int(rng.choice([2, 2, 2, 3, 4, 6]))
                A[e, rng.choice(g, size=r, replace=False)] = 1
                A[e] = np.minimum(A[e], 1)
            ids = rng.integers(0, n, size=(1024, 8)).astype(np.int32)
            ids[0] = np.arange(8)  # a few fixed ids; every expert is active at 8192 pairs w.h.p.
            for cl in (0, 1, 4):
                check_metro(ids, A, cl)


def test_id_out_of_range_error():
    A = make_placement(128, 8, 1.5, 7).matrix
    ids = gen_zipf_topk(128, 8, 256, 1.2, 1)
    ids[77, 3] = 128
    ids[200, 0] = -5
    for cl in (1, 8):
        with pytest.raises(pkg.ValidationError, match="token 77: expert id 128 out of range"):
            metro_dev(ids, A, cl)
        with pytest.raises(pkg.ValidationError, match="token 77: expert id 128 out of range"):
            eplb_dev(ids, A, cl)
    model = pkg.ModelSpec(128, 8, 64, 2, 1.0, 0.0, 1.0, 1)
    with pytest.raises(pkg.ValidationError, match="token 77: expert id 128 out of range"):
        pkg.aggregate_loads(pkg.TokenBatch.from_topk(ids, 8), model)


def test_active_expert_without_replica():
    A = np.array([[1, 1], [0, 0]], dtype=np.int8)
    with pytest.raises(AssertionError):
        metro_dev(np.array([[0, 1]], np.int32), A)
    with pytest.raises(AssertionError):
        eplb_dev(np.array([[0, 1]], np.int32), A)
    with pytest.raises(AssertionError):
        pkg.route_metro(pkg.ExpertLoadVector([1, 1]), pkg.PlacementMap(A, 1))
    # an inactive expert without replica is fine (reference only asserts on active ones)
    check_metro(np.array([[0, 0]], np.int32), A)


# ------------------------------------------------------------------ compat paths
def test_compat_huge_loads_and_parallel():
    rng = np.random.default_rng(77)
    for _ in range(60):
        n = int(rng.integers(1, 90))
        g = int(rng.integers(1, 40))
        A = (rng.random((n, g)) < 0.3).astype(np.int8)
        A[np.flatnonzero(A.sum(1) == 0), 0] = 1
        T = (rng.integers(0, 2 ** 40, size=n) * (rng.random(n) < 0.7)).astype(np.int64)
        choice, _, lam = oracle.route_metro(T, A)
        m = pkg.route_metro(pkg.ExpertLoadVector(T), pkg.PlacementMap(A, 1))
        assert m.lam == lam
        act = choice >= 0
        assert np.array_equal(np.flatnonzero(m.y.sum(1)), np.flatnonzero(act))
        assert (m.y[np.flatnonzero(act), choice[act]] == 1).all()
        x, _, elam = oracle.route_eplb(T, A)
        e = pkg.route_eplb(T, A)
        assert np.array_equal(e.x, x) and e.lam == elam
        seed = int(rng.integers(1000))
        active = [int(i) for i in np.flatnonzero(T)]
        np.random.default_rng(seed).shuffle(active)
        pc, _, plam = oracle.route_metro_order(T, A, active)
        p = pkg.route_metro_parallel(pkg.ExpertLoadVector(T), pkg.PlacementMap(A, 1), seed)
        assert p.lam == plam
        assert (p.y[np.flatnonzero(pc >= 0), pc[pc >= 0]] == 1).all()
        assert pkg.run_router("metro-parallel", T, A, seed=seed).lam == plam


def test_aggregate_loads_compat(shapes):
    c = shapes[0]
    model = pkg.ModelSpec(c["N"], c["k"], 64, 2, 1.0, 0.0, 1.0, 1)
    T = pkg.aggregate_loads(pkg.TokenBatch.from_topk(c["ids"], c["G"]), model)
    assert np.array_equal(T.loads, c["T"])
    assert np.array_equal(pkg.aggregate_loads(torch.from_numpy(c["ids"]).cuda(), model).loads, c["T"])
    assert pkg.aggregate_loads(pkg.TokenBatch(), model).total() == 0


# ------------------------------------------------------------------ graph + host e2e
def test_cuda_graph_replay(shapes):
    c = [s for s in shapes if s["name"] == "ds"][0]
    pl = DevicePlacement(c["A"])
    r = Router(pl, "metro")
    static_ids = torch.from_numpy(c["ids"]).cuda()
    out = r.alloc(static_ids.numel(), top_k=8)
    r.route(static_ids, out=out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        r.route(static_ids, out=out)
    for s in [x for x in shapes if x["name"] == "ds"]:
        static_ids.copy_(torch.from_numpy(s["ids"]).cuda())
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(out.choice.cpu().numpy(), s["metro_choice"])
        assert int(out.lam.item()) == s["metro_lam"]


def test_host_router_owned_buffers(shapes):
    for zc in (True, False):
        for c in shapes[:10]:
            pl = DevicePlacement(c["A"])
            hr = HostRouter(pl, max_pairs=c["ids"].size, zero_copy=zc)
            for rep in range(2):
                hr.ids.numpy()[:c["ids"].size] = c["ids"].reshape(-1)
                out = hr.run(c["ids"].size)
                n, g = c["N"], c["G"]
                assert out[0] == 0 and out[4] == c["metro_lam"]
                assert np.array_equal(out[8:8 + g], c["metro_counts"])
                assert np.array_equal(out[8 + g:8 + g + n], c["metro_choice"])
                assert np.array_equal(hr.pair_rank.numpy()[:c["ids"].size],
                                      oracle.pair_rank_metro(c["ids"].reshape(-1), c["metro_choice"]))


def test_host_router_e2e(shapes):
    for c in shapes[:12]:
        pl = DevicePlacement(c["A"])
        hr = HostRouter(pl, max_pairs=c["ids"].size)
        ids_h = torch.from_numpy(c["ids"].reshape(-1).copy()).pin_memory()
        pr = torch.empty(c["ids"].size, dtype=torch.int32).pin_memory()
        out = hr(ids_h, pr)
        n, g = c["N"], c["G"]
        assert out[0] == 0
        assert out[4] == c["metro_lam"]
        assert np.array_equal(out[8:8 + g], c["metro_counts"])
        assert np.array_equal(out[8 + g:8 + g + n], c["metro_choice"])
        assert np.array_equal(pr.numpy(), oracle.pair_rank_metro(c["ids"].reshape(-1), c["metro_choice"]))


def test_pdl_chain_in_one_graph(shapes):
    """Programmatic dependent launch inside a CUDA graph: each routing kernel
    reads ids written by the kernel right before it (a copy kernel standing in
    for the gating kernel), 64 layers back to back -- every layer must see its
    own batch.  The same with PDL off."""
    from paper_2512_09277_b200 import _native

    cs = [s for s in shapes if s["name"] == "ds"]
    pl = DevicePlacement(cs[0]["A"])
    r = Router(pl, "metro")
    src = [torch.from_numpy(s["ids"]).cuda() for s in cs]
    L = 64
    ids = torch.empty((L,) + tuple(src[0].shape), dtype=torch.int32, device="cuda")
    outs = [r.alloc(src[0].numel(), top_k=8) for _ in range(L)]
    for pdl in (1, 0):
        _native.lib().metro_set_pdl(pdl)
        try:
            ids.zero_()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for j in range(L):
                    ids[j].copy_(src[j % len(src)])  # the "producer" kernel of layer j
                    r.route(ids[j], out=outs[j])
            g.replay()
            torch.cuda.synchronize()
            for j in range(L):
                s = cs[j % len(cs)]
                assert np.array_equal(outs[j].choice.cpu().numpy(), s["metro_choice"]), (pdl, j)
                assert int(outs[j].lam.item()) == s["metro_lam"]
        finally:
            _native.lib().metro_set_pdl(1)


def test_bound_plan_eager_loop(shapes):
    """Router.bind (metro_route_plan_*): one plan per (buffers, batch size), the
    ids refilled in place between launches, METRO and EPLB, every cluster size --
    identical to route() and to the reference's golden outputs; route() with a
    reused result set (checked once) stays exact too."""
    from paper_2512_09277_b200 import _native

    for name in ("ds", "q30", "q235_200"):
        cs = [s for s in shapes if s["name"] == name]
        if not cs:
            continue
        pl = DevicePlacement(cs[0]["A"])
        for cl in (0, 1, 4):
            ids = torch.empty(cs[0]["ids"].shape, dtype=torch.int32, device="cuda")
            plan = Router(pl, "metro", cl).bind(ids)
            eplan = Router(pl, "eplb", cl).bind(ids, with_x=True)
            r = Router(pl, "metro", cl)
            reuse = r.alloc(ids.numel(), top_k=ids.shape[1])
            for s in cs:
                ids.copy_(torch.from_numpy(s["ids"]))
                o = plan().check()
                e = eplan().check()
                q = r.route(ids, out=reuse).check()
                assert np.array_equal(o.choice.cpu().numpy(), s["metro_choice"]), (name, cl)
                assert int(o.lam.item()) == s["metro_lam"]
                assert np.array_equal(o.pair_rank.cpu().numpy(), oracle.pair_rank_metro(s["ids"].reshape(-1),
                                                                                        s["metro_choice"]))
                assert np.array_equal(q.choice.cpu().numpy(), s["metro_choice"])
                assert np.array_equal(e.x.cpu().numpy(), s["eplb_x"])
                assert int(e.lam.item()) == s["eplb_lam"]
            plan.close()
            with pytest.raises(pkg.ValidationError):
                plan()
    # a plan is capturable like route()
    c = [s for s in shapes if s["name"] == "ds"][0]
    pl = DevicePlacement(c["A"])
    ids = torch.from_numpy(c["ids"]).cuda()
    plan = Router(pl, "metro").bind(ids)
    plan()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        plan_g = Router(pl, "metro").bind(ids, out=plan.out, stream=torch.cuda.current_stream())
        plan_g()
    plan.out.lam.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert int(plan.out.lam.item()) == c["metro_lam"]
    assert _native.lib() is not None
