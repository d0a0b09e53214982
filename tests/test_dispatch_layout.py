"""Dispatch layout after routing (include/dispatch_layout.h).

CPU: the oracle's layout reproduces the reference's assignment x (rows of
replica (i, g) = x[i, g], routing.py:41-52 / :64-69) on the golden shapes, and
the replica table matches its definition.  GPU (-m gpu): the sm_100a kernel is
bit-exact against the oracle for METRO and EPLB pair ranks at every cluster
size, on fuzz, ragged/empty/maximum sizes and the error cases.
"""

import os
import numpy as np
import pytest
import torch

import oracle
from paper_2512_09277_b200 import DevicePlacement, DispatchLayout, Router, ValidationError, replica_table
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement


def _rid_numpy(A):
    A = np.asarray(A) != 0
    n, g = A.shape
    rid = -np.ones((n, g), np.int32)
    base = np.zeros(g + 1, np.int32)
    r = 0
    for j in range(g):
        base[j] = r
        for i in range(n):
            if A[i, j]:
                rid[i, j] = r
                r += 1
    base[g] = r
    return rid, base


def _check_layout_props(ids, pr, A, row, off, x_ref):
    """rows of replica (i, g) = x_ref[i, g]; rows of a rank are a permutation of
    0..rows-1; pairs of one replica occupy its rows in ascending pair order."""
    rid, base = _rid_numpy(A)
    ids, pr = ids.reshape(-1), pr.reshape(-1)
    n, g = np.asarray(A).shape
    cnt = np.diff(off)
    for i in range(n):
        for j in range(g):
            if rid[i, j] >= 0:
                assert cnt[rid[i, j]] == x_ref[i, j]
            else:
                assert x_ref[i, j] == 0
    for j in range(g):
        sel = pr == j
        rows = np.sort(row[sel])
        assert (rows == np.arange(sel.sum())).all()
    key = rid[ids, pr]
    for r in np.unique(key):
        rr = row[key == r]
        assert (np.diff(rr) == 1).all()


def test_replica_table_matches_definition():
    rng = np.random.default_rng(0)
    for _ in range(20):
        n, g = rng.integers(1, 40), rng.integers(1, 20)
        A = (rng.random((n, g)) < 0.3).astype(np.int8)
        rid, base = replica_table(A)
        r2, b2 = _rid_numpy(A)
        assert (rid == r2).all() and (base == b2).all()
    with pytest.raises(ValidationError):
        replica_table(np.array([[2, 0]], np.int8))


def test_oracle_layout_known_answer():
    A = np.array([[1, 1, 0], [0, 1, 1], [1, 0, 1]], np.int8)
    row, off = oracle.dispatch_layout([0, 1, 2, 0, 1, 0], [0, 2, 2, 1, 1, 0], A)
    assert row.tolist() == [0, 0, 1, 0, 1, 1]
    assert off.tolist() == [0, 2, 2, 3, 4, 5, 6]
    with pytest.raises(oracle.OracleError):
        oracle.dispatch_layout([0, 5], [0, 0], A)
    with pytest.raises(oracle.OracleError):
        oracle.dispatch_layout([0, 1], [0, 0], A)  # expert 1 not on rank 0


def test_oracle_layout_reproduces_reference_x(shapes):
    for c in shapes[:12]:
        ids, A = c["ids"], c["A"]
        choice = c["metro_choice"]
        pm = oracle.pair_rank_metro(ids, choice)
        xm = np.zeros(A.shape, np.int64)
        act = choice >= 0
        xm[np.flatnonzero(act), choice[act]] = c["T"][act]
        row, off = oracle.dispatch_layout(ids, pm, A)
        _check_layout_props(ids, pm, A, row, off, xm)
        pe = oracle.pair_rank_eplb(ids, A)
        row, off = oracle.dispatch_layout(ids, pe, A)
        _check_layout_props(ids, pe, A, row, off, c["eplb_x"])


# ---------------------------------------------------------------- GPU parity


@pytest.fixture(scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.init()


def _dev_layout(ids, pr, A, cluster=0):
    pl = DevicePlacement(A)
    dl = DispatchLayout(pl, cluster)
    it = torch.as_tensor(np.ascontiguousarray(ids, np.int32)).cuda()
    pt = torch.as_tensor(np.ascontiguousarray(pr, np.int32)).cuda()
    out = dl(it, pt).check()
    P = int(np.size(ids))
    return out.pair_row.cpu().numpy()[:P], out.rep_off.cpu().numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("cluster", [0, 1, 2, 4, 8, 16])
def test_layout_golden_shapes(_cuda, shapes, cluster):
    for c in shapes[::3]:
        ids, A = c["ids"], c["A"]
        if cluster and ids.size > cluster * 8192:
            continue  # beyond the per-CTA slice limit: needs a larger cluster
        for pr in (oracle.pair_rank_metro(ids, c["metro_choice"]), oracle.pair_rank_eplb(ids, A)):
            r0, o0 = oracle.dispatch_layout(ids, pr, A)
            r1, o1 = _dev_layout(ids, pr, A, cluster)
            assert (o1 == o0).all(), c["name"]
            assert (r1 == r0.reshape(-1)).all(), c["name"]


@pytest.mark.gpu
def test_layout_after_device_routing(_cuda):
    """Router pair_rank -> layout, all on device; rows per replica = x."""
    A = make_placement(256, 8, 1.5, 7).matrix
    pl = DevicePlacement(A)
    dl = DispatchLayout(pl)
    for kind in ("metro", "eplb"):
        for B in (64, 1024, 8192):
            ids = gen_zipf_topk(256, 8, B, 1.2, 1000 + B, popularity_seed=7)
            it = torch.from_numpy(ids).cuda()
            rr = Router(pl, kind).route(it, pair_rank=True).check()
            out = dl(it, rr.pair_rank).check()
            pr = rr.pair_rank.cpu().numpy()
            r0, o0 = oracle.dispatch_layout(ids, pr, A)
            assert (out.rep_off.cpu().numpy() == o0).all()
            assert (out.pair_row.cpu().numpy()[: ids.size] == r0).all()


@pytest.mark.gpu
def test_layout_fuzz(_cuda):
    rng = np.random.default_rng(5)
    for it in range(120):
        n = int(rng.integers(1, 300))
        g = int(rng.integers(1, 130))
        A = (rng.random((n, g)) < min(1.0, 3.0 / g)).astype(np.int8)
        A[np.arange(n), rng.integers(0, g, n)] = 1
        if A.sum() > 4096:
            continue
        P = int(rng.integers(0, 5000))
        ids = rng.integers(0, n, P).astype(np.int32)
        # any valid pair rank: a random replica of the pair's expert
        reps = [np.flatnonzero(A[i]) for i in range(n)]
        pr = np.array([reps[e][rng.integers(0, len(reps[e]))] for e in ids], np.int32)
        cl = int(rng.choice([0, 1, 2, 4, 8, 16]))
        if P > cl * 8192 and cl:
            cl = 0
        r0, o0 = oracle.dispatch_layout(ids, pr, A)
        r1, o1 = _dev_layout(ids, pr, A, cl)
        assert (o1 == o0).all(), it
        assert (r1 == r0).all(), it


@pytest.mark.gpu
def test_layout_max_and_empty(_cuda):
    A = make_placement(256, 8, 1.5, 7).matrix
    ids = gen_zipf_topk(256, 8, 16384, 1.2, 3, popularity_seed=7)  # 131072 pairs: 16 x 8192
    pe = oracle.pair_rank_eplb(ids, A)
    r0, o0 = oracle.dispatch_layout(ids, pe, A)
    r1, o1 = _dev_layout(ids, pe, A)
    assert (o1 == o0).all() and (r1 == r0.reshape(-1)).all()
    r1, o1 = _dev_layout(np.zeros(0, np.int32), np.zeros(0, np.int32), A)
    assert (o1 == 0).all()
    with pytest.raises(ValidationError):
        _dev_layout(np.zeros(131073, np.int32), np.zeros(131073, np.int32), A)


@pytest.mark.gpu
def test_layout_errors(_cuda):
    A = np.array([[1, 1, 0], [0, 1, 1], [1, 0, 1]], np.int8)
    ids = np.array([0, 1, 2, 0, 1, 0] * 100, np.int32)
    pr = np.array([0, 2, 2, 1, 1, 0] * 100, np.int32)
    bad = ids.copy()
    bad[333] = 7
    with pytest.raises(ValidationError, match="token 333: expert id 7 out of range"):
        _dev_layout(bad, pr, A, 4)
    badr = pr.copy()
    badr[400] = 0  # pair 400 is expert 1, not hosted on rank 0
    with pytest.raises(ValidationError, match="token 400: rank 0 hosts no replica"):
        _dev_layout(ids, badr, A, 2)


# ---------------------------------------------------------------- fused METRO + layout
def _fused(ids, A, cluster=0):
    pl = DevicePlacement(A)
    dl = DispatchLayout(pl, cluster)
    it = torch.as_tensor(np.ascontiguousarray(ids, np.int32)).cuda()
    o, lo = dl.route_metro(it)
    o.check()
    P = int(np.size(ids))
    return (o.loads.cpu().numpy(), o.choice.cpu().numpy(), o.rank_counts.cpu().numpy(), int(o.lam.item()),
            o.pair_rank.cpu().numpy()[:P], lo.pair_row.cpu().numpy()[:P], lo.rep_off.cpu().numpy())


def _check_fused(ids, A, cluster=0):
    A = np.asarray(A, np.int8)
    T = oracle.aggregate_loads(ids, A.shape[0])
    choice, counts, lam = oracle.route_metro(T, A)
    pr = oracle.pair_rank_metro(ids, choice).reshape(-1)
    r0, o0 = oracle.dispatch_layout(ids, pr, A)
    loads, ch, cnt, lm, pr1, r1, o1 = _fused(ids, A, cluster)
    assert (loads == T).all() and (ch == choice).all() and (cnt == counts).all() and lm == lam
    assert (pr1 == pr).all()
    assert (o1 == o0).all()
    assert (r1 == r0.reshape(-1)).all()


@pytest.mark.gpu
@pytest.mark.parametrize("cluster", [0, 1, 2, 4, 8, 16])
def test_fused_route_layout_golden(_cuda, shapes, cluster):
    """metro_route_layout_v1 == metro_route_v1 + metro_dispatch_layout_v1 == the
    oracle, on every golden shape at every cluster size (fallback included)."""
    for c in shapes:
        _check_fused(c["ids"], c["A"], cluster)


@pytest.mark.gpu
def test_fused_route_layout_fuzz_and_edges(_cuda):
    rng = np.random.default_rng(11)
    for it in range(150):
        n = int(rng.integers(1, 400))
        g = int(rng.choice([1, 2, 3, 8, 16, 33, 100]))
        A = (rng.random((n, g)) < min(1.0, 3.0 / g)).astype(np.int8)
        A[np.arange(n), rng.integers(0, g, n)] = 1
        if A.sum() > 4096:
            continue
        B = int(rng.choice([0, 1, 5, 64, 255, 1024, 3000]))
        k = int(rng.integers(1, min(10, n) + 1))
        ids = rng.integers(0, n, (B, k)).astype(np.int32)  # duplicates allowed
        _check_fused(ids, A, int(rng.choice([0, 1, 2, 4, 8, 16])))
    # DeepSeek-V3 decode sweep through the auto plan
    A = make_placement(256, 8, 1.5, 7).matrix
    for B in (64, 256, 1024, 4096, 8192):
        _check_fused(gen_zipf_topk(256, 8, B, 1.2, 77 + B, popularity_seed=7), A)
    # an out-of-range id is reported like metro_route_v1
    ids = gen_zipf_topk(256, 8, 64, 1.2, 5, popularity_seed=7)
    ids[10, 3] = 999
    with pytest.raises(ValidationError, match="token 10: expert id 999 out of range"):
        _fused(ids, A)


@pytest.mark.gpu
def test_fused_route_layout_without_loads(_cuda):
    """out.loads is optional on the fused route + layout, as on Router.route."""
    import dataclasses

    A = make_placement(256, 8, 1.5, 7).matrix
    ids = torch.from_numpy(gen_zipf_topk(256, 8, 256, 1.2, 3, popularity_seed=7)).cuda()
    pl = DevicePlacement(A)
    lay = DispatchLayout(pl)
    ref, ref_lo = lay.route_metro(ids)
    out = dataclasses.replace(Router(pl, "metro").alloc(ids.numel(), top_k=8), loads=None)
    got, lo = lay.route_metro(ids, out=out)
    got.check()
    assert torch.equal(got.choice, ref.choice) and torch.equal(got.pair_rank, ref.pair_rank)
    assert torch.equal(lo.pair_row, ref_lo.pair_row) and torch.equal(lo.rep_off, ref_lo.rep_off)


@pytest.mark.gpu
@pytest.mark.parametrize("nrep", [31, 32, 33, 511, 512, 513, 1024])
def test_fused_route_layout_replica_count_boundaries(_cuda, nrep):
    """rep_off has nrep + 1 entries: replica counts at the one-replica-per-thread
    limit of the fused scan (512 threads) and at warp multiples (found by the
    soak: nrep == 512 lost rep_off[nrep])."""
    rng = np.random.default_rng(nrep)
    n, g = 256, 8
    A = np.zeros((n, g), np.int8)
    A[np.arange(n), np.arange(n) % g] = 1  # one replica each ...
    extra = nrep - n
    if extra < 0:
        n = nrep
        A = A[:n]
    else:
        free = np.argwhere(A == 0)
        pick = free[rng.choice(len(free), extra, replace=False)]
        A[pick[:, 0], pick[:, 1]] = 1  # ... plus extra replicas
    assert int(A.sum()) == nrep
    for B in (1, 255, 1024):
        ids = rng.integers(0, n, (B, 8 if n >= 8 else n)).astype(np.int32)
        for cluster in (0, 1, 4):
            _check_fused(ids, A, cluster)


@pytest.mark.gpu
def test_fused_route_layout_large_tables(_cuda):
    """Replica tables big enough that the plan shrinks the histogram copies: the
    sort scratch must not alias the partial rows that classify still reads (two
    soak instances, N > 512 experts x 65 ranks, that once routed wrong at R = 8),
    plus a fuzz over N in (512, 700] and multi-word masks."""
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "fused_regress.npz"))
    for i in (0, 1):
        ids, A = z[f"ids{i}"], z[f"A{i}"]
        for cluster in (0, 1, 2, 4, 8, 16):
            _check_fused(ids, A, cluster)
            T = oracle.aggregate_loads(ids, A.shape[0])
            choice, counts, lam = oracle.route_metro(T, A)
            o = Router(DevicePlacement(A), "metro", cluster).route(torch.from_numpy(ids).cuda()).check()
            assert (o.choice.cpu().numpy() == choice).all() and int(o.lam.item()) == lam
    rng = np.random.default_rng(5)
    for _ in range(40):
        n = int(rng.integers(513, 701))
        g = int(rng.choice([33, 65, 100]))
        A = (rng.random((n, g)) < rng.uniform(0.02, 0.1)).astype(np.int8)
        A[np.arange(n), rng.integers(0, g, n)] = 1
        if A.sum() > 4096:
            continue
        ids = rng.integers(0, n, (int(rng.choice([255, 1000, 3000])), int(rng.integers(1, 10)))).astype(np.int32)
        _check_fused(ids, A, int(rng.choice([0, 2, 4, 8, 16])))
