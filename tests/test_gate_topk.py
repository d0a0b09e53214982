"""Gating top-k fused with METRO routing (metro_route_scores_v1).

CPU: the oracle's top-k over the float32 gating scores reproduces the reference
generator's top-k ids (core.py:319-326) on every golden case.  GPU (-m gpu): the
fused kernel's ids equal the oracle's, and its routing outputs equal the oracle
routing of those ids -- golden cases at every cluster size, random scores with
forced ties (tie -> lower expert id), limits and argument errors.
"""

import numpy as np
import pytest
import torch

import oracle
from paper_2512_09277_b200 import DevicePlacement, Router, ValidationError
from paper_2512_09277_b200.placement import make_placement


def test_oracle_topk_matches_reference_generator(gate):
    for c in gate:
        assert (oracle.gate_topk(c["scores"], c["k"]) == c["ids"]).all(), (c["N"], c["k"])


def test_oracle_topk_ties_lower_id():
    sc = np.array([[1, 3, 3, 2, 3]], np.float32)
    assert oracle.gate_topk(sc, 4).tolist() == [[1, 2, 4, 3]]


def test_oracle_topk_signed_zero_and_nan():
    nan = np.float32("nan")
    # -0.0 == +0.0: the lower id wins; NaN ranks below every number, even -inf
    sc = np.array([[-0.0, 0.0, -1.0],
                   [0.0, -0.0, -1.0],
                   [nan, -np.inf, 1.0],
                   [nan, nan, -0.0]], np.float32)
    assert oracle.gate_topk(sc, 3).tolist() == [[0, 1, 2], [0, 1, 2], [2, 1, 0], [2, 0, 1]]
    assert oracle.gate_topk(sc, 1).tolist() == [[0], [0], [2], [2]]


def _signed_zero_nan_scores(rng, B, n):
    """Rows that stress the key order: +-0.0 mixes, NaNs and +-inf among a few
    distinct values, so the k-th boundary often falls inside a tie class."""
    vals = np.array([-0.0, 0.0, -0.0, 0.0, 1.0, -1.0, np.inf, -np.inf, np.nan, 0.5], np.float32)
    sc = vals[rng.integers(0, len(vals), size=(B, n))]
    # a quarter of the rows: all zeros of random sign (k = 1 picks the lowest id)
    z = rng.random(B) < 0.25
    sc[z] = np.where(rng.random((int(z.sum()), n)) < 0.5, np.float32(-0.0), np.float32(0.0))
    return sc


@pytest.fixture(scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.init()


def _fused(scores, k, A, cluster=0, whole_gpu=None):
    pl = DevicePlacement(A)
    r = Router(pl, "metro", cluster)
    st = torch.from_numpy(np.ascontiguousarray(scores, np.float32)).cuda()
    ids, out = r.route_scores(st, k, whole_gpu=whole_gpu)
    out.check()
    return ids.cpu().numpy(), out


def _check_routing(ids, out, A):
    loads = oracle.aggregate_loads(ids, A.shape[0])
    choice, counts, lam = oracle.route_metro(loads, A)
    assert (out.loads.cpu().numpy() == loads).all()
    assert (out.choice.cpu().numpy() == choice).all()
    assert (out.rank_counts.cpu().numpy() == counts).all()
    assert int(out.lam.item()) == lam
    pr = oracle.pair_rank_metro(ids, choice)
    assert (out.pair_rank.cpu().numpy() == pr.reshape(-1)).all()


@pytest.mark.gpu
@pytest.mark.parametrize("cluster", ["gpu", 0, 1, 2, 4, 8, 16])
def test_fused_gate_golden(_cuda, gate, cluster):
    for c in gate:
        A = make_placement(c["N"], c["G"], 1.5, 7).matrix
        if cluster == "gpu":
            ids, out = _fused(c["scores"], c["k"], A, whole_gpu=True)
        else:
            ids, out = _fused(c["scores"], c["k"], A, cluster, whole_gpu=False)
        assert (ids == c["ids"]).all(), (c["N"], c["k"], cluster)
        _check_routing(ids, out, A)


@pytest.mark.gpu
def test_fused_gate_random_with_ties(_cuda):
    rng = np.random.default_rng(9)
    for it in range(60):
        n = int(rng.choice([8, 33, 64, 100, 128, 200, 256, 300, 512]))
        g = int(rng.choice([2, 4, 8, 16, 32]))
        k = int(rng.integers(1, min(32, n) + 1))
        B = int(rng.integers(0, 1500))
        A = (rng.random((n, g)) < 2.0 / g).astype(np.int8)
        A[np.arange(n), rng.integers(0, g, n)] = 1
        if it % 3 == 0:  # heavy ties: small integer scores (incl. negatives)
            sc = rng.integers(-3, 4, size=(B, n)).astype(np.float32)
        else:
            sc = rng.standard_normal((B, n)).astype(np.float32)
        cl = int(rng.choice([-1, 0, 1, 4, 16]))
        ids, out = _fused(sc, k, A, max(cl, 0), whole_gpu=True if cl < 0 else (None if cl == 0 else False))
        ref = oracle.gate_topk(sc, k) if B else np.zeros((0, k), np.int32)
        assert (ids == ref).all(), it
        if B:
            _check_routing(ids, out, A)


@pytest.mark.gpu
def test_fused_gate_limits_and_errors(_cuda):
    A = make_placement(256, 8, 1.5, 7).matrix
    sc = np.random.default_rng(1).standard_normal((4096, 256)).astype(np.float32)
    for whole in (True, False, None):
        ids, out = _fused(sc, 8, A, whole_gpu=whole)
        assert (ids == oracle.gate_topk(sc, 8)).all()
        _check_routing(ids, out, A)
    # the workspace is left zeroed: repeated launches on one router agree
    pl = DevicePlacement(A)
    r = Router(pl, "metro")
    st = torch.from_numpy(sc[:1000]).cuda()
    for _ in range(3):
        ids, out = r.route_scores(st, 8)
        out.check()
        _check_routing(ids.cpu().numpy(), out, A)
    pl = DevicePlacement(A)
    r = Router(pl, "metro")
    with pytest.raises(ValidationError):
        r.route_scores(torch.zeros((4, 255), device="cuda"), 8)  # dimension mismatch
    with pytest.raises(ValidationError):
        r.route_scores(torch.zeros((4, 256), device="cuda"), 33)  # k > 32
    with pytest.raises(ValidationError):
        r.route_scores(torch.zeros((4, 256), device="cuda", dtype=torch.float64), 8)
    with pytest.raises(ValidationError):
        r.route_scores(torch.zeros((4, 256), device="cuda"), 8,
                       topk_ids=torch.empty((4, 8), dtype=torch.int64, device="cuda"))  # wrong dtype
    with pytest.raises(ValidationError):
        r.route_scores(torch.zeros((4, 256), device="cuda"), 8,
                       topk_ids=torch.empty((4, 7), dtype=torch.int32, device="cuda"))  # wrong size
    big = DevicePlacement(np.ones((600, 8), np.int8))
    with pytest.raises(ValidationError):
        Router(big, "metro").route_scores(torch.zeros((4, 600), device="cuda"), 8)  # N > 512


@pytest.mark.gpu
def test_fused_gate_whole_gpu_sequence(_cuda):
    """One router, consecutive whole-GPU launches of different sizes (1-16 routing
    CTAs, pair counts not a multiple of 4): the workspace handoff between the
    routing CTAs and the next launch's top-k grid, and an unaligned ids buffer."""
    rng = np.random.default_rng(21)
    A = make_placement(256, 8, 1.5, 7).matrix
    r = Router(DevicePlacement(A), "metro")
    for B in (1500, 3, 700, 4096, 65, 1, 2049):
        sc = rng.standard_normal((B, 256)).astype(np.float32)
        st = torch.from_numpy(sc).cuda()
        if B == 65:  # topk_ids 4 bytes past a 16-byte boundary: scalar pair-rank path
            buf = torch.empty(B * 6 + 1, dtype=torch.int32, device="cuda")
            ids, out = r.route_scores(st, 6, topk_ids=buf[1:].view(B, 6), whole_gpu=True)
        else:
            ids, out = r.route_scores(st, 6, whole_gpu=True)
        out.check()
        got = ids.cpu().numpy()
        assert (got == oracle.gate_topk(sc, 6)).all(), B
        _check_routing(got, out, A)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["gpu", 1, 4])
def test_fused_gate_signed_zero_and_nan(_cuda, variant):
    """Bit-exact ids vs the oracle on +-0.0 / NaN / +-inf rows, k = 1 and k at a
    tie boundary, both gating variants (whole GPU and one cluster)."""
    rng = np.random.default_rng(77)
    for n, g in ((256, 8), (128, 8), (64, 4), (320, 16)):
        A = make_placement(n, g, 1.5, 7).matrix
        for k in (1, 2, 8):
            for B in (1, 37, 700):
                sc = _signed_zero_nan_scores(rng, B, n)
                if variant == "gpu":
                    ids, out = _fused(sc, k, A, whole_gpu=True)
                else:
                    ids, out = _fused(sc, k, A, variant, whole_gpu=False)
                ref = oracle.gate_topk(sc, k)
                assert (ids == ref).all(), (n, k, B, variant)
                _check_routing(ids, out, A)
