"""Pin the CPU oracle (oracle/metro_oracle.c) to the reference's golden vectors.

Golden vectors come from the unmodified reference (tests/golden/make_golden.py).
When the reference is mounted (build container) the oracle is also checked
differentially against it on fresh random instances.
"""

import numpy as np
import pytest

import oracle


def test_oracle_shapes_golden(shapes):
    for c in shapes:
        T = oracle.aggregate_loads(c["ids"], c["N"])
        assert (T == c["T"]).all(), c["name"]
        choice, counts, lam = oracle.route_metro(T, c["A"])
        assert (choice == c["metro_choice"]).all(), c["name"]
        assert (counts == c["metro_counts"]).all()
        assert lam == c["metro_lam"]
        x, ecounts, elam = oracle.route_eplb(T, c["A"])
        assert (x == c["eplb_x"]).all()
        assert (ecounts == c["eplb_counts"]).all()
        assert elam == c["eplb_lam"]
        # per-pair conventions reproduce the reference's x exactly
        pr = oracle.pair_rank_metro(c["ids"], choice)
        xm = np.zeros_like(x)
        np.add.at(xm, (c["ids"].reshape(-1), pr.reshape(-1)), 1)
        assert (xm.sum(axis=0).max()) == c["metro_maxtok"]
        pe = oracle.pair_rank_eplb(c["ids"], c["A"])
        xe = np.zeros_like(x)
        np.add.at(xe, (c["ids"].reshape(-1), pe.reshape(-1)), 1)
        assert (xe == c["eplb_x"]).all()
        assert xe.sum(axis=0).max() == c["eplb_maxtok"]


def test_oracle_small_golden(small):
    for c in small:
        choice, counts, lam = oracle.route_metro(c["T"], c["A"])
        assert (choice == c["metro_choice"]).all(), c
        assert lam == c["metro_lam"]
        x, _, elam = oracle.route_eplb(c["T"], c["A"])
        assert (x == c["eplb_x"]).all()
        assert elam == c["eplb_lam"]


def test_oracle_known_answers():
    # pkg/tests/test_routing.py:42-56, :65-79
    x, _, lam = oracle.route_eplb([6], [[1, 1, 1]])
    assert x.tolist() == [[2, 2, 2]] and lam == 1
    x, _, _ = oracle.route_eplb([5], [[1, 1, 1]])
    assert x.tolist() == [[2, 2, 1]]
    assert oracle.route_eplb([8, 8], [[1, 1], [1, 1]])[2] == 2
    assert oracle.route_metro([8, 8], [[1, 1], [1, 1]])[2] == 1
    assert oracle.route_metro([0, 0], [[1, 1], [1, 1]])[2] == 0
    assert oracle.route_metro([1, 3, 8], [[1, 1, 0], [1, 0, 1], [0, 1, 1]])[2] == 2


def test_oracle_errors():
    with pytest.raises(oracle.OracleError) as ei:
        oracle.aggregate_loads([[0, 99]], 4)
    assert ei.value.code == oracle.oracle.ERR_ID_RANGE
    with pytest.raises(oracle.OracleError) as ei:
        oracle.route_metro([1, 1], [[1, 0], [0, 0]])
    assert ei.value.code == oracle.oracle.ERR_NO_REPLICA


def test_duplicate_ids_count_twice():
    # aggregate_loads does not enforce distinctness (SURVEY.md App. A probe)
    assert oracle.aggregate_loads([[1, 1]], 4).tolist() == [0, 2, 0, 0]


def test_oracle_differential_vs_reference(eproute_ref):
    """Fresh random instances: the oracle agrees with the imported reference."""
    from eproute import ExpertLoadVector, PlacementMap
    from eproute.routing import route_eplb, route_metro

    rng = np.random.default_rng(123)
    for _ in range(300):
        n = int(rng.integers(1, 80))
        g = int(rng.integers(1, 20))
        A = (rng.random((n, g)) < rng.uniform(0.1, 0.8)).astype(np.int8)
        for i in range(n):
            if not A[i].any():
                A[i, rng.integers(g)] = 1
        T = rng.integers(0, 6, size=n) * (rng.random(n) < 0.8)
        Tv, Am = ExpertLoadVector(T), PlacementMap(A, int(A.sum(axis=0).max()))
        rm, re = route_metro(Tv, Am), route_eplb(Tv, Am)
        choice, _, lam = oracle.route_metro(T, A)
        y = np.zeros_like(A)
        act = choice >= 0
        y[np.flatnonzero(act), choice[act]] = 1
        assert (y == rm.y).all() and lam == rm.lam
        x, _, elam = oracle.route_eplb(T, A)
        assert (x == re.x).all() and elam == re.lam
