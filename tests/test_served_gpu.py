"""Persistent host router (include/metro_serve.h, ``ServedRouter``) against the
oracle (-m gpu): the resident CTA must return exactly what metro_route_v1 and
the oracle return, for every golden shape, across back-to-back requests that
reuse the same pinned buffers (a stale host line would show up here), ragged
sizes, the reference's error cases, idle exit + transparent relaunch, and stop.
"""

import time

import numpy as np
import pytest
import torch

import oracle
from paper_2512_09277_b200 import DevicePlacement, ServedRouter, ValidationError
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.init()


def expect(ids, A):
    A = np.asarray(A, dtype=np.int8)
    T = oracle.aggregate_loads(ids, A.shape[0])
    choice, counts, lam = oracle.route_metro(T, A)
    return choice, counts, lam, oracle.pair_rank_metro(ids, choice).reshape(-1)


def check(sr, ids, A):
    G = A.shape[1]
    flat = np.ascontiguousarray(ids, dtype=np.int32).reshape(-1)
    sr.ids.numpy()[: flat.size] = flat
    out = sr.run(flat.size)
    choice, counts, lam, pair = expect(ids, A)
    assert int(out[0]) == 0, out[:4]
    assert int(out[4]) == lam
    assert np.array_equal(out[8:8 + G], counts)
    assert np.array_equal(out[8 + G:], choice)
    assert np.array_equal(sr.pair_rank.numpy()[: flat.size], pair)


def test_served_golden_shapes(shapes):
    # batches up to 32k pairs are staged in shared memory; B = 8192 (65,536 pairs)
    # reads the ids from host memory a second time for the pair ranks
    for c in shapes:
        pl = DevicePlacement(c["A"])
        with ServedRouter(pl, c["B"] * c["k"]) as sr:
            check(sr, c["ids"], c["A"])
            assert sr.launches == 1


def test_served_back_to_back_same_buffers():
    A = make_placement(256, 8, 1.5, 7).matrix
    pl = DevicePlacement(A)
    batches = [gen_zipf_topk(256, 8, 1024, 1.2, 2000 + s, popularity_seed=7) for s in range(40)]
    with ServedRouter(pl, 8192) as sr:
        for b in batches:  # every request overwrites the previous batch in place
            check(sr, b, A)
        assert sr.launches == 1


def test_served_ragged_sizes():
    rng = np.random.default_rng(5)
    A = make_placement(128, 8, 1.5, 7).matrix
    pl = DevicePlacement(A)
    with ServedRouter(pl, 5003) as sr:
        for B in (0, 1, 3, 7, 64, 333, 625):
            ids = rng.integers(0, 128, size=(B, 8)).astype(np.int32)
            check(sr, ids, A)
        ids = rng.integers(0, 128, size=5003).astype(np.int32)  # not a multiple of 4
        check(sr, ids, A)


def test_served_multiword_masks():
    rng = np.random.default_rng(9)
    for G in (16, 40, 128):
        N = 300
        A = (rng.random((N, G)) < 0.05).astype(np.int8)
        A[np.arange(N), rng.integers(0, G, N)] = 1
        pl = DevicePlacement(A)
        with ServedRouter(pl, 4096) as sr:
            for _ in range(3):
                ids = rng.integers(0, N, size=(512, 8)).astype(np.int32)
                check(sr, ids, A)


def test_served_errors_then_recovers():
    A = make_placement(128, 8, 1.5, 7).matrix
    pl = DevicePlacement(A)
    with ServedRouter(pl, 4096) as sr:
        ids = gen_zipf_topk(128, 8, 256, 1.2, 1000, popularity_seed=7)
        bad = ids.copy()
        bad[17, 3] = 128
        with pytest.raises(ValidationError, match="token 17: expert id 128 out of range"):
            sr.route(bad)
        check(sr, ids, A)  # the next request on the same server is clean
    A2 = A.copy()
    A2[5, :] = 0  # expert 5 without a replica: the reference asserts (routing.py:66, :99)
    A2[5, 0] = 0
    pl2 = DevicePlacement(A2)
    with ServedRouter(pl2, 4096) as sr:
        ids = np.full((4, 8), 5, dtype=np.int32)
        with pytest.raises(AssertionError):
            sr.route(ids)
        with pytest.raises(ValidationError):
            sr.run(4097)


def test_served_idle_exit_relaunch():
    A = make_placement(256, 8, 1.5, 7).matrix
    pl = DevicePlacement(A)
    with ServedRouter(pl, 8192, idle_timeout_us=2000) as sr:
        b0 = gen_zipf_topk(256, 8, 1024, 1.2, 1000, popularity_seed=7)
        check(sr, b0, A)
        l0 = sr.launches
        time.sleep(0.05)  # the resident CTA has left (2 ms idle timeout)
        torch.cuda.synchronize()  # a device-wide sync is not blocked by it
        b1 = gen_zipf_topk(256, 8, 1024, 1.2, 1001, popularity_seed=7)
        check(sr, b1, A)
        assert sr.launches == l0 + 1
        for s in range(5):  # races between the idle exit and the doorbell
            time.sleep(0.002)
            check(sr, gen_zipf_topk(256, 8, 1024, 1.2, 1100 + s, popularity_seed=7), A)
    assert sr.launches == 0  # closed


def test_served_empty_batches():
    A = make_placement(128, 8, 1.5, 7).matrix
    pl = DevicePlacement(A)
    with ServedRouter(pl, 0) as sr:  # a server sized for nothing still answers
        out = sr.run(0)
        assert int(out[0]) == 0 and int(out[4]) == 0
        assert (out[8:8 + 8] == 0).all() and (out[8 + 8:] == -1).all()
