"""Fused all-gather + METRO over peer memory (include/metro_exchange.h) against the
oracle (-m gpu).

All EP ranks run in this one process on one device ("virtual ranks", distinct
streams, each rank addressing the others' exchange buffers directly): the same
kernel and flag protocol as across NVLink peers.  Every rank must produce the
oracle's routing of the GLOBAL batch (rank-major token shards, as the
reference's source_gpu = j % G is a pure relabelling for the histogram), the
oracle's pair ranks for its own tokens, and, when asked, the gathered ids.
"""

import os

import numpy as np
import pytest
import torch

import oracle
from paper_2512_09277_b200 import DevicePlacement, NativeLibraryError, ValidationError
from paper_2512_09277_b200.dist import virtual_ranks
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.init()


def run_all(routers, shards, streams):
    """One exchange + route on every virtual rank, each on its own stream."""
    for r, (rt, ids) in enumerate(zip(routers, shards)):
        with torch.cuda.stream(streams[r]):
            rt.step(ids, stream=streams[r])
    torch.cuda.synchronize()


def check_rank(rt, ids_global, A, local_tokens, gathered=False):
    A = np.asarray(A, dtype=np.int8)
    T = oracle.aggregate_loads(ids_global, A.shape[0])
    choice, counts, lam = oracle.route_metro(T, A)
    o = rt.out
    o.check()
    assert np.array_equal(o.loads.cpu().numpy(), T)
    assert np.array_equal(o.choice.cpu().numpy(), choice)
    assert np.array_equal(o.rank_counts.cpu().numpy(), counts)
    assert int(o.lam.item()) == lam
    own = ids_global[rt.rank * local_tokens:(rt.rank + 1) * local_tokens]
    assert np.array_equal(o.pair_rank.cpu().numpy().reshape(own.shape), oracle.pair_rank_metro(own, choice))
    if gathered:
        assert np.array_equal(rt.gathered.cpu().numpy(), ids_global)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("gather", [False, True])
def test_fused_allgather_matches_oracle(world, gather):
    A = make_placement(256, 8, 1.5, 7).matrix
    pl = DevicePlacement(A)
    B, k = 1024, 8
    lt = B // world
    routers, bufs = virtual_ranks(pl, world, lt, k, gather_ids=gather)
    streams = [torch.cuda.Stream() for _ in range(world)]
    try:
        for call in range(5):  # consecutive calls: epochs and both buffer parities
            ids = gen_zipf_topk(256, k, B, 1.2, 3000 + call, popularity_seed=7)
            shards = [torch.from_numpy(ids[r * lt:(r + 1) * lt].copy()).cuda() for r in range(world)]
            run_all(routers, shards, streams)
            for rt in routers:
                check_rank(rt, ids, A, lt, gathered=gather)
    finally:
        for b in bufs:
            b.close()


def test_fused_allgather_baseline_shapes(shapes):
    for c in shapes:
        if c["B"] % 8 or c["B"] > 4096 or c["G"] > 32:
            continue
        world = 8
        lt = c["B"] // world
        pl = DevicePlacement(c["A"])
        routers, bufs = virtual_ranks(pl, world, lt, c["k"], gather_ids=True)
        streams = [torch.cuda.Stream() for _ in range(world)]
        try:
            shards = [torch.from_numpy(np.ascontiguousarray(c["ids"][r * lt:(r + 1) * lt])).cuda() for r in range(world)]
            run_all(routers, shards, streams)
            for rt in routers:
                check_rank(rt, c["ids"], c["A"], lt, gathered=True)
                assert int(rt.out.lam.item()) == c["metro_lam"]
        finally:
            for b in bufs:
                b.close()


def test_fused_allgather_bad_id_reported_on_every_rank():
    A = make_placement(128, 8, 1.5, 7).matrix
    pl = DevicePlacement(A)
    world, lt, k = 4, 64, 8
    routers, bufs = virtual_ranks(pl, world, lt, k)
    streams = [torch.cuda.Stream() for _ in range(world)]
    try:
        ids = gen_zipf_topk(128, k, world * lt, 1.2, 11, popularity_seed=7)
        ids[2 * lt + 5, 6] = 200  # a bad id on rank 2: global token 2*lt + 5
        ids[3 * lt + 1, 0] = 300  # and a later one on rank 3
        shards = [torch.from_numpy(ids[r * lt:(r + 1) * lt].copy()).cuda() for r in range(world)]
        run_all(routers, shards, streams)
        for rt in routers:
            with pytest.raises(ValidationError, match=f"token {2 * lt + 5}: expert id 200 out of range"):
                rt.out.check()
        # the next call on the same buffers is clean again
        ids2 = gen_zipf_topk(128, k, world * lt, 1.2, 12, popularity_seed=7)
        shards = [torch.from_numpy(ids2[r * lt:(r + 1) * lt].copy()).cuda() for r in range(world)]
        run_all(routers, shards, streams)
        for rt in routers:
            check_rank(rt, ids2, A, lt)
    finally:
        for b in bufs:
            b.close()


def test_fused_allgather_missing_peer_times_out(monkeypatch):
    monkeypatch.setenv("METRO_PEER_TIMEOUT_MS", "200")
    A = make_placement(128, 8, 1.5, 7).matrix
    pl = DevicePlacement(A)
    routers, bufs = virtual_ranks(pl, 2, 32, 8)
    try:
        ids = torch.from_numpy(gen_zipf_topk(128, 8, 32, 1.2, 1, popularity_seed=7)).cuda()
        routers[0].step(ids)  # rank 1 never joins
        torch.cuda.synchronize()
        with pytest.raises(NativeLibraryError, match="peer rank 1"):
            routers[0].out.check()
    finally:
        for b in bufs:
            b.close()


@pytest.mark.parametrize("world", [1, 4])
def test_fused_allgather_empty_local_batches(world):
    """No tokens anywhere: every rank reports an empty routing (λ 0), twice."""
    A = make_placement(128, 8, 1.5, 7).matrix
    pl = DevicePlacement(A)
    routers, bufs = virtual_ranks(pl, world, 0, 8, gather_ids=True)
    streams = [torch.cuda.Stream() for _ in range(world)]
    try:
        empty = [torch.zeros((0, 8), dtype=torch.int32, device="cuda") for _ in range(world)]
        for _ in range(2):
            run_all(routers, empty, streams)
            for rt in routers:
                rt.out.check()
                assert int(rt.out.lam.item()) == 0
                assert bool((rt.out.choice == -1).all())
    finally:
        for b in bufs:
            b.close()


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_fused_exchange_layout_matches_oracle(world, shapes):
    """metro_allgather_route_layout_v1: every rank's own pairs' rows in the
    GLOBAL (rank-major) dispatch layout and the replica offsets, from the
    exchanged histograms only -- bit-exact with the oracle's layout of the
    gathered batch under METRO (golden shapes + consecutive calls)."""
    from paper_2512_09277_b200 import DispatchLayout

    cases = [c for c in shapes if c["B"] % world == 0 and c["B"] * c["k"] // world <= 8192 and c["G"] <= 32]
    for c in cases[:6]:
        A = c["A"]
        pl = DevicePlacement(A)
        lay = DispatchLayout(pl)
        B, k = c["B"], c["k"]
        lt = B // world
        routers, bufs = virtual_ranks(pl, world, lt, k, layout=lay)
        streams = [torch.cuda.Stream() for _ in range(world)]
        try:
            for call in range(3):
                ids = c["ids"] if call == 0 else gen_zipf_topk(c["N"], k, B, 1.2, 4000 + call, popularity_seed=7)
                shards = [torch.from_numpy(np.ascontiguousarray(ids[r * lt:(r + 1) * lt])).cuda()
                          for r in range(world)]
                run_all(routers, shards, streams)
                T = oracle.aggregate_loads(ids, A.shape[0])
                choice, _, _ = oracle.route_metro(T, A)
                pr = oracle.pair_rank_metro(ids, choice).reshape(-1)
                row, off = oracle.dispatch_layout(ids, pr, A)
                row = np.asarray(row).reshape(-1)
                for rt in routers:
                    check_rank(rt, ids, A, lt)
                    lo = rt.layout_out
                    own = slice(rt.rank * lt * k, (rt.rank + 1) * lt * k)
                    assert np.array_equal(lo.pair_row.cpu().numpy()[:lt * k], row[own]), (c["name"], world, rt.rank)
                    assert np.array_equal(lo.rep_off.cpu().numpy(), off), (c["name"], world)
        finally:
            for b in bufs:
                b.close()
