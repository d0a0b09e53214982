"""N > 1 host logic on CPU: world_size-2 gloo processes.

Checks the rank-major all-gather of per-rank top-k ids (paper_2512_09277_b200.dist),
that routing the gathered batch equals routing the global batch (routing depends
only on the histogram), that each rank's own pair ranks are the right slice, and
the cross-rank agreement digest.  The oracle stands in for the device router
here (no GPU on this host); -m gpu tests cover the device router itself.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        from paper_2512_09277_b200.dist import allgather_topk, assert_ranks_agree, local_slice, shard_tokens
        from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement

        A = make_placement(256, 8, 1.5, 7).matrix
        results = []
        for seed in (1000, 1001, 1002):
            glob = gen_zipf_topk(256, 8, 1024, 1.2, seed, popularity_seed=7)
            mine = torch.from_numpy(shard_tokens(glob, world, rank).copy())
            gathered = allgather_topk(mine).numpy()
            assert np.array_equal(gathered, glob)
            T = oracle.aggregate_loads(gathered, 256)
            choice, counts, lam = oracle.route_metro(T, A)
            ref_choice, _, ref_lam = oracle.route_metro(oracle.aggregate_loads(glob, 256), A)
            assert np.array_equal(choice, ref_choice) and lam == ref_lam
            pr = oracle.pair_rank_metro(gathered, choice).reshape(-1)
            own = pr[local_slice(rank, 1024 // world, 8)].reshape(-1, 8)
            assert np.array_equal(own, choice[mine.numpy()])
            results.append(assert_ranks_agree(choice, counts, lam))
        # a deliberately different routing on one rank must be caught
        bad_choice = choice.copy()
        if rank == 1:
            bad_choice[0] = (bad_choice[0] + 1) % 8
        try:
            assert_ranks_agree(bad_choice, counts, lam)
            caught = False
        except RuntimeError:
            caught = True
        dist.destroy_process_group()
        q.put((rank, "ok", results, caught))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, "err", repr(e), False))


@pytest.mark.parametrize("world", [2])
def test_allgather_route_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, status, payload, caught in out:
        assert status == "ok", payload
        assert caught
    digests = [payload for _, _, payload, _ in sorted(out)]
    assert digests[0] == digests[1]
