"""The N > 1 product path across PROCESSES through the device router (-m gpu):
world_size-2 gloo process group, both ranks on the box's one GPU.

Each rank holds its own decode tokens; it (1) all-gathers them with
``allgather_topk`` (gloo staging: NCCL refuses two ranks on one device) and
routes the global batch with ``DistributedRouter`` (the NCCL-path class), and
(2) runs ``FusedAllGatherRouter`` with the global dispatch layout (histogram
exchange over CUDA IPC, one kernel).  Both must equal the oracle's routing of
the global batch, the pair ranks / rows of the rank's own tokens must match the
oracle's layout, and the ranks must agree (routing digest all-gathered).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), METRO_PEER_TIMEOUT_MS="20000")
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        from paper_2512_09277_b200 import DevicePlacement, DispatchLayout
        from paper_2512_09277_b200.dist import (DistributedRouter, FusedAllGatherRouter, assert_ranks_agree,
                                                shard_tokens)
        from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement

        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        A = make_placement(256, 8, 1.5, 7).matrix
        pl = DevicePlacement(A, dev)
        B, k = 1024, 8
        lt = B // world
        dr = DistributedRouter(pl, lt, k, "metro")
        fz = FusedAllGatherRouter(pl, lt, k, layout=DispatchLayout(pl))
        for call in range(3):
            glob = gen_zipf_topk(256, k, B, 1.2, 700 + call, popularity_seed=7)
            mine = torch.from_numpy(shard_tokens(glob, world, rank).copy()).to(dev)
            T = oracle.aggregate_loads(glob, 256)
            choice, counts, lam = oracle.route_metro(T, A)
            own = oracle.pair_rank_metro(glob, choice).reshape(-1)[rank * lt * k:(rank + 1) * lt * k]
            row, off = oracle.dispatch_layout(glob, oracle.pair_rank_metro(glob, choice), A)
            own_row = np.asarray(row).reshape(-1)[rank * lt * k:(rank + 1) * lt * k]
            # (1) all-gather + device router
            dr.local.copy_(mine)
            o = dr.step()
            torch.cuda.synchronize()
            o.check()
            assert np.array_equal(dr.gathered.cpu().numpy(), glob)
            assert np.array_equal(o.choice.cpu().numpy(), choice)
            assert int(o.lam.item()) == lam
            assert np.array_equal(dr.own_pair_rank().cpu().numpy(), own)
            assert_ranks_agree(o.choice.cpu().numpy(), o.rank_counts.cpu().numpy(), int(o.lam.item()))
            # (2) fused exchange + route + global dispatch layout
            f = fz.step(mine)
            torch.cuda.synchronize()
            f.check()
            assert np.array_equal(f.choice.cpu().numpy(), choice)
            assert np.array_equal(f.rank_counts.cpu().numpy(), counts)
            assert np.array_equal(f.pair_rank.cpu().numpy(), own)
            assert np.array_equal(fz.layout_out.pair_row.cpu().numpy()[:lt * k], own_row)
            assert np.array_equal(fz.layout_out.rep_off.cpu().numpy(), off)
            assert_ranks_agree(f.choice.cpu().numpy(), f.rank_counts.cpu().numpy(), int(f.lam.item()))
        dist.barrier()
        fz.close()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as ex:  # noqa: BLE001
        import traceback

        q.put((rank, repr(ex) + traceback.format_exc()[-800:]))


def test_two_process_device_routing():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
