"""FusedAllGatherRouter across PROCESSES (-m gpu): two ranks, one process each,
exchange buffers mapped with CUDA IPC handles all-gathered over a gloo group,
the fused kernel's LL exchange between the processes.  Both processes share the
one GPU of the test box (their contexts time-slice, so this checks the plumbing
and the protocol, not speed), and each must produce the oracle's routing of the
global batch and the pair ranks of its own tokens.
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
        from paper_2512_09277_b200 import DevicePlacement
        from paper_2512_09277_b200.dist import FusedAllGatherRouter
        from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement

        torch.cuda.set_device(0)
        A = make_placement(256, 8, 1.5, 7).matrix
        pl = DevicePlacement(A, torch.device("cuda", 0))
        B, k = 256, 8
        lt = B // world
        fz = FusedAllGatherRouter(pl, lt, k, gather_ids=True)
        for call in range(3):
            ids = gen_zipf_topk(256, k, B, 1.2, 500 + call, popularity_seed=7)
            mine = torch.from_numpy(ids[rank * lt:(rank + 1) * lt].copy()).cuda()
            out = fz.step(mine)
            torch.cuda.synchronize()
            out.check()
            T = oracle.aggregate_loads(ids, 256)
            choice, counts, lam = oracle.route_metro(T, A)
            assert np.array_equal(out.choice.cpu().numpy(), choice)
            assert np.array_equal(out.rank_counts.cpu().numpy(), counts)
            assert int(out.lam.item()) == lam
            own = ids[rank * lt:(rank + 1) * lt]
            assert np.array_equal(out.pair_rank.cpu().numpy().reshape(own.shape), oracle.pair_rank_metro(own, choice))
            assert np.array_equal(fz.gathered.cpu().numpy(), ids)
        dist.barrier()
        fz.close()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as ex:  # noqa: BLE001
        q.put((rank, repr(ex)))


def test_fused_allgather_two_processes():
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
