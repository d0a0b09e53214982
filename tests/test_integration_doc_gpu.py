"""INTEGRATION.md §3 as written (-m gpu): the serving-side snippets run and agree
with the oracle, so the guide a maintainer follows is the tested path."""

import numpy as np
import pytest
import torch

import oracle
from paper_2512_09277_b200 import DevicePlacement, Router
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.init()


def test_integration_section3_snippets():
    device = torch.device("cuda", 0)
    A = make_placement(256, 8, 1.5, 7).matrix
    B, k = 256, 8
    topk = gen_zipf_topk(256, k, B, 1.2, 77, popularity_seed=7)
    topk_ids = torch.from_numpy(topk).to(device)

    # device fast path
    placement = DevicePlacement(A, device)
    router = Router(placement, "metro")
    out = router.alloc(num_pairs=B * k, top_k=k)
    router.route(topk_ids, out=out)
    out.check()
    T = oracle.aggregate_loads(topk, 256)
    choice, counts, lam = oracle.route_metro(T, A)
    assert np.array_equal(out.choice.cpu().numpy(), choice) and int(out.lam.item()) == lam

    # gating fused with routing
    scores = torch.randn((B, 256), device=device)
    ids, out2 = router.route_scores(scores, top_k=k)
    out2.check()
    ref_ids = oracle.gate_topk(scores.cpu().numpy(), k)
    assert np.array_equal(ids.cpu().numpy(), ref_ids)
    c2, _, l2 = oracle.route_metro(oracle.aggregate_loads(ref_ids, 256), A)
    assert np.array_equal(out2.choice.cpu().numpy(), c2) and int(out2.lam.item()) == l2

    # dispatch layout and the rank's expert FFN
    from paper_2512_09277_b200.dispatch import DispatchLayout
    from paper_2512_09277_b200.moe import ExpertFFN, RankMoE

    lay = DispatchLayout(placement)
    res = lay(topk_ids, out.pair_rank)
    res.check()
    g = int(np.argmax(counts))
    ffn = ExpertFFN(lay.slots(g), 7168, 2048, device, dtype="fp8")
    layer = RankMoE(placement, "metro", g, ffn, max_pairs=B * k, top_k=k)
    hidden = torch.randn((B, 7168), device=device).to(torch.bfloat16)
    y = layer(topk_ids, hidden)
    torch.cuda.synchronize()
    rows = int(layer.counts[2].item())
    assert rows == int((out.pair_rank.cpu().numpy() == g).sum())
    assert torch.isfinite(y[:rows].float()).all()

    # METRO routing and its layout in one launch
    out3, res3 = lay.route_metro(topk_ids)
    out3.check()
    assert torch.equal(out3.pair_rank.reshape(-1)[:B * k], out.pair_rank.reshape(-1)[:B * k])
    assert torch.equal(res3.pair_row.reshape(-1)[:B * k], res.pair_row.reshape(-1)[:B * k])
    assert torch.equal(res3.rep_off, res.rep_off)

    # eager callers: a bound launch plan
    buf = topk_ids.clone()
    out4 = router.alloc(num_pairs=B * k, top_k=k)
    launch = router.bind(buf, out4)
    launch()
    out4.check()
    assert torch.equal(out4.choice, out.choice) and torch.equal(out4.pair_rank, out.pair_rank)


def test_integration_fused_exchange_layout_snippet():
    """§3's FusedAllGatherRouter(..., layout=lay) on one rank (world 1): its own
    pairs' rows equal the layout of the whole batch."""
    import torch.distributed as dist

    from paper_2512_09277_b200.dispatch import DispatchLayout
    from paper_2512_09277_b200.dist import FusedAllGatherRouter

    device = torch.device("cuda", 0)
    A = make_placement(256, 8, 1.5, 7).matrix
    B, k = 256, 8
    topk = gen_zipf_topk(256, k, B, 1.2, 78, popularity_seed=7)
    topk_ids = torch.from_numpy(topk).to(device)
    placement = DevicePlacement(A, device)
    lay = DispatchLayout(placement)
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("gloo", init_method="tcp://127.0.0.1:29631", rank=0, world_size=1)
    try:
        fzl = FusedAllGatherRouter(placement, local_tokens=B, top_k=k, layout=lay)
        out = fzl.step(topk_ids)
        out.check()
        T = oracle.aggregate_loads(topk, 256)
        choice, counts, lam = oracle.route_metro(T, A)
        row, off = oracle.dispatch_layout(topk, oracle.pair_rank_metro(topk, choice), A)
        assert np.array_equal(out.choice.cpu().numpy(), choice)
        assert np.array_equal(fzl.layout_out.pair_row.cpu().numpy()[:B * k], np.asarray(row).reshape(-1))
        assert np.array_equal(fzl.layout_out.rep_off.cpu().numpy()[:len(off)], off)
        fzl.close()
    finally:
        if own:
            dist.destroy_process_group()
