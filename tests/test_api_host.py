"""Host-side logic of the drop-in API (no GPU needed)."""

import numpy as np
import pytest

import paper_2512_09277_b200 as pkg
from paper_2512_09277_b200 import routing


def test_reference_names_exported(eproute_ref):
    missing = [n for n in eproute_ref.__all__ if not hasattr(pkg, n)]
    # the cost model (CostProfile / LayerTiming) is outside the routing hot path;
    # the trace / placement JSONL IO is built (io.py)
    allowed = {"CostProfile", "LayerTiming"}
    assert set(missing) <= allowed, missing


def test_dimension_mismatch_message():
    with pytest.raises(pkg.ValidationError, match="dimension mismatch: T has 2 experts, A has 1"):
        pkg.route_eplb(pkg.ExpertLoadVector(np.array([1, 2])), pkg.PlacementMap(np.ones((1, 2)), 1))
    with pytest.raises(pkg.ValidationError, match="dimension mismatch"):
        pkg.route_metro(np.array([1, 2, 3]), np.ones((2, 2)))


def test_unknown_router_kind():
    with pytest.raises(pkg.ValidationError, match="unknown router"):
        pkg.run_router("bogus", pkg.ExpertLoadVector([1]), pkg.PlacementMap([[1]], 1))


def test_cpu_quality_oracles_are_out_of_scope():
    for kind in ("optimal", "bruteforce"):
        with pytest.raises(NotImplementedError):
            pkg.run_router(kind, pkg.ExpertLoadVector([1]), pkg.PlacementMap([[1]], 1))


def test_no_cpu_fallback():
    """Without a GPU the product path raises instead of computing on the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(pkg.NativeLibraryError):
        pkg.route_metro(pkg.ExpertLoadVector([3, 1]), pkg.PlacementMap([[1, 1], [1, 0]], 1))
    with pytest.raises(pkg.NativeLibraryError):
        pkg.aggregate_loads(np.array([[0, 1]]), pkg.ModelSpec(2, 2, 8, 2, 1.0, 0.0, 1.0, 1))


def test_rank_compress_preserves_order():
    T = np.array([0, 5, 2 ** 40, 7, 2 ** 40, 0, 2 ** 35], dtype=np.int64)
    c = routing._rank_compress(T)
    assert c.max() < 2 ** 32
    assert ((c > 0) == (T > 0)).all()
    for i in range(len(T)):
        for j in range(len(T)):
            assert (T[i] < T[j]) == (c[i] < c[j])
    small = np.array([0, 3, 9])
    assert routing._rank_compress(small) is small


def test_lambda_of_and_validate():
    a = pkg.RoutingAssignment(x=np.zeros((2, 2)), y=np.zeros((2, 2)), lam=0)
    assert pkg.lambda_of(a) == 0
    A = pkg.PlacementMap(np.array([[1, 0], [0, 1]]), 1)
    bad = pkg.RoutingAssignment(x=np.array([[0, 3], [0, 0]]), y=np.array([[0, 1], [0, 0]]), lam=1)
    rep = pkg.validate_assignment(bad, A, pkg.ExpertLoadVector(np.array([3, 0])))
    assert "constraint_3_placement" in rep.violations
    with pytest.raises(pkg.ValidationError, match="dimension mismatch"):
        pkg.validate_assignment(pkg.RoutingAssignment(np.zeros((3, 2)), np.zeros((3, 2)), 0), A,
                                pkg.ExpertLoadVector(np.zeros(2)))


def test_token_batch_roundtrip():
    ids = np.array([[3, 1], [0, 2], [1, 3]], dtype=np.int32)
    b = pkg.TokenBatch.from_topk(ids, 2)
    assert [t.source_gpu for t in b.tokens] == [0, 1, 0]
    assert np.array_equal(b.topk_ids(2), ids)
    assert b.max_tokens_per_source_gpu(2) == 2


def test_moe_item_bound_checked_on_host():
    """an explicit max_item_tokens below a host item's token count is
    rejected before launch (it would select the 64-token tiling); numpy items with
    an explicit bound are converted (no AttributeError)."""
    from paper_2512_09277_b200 import moe
    items = np.array([[0, 0, 0, 100], [1, 0, 100, 30]], np.int32)
    t, bound = moe._items_and_bound(items, None)
    assert bound == 100 and tuple(t.shape) == (2, 4)
    t, bound = moe._items_and_bound(items, 256)
    assert bound == 256 and t.dtype == __import__("torch").int32
    with pytest.raises(pkg.ValidationError, match="above max_item_tokens"):
        moe._items_and_bound(items, 64)
