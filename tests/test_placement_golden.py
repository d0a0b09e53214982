"""The package's cold-path generators reproduce the reference's outputs exactly."""

import numpy as np

from paper_2512_09277_b200 import (
    ExpertLoadVector, eplb_place, eplb_replicate, gen_zipf_topk, make_placement, zipf_popularity,
)
from conftest import GOLDEN


def test_placement_golden():
    z = np.load(f"{GOLDEN}/placement.npz")
    for j in range(int(z["count"])):
        n, g = (int(v) for v in z[f"p{j}_meta"])
        ratio = float(z[f"p{j}_ratio"])
        probs = zipf_popularity(n, 1.2, 7)
        assert np.array_equal(probs, z[f"p{j}_probs"])
        hist = ExpertLoadVector(np.round(probs * 1e6).astype(np.int64))
        plan = eplb_replicate(hist, ratio, g)
        assert np.array_equal(plan.replica_counts, z[f"p{j}_counts"])
        A = eplb_place(plan, hist, g)
        assert np.array_equal(A.matrix, z[f"p{j}_A"])


def test_shapes_inputs_reproduced(shapes):
    for c in shapes:
        A = make_placement(c["N"], c["G"], c["ratio"], 7)
        assert np.array_equal(A.matrix, c["A"]), c["name"]
        ids = gen_zipf_topk(c["N"], c["k"], c["B"], c["skew"], c["seed"], popularity_seed=7)
        assert np.array_equal(ids, c["ids"]), c["name"]
        assert np.array_equal(c["src"], np.arange(c["B"]) % c["G"])


def test_generators_vs_reference(eproute_ref):
    from eproute import ClusterSpec, ModelSpec
    from eproute.core import gen_zipf_trace
    from eproute.placement import eplb_place as rplace, eplb_replicate as rrep

    rng = np.random.default_rng(5)
    for _ in range(40):
        n = int(rng.choice([8, 16, 32, 64, 128]))
        g = int(rng.choice([2, 4, 8]))
        ratios = [r for r in (1.0, 1.125, 1.25, 1.5, 2.0) if round(n * r) % g == 0 and round(n * r) <= n * g]
        ratio = float(rng.choice(ratios))
        hist = ExpertLoadVector(rng.integers(0, 10_000, size=n))
        ours = eplb_place(eplb_replicate(hist, ratio, g), hist, g)
        ref = rplace(rrep(eproute_ref.ExpertLoadVector(hist.loads), ratio, g),
                     eproute_ref.ExpertLoadVector(hist.loads), g)
        assert np.array_equal(ours.matrix, ref.matrix)
        k = int(rng.integers(1, min(8, n) + 1))
        seed = int(rng.integers(1 << 30))
        b = gen_zipf_trace(ModelSpec(n, k, 64, 2, 1.0, 0.0, 1.0, 1), ClusterSpec(g, 1, 1, 1, 0, 0), 3, 1.1, seed)
        ids = np.array([t.expert_ids for t in b.tokens], dtype=np.int32)
        assert np.array_equal(gen_zipf_topk(n, k, 3 * g, 1.1, seed), ids)
