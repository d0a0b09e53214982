"""Generate golden vectors for the METRO routing path from the UNMODIFIED reference.

Run in the build container (the reference only exists there):

    python tests/golden/make_golden.py

It imports ``eproute`` from ``/root/reference/pkg/src`` and the reference's own
test fixtures (``/root/reference/pkg/tests/conftest.py``: ``make_placement``,
``random_small_instance``, ``random_dominance_instance``), runs the reference
functions and stores inputs + outputs as compressed ``.npz`` fixtures next to
this script.  The GPU box never reads ``/root/reference``; it only reads these
committed files.

Fixtures
--------
``shapes.npz``   BASELINE.json shapes (Qwen3-30B, DeepSeek-V3 + batch sweep +
                 skew sweep, Qwen3-235B at 3 ratios): placement A (make_placement,
                 conftest.py:48-53), top-k ids (gen_zipf_trace, core.py:295-329),
                 loads T (aggregate_loads, core.py:236-244), METRO choice/counts/lam
                 (route_metro, routing.py:105-113), EPLB x/lam (route_eplb,
                 routing.py:55-72).
``small.npz``    reference test families: random_small_instance (conftest.py:56-71)
                 and random_dominance_instance (conftest.py:74-91) as (T, A) pairs
                 with METRO and EPLB outputs.
``placement.npz`` zipf_popularity / eplb_replicate / eplb_place outputs used to pin
                 the package's cold-path placement + synthetic-trace generator.
``gate.npz``     the gating scores behind gen_zipf_trace's top-k (core.py:316-326:
                 log(popularity) + Gumbel noise from the same seeded stream), as
                 float32, with the reference's top-k ids for the same batch -- pins
                 the fused gating top-k (metro_route_scores_v1) and its oracle.

``python make_golden.py gate`` rewrites gate.npz only.
"""

from __future__ import annotations

import importlib.util
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_CONFTEST = "/root/reference/pkg/tests/conftest.py"
HERE = os.path.dirname(os.path.abspath(__file__))

sys.path.insert(0, REF_SRC)
import eproute  # noqa: E402
from eproute import ClusterSpec, ExpertLoadVector, ModelSpec, PlacementMap  # noqa: E402
from eproute.core import aggregate_loads, gen_zipf_trace, zipf_popularity  # noqa: E402
from eproute.placement import eplb_place, eplb_replicate  # noqa: E402
from eproute.routing import route_eplb, route_metro  # noqa: E402

_spec = importlib.util.spec_from_file_location("ref_conftest", REF_CONFTEST)
ref_conftest = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(ref_conftest)

HISTORY_SEED = 7  # make_placement(N, G, ratio, history_seed=7)


def model(n: int, k: int) -> ModelSpec:
    return ModelSpec(n, k, 4096, 2, 1e6, 0.0, 1e6, 1)


def cluster(g: int) -> ClusterSpec:
    return ClusterSpec(g, 1e12, 1e12, 1e11, 0.0, 0.0)


def choice_of(a, loads) -> np.ndarray:
    """Recover per-expert choice (-1 = inactive) from a single-replica y."""
    n, _ = a.y.shape
    ch = np.full(n, -1, dtype=np.int32)
    rows, cols = np.nonzero(a.y)
    ch[rows] = cols
    assert ((ch >= 0) == (loads > 0)).all()
    return ch


# (name, N, k, G, ratio, B, skew, seeds)
SHAPES = [
    ("q30", 128, 8, 8, 1.5, 256, 1.2, range(1000, 1008)),
    ("ds", 256, 8, 8, 1.5, 1024, 1.2, range(1000, 1008)),
    ("ds_b64", 256, 8, 8, 1.5, 64, 1.2, range(1000, 1006)),
    ("ds_b128", 256, 8, 8, 1.5, 128, 1.2, range(1000, 1004)),
    ("ds_b256", 256, 8, 8, 1.5, 256, 1.2, range(1000, 1004)),
    ("ds_b512", 256, 8, 8, 1.5, 512, 1.2, range(1000, 1004)),
    ("ds_b2048", 256, 8, 8, 1.5, 2048, 1.2, range(1000, 1002)),
    ("ds_b4096", 256, 8, 8, 1.5, 4096, 1.2, range(1000, 1001)),
    ("ds_b8192", 256, 8, 8, 1.5, 8192, 1.2, range(1000, 1001)),
    ("ds_skew05", 256, 8, 8, 1.5, 1024, 0.5, range(1000, 1003)),
    ("ds_skew20", 256, 8, 8, 1.5, 1024, 2.0, range(1000, 1003)),
    ("q235_125", 128, 8, 16, 1.25, 1024, 1.2, range(1000, 1003)),
    ("q235_150", 128, 8, 16, 1.5, 1024, 1.2, range(1000, 1003)),
    ("q235_200", 128, 8, 16, 2.0, 1024, 1.2, range(1000, 1003)),
]


def make_shapes() -> dict:
    out = {}
    idx = 0
    for name, n, k, g, ratio, b, skew, seeds in SHAPES:
        A = ref_conftest.make_placement(n, g, ratio, history_seed=HISTORY_SEED)
        A.validate()
        for seed in seeds:
            batch = gen_zipf_trace(model(n, k), cluster(g), b // g, skew, seed,
                                   popularity_seed=HISTORY_SEED)
            ids = np.array([t.expert_ids for t in batch.tokens], dtype=np.int32).reshape(b, k)
            src = np.array([t.source_gpu for t in batch.tokens], dtype=np.int32)
            T = aggregate_loads(batch, model(n, k))
            m = route_metro(T, A)
            e = route_eplb(T, A)
            p = f"c{idx}_"
            out[p + "meta"] = np.array([n, k, g, b, seed], dtype=np.int64)
            out[p + "ratio_skew"] = np.array([ratio, skew], dtype=np.float64)
            out[p + "name"] = np.array(name)
            out[p + "A"] = A.matrix.astype(np.int8)
            out[p + "slots"] = np.array(A.slots_per_gpu, dtype=np.int64)
            out[p + "ids"] = ids
            out[p + "src"] = src
            out[p + "T"] = T.loads.astype(np.int64)
            out[p + "metro_choice"] = choice_of(m, T.loads)
            out[p + "metro_counts"] = m.y.sum(axis=0).astype(np.int64)
            out[p + "metro_lam"] = np.array(m.lam, dtype=np.int64)
            out[p + "metro_maxtok"] = np.array(m.max_tokens_per_gpu(), dtype=np.int64)
            out[p + "eplb_x"] = e.x.astype(np.int32)
            out[p + "eplb_counts"] = e.y.sum(axis=0).astype(np.int64)
            out[p + "eplb_lam"] = np.array(e.lam, dtype=np.int64)
            out[p + "eplb_maxtok"] = np.array(e.max_tokens_per_gpu(), dtype=np.int64)
            idx += 1
    out["count"] = np.array(idx, dtype=np.int64)
    return out


def make_small(num_small: int = 1500, num_dom: int = 400) -> dict:
    """Ragged (T, A) instances stored as concatenations + offsets."""
    Ts, As, shapes, fam = [], [], [], []
    rng = np.random.default_rng(20251209)
    for _ in range(num_small):
        T, A = ref_conftest.random_small_instance(rng, max_active=10, max_g=4)
        Ts.append(T.loads); As.append(A.matrix); shapes.append(A.matrix.shape); fam.append(0)
    rng = np.random.default_rng(977)
    for _ in range(num_small // 3):
        T, A = ref_conftest.random_small_instance(rng, max_active=24, max_g=12)
        Ts.append(T.loads); As.append(A.matrix); shapes.append(A.matrix.shape); fam.append(1)
    rng = np.random.default_rng(0)  # test_acceptance.py:52 uses seed 0 for this family
    for _ in range(num_dom):
        T, A = ref_conftest.random_dominance_instance(rng)
        Ts.append(T.loads); As.append(A.matrix); shapes.append(A.matrix.shape); fam.append(2)
    # hand-derived known answers from pkg/tests/test_routing.py
    hand = [
        ([[1, 1, 1]], [6]), ([[1, 1, 1]], [5]), ([[1, 1], [1, 1]], [8, 8]),
        ([[1, 1], [1, 1]], [0, 0]), ([[1, 1, 0], [1, 0, 1], [0, 1, 1]], [1, 3, 8]),
        ([[1, 0, 0], [0, 1, 0], [0, 0, 1]], [4, 9, 2]), ([[1, 1]], [0]), ([[1, 1, 1]], [9]),
        ([[1, 1], [1, 1]], [4, 4]), ([[1, 1], [1, 1]], [3, 3]), ([[1, 1], [1, 1]], [5, 3]),
        ([[1, 1, 0], [0, 0, 1]], [5, 0]),
    ]
    for mat, loads in hand:
        mat = np.asarray(mat, dtype=np.int8)
        Ts.append(np.asarray(loads, dtype=np.int64)); As.append(mat); shapes.append(mat.shape); fam.append(3)
    # large / adversarial loads: T up to 2**40 (accepted by the reference), ties everywhere
    rng = np.random.default_rng(4242)
    for _ in range(60):
        n = int(rng.integers(1, 64)); g = int(rng.integers(1, 33))
        mat = (rng.random((n, g)) < rng.uniform(0.05, 0.9)).astype(np.int8)
        for i in range(n):
            if mat[i].sum() == 0:
                mat[i, rng.integers(g)] = 1
        kind = rng.integers(3)
        if kind == 0:
            loads = rng.integers(0, 3, size=n)
        elif kind == 1:
            loads = rng.integers(0, 2 ** 40, size=n) * (rng.random(n) < 0.7)
        else:
            loads = np.full(n, int(rng.integers(1, 5)))
        Ts.append(loads.astype(np.int64)); As.append(mat); shapes.append(mat.shape); fam.append(4)

    metro_choice, metro_lam, eplb_x, eplb_lam = [], [], [], []
    for T, A in zip(Ts, As):
        Tv = ExpertLoadVector(T)
        Am = PlacementMap(matrix=A, slots_per_gpu=int(A.sum(axis=0).max()) if A.size else 0)
        m = route_metro(Tv, Am)
        e = route_eplb(Tv, Am)
        metro_choice.append(choice_of(m, Tv.loads)); metro_lam.append(m.lam)
        eplb_x.append(e.x.reshape(-1)); eplb_lam.append(e.lam)
    shapes = np.array(shapes, dtype=np.int64)
    return {
        "shapes": shapes,
        "family": np.array(fam, dtype=np.int64),
        "T": np.concatenate(Ts).astype(np.int64),
        "A": np.concatenate([a.reshape(-1) for a in As]).astype(np.int8),
        "metro_choice": np.concatenate(metro_choice).astype(np.int32),
        "metro_lam": np.array(metro_lam, dtype=np.int64),
        "eplb_x": np.concatenate(eplb_x).astype(np.int64),
        "eplb_lam": np.array(eplb_lam, dtype=np.int64),
    }


def make_placement_golden() -> dict:
    out = {}
    cases = [(128, 8, 1.5), (256, 8, 1.5), (128, 16, 1.25), (128, 16, 1.5), (128, 16, 2.0),
             (128, 8, 1.25), (64, 4, 1.0), (32, 8, 1.5)]
    for j, (n, g, ratio) in enumerate(cases):
        probs = zipf_popularity(n, 1.2, HISTORY_SEED)
        history = ExpertLoadVector(np.round(probs * 1e6).astype(np.int64))
        plan = eplb_replicate(history, ratio, g)
        A = eplb_place(plan, history, g)
        out[f"p{j}_meta"] = np.array([n, g], dtype=np.int64)
        out[f"p{j}_ratio"] = np.array(ratio)
        out[f"p{j}_probs"] = probs
        out[f"p{j}_counts"] = plan.replica_counts
        out[f"p{j}_A"] = A.matrix.astype(np.int8)
    out["count"] = np.array(len(cases))
    return out


GATE_CASES = [  # (N, k, G, tokens per GPU, skew, seed)
    (128, 8, 8, 32, 1.2, 1000),   # Qwen3-30B-A3B, B=256
    (256, 8, 8, 32, 1.2, 1000),   # DeepSeek-V3, B=256
    (256, 8, 8, 8, 0.5, 1001),    # DeepSeek-V3, flatter popularity
    (512, 8, 8, 8, 1.2, 1002),    # N at the kernel limit
    (64, 1, 4, 16, 1.2, 1003),    # top-1
    (64, 32, 4, 4, 2.0, 1004),    # top-32, strong skew
]


def make_gate() -> dict:
    out = {}
    for j, (n, k, g, tpg, skew, seed) in enumerate(GATE_CASES):
        batch = gen_zipf_trace(model(n, k), cluster(g), tpg, skew, seed, popularity_seed=HISTORY_SEED)
        ids = np.array([t.expert_ids for t in batch.tokens], dtype=np.int32).reshape(-1, k)
        # the same scores the generator ranks (core.py:316-322, same seeded stream)
        probs = zipf_popularity(n, skew, HISTORY_SEED)
        rng = np.random.default_rng(seed)
        keys = np.log(probs)[None, :] + rng.gumbel(size=(tpg * g, n))
        assert (np.argsort(-keys, axis=1, kind="stable")[:, :k] == ids).all()
        out[f"g{j}_meta"] = np.array([n, k, g, tpg * g, seed], dtype=np.int64)
        out[f"g{j}_scores"] = keys.astype(np.float32)
        out[f"g{j}_ids"] = ids
    out["count"] = np.array(len(GATE_CASES))
    return out


def main() -> None:
    if sys.argv[1:] == ["gate"]:
        np.savez_compressed(os.path.join(HERE, "gate.npz"), **make_gate())
        print("wrote gate.npz")
        return
    np.savez_compressed(os.path.join(HERE, "gate.npz"), **make_gate())
    np.savez_compressed(os.path.join(HERE, "shapes.npz"), **make_shapes())
    np.savez_compressed(os.path.join(HERE, "small.npz"), **make_small())
    np.savez_compressed(os.path.join(HERE, "placement.npz"), **make_placement_golden())
    with open(os.path.join(HERE, "PROVENANCE.txt"), "w") as f:
        f.write(
            "Generated by tests/golden/make_golden.py from the unmodified reference\n"
            f"eproute {eproute.__version__} at {REF_SRC} with numpy {np.__version__}.\n"
        )
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
