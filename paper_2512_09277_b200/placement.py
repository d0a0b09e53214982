"""Cold-path inputs of the router: EPLB-style replication + placement, and the
synthetic Zipf decode batches the benchmarks route.

These run on the host once per rebalance window / per benchmark input, never on
the per-layer path.  They restate the reference so the framework is usable
without it, and are pinned to the reference's outputs by
tests/test_placement_golden.py:

  zipf_popularity  reference core.py:283-292
  gen_zipf_trace   reference core.py:295-329  (gen_zipf_topk: same stream, array output)
  eplb_replicate   reference placement.py:36-80
  eplb_place       reference placement.py:83-128
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .core import ConfigurationError, ExpertLoadVector, PlacementMap, TokenBatch, ValidationError


@dataclass
class ReplicationPlan:
    """Replica count per expert for a target replication ratio."""

    replica_counts: np.ndarray
    replication_ratio: float

    def __post_init__(self):
        self.replica_counts = np.asarray(self.replica_counts, dtype=np.int64)
        if (self.replica_counts < 1).any():
            raise ValidationError("every expert needs at least one replica")

    @property
    def total_slots(self) -> int:
        return int(self.replica_counts.sum())


def zipf_popularity(num_experts: int, skew: float, seed: int) -> np.ndarray:
    """Zipf(skew) expert probabilities; the rank -> expert map is a seeded permutation."""
    if skew < 0:
        raise ValidationError("skew must be >= 0")
    perm = np.random.default_rng(seed).permutation(num_experts)
    w = np.arange(1, num_experts + 1, dtype=np.float64) ** (-skew)
    probs = np.empty(num_experts, dtype=np.float64)
    probs[perm] = w / w.sum()
    return probs


def gen_zipf_topk(num_experts: int, top_k: int, num_tokens: int, skew: float, seed: int,
                  popularity_seed: Optional[int] = None) -> np.ndarray:
    """[num_tokens, top_k] int32 distinct expert ids per token, Gumbel top-k race.

    Same random stream and selection as the reference generator, so the ids are
    identical to ``gen_zipf_trace(...)`` for the same seeds (row j = token j,
    ids in descending key order).
    """
    if num_tokens < 0:
        raise ValidationError("tokens_per_gpu must be >= 0")
    pop = seed if popularity_seed is None else popularity_seed
    logp = np.log(zipf_popularity(num_experts, skew, pop))
    if num_tokens == 0:
        return np.zeros((0, top_k), dtype=np.int32)
    rng = np.random.default_rng(seed)
    keys = logp[None, :] + rng.gumbel(size=(num_tokens, num_experts))
    part = np.argpartition(-keys, top_k - 1, axis=1)[:, :top_k]
    sel = np.take_along_axis(keys, part, axis=1)
    desc = np.argsort(-sel, axis=1)
    return np.take_along_axis(part, desc, axis=1).astype(np.int32)


def gen_zipf_trace(model, cluster, tokens_per_gpu: int, skew: float, seed: int,
                   popularity_seed: Optional[int] = None) -> TokenBatch:
    """TokenBatch form of gen_zipf_topk (token j comes from rank j % G)."""
    g = int(cluster.num_gpus)
    ids = gen_zipf_topk(model.num_experts, model.top_k, tokens_per_gpu * g, skew, seed, popularity_seed)
    return TokenBatch.from_topk(ids, g)


def eplb_replicate(history: ExpertLoadVector, ratio: float, num_gpus: int) -> ReplicationPlan:
    """round(N * ratio) slots: one base replica per expert, extras by largest
    remainder of the load-proportional quota, capped at one replica per rank."""
    if ratio < 1:
        raise ConfigurationError("replication ratio must be >= 1")
    loads = np.asarray(getattr(history, "loads", history), dtype=np.int64)
    n = loads.shape[0]
    total = round(n * ratio)
    if total % num_gpus:
        raise ConfigurationError(
            f"round(N*ratio)={total} is not divisible by G={num_gpus}; "
            "memory-balanced placement is impossible"
        )
    if total > n * num_gpus:
        raise ConfigurationError("more slots requested than expert-GPU pairs")
    extras = total - n
    lf = loads.astype(np.float64)
    s = lf.sum()
    quotas = np.full(n, extras / n) if s == 0 else extras * lf / s
    whole = np.floor(quotas)
    counts = np.minimum(1 + whole.astype(np.int64), num_gpus)
    frac = quotas - whole
    order = np.lexsort((np.arange(n), -frac))  # largest remainder, then lower id
    left = extras - int(counts.sum() - n)
    while left > 0:
        room = order[counts[order] < num_gpus]
        if room.size == 0:
            raise ConfigurationError("cannot place all slots: every expert is at the GPU cap")
        take = room[:left]
        counts[take] += 1
        left -= take.size
    return ReplicationPlan(replica_counts=counts, replication_ratio=ratio)


def eplb_place(plan: ReplicationPlan, history: ExpertLoadVector, num_gpus: int) -> PlacementMap:
    """Heaviest expected replica first onto the least-loaded rank that has a free
    slot and does not host the expert yet; ties -> lower expert id, lower rank."""
    loads = np.asarray(getattr(history, "loads", history), dtype=np.int64)
    n = loads.shape[0]
    r = plan.replica_counts
    if r.shape[0] != n:
        raise ValidationError("plan and history dimensions disagree")
    if plan.total_slots % num_gpus:
        raise ConfigurationError("total slots not divisible by GPU count")
    slots = plan.total_slots // num_gpus
    expert = np.repeat(np.arange(n), r)
    expected = loads[expert] / r[expert]
    seq = np.lexsort((expert, -expected))
    A = np.zeros((n, num_gpus), dtype=np.int8)
    rank_load = np.zeros(num_gpus, dtype=np.float64)
    used = np.zeros(num_gpus, dtype=np.int64)
    for j in seq:
        i = expert[j]
        ok = (used < slots) & (A[i] == 0)
        if not ok.any():
            raise ConfigurationError(f"no feasible GPU left for a replica of expert {i}")
        best = int(np.argmin(np.where(ok, rank_load, np.inf)))
        A[i, best] = 1
        rank_load[best] += expected[j]
        used[best] += 1
    pm = PlacementMap(matrix=A, slots_per_gpu=slots)
    pm.validate()
    return pm


def make_placement(num_experts: int, num_ranks: int, ratio: float, history_seed: int = 7,
                   skew: float = 1.2) -> PlacementMap:
    """Placement from a synthetic Zipf history, as the reference tests build it
    (reference pkg/tests/conftest.py:48-53)."""
    probs = zipf_popularity(num_experts, skew, history_seed)
    hist = ExpertLoadVector(np.round(probs * 1e6).astype(np.int64))
    return eplb_place(eplb_replicate(hist, ratio, num_ranks), hist, num_ranks)
