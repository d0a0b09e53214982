"""Domain types of the routing API, kept name- and field-compatible with the
reference package so callers can switch imports (``eproute`` -> this package).

Reference: /root/reference/pkg/src/eproute/core.py
  ValidationError / ConfigurationError   core.py:14-19
  ClusterSpec, ModelSpec                 core.py:32-81
  PlacementMap                           core.py:84-119
  ExpertLoadVector                       core.py:122-140
  Token, TokenBatch                      core.py:143-176
  RoutingAssignment                      core.py:179-193
  aggregate_loads                        core.py:236-244  (here: sm_100a histogram)
  validate_assignment                    core.py:247-280

Objects of the reference's own classes are accepted wherever these types are
(duck-typed on ``.matrix`` / ``.loads`` / ``.tokens``).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np


class ValidationError(ValueError):
    """An input violates a structural invariant (reference core.py:14-15)."""


class ConfigurationError(ValueError):
    """Requested settings are internally inconsistent (reference core.py:18-19)."""


@dataclass(frozen=True)
class ClusterSpec:
    """One NVLink domain of GPUs (only ``num_gpus`` matters on the routing path)."""

    num_gpus: int
    hbm_bandwidth: float
    peak_flops: float
    link_bandwidth: float
    collective_launch_overhead: float
    link_base_latency: float

    def __post_init__(self):
        if self.num_gpus < 1:
            raise ValidationError("num_gpus must be >= 1")
        for name in ("hbm_bandwidth", "peak_flops", "link_bandwidth"):
            if getattr(self, name) <= 0:
                raise ValidationError(f"{name} must be positive")
        for name in ("collective_launch_overhead", "link_base_latency"):
            if getattr(self, name) < 0:
                raise ValidationError(f"{name} must be non-negative")


@dataclass(frozen=True)
class ModelSpec:
    """MoE geometry (``num_experts`` and ``top_k`` drive routing)."""

    num_experts: int
    top_k: int
    hidden_dim: int
    dtype_bytes: int
    expert_weight_bytes: float
    dense_weight_bytes: float
    flops_per_token_per_expert: float
    num_moe_layers: int

    def __post_init__(self):
        if not 1 <= self.top_k <= self.num_experts:
            raise ValidationError("top_k must be in [1, num_experts]")
        positive = ("num_experts", "hidden_dim", "dtype_bytes", "expert_weight_bytes",
                    "flops_per_token_per_expert", "num_moe_layers")
        for name in positive:
            if getattr(self, name) <= 0:
                raise ValidationError(f"{name} must be positive")
        if self.dense_weight_bytes < 0:
            raise ValidationError("dense_weight_bytes must be non-negative")


@dataclass
class PlacementMap:
    """Binary expert x EP-rank replica matrix A[N, G] with equal slots per rank."""

    matrix: np.ndarray
    slots_per_gpu: int

    def __post_init__(self):
        self.matrix = np.asarray(self.matrix, dtype=np.int8)
        if self.matrix.ndim != 2:
            raise ValidationError("placement matrix must be 2-dimensional")

    @property
    def num_experts(self) -> int:
        return int(self.matrix.shape[0])

    @property
    def num_gpus(self) -> int:
        return int(self.matrix.shape[1])

    def replicas(self, expert: int) -> List[int]:
        """Ranks hosting ``expert`` in ascending order (the greedy's tie-break scan)."""
        return np.flatnonzero(self.matrix[expert]).tolist()

    def validate(self) -> None:
        m = self.matrix
        if ((m != 0) & (m != 1)).any():
            raise ValidationError("placement matrix must be binary")
        per_expert = m.sum(axis=1)
        empty = np.flatnonzero(per_expert < 1)
        if empty.size:
            raise ValidationError(f"expert {int(empty[0])} has no replica")
        per_rank = m.sum(axis=0)
        if (per_rank != self.slots_per_gpu).any():
            raise ValidationError(
                f"per-GPU slot counts {per_rank.tolist()} != slots_per_gpu={self.slots_per_gpu}"
            )


@dataclass
class ExpertLoadVector:
    """T[N]: (token, expert) selections per logical expert in one batch."""

    loads: np.ndarray

    def __post_init__(self):
        self.loads = np.asarray(self.loads, dtype=np.int64)
        if self.loads.ndim != 1:
            raise ValidationError("loads must be 1-dimensional")
        if (self.loads < 0).any():
            raise ValidationError("loads must be non-negative")

    @property
    def num_experts(self) -> int:
        return int(self.loads.shape[0])

    def total(self) -> int:
        return int(self.loads.sum())


@dataclass(frozen=True)
class Token:
    source_gpu: int
    expert_ids: Tuple[int, ...]


@dataclass
class TokenBatch:
    """A decode batch: per token its source rank and top-k expert ids."""

    tokens: List[Token] = field(default_factory=list)

    def __len__(self) -> int:
        return len(self.tokens)

    def validate(self, model: ModelSpec, cluster: ClusterSpec) -> None:
        for idx, tok in enumerate(self.tokens):
            if not 0 <= tok.source_gpu < cluster.num_gpus:
                raise ValidationError(f"token {idx}: source_gpu {tok.source_gpu} out of range")
            if len(tok.expert_ids) != model.top_k:
                raise ValidationError(
                    f"token {idx}: expected {model.top_k} expert ids, got {len(tok.expert_ids)}"
                )
            if len(set(tok.expert_ids)) != len(tok.expert_ids):
                raise ValidationError(f"token {idx}: expert ids must be distinct")
            for e in tok.expert_ids:
                if not 0 <= e < model.num_experts:
                    raise ValidationError(f"token {idx}: expert id {e} out of range")

    def max_tokens_per_source_gpu(self, num_gpus: int) -> int:
        if not num_gpus:
            return 0
        src = np.fromiter((t.source_gpu for t in self.tokens), dtype=np.int64, count=len(self.tokens))
        return int(np.bincount(src, minlength=num_gpus).max()) if src.size else 0

    # --- array views used by the device path -------------------------------
    def topk_ids(self, top_k: int) -> np.ndarray:
        """[B, k] int32 row-major ids (the device layout of the batch)."""
        if not self.tokens:
            return np.zeros((0, top_k), dtype=np.int32)
        flat = [e for t in self.tokens for e in t.expert_ids]
        if len(flat) != len(self.tokens) * top_k:
            # ragged batch: keep row-major order, callers use the flat view
            return np.asarray(flat, dtype=np.int64).astype(np.int32, copy=False)
        return np.asarray(flat, dtype=np.int64).reshape(len(self.tokens), top_k).astype(np.int32)

    @classmethod
    def from_topk(cls, ids: np.ndarray, num_gpus: int) -> "TokenBatch":
        """Inverse of topk_ids(); token j comes from rank j % G (reference core.py:328)."""
        ids = np.asarray(ids)
        return cls([Token(j % num_gpus, tuple(int(e) for e in row)) for j, row in enumerate(ids)])


@dataclass
class RoutingAssignment:
    """Router output: token split x[N, G], activations y[N, G], objective lam."""

    x: np.ndarray
    y: np.ndarray
    lam: int

    def __post_init__(self):
        self.x = np.asarray(self.x, dtype=np.int64)
        self.y = np.asarray(self.y, dtype=np.int8)
        self.lam = int(self.lam)

    def max_tokens_per_gpu(self) -> int:
        return int(self.x.sum(axis=0).max()) if self.x.size else 0


@dataclass
class ValidationReport:
    violations: List[str] = field(default_factory=list)

    @property
    def ok(self) -> bool:
        return not self.violations


def validate_assignment(a, A, T, require_single_replica: bool = False) -> ValidationReport:
    """Routing-constraint check (reference core.py:247-280), numpy on the host."""
    mat = np.asarray(A.matrix)
    loads = np.asarray(T.loads, dtype=np.int64)
    n, g = mat.shape
    if a.x.shape != (n, g) or a.y.shape != (n, g) or loads.shape[0] != n:
        raise ValidationError(
            f"dimension mismatch: x {a.x.shape}, y {a.y.shape}, A {(n, g)}, T {loads.shape[0]}"
        )
    rep = ValidationReport()
    col = a.y.sum(axis=0)
    checks = [
        ("constraint_1_activation_bound", (col > a.lam).any()),
        ("constraint_2_token_conservation", (a.x.sum(axis=1) != loads).any()),
        ("constraint_3_placement", (a.x[mat == 0] != 0).any() or (a.y[mat == 0] != 0).any()),
        ("constraint_4_activation_link", (a.x > loads[:, None] * a.y).any()),
        ("variable_domain", (a.x < 0).any() or not np.isin(a.y, (0, 1)).all()),
        ("lambda_mismatch", a.lam != (int(col.max()) if a.y.size else 0)),
    ]
    if require_single_replica:
        checks.append(("single_replica_form", ((a.x > 0).sum(axis=1) > 1).any()))
    rep.violations.extend(name for name, bad in checks if bad)
    return rep
