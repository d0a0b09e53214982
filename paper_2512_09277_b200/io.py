"""On-disk formats either side of the routing path:
line-delimited JSON traces, placements and assignments, format-compatible with
the reference so traces recorded for / by it drive this router unchanged.

  Trace / TraceBatch / TraceFormatError   reference core.py:22-29, :196-222
  save_trace / load_trace                 reference core.py:332-400
  save_placement / load_placement         reference placement.py:131-171
  save_assignment                         reference routing.py:236-244 (in routing.py)

``load_trace_topk`` additionally returns each batch as the int32 [B, k] array
the device router consumes, without building Python Token objects.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .core import PlacementMap, Token, TokenBatch, ValidationError

PHASES = ("prefill", "decode")
_SEP = (",", ":")


class TraceFormatError(ValueError):
    """Malformed trace file; ``line`` is the 1-based offending line (or None)."""

    def __init__(self, message: str, line: Optional[int] = None):
        self.line = line
        super().__init__(f"line {line}: {message}" if line is not None else message)


@dataclass
class TraceBatch:
    layer: int
    phase: str
    batch: TokenBatch


@dataclass
class Trace:
    num_experts: int
    num_gpus: int
    top_k: int
    batches: List[TraceBatch] = field(default_factory=list)

    def validate(self, model, cluster) -> None:
        if self.num_experts != model.num_experts or self.top_k != model.top_k:
            raise ValidationError("trace header does not match model spec")
        if self.num_gpus != cluster.num_gpus:
            raise ValidationError("trace header does not match cluster spec")
        for tb in self.batches:
            if not 0 <= tb.layer < model.num_moe_layers:
                raise ValidationError(f"layer index {tb.layer} out of range")
            if tb.phase not in PHASES:
                raise ValidationError(f"unknown phase {tb.phase!r}")
            tb.batch.validate(model, cluster)


def save_trace(trace: Trace, path) -> None:
    with open(path, "w", encoding="utf-8") as f:
        f.write(json.dumps({"header": {"N": trace.num_experts, "G": trace.num_gpus, "k": trace.top_k}},
                           separators=_SEP) + "\n")
        for tb in trace.batches:
            toks = [{"src": t.source_gpu, "experts": list(t.expert_ids)} for t in tb.batch.tokens]
            f.write(json.dumps({"layer": tb.layer, "phase": tb.phase, "tokens": toks}, separators=_SEP) + "\n")


def _records(path):
    with open(path, "r", encoding="utf-8") as f:
        for lineno, line in enumerate(f, start=1):
            line = line.strip()
            if not line:
                continue
            try:
                yield lineno, json.loads(line)
            except json.JSONDecodeError as exc:
                raise TraceFormatError(f"invalid JSON: {exc}", lineno) from exc


def _parse(path, want_arrays: bool):
    header = None
    batches, arrays = [], []
    for lineno, rec in _records(path):
        if header is None:
            h = rec.get("header")
            if not isinstance(h, dict):
                raise TraceFormatError("first record must be the header", lineno)
            try:
                header = (int(h["N"]), int(h["G"]), int(h["k"]))
            except KeyError as exc:
                raise TraceFormatError(f"header missing field {exc}", lineno) from exc
            continue
        n, g, k = header
        try:
            layer, phase, raw = int(rec["layer"]), rec["phase"], rec["tokens"]
        except KeyError as exc:
            raise TraceFormatError(f"batch record missing field {exc}", lineno) from exc
        if phase not in PHASES:
            raise TraceFormatError(f"unknown phase {phase!r}", lineno)
        src = np.empty(len(raw), dtype=np.int64)
        ids = np.empty((len(raw), k), dtype=np.int64)
        for j, t in enumerate(raw):
            e = [int(v) for v in t["experts"]]
            if len(e) != k:
                raise TraceFormatError(f"expected {k} expert ids, got {len(e)}", lineno)
            s = int(t["src"])
            if not 0 <= s < g:
                raise TraceFormatError(f"source gpu {s} out of range", lineno)
            for v in e:
                if not 0 <= v < n:
                    raise TraceFormatError(f"expert id {v} out of range", lineno)
            src[j] = s
            ids[j] = e
        if want_arrays:
            arrays.append((layer, phase, ids.astype(np.int32), src.astype(np.int32)))
        else:
            toks = [Token(int(s), tuple(int(v) for v in row)) for s, row in zip(src, ids)]
            batches.append(TraceBatch(layer, phase, TokenBatch(toks)))
    return header, batches, arrays


def load_trace(path) -> Trace:
    header, batches, _ = _parse(path, False)
    if header is None:  # a file with no records is an empty trace
        return Trace(0, 0, 0)
    return Trace(*header, batches=batches)


def load_trace_topk(path):
    """[(layer, phase, topk_ids int32 [B, k], source_gpu int32 [B])] + (N, G, k)."""
    header, _, arrays = _parse(path, True)
    return (header or (0, 0, 0)), arrays


def save_placement(placement: PlacementMap, path) -> None:
    with open(path, "w", encoding="utf-8") as f:
        f.write(json.dumps({"header": {"N": placement.num_experts, "G": placement.num_gpus,
                                       "slots_per_gpu": placement.slots_per_gpu}}, separators=_SEP) + "\n")
        for i in range(placement.num_experts):
            f.write(json.dumps({"expert": i, "gpus": placement.replicas(i)}, separators=_SEP) + "\n")


def load_placement(path) -> PlacementMap:
    header, rows = None, {}
    with open(path, "r", encoding="utf-8") as f:
        for lineno, line in enumerate(f, start=1):
            line = line.strip()
            if not line:
                continue
            rec = json.loads(line)
            if header is None:
                header = rec.get("header")
                if not isinstance(header, dict):
                    raise ValidationError(f"line {lineno}: first record must be the header")
                continue
            rows[int(rec["expert"])] = [int(g) for g in rec["gpus"]]
    if header is None:
        raise ValidationError("placement file has no header record")
    mat = np.zeros((int(header["N"]), int(header["G"])), dtype=np.int8)
    for i, gpus in rows.items():
        mat[i, gpus] = 1
    pm = PlacementMap(matrix=mat, slots_per_gpu=int(header["slots_per_gpu"]))
    pm.validate()
    return pm
