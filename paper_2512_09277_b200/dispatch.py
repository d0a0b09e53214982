"""Dispatch layout after routing: where each
(token, slot) pair lands in its serving EP rank's receive buffer, and the
per-replica row ranges the grouped expert GEMM consumes.

The reference ends at the assignment x (routing.py:41-52 METRO, :64-69 EPLB;
simulate.py:87-88 prices a rank's tokens from it).  The layout materialises
exactly those counts -- rank g holds x[i, g] rows of expert i -- in a fixed
order: rows grouped by the rank's local expert slot (ascending expert id), pairs
in row-major order inside a slot.  Computed on device by
``metro_dispatch_layout_v1`` (include/dispatch_layout.h); no CPU fallback.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np
import torch

from . import _native
from .core import ValidationError
from .device import DevicePlacement, RouteResult, Router, _ptr, raise_status


def replica_table(A) -> Tuple[np.ndarray, np.ndarray]:
    """(rid_tab [N, G] int32, slot_base [G + 1] int32) of a binary placement:
    replicas numbered rank-major, by local slot inside a rank; -1 = no replica."""
    mat = np.ascontiguousarray(np.asarray(getattr(A, "matrix", A)), dtype=np.int8)
    if mat.ndim != 2:
        raise ValidationError("placement matrix must be 2-dimensional")
    n, g = mat.shape
    rid = np.empty((n, g), np.int32)
    base = np.empty(g + 1, np.int32)
    rc = _native.lib().metro_replica_table(mat.ctypes.data, n, g, rid.ctypes.data, base.ctypes.data)
    _native.check_rc(rc, "metro_replica_table")
    return rid, base


@dataclass
class LayoutResult:
    """Device outputs of one dispatch-layout launch (int32 CUDA tensors)."""

    pair_row: torch.Tensor   # [num_pairs] row inside the serving rank's buffer
    rep_off: torch.Tensor    # [nrep + 1] exclusive row prefix per replica (rid order)
    status: torch.Tensor     # [4]
    top_k: int = 1

    def check(self) -> "LayoutResult":
        """Synchronise on status; raise ValidationError on a bad pair."""
        raise_status(self.status.cpu().numpy(), self.top_k)
        return self


class DispatchLayout:
    """Builds dispatch layouts for one placement on its device.

    ``slot_base[g]`` is rank g's first replica id; rank g's local slot s is
    replica ``slot_base[g] + s`` and holds rows
    ``[rep_off[slot_base[g] + s], rep_off[slot_base[g] + s + 1]) - rep_off[slot_base[g]]``.
    """

    def __init__(self, placement: DevicePlacement, cluster_ctas: int = 0):
        self.placement = placement
        self.cluster_ctas = int(cluster_ctas)
        mat = placement.matrix
        self.rid_host, self.slot_base_host = replica_table(mat)
        self.nrep = int(self.slot_base_host[-1])
        if not 1 <= self.nrep <= 4096:
            raise ValidationError(f"{self.nrep} replicas outside the dispatch-layout limit (1..4096)")
        dev = placement.device
        self.rid_tab = torch.from_numpy(self.rid_host.reshape(-1)).to(dev)
        self.slot_base = torch.from_numpy(self.slot_base_host).to(dev)

    def slots(self, rank: int) -> int:
        return int(self.slot_base_host[rank + 1] - self.slot_base_host[rank])

    def __call__(self, topk_ids: torch.Tensor, pair_rank: torch.Tensor, out: Optional[LayoutResult] = None,
                 stream: Optional[torch.cuda.Stream] = None) -> LayoutResult:
        pl = self.placement
        ids = topk_ids.reshape(-1)
        pr = pair_rank.reshape(-1)
        for name, t in (("topk_ids", ids), ("pair_rank", pr)):
            if t.dtype != torch.int32 or t.device != pl.device or not t.is_contiguous():
                raise ValidationError(f"{name} must be a contiguous int32 tensor on {pl.device}")
        if ids.numel() != pr.numel():
            raise ValidationError(f"topk_ids has {ids.numel()} pairs, pair_rank {pr.numel()}")
        P = ids.numel()
        if out is None:
            out = LayoutResult(
                pair_row=torch.empty(max(P, 1), dtype=torch.int32, device=pl.device),
                rep_off=torch.empty(self.nrep + 1, dtype=torch.int32, device=pl.device),
                status=torch.empty(4, dtype=torch.int32, device=pl.device),
                top_k=topk_ids.shape[-1] if topk_ids.dim() == 2 else 1,
            )
        else:  # the kernel writes through raw pointers: a caller's buffers must fit
            for name, t, n in (("pair_row", out.pair_row, P), ("rep_off", out.rep_off, self.nrep + 1),
                               ("status", out.status, 4)):
                if (not isinstance(t, torch.Tensor) or t.dtype != torch.int32 or t.device != pl.device
                        or not t.is_contiguous() or t.numel() < n):
                    raise ValidationError(f"out.{name} must be a contiguous int32 tensor of >= {n} elements "
                                          f"on {pl.device}")
        s = stream if stream is not None else torch.cuda.current_stream(pl.device)
        rc = _native.lib().metro_dispatch_layout_v1(
            ids.data_ptr() if P else None, pr.data_ptr() if P else None, P,
            self.rid_tab.data_ptr(), self.slot_base.data_ptr(), pl.num_experts, pl.num_ranks, self.nrep,
            out.pair_row.data_ptr(), out.rep_off.data_ptr(), out.status.data_ptr(), self.cluster_ctas,
            ctypes.c_void_p(s.cuda_stream))
        _native.check_rc(rc, "metro_dispatch_layout_v1")
        return out

    def alloc(self, num_pairs: int, top_k: int = 1) -> LayoutResult:
        dev = self.placement.device
        return LayoutResult(pair_row=torch.empty(max(num_pairs, 1), dtype=torch.int32, device=dev),
                            rep_off=torch.empty(self.nrep + 1, dtype=torch.int32, device=dev),
                            status=torch.empty(4, dtype=torch.int32, device=dev), top_k=top_k)

    def route_metro(self, topk_ids: torch.Tensor, out: Optional[RouteResult] = None,
                    layout_out: Optional[LayoutResult] = None, stream: Optional[torch.cuda.Stream] = None
                    ) -> Tuple[RouteResult, LayoutResult]:
        """METRO routing AND its dispatch layout in one launch
        (metro_route_layout_v1): the same outputs as ``Router(placement,
        "metro").route(ids)`` followed by ``self(ids, pair_rank)``.  The layout's
        status words are the routing's (``layout_out.status`` is ``out.status``)."""
        pl = self.placement
        router = Router(pl, "metro", self.cluster_ctas)
        ids = topk_ids.reshape(-1) if topk_ids.is_contiguous() else topk_ids.contiguous().reshape(-1)
        if ids.dtype != torch.int32 or ids.device != pl.device:
            raise ValidationError(f"topk_ids must be an int32 tensor on {pl.device}")
        P = ids.numel()
        top_k = topk_ids.shape[-1] if topk_ids.dim() == 2 else 1
        if out is None:
            out = router.alloc(max(P, 1), pair_rank=True, top_k=top_k)
        else:
            router._check_out(out, P)
            if out.pair_rank is None:
                raise ValidationError("out.pair_rank is required by the fused layout")
        if layout_out is None:
            layout_out = self.alloc(P, top_k)
        else:
            for name, t, n in (("pair_row", layout_out.pair_row, P), ("rep_off", layout_out.rep_off, self.nrep + 1)):
                if (not isinstance(t, torch.Tensor) or t.dtype != torch.int32 or t.device != pl.device
                        or not t.is_contiguous() or t.numel() < n):
                    raise ValidationError(f"layout_out.{name} must be a contiguous int32 tensor of >= {n} "
                                          f"elements on {pl.device}")
        layout_out.status = out.status
        s = stream if stream is not None else torch.cuda.current_stream(pl.device)
        rc = _native.lib().metro_route_layout_v1(
            ids.data_ptr() if P else None, P, pl.mask.data_ptr(), pl.num_experts, pl.num_ranks,
            self.rid_tab.data_ptr(), self.slot_base.data_ptr(), self.nrep, _ptr(out.loads),
            out.choice.data_ptr(), out.rank_counts.data_ptr(), out.lam.data_ptr(), out.pair_rank.data_ptr(),
            layout_out.pair_row.data_ptr(), layout_out.rep_off.data_ptr(), out.status.data_ptr(),
            self.cluster_ctas, ctypes.c_void_p(s.cuda_stream))
        _native.check_rc(rc, "metro_route_layout_v1")
        return out, layout_out

    def rank_groups(self, rep_off: np.ndarray, rank: int) -> List[Tuple[int, int, int]]:
        """(local slot, first row, rows) of every non-empty replica on ``rank``
        (host view of a layout, e.g. to build K3 work items)."""
        b0, b1 = int(self.slot_base_host[rank]), int(self.slot_base_host[rank + 1])
        base = int(rep_off[b0])
        out = []
        for s, r in enumerate(range(b0, b1)):
            n = int(rep_off[r + 1] - rep_off[r])
            if n:
                out.append((s, int(rep_off[r]) - base, n))
        return out

    def rank_rows(self, rep_off: np.ndarray, rank: int) -> int:
        return int(rep_off[self.slot_base_host[rank + 1]] - rep_off[self.slot_base_host[rank]])
