"""Device fast path: placement bitmasks resident in HBM, routing on CUDA tensors.

This is the serving-side interface (what a MoE layer calls once per decode
step): device-resident ``topk_ids`` in, device tensors out, stream-ordered, no
host synchronisation, CUDA-graph capturable.  The reference-compatible numpy
API in ``routing.py`` is a thin host wrapper over the same kernels.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _native
from .core import ValidationError


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream(device: torch.device, stream: Optional[torch.cuda.Stream] = None) -> int:
    if stream is not None:
        return stream.cuda_stream
    # the raw handle of the device's current stream without building a Stream object
    return torch._C._cuda_getCurrentRawStream(device.index)


def _require_cuda(t: torch.Tensor, name: str, dtype: torch.dtype) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValidationError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ValidationError(f"{name} must be {dtype}, got {t.dtype}")
    return t.contiguous()


def pack_placement(matrix) -> np.ndarray:
    """Binary A[N, G] -> rank bitmasks [N, W] uint32 (C-ABI metro_pack_placement)."""
    mat = np.ascontiguousarray(np.asarray(getattr(matrix, "matrix", matrix)))
    if mat.ndim != 2:
        raise ValidationError("placement matrix must be 2-dimensional")
    if mat.dtype != np.int8:
        if ((mat != 0) & (mat != 1)).any():
            raise ValidationError("placement matrix must be binary")
        mat = mat.astype(np.int8)
    n, g = mat.shape
    L = _native.lib()
    w = max(1, L.metro_mask_words(max(g, 1)))
    mask = np.zeros((n, w), dtype=np.uint32)
    rc = L.metro_pack_placement(mat.ctypes.data, n, g, mask.ctypes.data)
    if rc == _native.ENOTBINARY:
        raise ValidationError("placement matrix must be binary")
    _native.check_rc(rc, "metro_pack_placement")
    return mask


class DevicePlacement:
    """One layer's EPLB placement as per-expert rank bitmasks in HBM.

    Uploaded once per rebalance window (cold path, reference placement.py:83-128
    builds A); every routing launch reads N * W * 4 bytes of it.
    """

    def __init__(self, A, device=None):
        mat = np.asarray(getattr(A, "matrix", A))
        if mat.ndim != 2:
            raise ValidationError("placement matrix must be 2-dimensional")
        n, g = mat.shape
        if not (1 <= n <= _native.MAX_N and 1 <= g <= _native.MAX_G):
            raise ValidationError(
                f"placement {n}x{g} outside the sm_100a kernel limits "
                f"(1 <= N <= {_native.MAX_N}, 1 <= G <= {_native.MAX_G})"
            )
        d = torch.device(device) if device is not None else torch.device("cuda")
        if d.type == "cuda" and d.index is None:  # normalise "cuda" to "cuda:<current>"
            d = torch.device("cuda", torch.cuda.current_device())
        self.device = d
        mask = pack_placement(mat)
        self.num_experts, self.num_ranks, self.words = n, g, mask.shape[1]
        self.mask_host = mask
        self.mask = torch.from_numpy(mask.view(np.int32)).to(self.device)
        self.replica_counts = np.asarray(mat != 0).sum(axis=1)
        self.matrix = np.ascontiguousarray(mat, dtype=np.int8)


@dataclass(frozen=True)
class RouteResult:
    """Device outputs of one routing launch (all int32 CUDA tensors).

    loads[N]; choice[N] (METRO; -1 inactive) or x[N, G] (EPLB); rank_counts[G];
    lam[1]; pair_rank[num_pairs] (optional); status[4] (see metro_route.h).
    Frozen: Router.route() validates a reused result set once, so its tensors
    cannot be swapped afterwards (the kernels write through raw pointers).
    """

    kind: str
    loads: Optional[torch.Tensor]
    choice: Optional[torch.Tensor]
    x: Optional[torch.Tensor]
    rank_counts: torch.Tensor
    lam: torch.Tensor
    pair_rank: Optional[torch.Tensor]
    status: torch.Tensor
    top_k: int = 1

    def check(self) -> "RouteResult":
        """Synchronise on status and raise the reference's exception on error."""
        raise_status(self.status.cpu().numpy(), self.top_k)
        return self


def raise_status(status: np.ndarray, top_k: int = 1) -> None:
    code = int(status[0])
    if code == _native.OK:
        return
    if code == _native.ERR_ID_RANGE:
        pair = int(np.uint32(status[1])) | (int(np.uint32(status[2])) << 32)
        raise ValidationError(f"token {pair // max(top_k, 1)}: expert id {int(status[3])} out of range")
    if code == _native.ERR_NO_REPLICA:
        # reference: `assert gpus` / `assert best >= 0` (routing.py:66, :99)
        raise AssertionError("placement invariant: every expert has a replica")
    if code == _native.ERR_LOAD_RANGE:
        raise ValidationError("load does not fit the device loads path")
    if code == _native.ERR_PEER_TIMEOUT:
        raise _native.NativeLibraryError(f"peer rank {int(status[1])} did not join the exchange (timeout)")
    if code == _native.ERR_PAIR_RANK:
        pair = int(np.uint32(status[1])) | (int(np.uint32(status[2])) << 32)
        raise ValidationError(f"token {pair // max(top_k, 1)}: rank {int(status[3])} hosts no replica of its expert")
    raise _native.NativeLibraryError(f"unknown kernel status {code}")


class Router:
    """Routes device-resident top-k ids against one DevicePlacement.

    ``kind`` is ``"metro"`` (routing.py:105-113) or ``"eplb"`` (routing.py:55-72).
    ``cluster_ctas`` = CTAs in the thread-block cluster (0 = auto by batch size).
    """

    KINDS = ("metro", "eplb")

    def __init__(self, placement: DevicePlacement, kind: str = "metro", cluster_ctas: int = 0):
        if kind not in self.KINDS:
            raise ValidationError(f"unknown device router kind {kind!r}; expected one of {self.KINDS}")
        self.placement = placement
        self.kind = kind
        self.cluster_ctas = int(cluster_ctas)
        self._checked = None
        self._checked_ref = None  # keeps the checked result alive so its id() stays unique

    def bind(self, topk_ids: torch.Tensor, out: Optional[RouteResult] = None, pair_rank: bool = True,
             with_x: bool = False, stream: Optional[torch.cuda.Stream] = None) -> "RoutePlan":
        """A launch plan for fixed buffers (metro_route_plan_create_v1): validation,
        cluster plan and kernel choice happen here once; ``plan()`` then launches
        one layer with a single two-argument C call -- the eager serving loop
        that refills ``topk_ids`` in place each step.  Same outputs as route()."""
        ids = _require_cuda(topk_ids, "topk_ids", torch.int32)
        if ids.data_ptr() != topk_ids.data_ptr():
            raise ValidationError("bind() needs a contiguous topk_ids buffer (it is read in place each launch)")
        if ids.device != self.placement.device:
            raise ValidationError(f"topk_ids on {ids.device}, placement on {self.placement.device}")
        top_k = ids.shape[-1] if ids.dim() >= 2 else 1
        num_pairs = ids.numel()
        if out is None:
            out = self.alloc(num_pairs, pair_rank=pair_rank, with_x=with_x, top_k=top_k)
        else:
            self._check_out(out, num_pairs)
        return RoutePlan(self, ids, out, _stream(self.placement.device, stream))

    def alloc(self, num_pairs: int, pair_rank: bool = True, with_x: bool = False, top_k: int = 1) -> RouteResult:
        dev = self.placement.device
        n, g = self.placement.num_experts, self.placement.num_ranks
        i32 = dict(dtype=torch.int32, device=dev)
        return RouteResult(
            kind=self.kind,
            loads=torch.empty(n, **i32),
            choice=torch.empty(n, **i32) if self.kind == "metro" else None,
            x=torch.empty((n, g), **i32) if (self.kind == "eplb" and with_x) else None,
            rank_counts=torch.empty(g, **i32),
            lam=torch.empty(1, **i32),
            pair_rank=torch.empty(num_pairs, **i32) if pair_rank else None,
            status=torch.zeros(4, **i32),
            top_k=top_k,
        )

    def _check_out(self, out: RouteResult, num_pairs: int) -> None:
        """A caller-supplied result set must hold this launch's outputs (the kernel
        writes through raw pointers): int32 on the placement's device, sized for
        N experts, G ranks and ``num_pairs`` pair ranks."""
        p = self.placement
        need = [("loads", out.loads, p.num_experts), ("rank_counts", out.rank_counts, p.num_ranks),
                ("lam", out.lam, 1), ("status", out.status, 4), ("pair_rank", out.pair_rank, num_pairs)]
        if self.kind == "metro":
            need.append(("choice", out.choice, p.num_experts))
        else:
            need.append(("x", out.x, p.num_experts * p.num_ranks))
        for name, t, n in need:
            if t is None:
                if name in ("loads", "pair_rank", "x"):
                    continue  # optional outputs
                raise ValidationError(f"out.{name} is missing")
            if t.dtype != torch.int32 or t.device != p.device or not t.is_contiguous() or t.numel() < n:
                raise ValidationError(f"out.{name} must be a contiguous int32 tensor of >= {n} elements on {p.device}")

    def route(self, topk_ids: torch.Tensor, out: Optional[RouteResult] = None, pair_rank: bool = True,
              with_x: bool = False, stream: Optional[torch.cuda.Stream] = None) -> RouteResult:
        """Launch one routing kernel on ``stream`` (default: current stream)."""
        ids = _require_cuda(topk_ids, "topk_ids", torch.int32)
        if ids.device != self.placement.device:
            raise ValidationError(f"topk_ids on {ids.device}, placement on {self.placement.device}")
        top_k = ids.shape[-1] if ids.dim() >= 2 else 1
        num_pairs = ids.numel()
        if out is None:
            out = self.alloc(num_pairs, pair_rank=pair_rank, with_x=with_x, top_k=top_k)
        elif self._checked != (id(out), num_pairs):
            # a result set is checked once per batch size; RouteResult's tensors are
            # fixed at construction (replacing one means a new RouteResult)
            self._check_out(out, num_pairs)
            self._checked = (id(out), num_pairs)
            self._checked_ref = out
        L = _native.lib()
        p = self.placement
        s = _stream(p.device, stream)
        if self.kind == "metro":
            rc = L.metro_route_v1(
                ids.data_ptr(), num_pairs, p.mask.data_ptr(), p.num_experts, p.num_ranks,
                _ptr(out.loads), out.choice.data_ptr(), out.rank_counts.data_ptr(), out.lam.data_ptr(),
                _ptr(out.pair_rank), out.status.data_ptr(), self.cluster_ctas, s,
            )
        else:
            rc = L.eplb_route_v1(
                ids.data_ptr(), num_pairs, p.mask.data_ptr(), p.num_experts, p.num_ranks,
                _ptr(out.loads), _ptr(out.x), out.rank_counts.data_ptr(), out.lam.data_ptr(),
                _ptr(out.pair_rank), out.status.data_ptr(), self.cluster_ctas, s,
            )
        _native.check_rc(rc, f"{self.kind}_route_v1")
        return out


    def route_scores(self, scores: torch.Tensor, top_k: int, out: Optional[RouteResult] = None,
                     topk_ids: Optional[torch.Tensor] = None, pair_rank: bool = True,
                     stream: Optional[torch.cuda.Stream] = None, whole_gpu: Optional[bool] = None):
        """Gating top-k fused with METRO (metro_route_scores_v1): ``scores`` fp32
        [B, N] router scores of the all-gathered tokens -> (topk_ids int32 [B, k],
        RouteResult).  Each token's ids are its k largest scores, largest first,
        ties to the lower expert id (the reference generator's order,
        core.py:319-326).

        ``whole_gpu=True``: every SM takes top-k for 32 tokens, then dependent
        routing CTAs route from the summed counts (a zeroed workspace owned by
        this Router; use one Router per stream).  ``False``: the routing cluster also takes the top-k.  ``None``
        (default): the library picks by batch size."""
        if self.kind != "metro":
            raise ValidationError("route_scores is the METRO router's fused gating entry point")
        p = self.placement
        if scores.dtype != torch.float32 or scores.dim() != 2 or not scores.is_cuda or not scores.is_contiguous():
            raise ValidationError("scores must be a contiguous float32 CUDA tensor [tokens, experts]")
        if scores.device != p.device:
            raise ValidationError(f"scores on {scores.device}, placement on {p.device}")
        B, n = scores.shape
        if n != p.num_experts:
            raise ValidationError(f"dimension mismatch: scores have {n} experts, A has {p.num_experts}")
        k = int(top_k)
        if topk_ids is None:
            topk_ids = torch.empty((B, k), dtype=torch.int32, device=p.device)
        elif (topk_ids.dtype != torch.int32 or not topk_ids.is_cuda or topk_ids.device != p.device
              or not topk_ids.is_contiguous() or topk_ids.numel() != B * k):
            raise ValidationError(f"topk_ids must be a contiguous int32 tensor of {B}x{k} on {p.device}")
        if out is None:
            out = self.alloc(B * k, pair_rank=pair_rank, top_k=k)
        else:
            self._check_out(out, B * k)
        s = _stream(p.device, stream)
        ws = None
        cl = self.cluster_ctas
        if whole_gpu is True:
            cl = -1
        elif whole_gpu is None and cl != 0:
            pass  # an explicit cluster size on the Router selects the cluster variant
        if whole_gpu is not False:
            if getattr(self, "_gate_ws", None) is None:
                nb = _native.lib().metro_scores_workspace_bytes(p.num_experts)
                self._gate_ws = torch.zeros(nb, dtype=torch.uint8, device=p.device)
            ws = self._gate_ws.data_ptr()
        rc = _native.lib().metro_route_scores_v1(
            scores.data_ptr(), B, k, p.mask.data_ptr(), p.num_experts, p.num_ranks, topk_ids.data_ptr(),
            _ptr(out.loads), out.choice.data_ptr(), out.rank_counts.data_ptr(), out.lam.data_ptr(),
            _ptr(out.pair_rank), out.status.data_ptr(), ws, cl, s)
        _native.check_rc(rc, "metro_route_scores_v1")
        return topk_ids, out


class RoutePlan:
    """One routing launch planned for fixed buffers (Router.bind).  Calling it
    launches the kernel on the bound stream and returns ``out``; refill
    ``topk_ids`` in place between calls.  Holds its buffers alive; ``close()``
    frees the C plan (also on garbage collection)."""

    def __init__(self, router: Router, ids: torch.Tensor, out: RouteResult, stream: int):
        p = router.placement
        L = _native.lib()
        h = ctypes.c_void_p()
        kind = _native.PLAN_METRO if router.kind == "metro" else _native.PLAN_EPLB
        rc = L.metro_route_plan_create_v1(
            kind, ids.data_ptr(), ids.numel(), p.mask.data_ptr(), p.num_experts, p.num_ranks, _ptr(out.loads),
            _ptr(out.choice), _ptr(out.x), out.rank_counts.data_ptr(), out.lam.data_ptr(), _ptr(out.pair_rank),
            out.status.data_ptr(), router.cluster_ctas, ctypes.byref(h))
        _native.check_rc(rc, "metro_route_plan_create_v1")
        self.topk_ids, self.out, self.placement = ids, out, p
        self._h = h
        self._launch = L.metro_route_plan_launch_v1
        self._args = (h, ctypes.c_void_p(stream))
        self._destroy = L.metro_route_plan_destroy_v1

    def __call__(self) -> RouteResult:
        rc = self._launch(*self._args)
        if rc:
            _native.check_rc(rc, "metro_route_plan_launch_v1")
        return self.out

    def close(self) -> None:
        if self._h is not None:
            self._destroy(self._h)
            self._h = None
            self._args = (ctypes.c_void_p(0), self._args[1])  # a later call reports METRO_EARG

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def aggregate_loads_device(topk_ids: torch.Tensor, num_experts: int, cluster_ctas: int = 0,
                           stream: Optional[torch.cuda.Stream] = None):
    """T[N] int32 on device + status[4] (metro_aggregate_loads_v1)."""
    ids = _require_cuda(topk_ids, "topk_ids", torch.int32)
    loads = torch.empty(num_experts, dtype=torch.int32, device=ids.device)
    status = torch.zeros(4, dtype=torch.int32, device=ids.device)
    rc = _native.lib().metro_aggregate_loads_v1(
        ids.data_ptr(), ids.numel(), num_experts, loads.data_ptr(), status.data_ptr(), cluster_ctas,
        _stream(ids.device, stream),
    )
    _native.check_rc(rc, "metro_aggregate_loads_v1")
    return loads, status


class HostRouter:
    """End-to-end METRO from host (pinned) buffers through metro_route_host_v1.

    Each call moves the ids host -> device, routes, moves choice / rank_counts /
    lam / status (+ pair_rank) device -> host and synchronises -- the
    reference-facing call a CPU-resident caller makes.  ``zero_copy=True`` lets
    the kernel read/write the pinned host buffers directly over PCIe (no copy
    engine round trips); ``False`` uses explicit cudaMemcpyAsync H2D / D2H.

    The router owns its pinned buffers: write the batch into ``ids`` (int32,
    row-major [B, k] flattened) and call ``run(num_pairs)``; results land in
    ``out`` ([status 4 | lam | pad 3 | rank_counts G | choice N]) and
    ``pair_rank``.  ``__call__(ids_host, pair_rank_host)`` is the convenience form
    for caller-owned pinned tensors.
    """

    def __init__(self, placement: DevicePlacement, max_pairs: int, cluster_ctas: int = 0,
                 zero_copy: bool = True):
        self.placement = placement
        self.cluster_ctas = int(cluster_ctas)
        L = _native.lib()
        n, g = placement.num_experts, placement.num_ranks
        self.max_pairs = max_pairs
        self.ws = torch.empty(L.metro_host_workspace_bytes(max_pairs, n, g), dtype=torch.uint8,
                              device=placement.device)
        self.ids = torch.zeros(max_pairs, dtype=torch.int32).pin_memory()
        self.out = torch.zeros(8 + g + n, dtype=torch.int32).pin_memory()
        self.pair_rank = torch.zeros(max_pairs, dtype=torch.int32).pin_memory()
        self.stream = torch.cuda.Stream(placement.device)
        self.flags = (_native.HOST_ZEROCOPY if zero_copy else 0)
        self._fn = L.metro_route_host_v1
        self._npairs = ctypes.c_int64(max_pairs)
        self._args = (
            ctypes.c_void_p(self.ids.data_ptr()), self._npairs, ctypes.c_void_p(placement.mask.data_ptr()),
            ctypes.c_int32(n), ctypes.c_int32(g), ctypes.c_void_p(self.ws.data_ptr()),
            ctypes.c_void_p(self.out.data_ptr()), ctypes.c_void_p(self.pair_rank.data_ptr()),
            ctypes.c_int32(self.cluster_ctas), ctypes.c_int32(self.flags | _native.HOST_STABLE_BUFFERS),
            ctypes.c_void_p(self.stream.cuda_stream),
        )
        self._out_np = self.out.numpy()

    def run(self, num_pairs: int) -> np.ndarray:
        """Route ids[:num_pairs] (already written into self.ids); synchronous."""
        if not 0 <= num_pairs <= self.max_pairs:
            raise ValidationError("batch larger than the HostRouter workspace")
        self._npairs.value = num_pairs
        rc = self._fn(*self._args)
        if rc:
            _native.check_rc(rc, "metro_route_host_v1")
        return self._out_np

    def __call__(self, ids_host: torch.Tensor, pair_rank_host: Optional[torch.Tensor] = None) -> np.ndarray:
        if ids_host.is_cuda or ids_host.dtype != torch.int32 or not ids_host.is_contiguous():
            raise ValidationError("ids_host must be a contiguous int32 CPU tensor (pinned for speed)")
        if ids_host.numel() > self.max_pairs:
            raise ValidationError("batch larger than the HostRouter workspace")
        p = self.placement
        rc = _native.lib().metro_route_host_v1(
            ids_host.data_ptr(), ids_host.numel(), p.mask.data_ptr(), p.num_experts, p.num_ranks,
            self.ws.data_ptr(), self.out.data_ptr(),
            None if pair_rank_host is None else pair_rank_host.data_ptr(), self.cluster_ctas,
            self.flags, self.stream.cuda_stream,
        )
        _native.check_rc(rc, "metro_route_host_v1")
        return self._out_np


class ServedRouter:
    """End-to-end METRO for host callers through a persistent router
    (include/metro_serve.h): one resident CTA waits on a doorbell in pinned host
    memory, so a call costs two PCIe round trips plus the routing itself instead
    of a kernel launch + stream synchronise (``HostRouter``).

    Same buffers and result layout as ``HostRouter``: write the batch into
    ``ids`` and call ``run(num_pairs)``; results land in ``out`` ([status 4 |
    lam | pad 3 | rank_counts G | choice N]) and ``pair_rank``.  The resident
    CTA occupies one SM and exits by itself after ``idle_timeout_us`` without a
    request (the next call relaunches it), so a device-wide synchronise
    elsewhere waits at most that long.  ``close()`` (or the context manager)
    stops it.  One ServedRouter per placement; not thread-safe (one caller at a
    time).
    """

    def __init__(self, placement: DevicePlacement, max_pairs: int, idle_timeout_us: int = 200_000):
        self.placement = placement
        self.max_pairs = int(max_pairs)
        L = _native.lib()
        n, g = placement.num_experts, placement.num_ranks
        self.ids = torch.zeros(max(self.max_pairs, 4), dtype=torch.int32).pin_memory()
        self.out = torch.zeros(8 + g + n, dtype=torch.int32).pin_memory()
        self.pair_rank = torch.zeros(max(self.max_pairs, 4), dtype=torch.int32).pin_memory()
        self._out_np = self.out.numpy()
        h = ctypes.c_void_p()
        with torch.cuda.device(placement.device):
            rc = L.metro_server_create_v1(placement.mask.data_ptr(), n, g, self.max_pairs, int(idle_timeout_us),
                                          ctypes.byref(h))
        _native.check_rc(rc, "metro_server_create_v1")
        self._h = h
        self._fn = L.metro_server_route_v1
        self._args = [h, ctypes.c_void_p(self.ids.data_ptr()), ctypes.c_int64(0),
                      ctypes.c_void_p(self.out.data_ptr()), ctypes.c_void_p(self.pair_rank.data_ptr())]

    def run(self, num_pairs: int) -> np.ndarray:
        """Route ids[:num_pairs] (already written into self.ids); synchronous."""
        if self._h is None:
            raise ValidationError("ServedRouter is closed")
        if not 0 <= num_pairs <= self.max_pairs:
            raise ValidationError("batch larger than the ServedRouter capacity")
        self._args[2].value = num_pairs
        rc = self._fn(*self._args)
        if rc:
            _native.check_rc(rc, "metro_server_route_v1")
        return self._out_np

    def route(self, topk_ids) -> np.ndarray:
        """Copy a host batch (numpy / CPU tensor, [B, k] int) into the pinned
        buffer and route it; returns ``out`` (raises on a data error, like the
        reference's ValidationError / AssertionError)."""
        a = np.ascontiguousarray(np.asarray(topk_ids, dtype=np.int32)).reshape(-1)
        if a.size > self.max_pairs:
            raise ValidationError("batch larger than the ServedRouter capacity")
        self.ids.numpy()[: a.size] = a
        out = self.run(a.size)
        raise_status(out[:4], topk_ids.shape[-1] if getattr(topk_ids, "ndim", 1) >= 2 else 1)
        return out

    @property
    def launches(self) -> int:
        """Launches of the resident CTA (1 + relaunches after idle exits)."""
        return int(_native.lib().metro_server_launches(self._h)) if self._h is not None else 0

    def close(self) -> None:
        if self._h is not None:
            rc = _native.lib().metro_server_destroy_v1(self._h)
            self._h = None
            _native.check_rc(rc, "metro_server_destroy_v1")

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
