"""K3: the memory-bound grouped expert FFN that consumes a routing decision.

Used to measure what the routing buys: the weight bytes one EP rank streams
from HBM per MoE layer are proportional to its activated replicas (lambda).
The reference only models this (costmodel.py:83-94 memory_time); here the
bytes are moved by a tcgen05 grouped GEMM (csrc/moe_gemm.cu, include/moe_gemm.h).

Expert FFN (DeepSeek-V3 geometry by default, bf16):
    H = silu(X W_gate^T) * (X W_up^T)       W1 = [W_gate; W_up]  [2I, D]
    Y = H W_down^T                          W2                   [D, I]
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _native
from .core import ValidationError

BM = 128      # weight rows per tile
MAXN = 256    # tokens per work item (wide GEMM tiling; moe_item_tokens() for the items we build)


def _lib():
    L = _native.lib()
    if not hasattr(L, "_moe_bound"):
        import ctypes

        P, i32 = ctypes.c_void_p, ctypes.c_int32
        L.moe_grouped_gemm_v1.argtypes = [P, i32, i32, i32, P, i32, P, i32, P, i32, P]
        L.moe_grouped_gemm_v1.restype = ctypes.c_int
        L.moe_grouped_gemm_v2.argtypes = [P, i32, i32, i32, P, i32, P, i32, i32, P, i32, P]
        L.moe_grouped_gemm_v2.restype = ctypes.c_int
        L.moe_grouped_gemm_dev_v2.argtypes = [P, i32, i32, i32, P, i32, P, i32, P, i32, P, i32, P]
        L.moe_grouped_gemm_dev_v2.restype = ctypes.c_int
        L.moe_item_tokens.argtypes = []
        L.moe_item_tokens.restype = ctypes.c_int32
        L.moe_grouped_gemm_fp8_v1.argtypes = [P, P, i32, i32, i32, P, P, i32, P, i32, P, i32, P, i32, P]
        L.moe_grouped_gemm_fp8_v1.restype = ctypes.c_int
        L.moe_quantize_rows_fp8_v1.argtypes = [P, i32, i32, P, P, P, P]
        L.moe_quantize_rows_fp8_v1.restype = ctypes.c_int
        L.moe_silu_mul_fp8_v1.argtypes = [P, i32, i32, P, P, P, P]
        L.moe_silu_mul_fp8_v1.restype = ctypes.c_int
        L.moe_silu_mul_v1.argtypes = [P, i32, i32, P, P]
        L.moe_silu_mul_v1.restype = ctypes.c_int
        L.moe_grouped_gemm_dev_v1.argtypes = [P, i32, i32, i32, P, i32, P, i32, P, P, i32, P]
        L.moe_grouped_gemm_dev_v1.restype = ctypes.c_int
        L.moe_layout_items_v1.argtypes = [P, P, i32, i32, i32, P, i32, P, i32, P, P]
        L.moe_layout_items_v1.restype = ctypes.c_int
        L.moe_gather_rows_v1.argtypes = [P, i32, i32, P, P, ctypes.c_int64, i32, P, i32, P]
        L.moe_gather_rows_v1.restype = ctypes.c_int
        L.moe_silu_mul_dev_v1.argtypes = [P, i32, i32, P, P, P]
        L.moe_silu_mul_dev_v1.restype = ctypes.c_int
        L.moe_last_cuda_error.argtypes = []
        L.moe_last_cuda_error.restype = ctypes.c_int
        L._moe_bound = True
    return L


def _check(rc: int, what: str) -> None:
    if rc == _native.OK:
        return
    if rc == _native.ECUDA:
        raise _native.NativeLibraryError(f"{what}: CUDA error {_lib().moe_last_cuda_error()}")
    raise ValidationError(f"{what}: {_lib().metro_strerror(rc).decode()}")


def item_tokens() -> int:
    """Tokens per work item of the items this package builds (build_items and
    moe_layout_items_v1): the narrow, deeper-pipelined GEMM tiling."""
    return int(_lib().moe_item_tokens())


def build_items(groups: Sequence[Tuple[int, int, int]], M: int) -> np.ndarray:
    """Work items for groups of (expert slot e, first token row t0, token count n):
    every 128-row block of W[e] x every <= item_tokens() chunk of the group."""
    if M % BM:
        raise ValidationError(f"M={M} must be a multiple of {BM}")
    out = []
    for e, t0, n in groups:
        # token chunks of one weight block are adjacent, so the CTAs that run them
        # concurrently share the block's HBM read through L2
        ch = item_tokens()
        for mb in range(M // BM):
            for c0 in range(0, n, ch):
                out.append((e, mb, t0 + c0, min(ch, n - c0)))
    return np.asarray(out, dtype=np.int32).reshape(-1, 4)


def _items_and_bound(items, max_item_tokens):
    """(items as a tensor, token bound).  Host items: the bound is their largest
    token count, and an explicit bound below it is rejected (a bound <= item_tokens()
    selects the 64-token tiling).  Device items are not read back: without an
    explicit bound the wide tiling (any count <= 256) runs, and the kernel clamps
    every count to its tiling as a memory-safety guard (moe_gemm.cu load_item)."""
    if isinstance(items, torch.Tensor) and items.is_cuda:
        return items, (MAXN if max_item_tokens is None else int(max_item_tokens))
    a = np.asarray(items.cpu() if isinstance(items, torch.Tensor) else items).reshape(-1, 4)
    most = int(a[:, 3].max()) if len(a) else 1
    if max_item_tokens is None:
        max_item_tokens = most
    elif most > int(max_item_tokens):
        raise ValidationError(f"an item has {most} tokens, above max_item_tokens={int(max_item_tokens)}")
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)), int(max_item_tokens)


def _check_host_items(items: torch.Tensor, E: int, M: int, T: int) -> None:
    """Host items must address existing experts, row blocks and token rows (the
    kernel drops stores past T as a guard, but an item outside the problem is a
    caller error)."""
    if items.is_cuda or items.numel() == 0:
        return
    a = items.numpy()
    e, mb, t0, n = a[:, 0], a[:, 1], a[:, 2], a[:, 3]
    if (e < 0).any() or (e >= E).any() or (mb < 0).any() or (mb >= M // BM).any() or (t0 < 0).any() \
            or (n < 0).any() or (t0.astype(np.int64) + n > T).any():
        raise ValidationError("an item addresses an expert / row block / token range outside W and X")


def _check_out(Y: Optional[torch.Tensor], T: int, M: int, device) -> None:
    if Y is not None and (Y.dtype != torch.bfloat16 or Y.device != device or not Y.is_contiguous()
                          or Y.dim() != 2 or tuple(Y.shape) != (T, M)):
        raise ValidationError(f"Y must be a contiguous bfloat16 [{T}, {M}] tensor on {device}")


def grouped_gemm(W: torch.Tensor, X: torch.Tensor, items, Y: torch.Tensor = None,
                 num_ctas: int = 0, max_item_tokens: int = None) -> torch.Tensor:
    """Y[t, m] = sum_k W[e][m, k] X[t, k] for every item (bf16 in/out, fp32 accumulate).

    ``max_item_tokens`` bounds the items' token counts: <= item_tokens() selects
    the deeper-pipelined narrow tiling.  Taken from host items; device items
    without it use the wide tiling (any count <= 256)."""
    items, max_item_tokens = _items_and_bound(items, max_item_tokens)
    if W.dtype != torch.bfloat16 or X.dtype != torch.bfloat16:
        raise ValidationError("W and X must be bfloat16")
    if W.dim() != 3 or X.dim() != 2 or W.shape[2] != X.shape[1]:
        raise ValidationError(f"shape mismatch: W {tuple(W.shape)}, X {tuple(X.shape)}")
    if not (W.is_cuda and X.device == W.device and W.is_contiguous() and X.is_contiguous()):
        raise ValidationError("W and X must be contiguous CUDA tensors on one device")
    E, M, K = W.shape
    T = X.shape[0]
    _check_host_items(items, E, M, T)
    _check_out(Y, T, M, W.device)
    items = items.to(device=W.device, dtype=torch.int32).contiguous()
    if Y is None:
        Y = torch.empty((T, M), dtype=torch.bfloat16, device=W.device)
    rc = _lib().moe_grouped_gemm_v2(W.data_ptr(), E, M, K, X.data_ptr(), T, items.data_ptr(),
                                    items.shape[0], int(max_item_tokens), Y.data_ptr(), num_ctas,
                                    torch.cuda.current_stream(W.device).cuda_stream)
    _check(rc, "moe_grouped_gemm_v2")
    return Y


def silu_mul(GU: torch.Tensor, H: torch.Tensor = None) -> torch.Tensor:
    T, I2 = GU.shape
    I = I2 // 2
    if H is None:
        H = torch.empty((T, I), dtype=torch.bfloat16, device=GU.device)
    rc = _lib().moe_silu_mul_v1(GU.data_ptr(), T, I, H.data_ptr(),
                                torch.cuda.current_stream(GU.device).cuda_stream)
    _check(rc, "moe_silu_mul_v1")
    return H


@dataclass
class RankWorkload:
    """What one EP rank computes for one MoE layer under a routing decision."""

    groups: List[Tuple[int, int, int]]   # (local expert slot, t0, n tokens)
    tokens: int                          # rows of X on this rank
    activated: int                       # activated replicas (= len(groups))


def rank_workload_metro(choice: np.ndarray, loads: np.ndarray, A: np.ndarray, rank: int) -> RankWorkload:
    """METRO: every token of expert e goes to rank choice[e] (routing.py:49)."""
    slots = np.cumsum(A[:, rank]) - 1          # local slot index of each hosted expert
    groups, t = [], 0
    for e in np.flatnonzero((choice == rank) & (loads > 0)):
        n = int(loads[e])
        groups.append((int(slots[e]), t, n))
        t += n
    return RankWorkload(groups, t, len(groups))


def rank_workload_eplb(x: np.ndarray, A: np.ndarray, rank: int) -> RankWorkload:
    """EPLB: x[e][rank] tokens of expert e on this rank (routing.py:67-69)."""
    slots = np.cumsum(A[:, rank]) - 1
    groups, t = [], 0
    for e in np.flatnonzero(x[:, rank] > 0):
        n = int(x[e, rank])
        groups.append((int(slots[e]), t, n))
        t += n
    return RankWorkload(groups, t, len(groups))


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def quantize_weights_fp8(W: torch.Tensor):
    """bf16 W [E, M, K] -> (E4M3 bytes uint8 [E, M, K], f32 scale [E, M / 128]):
    one scale per (expert, 128-row block) = max |w| / 448 (weight loading, cold)."""
    E, M, K = W.shape
    if M % BM:
        raise ValidationError(f"M={M} must be a multiple of {BM}")
    blk = W.float().view(E, M // BM, BM, K)
    s = (blk.abs().amax(dim=(2, 3)) / 448.0).clamp_min(torch.finfo(torch.float32).tiny)
    q = (blk / s[:, :, None, None]).to(torch.float8_e4m3fn).view(torch.uint8).view(E, M, K)
    return q.contiguous(), s.contiguous()


def dequantize_fp8(q: torch.Tensor, scale: torch.Tensor, rows_per_scale: int) -> torch.Tensor:
    """E4M3 bytes + scales -> f32 (test reference)."""
    v = q.view(torch.float8_e4m3fn).float()
    return v * scale.repeat_interleave(rows_per_scale, dim=-1)[..., None]


def quantize_rows_fp8(X: torch.Tensor, X8: torch.Tensor = None, xs: torch.Tensor = None, rows_dev=None):
    """bf16 [T, K] -> (E4M3 uint8 [T, K], f32 [T]) with one scale per row (device)."""
    T, K = X.shape
    if X8 is None:
        X8 = torch.empty((T, K), dtype=torch.uint8, device=X.device)
    if xs is None:
        xs = torch.empty(T, dtype=torch.float32, device=X.device)
    _check(_lib().moe_quantize_rows_fp8_v1(X.data_ptr(), T, K, X8.data_ptr(), xs.data_ptr(),
                                            None if rows_dev is None else rows_dev.data_ptr(),
                                            _stream_ptr(X.device)), "moe_quantize_rows_fp8_v1")
    return X8, xs


def silu_mul_fp8(GU: torch.Tensor, H8: torch.Tensor = None, hs: torch.Tensor = None, rows_dev=None):
    """silu(gate) * up of GU [T, 2I] (bf16) -> (E4M3 uint8 [T, I], f32 [T])."""
    T, I2 = GU.shape
    I = I2 // 2
    if H8 is None:
        H8 = torch.empty((T, I), dtype=torch.uint8, device=GU.device)
    if hs is None:
        hs = torch.empty(T, dtype=torch.float32, device=GU.device)
    _check(_lib().moe_silu_mul_fp8_v1(GU.data_ptr(), T, I, H8.data_ptr(), hs.data_ptr(),
                                       None if rows_dev is None else rows_dev.data_ptr(),
                                       _stream_ptr(GU.device)), "moe_silu_mul_fp8_v1")
    return H8, hs


def grouped_gemm_fp8(W8: torch.Tensor, w_scale: torch.Tensor, X8: torch.Tensor, x_scale: torch.Tensor, items,
                     Y: torch.Tensor = None, num_ctas: int = 0, max_item_tokens: int = None,
                     n_items_dev: torch.Tensor = None) -> torch.Tensor:
    """Y[t, m] = w_scale[e, m / 128] * x_scale[t] * sum_k W8[e][m, k] X8[t, k] (E4M3 in, bf16 out)."""
    if W8.dtype != torch.uint8 or X8.dtype != torch.uint8:
        raise ValidationError("W8 and X8 must be E4M3 bytes (uint8)")
    if W8.dim() != 3 or X8.dim() != 2 or W8.shape[2] != X8.shape[1]:
        raise ValidationError(f"shape mismatch: W8 {tuple(W8.shape)}, X8 {tuple(X8.shape)}")
    if not (W8.is_cuda and X8.device == W8.device and W8.is_contiguous() and X8.is_contiguous()):
        raise ValidationError("W8 and X8 must be contiguous CUDA tensors on one device")
    E, M, K = W8.shape
    T = X8.shape[0]
    for name, t, n in (("w_scale", w_scale, E * (M // BM)), ("x_scale", x_scale, T)):
        if t.dtype != torch.float32 or t.device != W8.device or not t.is_contiguous() or t.numel() < n:
            raise ValidationError(f"{name} must be a contiguous float32 tensor of >= {n} elements on {W8.device}")
    items, max_item_tokens = _items_and_bound(items, max_item_tokens)
    _check_host_items(items, E, M, T)
    _check_out(Y, T, M, W8.device)
    items = items.to(device=W8.device, dtype=torch.int32).contiguous()
    if Y is None:
        Y = torch.empty((T, M), dtype=torch.bfloat16, device=W8.device)
    rc = _lib().moe_grouped_gemm_fp8_v1(W8.data_ptr(), w_scale.data_ptr(), E, M, K, X8.data_ptr(),
                                        x_scale.data_ptr(), T, items.data_ptr(), items.shape[0],
                                        None if n_items_dev is None else n_items_dev.data_ptr(),
                                        int(max_item_tokens), Y.data_ptr(), num_ctas, _stream_ptr(W8.device))
    _check(rc, "moe_grouped_gemm_fp8_v1")
    return Y


class ExpertFFN:
    """The experts hosted by one EP rank (random init: no checkpoints).

    ``dtype`` "bf16" or "fp8" (E4M3 weights with a scale per 128-row block, E4M3
    activations with a scale per token: DeepSeek-V3 ships FP8 experts)."""

    def __init__(self, slots: int, hidden: int, inter: int, device, seed: int = 0, dtype: str = "bf16"):
        if dtype not in ("bf16", "fp8"):
            raise ValidationError(f"unknown expert dtype {dtype!r}")
        g = torch.Generator(device=device).manual_seed(seed)
        self.slots, self.hidden, self.inter, self.dtype = slots, hidden, inter, dtype
        self.W1 = (torch.randn((slots, 2 * inter, hidden), generator=g, device=device) * hidden ** -0.5).to(torch.bfloat16)
        self.W2 = (torch.randn((slots, hidden, inter), generator=g, device=device) * inter ** -0.5).to(torch.bfloat16)
        if dtype == "fp8":
            self.W1q, self.W1s = quantize_weights_fp8(self.W1)
            self.W2q, self.W2s = quantize_weights_fp8(self.W2)
            del self.W1, self.W2  # the FP8 copies are the weights
            self.W1 = self.W2 = None

    def weight_bytes(self, activated: int) -> int:
        per = 2 * self.inter * self.hidden + self.hidden * self.inter
        return activated * per * (1 if self.dtype == "fp8" else 2)

    def plan(self, wl: RankWorkload, device):
        it1 = torch.from_numpy(build_items(wl.groups, 2 * self.inter)).to(device)
        it2 = torch.from_numpy(build_items(wl.groups, self.hidden)).to(device)
        return it1, it2

    def forward(self, X: torch.Tensor, items1: torch.Tensor, items2: torch.Tensor, bufs=None) -> torch.Tensor:
        T = X.shape[0]
        if self.dtype == "fp8":
            nt = item_tokens()
            if bufs is None:
                bufs = (torch.empty((T, 2 * self.inter), dtype=torch.bfloat16, device=X.device),
                        None, torch.empty((T, self.hidden), dtype=torch.bfloat16, device=X.device))
            GU, _, Y = bufs
            X8, xs = quantize_rows_fp8(X)
            grouped_gemm_fp8(self.W1q, self.W1s, X8, xs, items1, GU, max_item_tokens=nt)
            H8, hs = silu_mul_fp8(GU)
            grouped_gemm_fp8(self.W2q, self.W2s, H8, hs, items2, Y, max_item_tokens=nt)
            return Y
        if bufs is None:
            bufs = (torch.empty((T, 2 * self.inter), dtype=torch.bfloat16, device=X.device),
                    torch.empty((T, self.inter), dtype=torch.bfloat16, device=X.device),
                    torch.empty((T, self.hidden), dtype=torch.bfloat16, device=X.device))
        GU, H, Y = bufs
        nt = item_tokens()  # plan() builds items with build_items
        grouped_gemm(self.W1, X, items1, GU, max_item_tokens=nt)
        silu_mul(GU, H)
        grouped_gemm(self.W2, H, items2, Y, max_item_tokens=nt)
        return Y


class RankMoE:
    """One EP rank's MoE layer, entirely on device and graph-capturable:

        route (METRO / EPLB, pair ranks)      metro_route_v1 / eplb_route_v1
        -> dispatch layout                    metro_dispatch_layout_v1
           (METRO: both in ONE launch,        metro_route_layout_v1)
        -> the rank's K3 work items           moe_layout_items_v1
        -> receive buffer (token rows)        moe_gather_rows_v1
        -> expert FFN                         moe_grouped_gemm_dev_v1, silu, GEMM

    No host round trip: item and row counts stay on device.  Buffers are sized
    for the worst case (every pair of ``max_pairs`` on this rank).  The combine
    back to token order is the EP all-to-all's job and out of scope.
    """

    def __init__(self, placement, kind: str, rank: int, ffn: "ExpertFFN", max_pairs: int, top_k: int,
                 cluster_ctas: int = 0):
        from .device import Router
        from .dispatch import DispatchLayout

        dev = placement.device
        self.kind, self.rank, self.ffn, self.top_k = kind, int(rank), ffn, int(top_k)
        self.router = Router(placement, kind, cluster_ctas)
        self.layout = DispatchLayout(placement, cluster_ctas)
        slots = self.layout.slots(self.rank)
        if slots > ffn.slots:
            raise ValidationError(f"rank {rank} hosts {slots} experts but the FFN has {ffn.slots} slots")
        self.max_pairs = int(max_pairs)
        self.rows_cap = max(1, self.max_pairs)
        chunks = slots + self.rows_cap // item_tokens() + 1
        self.cap1 = chunks * (2 * ffn.inter // BM)
        self.cap2 = chunks * (ffn.hidden // BM)
        self.route_out = self.router.alloc(self.max_pairs, pair_rank=True, top_k=self.top_k)
        i32 = dict(dtype=torch.int32, device=dev)
        from .dispatch import LayoutResult

        self.layout_out = LayoutResult(pair_row=torch.empty(self.rows_cap, **i32),
                                       rep_off=torch.empty(self.layout.nrep + 1, **i32),
                                       status=torch.zeros(4, **i32), top_k=self.top_k)
        self.items1 = torch.empty((self.cap1, 4), **i32)
        self.items2 = torch.empty((self.cap2, 4), **i32)
        self.counts = torch.zeros(3, **i32)
        bf = dict(dtype=torch.bfloat16, device=dev)
        self.X = torch.zeros((self.rows_cap, ffn.hidden), **bf)
        self.GU = torch.empty((self.rows_cap, 2 * ffn.inter), **bf)
        self.H = torch.empty((self.rows_cap, ffn.inter), **bf)
        self.Y = torch.empty((self.rows_cap, ffn.hidden), **bf)
        if ffn.dtype == "fp8":  # E4M3 rows + per-row scales of the GEMM inputs
            u8 = dict(dtype=torch.uint8, device=dev)
            self.X8 = torch.empty((self.rows_cap, ffn.hidden), **u8)
            self.xs = torch.empty(self.rows_cap, dtype=torch.float32, device=dev)
            self.H8 = torch.empty((self.rows_cap, ffn.inter), **u8)
            self.hs = torch.empty(self.rows_cap, dtype=torch.float32, device=dev)

    def __call__(self, topk_ids: torch.Tensor, hidden: torch.Tensor, stream=None) -> torch.Tensor:
        """topk_ids int32 [B, k] (all-gathered), hidden bf16 [B, D] -> Y [rows_cap, D]
        (the first ``counts[2]`` rows are this rank's outputs, dispatch-layout order)."""
        import ctypes

        if topk_ids.numel() > self.max_pairs:
            raise ValidationError(f"{topk_ids.numel()} pairs > max_pairs {self.max_pairs}")
        if hidden.dtype != torch.bfloat16 or hidden.shape[-1] != self.ffn.hidden or not hidden.is_contiguous():
            raise ValidationError("hidden must be a contiguous bf16 [B, hidden] tensor")
        s = stream if stream is not None else torch.cuda.current_stream(self.X.device)
        sp = ctypes.c_void_p(s.cuda_stream)
        L = _lib()
        P = topk_ids.numel()
        ids = topk_ids.reshape(-1)
        if self.kind == "metro":  # routing + its dispatch layout in one launch
            rr, self.layout_out = self.layout.route_metro(topk_ids, out=self.route_out,
                                                          layout_out=self.layout_out, stream=s)
            pr = rr.pair_rank[:P]
        else:
            rr = self.router.route(topk_ids, out=self.route_out, stream=s)
            pr = rr.pair_rank[:P]
            self.layout_out = self.layout(ids, pr, out=self.layout_out, stream=s)
        lo = self.layout_out
        _check(L.moe_layout_items_v1(lo.rep_off.data_ptr(), self.layout.slot_base.data_ptr(), self.rank,
                                     2 * self.ffn.inter, self.ffn.hidden, self.items1.data_ptr(), self.cap1,
                                     self.items2.data_ptr(), self.cap2, self.counts.data_ptr(), sp),
               "moe_layout_items_v1")
        _check(L.moe_gather_rows_v1(hidden.data_ptr(), self.ffn.hidden * 2, self.top_k, pr.data_ptr(),
                                    lo.pair_row.data_ptr(), P, self.rank, self.X.data_ptr(), self.rows_cap, sp),
               "moe_gather_rows_v1")
        f = self.ffn
        nt = item_tokens()  # moe_layout_items_v1 chunks at this many tokens
        if f.dtype == "fp8":
            rows = self.counts[2:].data_ptr()
            _check(L.moe_quantize_rows_fp8_v1(self.X.data_ptr(), self.rows_cap, f.hidden, self.X8.data_ptr(),
                                              self.xs.data_ptr(), rows, sp), "moe_quantize_rows_fp8_v1")
            _check(L.moe_grouped_gemm_fp8_v1(f.W1q.data_ptr(), f.W1s.data_ptr(), f.slots, 2 * f.inter, f.hidden,
                                             self.X8.data_ptr(), self.xs.data_ptr(), self.rows_cap,
                                             self.items1.data_ptr(), self.cap1, self.counts.data_ptr(), nt,
                                             self.GU.data_ptr(), 0, sp), "moe_grouped_gemm_fp8_v1")
            _check(L.moe_silu_mul_fp8_v1(self.GU.data_ptr(), self.rows_cap, f.inter, self.H8.data_ptr(),
                                         self.hs.data_ptr(), rows, sp), "moe_silu_mul_fp8_v1")
            _check(L.moe_grouped_gemm_fp8_v1(f.W2q.data_ptr(), f.W2s.data_ptr(), f.slots, f.hidden, f.inter,
                                             self.H8.data_ptr(), self.hs.data_ptr(), self.rows_cap,
                                             self.items2.data_ptr(), self.cap2, self.counts[1:].data_ptr(), nt,
                                             self.Y.data_ptr(), 0, sp), "moe_grouped_gemm_fp8_v1")
            return self.Y
        _check(L.moe_grouped_gemm_dev_v2(f.W1.data_ptr(), f.slots, 2 * f.inter, f.hidden, self.X.data_ptr(),
                                         self.rows_cap, self.items1.data_ptr(), self.cap1,
                                         self.counts.data_ptr(), nt, self.GU.data_ptr(), 0, sp),
               "moe_grouped_gemm_dev_v2")
        _check(L.moe_silu_mul_dev_v1(self.GU.data_ptr(), self.rows_cap, f.inter, self.H.data_ptr(),
                                     self.counts[2:].data_ptr(), sp), "moe_silu_mul_dev_v1")
        _check(L.moe_grouped_gemm_dev_v2(f.W2.data_ptr(), f.slots, f.hidden, f.inter, self.H.data_ptr(),
                                         self.rows_cap, self.items2.data_ptr(), self.cap2,
                                         self.counts[1:].data_ptr(), nt, self.Y.data_ptr(), 0, sp),
               "moe_grouped_gemm_dev_v2")
        return self.Y
