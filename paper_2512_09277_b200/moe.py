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
from typing import List, Sequence, Tuple

import numpy as np
import torch

from . import _native
from .core import ValidationError

BM = 128      # weight rows per tile
MAXN = 256    # tokens per work item


def _lib():
    L = _native.lib()
    if not hasattr(L, "_moe_bound"):
        import ctypes

        P, i32 = ctypes.c_void_p, ctypes.c_int32
        L.moe_grouped_gemm_v1.argtypes = [P, i32, i32, i32, P, i32, P, i32, P, i32, P]
        L.moe_grouped_gemm_v1.restype = ctypes.c_int
        L.moe_silu_mul_v1.argtypes = [P, i32, i32, P, P]
        L.moe_silu_mul_v1.restype = ctypes.c_int
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


def build_items(groups: Sequence[Tuple[int, int, int]], M: int) -> np.ndarray:
    """Work items for groups of (expert slot e, first token row t0, token count n):
    every 128-row block of W[e] x every <=256-token chunk of the group."""
    if M % BM:
        raise ValidationError(f"M={M} must be a multiple of {BM}")
    out = []
    for e, t0, n in groups:
        # token chunks of one weight block are adjacent, so the CTAs that run them
        # concurrently share the block's HBM read through L2
        for mb in range(M // BM):
            for c0 in range(0, n, MAXN):
                out.append((e, mb, t0 + c0, min(MAXN, n - c0)))
    return np.asarray(out, dtype=np.int32).reshape(-1, 4)


def grouped_gemm(W: torch.Tensor, X: torch.Tensor, items: torch.Tensor, Y: torch.Tensor = None,
                 num_ctas: int = 0) -> torch.Tensor:
    """Y[t, m] = sum_k W[e][m, k] X[t, k] for every item (bf16 in/out, fp32 accumulate)."""
    if W.dtype != torch.bfloat16 or X.dtype != torch.bfloat16:
        raise ValidationError("W and X must be bfloat16")
    if W.dim() != 3 or X.dim() != 2 or W.shape[2] != X.shape[1]:
        raise ValidationError(f"shape mismatch: W {tuple(W.shape)}, X {tuple(X.shape)}")
    E, M, K = W.shape
    T = X.shape[0]
    items = items.to(device=W.device, dtype=torch.int32).contiguous()
    if Y is None:
        Y = torch.empty((T, M), dtype=torch.bfloat16, device=W.device)
    rc = _lib().moe_grouped_gemm_v1(W.data_ptr(), E, M, K, X.data_ptr(), T, items.data_ptr(),
                                    items.shape[0], Y.data_ptr(), num_ctas,
                                    torch.cuda.current_stream(W.device).cuda_stream)
    _check(rc, "moe_grouped_gemm_v1")
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


class ExpertFFN:
    """The experts hosted by one EP rank (bf16, random init: no checkpoints)."""

    def __init__(self, slots: int, hidden: int, inter: int, device, seed: int = 0):
        g = torch.Generator(device=device).manual_seed(seed)
        self.slots, self.hidden, self.inter = slots, hidden, inter
        self.W1 = (torch.randn((slots, 2 * inter, hidden), generator=g, device=device) * hidden ** -0.5).to(torch.bfloat16)
        self.W2 = (torch.randn((slots, hidden, inter), generator=g, device=device) * inter ** -0.5).to(torch.bfloat16)

    def weight_bytes(self, activated: int) -> int:
        return activated * (self.W1[0].numel() + self.W2[0].numel()) * 2

    def plan(self, wl: RankWorkload, device):
        it1 = torch.from_numpy(build_items(wl.groups, 2 * self.inter)).to(device)
        it2 = torch.from_numpy(build_items(wl.groups, self.hidden)).to(device)
        return it1, it2

    def forward(self, X: torch.Tensor, items1: torch.Tensor, items2: torch.Tensor, bufs=None) -> torch.Tensor:
        T = X.shape[0]
        if bufs is None:
            bufs = (torch.empty((T, 2 * self.inter), dtype=torch.bfloat16, device=X.device),
                    torch.empty((T, self.inter), dtype=torch.bfloat16, device=X.device),
                    torch.empty((T, self.hidden), dtype=torch.bfloat16, device=X.device))
        GU, H, Y = bufs
        grouped_gemm(self.W1, X, items1, GU)
        silu_mul(GU, H)
        grouped_gemm(self.W2, H, items2, Y)
        return Y
