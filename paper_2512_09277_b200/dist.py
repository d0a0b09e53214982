"""Multi-GPU METRO: one process per GPU, global top-k knowledge by all-gather.

The reference models this step only as a cost (costmodel.py:102-119, chosen for
the greedy routers at simulate.py:33, :69-70, :81); the paper replaces the
dispatch all-to-all with an all-gather so every EP rank can run the identical,
deterministic routing.  Here each rank holds the top-k ids of
its own decode tokens [B/P, k]; one NCCL all-gather over NVLink builds the
global [B, k] batch (rank-major) on every rank, then the sm_100a router runs on
it.  Routing outputs depend only on the per-expert histogram, so every rank
produces identical choice / rank_counts / lam without a broadcast; pair_rank of
this rank's own tokens is the slice [rank * B/P, (rank + 1) * B/P).
"""

from __future__ import annotations

import hashlib
from typing import Optional

import numpy as np
import torch
import torch.distributed as dist

from .device import DevicePlacement, RouteResult, Router


def allgather_topk(local_ids: torch.Tensor, out: Optional[torch.Tensor] = None, group=None) -> torch.Tensor:
    """[B/P, k] per rank -> [P * B/P, k] on every rank, rank-major (NCCL or gloo)."""
    world = dist.get_world_size(group)
    local = local_ids.contiguous()
    if out is None:
        out = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype,
                          device=local.device)
    if local.is_cuda:
        dist.all_gather_into_tensor(out, local, group=group)
    else:  # gloo: list form
        parts = list(out.chunk(world, dim=0))
        dist.all_gather(parts, local, group=group)
    return out


def local_slice(rank: int, local_tokens: int, top_k: int) -> slice:
    """Flat pair range of this rank's tokens inside the gathered batch."""
    return slice(rank * local_tokens * top_k, (rank + 1) * local_tokens * top_k)


def shard_tokens(global_ids: np.ndarray, world: int, rank: int) -> np.ndarray:
    """Contiguous token shard of a global batch (inverse of the rank-major gather)."""
    b = global_ids.shape[0]
    if b % world:
        raise ValueError(f"global batch {b} not divisible by world size {world}")
    per = b // world
    return global_ids[rank * per:(rank + 1) * per]


def routing_digest(choice: np.ndarray, counts: np.ndarray, lam: int) -> int:
    """64-bit digest of a routing decision (cross-rank agreement check)."""
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(choice, dtype=np.int32).tobytes())
    h.update(np.ascontiguousarray(counts, dtype=np.int32).tobytes())
    h.update(int(lam).to_bytes(8, "little", signed=True))
    return int.from_bytes(h.digest()[:8], "little", signed=True)


def assert_ranks_agree(choice: np.ndarray, counts: np.ndarray, lam: int, group=None,
                       device: Optional[torch.device] = None) -> int:
    """All ranks must hold the same routing; returns the digest."""
    d = routing_digest(choice, counts, lam)
    t = torch.tensor([d], dtype=torch.int64, device=device)
    world = dist.get_world_size(group)
    allv = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(allv, t, group=group)
    vals = {int(v.item()) for v in allv}
    if len(vals) != 1:
        raise RuntimeError(f"ranks disagree on the routing: {sorted(vals)}")
    return d


class DistributedRouter:
    """All-gather + route for one MoE layer, capturable as one CUDA graph.

    ``local_tokens`` decode tokens (top_k ids each) live on this rank; the
    global batch is world * local_tokens tokens.
    """

    def __init__(self, placement: DevicePlacement, local_tokens: int, top_k: int, kind: str = "metro",
                 cluster_ctas: int = 0, group=None, pair_rank: bool = True):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        dev = placement.device
        self.local_tokens, self.top_k = local_tokens, top_k
        self.local = torch.zeros((local_tokens, top_k), dtype=torch.int32, device=dev)
        self.gathered = torch.zeros((self.world * local_tokens, top_k), dtype=torch.int32, device=dev)
        self.router = Router(placement, kind, cluster_ctas)
        self.out: RouteResult = self.router.alloc(self.gathered.numel(), pair_rank=pair_rank, top_k=top_k)
        self.graph: Optional[torch.cuda.CUDAGraph] = None

    def step(self) -> RouteResult:
        """Eager: all-gather self.local, route the global batch (stream-ordered)."""
        if self.world > 1:
            allgather_topk(self.local, self.gathered, self.group)
        else:
            self.gathered.copy_(self.local)
        self.router.route(self.gathered, out=self.out)
        return self.out

    def capture(self, warmup: int = 3) -> torch.cuda.CUDAGraph:
        s = torch.cuda.Stream(self.local.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self.step()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.step()
        self.graph = g
        return g

    def replay(self) -> RouteResult:
        assert self.graph is not None, "capture() first"
        self.graph.replay()
        return self.out

    def own_pair_rank(self) -> torch.Tensor:
        """EP rank serving each (token, slot) of this rank's own tokens."""
        return self.out.pair_rank[local_slice(self.rank, self.local_tokens, self.top_k)]
