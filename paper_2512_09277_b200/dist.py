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
    if local.is_cuda and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, local, group=group)
    elif not local.is_cuda:  # gloo: list form
        parts = list(out.chunk(world, dim=0))
        dist.all_gather(parts, local, group=group)
    else:  # CUDA tensors over gloo (ranks sharing a GPU): staged through host memory
        parts = [torch.empty_like(local, device="cpu") for _ in range(world)]
        dist.all_gather(parts, local.cpu(), group=group)
        out.copy_(torch.cat(parts, dim=0))
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


class ExchangeRoute:
    """One EP rank's fused all-gather + METRO launch (include/metro_exchange.h).

    The rank's exchange buffer and the device-visible addresses of every rank's
    buffer are given (``peer_ptrs[rank]`` is the own one).  Use
    ``FusedAllGatherRouter`` (one process per GPU, CUDA IPC over the process
    group) or ``virtual_ranks`` (all ranks in one process on one device, for
    tests and single-GPU measurement) to build them.
    """

    def __init__(self, placement: DevicePlacement, rank: int, world: int, local_tokens: int, top_k: int,
                 peer_ptrs, max_local_pairs: int, gather_ids: bool = False, layout=None):
        import ctypes

        from . import _native

        if not 1 <= world <= 32 or not 0 <= rank < world:
            raise ValueError(f"rank {rank} / world {world} outside 1..32")
        self.placement, self.rank, self.world = placement, rank, world
        self.local_tokens, self.top_k = local_tokens, top_k
        self.local_pairs = local_tokens * top_k
        self.max_local_pairs = max_local_pairs
        dev = placement.device
        i32 = dict(dtype=torch.int32, device=dev)
        n, g = placement.num_experts, placement.num_ranks
        self.local = torch.zeros((local_tokens, top_k), **i32)
        self.out = RouteResult(kind="metro", loads=torch.empty(n, **i32), choice=torch.empty(n, **i32), x=None,
                               rank_counts=torch.empty(g, **i32), lam=torch.empty(1, **i32),
                               pair_rank=torch.empty(self.local_pairs, **i32), status=torch.zeros(4, **i32),
                               top_k=top_k)
        self.gathered = torch.zeros((world * local_tokens, top_k), **i32) if gather_ids else None
        self._peers = (ctypes.c_void_p * world)(*[int(p) for p in peer_ptrs])
        self._fn = _native.lib().metro_allgather_route_v1
        # optional dispatch layout of the global batch (metro_allgather_route_layout_v1):
        # this rank's pairs' rows in their serving ranks' receive buffers + rep_off
        self.layout = layout
        self.layout_out = None
        if layout is not None:
            if gather_ids:
                raise ValueError("the fused layout exchanges histograms only (gather_ids=False)")
            self.layout_out = layout.alloc(self.local_pairs, top_k)
            self.layout_out.status = self.out.status
            self._fn_layout = _native.lib().metro_allgather_route_layout_v1

    def step(self, local_ids: Optional[torch.Tensor] = None,
             stream: Optional[torch.cuda.Stream] = None) -> RouteResult:
        """One layer: exchange + route (stream-ordered, graph-capturable).  Every
        rank must call it the same number of times, in the same order."""
        from . import _native

        ids = self.local if local_ids is None else local_ids
        p = self.placement
        if ids.numel() != self.local_pairs or ids.dtype != torch.int32 or not ids.is_cuda or ids.device != p.device:
            raise ValueError(f"local_ids must be int32 [local_tokens, top_k] on {p.device}")
        ids = ids.contiguous()
        s = (stream if stream is not None else torch.cuda.current_stream(p.device)).cuda_stream
        o = self.out
        if self.layout is not None:
            lo, lay = self.layout_out, self.layout
            rc = self._fn_layout(ids.data_ptr(), self.local_pairs, self.rank, self.world, self._peers,
                                 self.max_local_pairs, p.mask.data_ptr(), p.num_experts, p.num_ranks,
                                 lay.rid_tab.data_ptr(), lay.slot_base.data_ptr(), lay.nrep, o.loads.data_ptr(),
                                 o.choice.data_ptr(), o.rank_counts.data_ptr(), o.lam.data_ptr(),
                                 o.pair_rank.data_ptr(), lo.pair_row.data_ptr(), lo.rep_off.data_ptr(),
                                 o.status.data_ptr(), s)
            _native.check_rc(rc, "metro_allgather_route_layout_v1")
            return o
        rc = self._fn(ids.data_ptr(), self.local_pairs, self.rank, self.world, self._peers, self.max_local_pairs,
                      p.mask.data_ptr(), p.num_experts, p.num_ranks, o.loads.data_ptr(), o.choice.data_ptr(),
                      o.rank_counts.data_ptr(), o.lam.data_ptr(), o.pair_rank.data_ptr(),
                      None if self.gathered is None else self.gathered.data_ptr(), o.status.data_ptr(), s)
        _native.check_rc(rc, "metro_allgather_route_v1")
        return o


class _ExchangeBuffer:
    """A zeroed exchange buffer from metro_exchange_alloc (freed on close)."""

    def __init__(self, nbytes: int, device: torch.device):
        import ctypes

        from . import _native

        self.ptr = ctypes.c_void_p()
        with torch.cuda.device(device):
            _native.check_rc(_native.lib().metro_exchange_alloc(nbytes, ctypes.byref(self.ptr)),
                             "metro_exchange_alloc")
        self.device = device

    def close(self):
        from . import _native

        if self.ptr:
            with torch.cuda.device(self.device):
                _native.lib().metro_exchange_free(self.ptr)
            self.ptr = None


def exchange_bytes(placement: DevicePlacement, world: int, max_local_pairs: int) -> int:
    from . import _native

    return int(_native.lib().metro_exchange_bytes(placement.num_experts, world, max_local_pairs))


def virtual_ranks(placement: DevicePlacement, world: int, local_tokens: int, top_k: int,
                  gather_ids: bool = False, layout=None):
    """``world`` EP ranks in ONE process on ONE device, each with its own exchange
    buffer, addressing the others' buffers directly: the same kernel and protocol
    as across GPUs (peer addresses are plain device addresses here).  Launch the
    ranks' steps on distinct streams -- they wait for each other.  Returns
    (routers, buffers); close the buffers when done."""
    max_local = -(-local_tokens * top_k // 4) * 4
    nbytes = exchange_bytes(placement, world, max_local)
    bufs = [_ExchangeBuffer(nbytes, placement.device) for _ in range(world)]
    ptrs = [b.ptr.value for b in bufs]
    routers = [ExchangeRoute(placement, r, world, local_tokens, top_k, ptrs, max_local, gather_ids, layout)
               for r in range(world)]
    return routers, bufs


class FusedAllGatherRouter(ExchangeRoute):
    """Fused all-gather + METRO over NVLink peer memory, one process per GPU.

    The exchange buffers are allocated per rank and mapped into every peer with
    CUDA IPC handles all-gathered over ``group`` (``torch.distributed`` is the
    plumbing; the exchange itself is the kernel's P2P stores).  Replaces
    ``DistributedRouter``'s NCCL all-gather + route with one launch.
    """

    def __init__(self, placement: DevicePlacement, local_tokens: int, top_k: int, group=None,
                 gather_ids: bool = False, layout=None):
        import ctypes

        from . import _native

        world, rank = dist.get_world_size(group), dist.get_rank(group)
        max_local = -(-local_tokens * top_k // 4) * 4
        self._buf = _ExchangeBuffer(exchange_bytes(placement, world, max_local), placement.device)
        L = _native.lib()
        h = ctypes.create_string_buffer(64)
        _native.check_rc(L.metro_ipc_get_handle(self._buf.ptr, h), "metro_ipc_get_handle")
        handles = [None] * world
        dist.all_gather_object(handles, bytes(h.raw), group=group)
        self._opened = []
        ptrs = []
        with torch.cuda.device(placement.device):
            for q in range(world):
                if q == rank:
                    ptrs.append(self._buf.ptr.value)
                    continue
                p = ctypes.c_void_p()
                _native.check_rc(L.metro_ipc_open_handle(ctypes.create_string_buffer(handles[q], 64),
                                                         ctypes.byref(p)), "metro_ipc_open_handle")
                self._opened.append(p)
                ptrs.append(p.value)
        super().__init__(placement, rank, world, local_tokens, top_k, ptrs, max_local, gather_ids, layout)
        dist.barrier(group=group)

    def close(self):
        from . import _native

        for p in self._opened:
            _native.lib().metro_ipc_close_handle(p)
        self._opened = []
        self._buf.close()
