"""Reference-compatible routing API, executed by the sm_100a kernels.

Drop-in for /root/reference/pkg/src/eproute/routing.py (+ core.aggregate_loads):
same names, argument meaning, return types and exceptions.  Every call runs on
the GPU through include/metro_route.h; there is no CPU fallback.

  ROUTER_KINDS          routing.py:24
  _check_dims           routing.py:29-33   -> ValidationError("dimension mismatch ...")
  lambda_of             routing.py:36-38
  route_eplb            routing.py:55-72   -> eplb_route_from_loads_v1
  route_metro           routing.py:105-113 -> metro_route_from_loads_v1
  route_metro_parallel  routing.py:116-128 -> metro_route_ordered_v1 (seeded numpy shuffle
                                              on the host, exactly as the reference)
  run_router            routing.py:219-233
  aggregate_loads       core.py:236-244    -> metro_aggregate_loads_v1

``optimal`` / ``bruteforce`` are the reference's CPU quality oracles
(max-flow / exhaustive search); they are outside the B200 hot path (DESIGN.md
§6) and raise NotImplementedError here.
"""

from __future__ import annotations

import json

import numpy as np
import torch

from . import _native
from .core import ExpertLoadVector, RoutingAssignment, TokenBatch, ValidationError
from .device import DevicePlacement, _stream, aggregate_loads_device, raise_status

ROUTER_KINDS = ("eplb", "metro", "metro-parallel", "optimal", "bruteforce")
DEVICE_KINDS = ("eplb", "metro", "metro-parallel")


def _loads_of(T) -> np.ndarray:
    return np.asarray(getattr(T, "loads", T), dtype=np.int64)


def _matrix_of(A) -> np.ndarray:
    return np.asarray(getattr(A, "matrix", A))


def _check_dims(loads: np.ndarray, mat: np.ndarray) -> None:
    if loads.shape[0] != mat.shape[0]:
        raise ValidationError(
            f"dimension mismatch: T has {loads.shape[0]} experts, A has {mat.shape[0]}"
        )


def lambda_of(a: RoutingAssignment) -> int:
    """Maximum activated-replica count over EP ranks."""
    return int(a.y.sum(axis=0).max()) if a.y.size else 0


def _device() -> torch.device:
    _native.lib()  # fail loudly before anything else if the library is missing
    if not torch.cuda.is_available():
        raise _native.NativeLibraryError("no CUDA device: the B200 routing path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _rank_compress(loads: np.ndarray) -> np.ndarray:
    """Order-preserving relabel of loads >= 2^32 (the greedy only compares T)."""
    if loads.size == 0 or loads.max() < (1 << 32):
        return loads
    pos = loads > 0
    uniq = np.unique(loads[pos])
    out = np.zeros_like(loads)
    out[pos] = np.searchsorted(uniq, loads[pos]) + 1
    return out


def _empty(n: int, g: int) -> RoutingAssignment:
    return RoutingAssignment(x=np.zeros((n, g), np.int64), y=np.zeros((n, g), np.int8), lam=0)


def _degenerate(loads: np.ndarray, mat: np.ndarray):
    """Shapes the kernels do not launch for: nothing active, or no ranks at all."""
    n, g = mat.shape
    if n == 0 or not (loads > 0).any():
        return _empty(n, g)
    if g == 0:
        raise AssertionError("placement invariant: every expert has a replica")
    return None


def _from_choice(loads: np.ndarray, choice: np.ndarray, n: int, g: int, lam: int) -> RoutingAssignment:
    x = np.zeros((n, g), np.int64)
    y = np.zeros((n, g), np.int8)
    act = np.flatnonzero(choice >= 0)
    x[act, choice[act]] = loads[act]
    y[act, choice[act]] = 1
    return RoutingAssignment(x=x, y=y, lam=lam)


def _run_metro(loads: np.ndarray, mat: np.ndarray, order=None) -> RoutingAssignment:
    dev = _device()
    n, g = mat.shape
    placement = DevicePlacement(mat, dev)
    i32 = dict(dtype=torch.int32, device=dev)
    out = torch.empty(n + g + 1 + 4, **i32)
    choice, counts, lam, status = out[:n], out[n:n + g], out[n + g:n + g + 1], out[n + g + 1:]
    L = _native.lib()
    s = _stream(dev)
    if order is None:
        t_dev = torch.from_numpy(_rank_compress(loads)).to(dev)
        rc = L.metro_route_from_loads_v1(
            t_dev.data_ptr(), placement.mask.data_ptr(), n, g, choice.data_ptr(),
            counts.data_ptr(), lam.data_ptr(), status.data_ptr(), s,
        )
        what = "metro_route_from_loads_v1"
    else:
        o_dev = torch.from_numpy(np.ascontiguousarray(order, dtype=np.int32)).to(dev)
        rc = L.metro_route_ordered_v1(
            o_dev.data_ptr(), len(order), placement.mask.data_ptr(), n, g, choice.data_ptr(),
            counts.data_ptr(), lam.data_ptr(), status.data_ptr(), s,
        )
        what = "metro_route_ordered_v1"
    _native.check_rc(rc, what)
    host = out.cpu().numpy()
    raise_status(host[n + g + 1:])
    return _from_choice(loads, host[:n].astype(np.int64), n, g, int(host[n + g]))


def route_metro(T, A) -> RoutingAssignment:
    """METRO greedy: one replica per active expert, canonical order, lowest-rank ties."""
    loads, mat = _loads_of(T), _matrix_of(A)
    _check_dims(loads, mat)
    _device()
    deg = _degenerate(loads, mat)
    if deg is not None:
        return deg
    return _run_metro(loads, mat)


def route_metro_parallel(T, A, seed: int) -> RoutingAssignment:
    """Greedy under the reference's seeded serialisation order (routing.py:124-128)."""
    loads, mat = _loads_of(T), _matrix_of(A)
    _check_dims(loads, mat)
    _device()
    active = [int(i) for i in np.flatnonzero(loads)]
    rng = np.random.default_rng(seed)
    rng.shuffle(active)
    deg = _degenerate(loads, mat)
    if deg is not None:
        return deg
    return _run_metro(loads, mat, order=active)


def route_eplb(T, A) -> RoutingAssignment:
    """EPLB even split; remainder tokens to replicas in ascending rank id."""
    loads, mat = _loads_of(T), _matrix_of(A)
    _check_dims(loads, mat)
    dev = _device()
    deg = _degenerate(loads, mat)
    if deg is not None:
        return deg
    n, g = mat.shape
    placement = DevicePlacement(mat, dev)
    t_dev = torch.from_numpy(np.ascontiguousarray(loads)).to(dev)
    x = torch.empty((n, g), dtype=torch.int64, device=dev)
    small = torch.empty(g + 1 + 4, dtype=torch.int32, device=dev)
    counts, lam, status = small[:g], small[g:g + 1], small[g + 1:]
    rc = _native.lib().eplb_route_from_loads_v1(
        t_dev.data_ptr(), placement.mask.data_ptr(), n, g, x.data_ptr(), counts.data_ptr(),
        lam.data_ptr(), status.data_ptr(), _stream(dev),
    )
    _native.check_rc(rc, "eplb_route_from_loads_v1")
    host_small = small.cpu().numpy()
    raise_status(host_small[g + 1:])
    xh = x.cpu().numpy()
    return RoutingAssignment(x=xh, y=(xh > 0).astype(np.int8), lam=int(host_small[g]))


def route_optimal(T, A) -> RoutingAssignment:
    raise NotImplementedError(
        "router 'optimal' (binary search + max-flow, reference routing.py:131-159) is a CPU "
        "quality oracle outside the B200 routing path; see DESIGN.md §6"
    )


def route_bruteforce(T, A, guard: int = 10 ** 6) -> RoutingAssignment:
    raise NotImplementedError(
        "router 'bruteforce' (reference routing.py:162-216) is a CPU quality oracle outside the "
        "B200 routing path; see DESIGN.md §6"
    )


def run_router(kind: str, T, A, seed: int = 0) -> RoutingAssignment:
    """Dispatch by name (routing.py:219-233)."""
    if kind == "eplb":
        return route_eplb(T, A)
    if kind == "metro":
        return route_metro(T, A)
    if kind == "metro-parallel":
        return route_metro_parallel(T, A, seed)
    if kind == "optimal":
        return route_optimal(T, A)
    if kind == "bruteforce":
        return route_bruteforce(T, A)
    raise ValidationError(f"unknown router kind {kind!r}; expected one of {ROUTER_KINDS}")


def aggregate_loads(batch, model) -> ExpertLoadVector:
    """Per-expert (token, slot) counts on the GPU (reference core.py:236-244).

    ``batch`` may be a TokenBatch, a host array of ids or a CUDA int32 tensor.
    Out-of-range ids raise ValidationError("token t: expert id e out of range").
    """
    n = int(model.num_experts)
    k = int(getattr(model, "top_k", 1))
    dev = _device()
    offsets = None
    if isinstance(batch, torch.Tensor):
        ids = batch.to(dev, dtype=torch.int32).contiguous()
    else:
        if isinstance(batch, TokenBatch) or hasattr(batch, "tokens"):
            lens = np.fromiter((len(t.expert_ids) for t in batch.tokens), dtype=np.int64,
                               count=len(batch.tokens))
            flat = np.fromiter((e for t in batch.tokens for e in t.expert_ids), dtype=np.int64,
                               count=int(lens.sum()))
            offsets = np.concatenate([[0], np.cumsum(lens)])
        else:
            flat = np.asarray(batch, dtype=np.int64).reshape(-1)
        bad = (flat < -(1 << 31)) | (flat >= (1 << 31))
        if bad.any():  # ids beyond int32 cannot be in range; report like the reference
            p = int(np.flatnonzero(bad)[0])
            t = int(np.searchsorted(offsets, p, side="right") - 1) if offsets is not None else p // k
            raise ValidationError(f"token {t}: expert id {int(flat[p])} out of range")
        ids = torch.from_numpy(flat.astype(np.int32)).to(dev)
    if ids.numel() == 0:
        return ExpertLoadVector(np.zeros(n, np.int64))
    loads, status = aggregate_loads_device(ids, n)
    st = status.cpu().numpy()
    if int(st[0]) == _native.ERR_ID_RANGE and offsets is not None:
        p = int(np.uint32(st[1])) | (int(np.uint32(st[2])) << 32)
        t = int(np.searchsorted(offsets, p, side="right") - 1)
        raise ValidationError(f"token {t}: expert id {int(st[3])} out of range")
    raise_status(st, k)
    return ExpertLoadVector(loads.cpu().numpy().astype(np.int64))


def save_assignment(a: RoutingAssignment, path) -> None:
    """Assignment export in the reference's JSONL format (routing.py:236-244)."""
    with open(path, "w", encoding="utf-8") as f:
        for i, g in zip(*np.nonzero(a.x)):
            f.write(json.dumps({"expert": int(i), "gpu": int(g), "tokens": int(a.x[i, g])},
                               separators=(",", ":")) + "\n")
        f.write(json.dumps({"lambda": a.lam, "max_tokens_per_gpu": a.max_tokens_per_gpu()},
                           separators=(",", ":")) + "\n")
