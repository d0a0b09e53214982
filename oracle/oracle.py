"""ctypes wrapper over oracle/_build/libmetro_oracle.so (test infrastructure only)."""

from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libmetro_oracle.so")
_lib: Optional[ctypes.CDLL] = None

ERR_ID_RANGE = 1
ERR_NO_REPLICA = 2


class OracleError(RuntimeError):
    def __init__(self, code: int, detail: str = ""):
        self.code = code
        super().__init__(f"oracle error {code}{': ' + detail if detail else ''}")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no GPU needed)."""
    src = os.path.join(_HERE, "metro_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        i32, i64 = ctypes.c_int32, ctypes.c_int64
        L.oracle_aggregate_loads.argtypes = [P, i64, i32, P, P]
        L.oracle_route_metro.argtypes = [P, P, i32, i32, P, P, P]
        L.oracle_route_metro_order.argtypes = [P, P, i32, i32, P, i32, P, P, P]
        L.oracle_route_eplb.argtypes = [P, P, i32, i32, P, P, P]
        L.oracle_pair_rank_metro.argtypes = [P, i64, P, P]
        L.oracle_pair_rank_metro.restype = None
        L.oracle_pair_rank_eplb.argtypes = [P, i64, P, i32, i32, P]
        L.oracle_metro_layer.argtypes = [P, i64, P, i32, i32, P, P, P, P, P]
        L.oracle_dispatch_layout.argtypes = [P, P, i64, P, i32, i32, P, P, P]
        L.oracle_gate_topk.argtypes = [P, i64, i32, i32, P]
        L.oracle_gate_topk.restype = None
        _lib = L
    return _lib


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def _c(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


def aggregate_loads(ids, num_experts: int) -> np.ndarray:
    ids = _c(ids, np.int32).reshape(-1)
    loads = np.zeros(num_experts, dtype=np.int64)
    bad = np.zeros(1, dtype=np.int64)
    rc = lib().oracle_aggregate_loads(_p(ids), ids.size, num_experts, _p(loads), _p(bad))
    if rc:
        raise OracleError(rc, f"pair {int(bad[0])}")
    return loads


def route_metro(loads, A) -> Tuple[np.ndarray, np.ndarray, int]:
    """Returns (choice[N] int32 with -1 for inactive, rank_counts[G] int64, lam)."""
    loads = _c(loads, np.int64)
    A = _c(A, np.int8)
    n, g = A.shape
    choice = np.empty(n, dtype=np.int32)
    counts = np.zeros(g, dtype=np.int64)
    lam = np.zeros(1, dtype=np.int64)
    rc = lib().oracle_route_metro(_p(loads), _p(A), n, g, _p(choice), _p(counts), _p(lam))
    if rc:
        raise OracleError(rc)
    return choice, counts, int(lam[0])


def route_metro_order(loads, A, order) -> Tuple[np.ndarray, np.ndarray, int]:
    loads = _c(loads, np.int64)
    A = _c(A, np.int8)
    order = _c(order, np.int32)
    n, g = A.shape
    choice = np.empty(n, dtype=np.int32)
    counts = np.zeros(g, dtype=np.int64)
    lam = np.zeros(1, dtype=np.int64)
    rc = lib().oracle_route_metro_order(
        _p(loads), _p(A), n, g, _p(order), order.size, _p(choice), _p(counts), _p(lam)
    )
    if rc:
        raise OracleError(rc)
    return choice, counts, int(lam[0])


def route_eplb(loads, A) -> Tuple[np.ndarray, np.ndarray, int]:
    """Returns (x[N,G] int64, rank_counts[G] int64, lam)."""
    loads = _c(loads, np.int64)
    A = _c(A, np.int8)
    n, g = A.shape
    x = np.zeros((n, g), dtype=np.int64)
    counts = np.zeros(g, dtype=np.int64)
    lam = np.zeros(1, dtype=np.int64)
    rc = lib().oracle_route_eplb(_p(loads), _p(A), n, g, _p(x), _p(counts), _p(lam))
    if rc:
        raise OracleError(rc)
    return x, counts, int(lam[0])


def pair_rank_metro(ids, choice) -> np.ndarray:
    ids = _c(ids, np.int32)
    choice = _c(choice, np.int32)
    out = np.empty(ids.shape, dtype=np.int32)
    lib().oracle_pair_rank_metro(_p(ids), ids.size, _p(choice), _p(out))
    return out


def pair_rank_eplb(ids, A) -> np.ndarray:
    ids = _c(ids, np.int32)
    A = _c(A, np.int8)
    n, g = A.shape
    out = np.empty(ids.shape, dtype=np.int32)
    rc = lib().oracle_pair_rank_eplb(_p(ids), ids.size, _p(A), n, g, _p(out))
    if rc:
        raise OracleError(rc)
    return out


def metro_layer(ids, A, out=None):
    """aggregate_loads -> route_metro -> pair_rank in one C call (CPU baseline)."""
    ids = _c(ids, np.int32)
    A = _c(A, np.int8)
    n, g = A.shape
    if out is None:
        out = (
            np.zeros(n, dtype=np.int64),
            np.empty(n, dtype=np.int32),
            np.zeros(g, dtype=np.int64),
            np.zeros(1, dtype=np.int64),
            np.empty(ids.shape, dtype=np.int32),
        )
    loads, choice, counts, lam, pr = out
    rc = lib().oracle_metro_layer(
        _p(ids), ids.size, _p(A), n, g, _p(loads), _p(choice), _p(counts), _p(lam), _p(pr)
    )
    if rc:
        raise OracleError(rc)
    return out


def dispatch_layout(ids, pair_rank, A) -> Tuple[np.ndarray, np.ndarray]:
    """(pair_row [P], rep_off [nrep + 1]) -- see oracle_dispatch_layout."""
    ids = _c(ids, np.int32).reshape(-1)
    pr = _c(pair_rank, np.int32).reshape(-1)
    A = _c(A, np.int8)
    N, G = A.shape
    nrep = int((A != 0).sum())
    row = np.empty(ids.size, np.int32)
    off = np.empty(nrep + 1, np.int32)
    bad = np.zeros(1, np.int64)
    rc = lib().oracle_dispatch_layout(_p(ids), _p(pr), ids.size, _p(A), N, G, _p(row), _p(off), _p(bad))
    if rc:
        raise OracleError(rc, f"pair {int(bad[0])}")
    return row, off


def gate_topk(scores, k: int) -> np.ndarray:
    """int32 [T, k]: each row's k largest scores' expert ids, largest first."""
    sc = _c(scores, np.float32)
    T, N = sc.shape
    if not 1 <= k <= N:
        raise OracleError(3, "k out of range")
    ids = np.empty((T, k), np.int32)
    lib().oracle_gate_topk(_p(sc), T, N, k, _p(ids))
    return ids
