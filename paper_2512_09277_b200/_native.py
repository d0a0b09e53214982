"""ctypes binding of the sm_100a routing library (include/metro_route.h).

The library is the product: there is no CPU fallback.  If the shared object is
missing or cannot be loaded, every routing call raises ``NativeLibraryError``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "_lib")
# METRO_B200_LIB: load another build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("METRO_B200_LIB") or os.path.join(LIB_DIR, "libmetro_b200.so")
CSRC = os.path.join(_HERE, "csrc")

ABI_VERSION = 1

# status / return codes (include/metro_route.h)
OK = 0
ERR_ID_RANGE = 1
ERR_NO_REPLICA = 2
ERR_LOAD_RANGE = 3
ERR_PAIR_RANK = 4
ERR_PEER_TIMEOUT = 5
EARG = -1
EDIMS = -2
ECUDA = -3
ENOTBINARY = -4
ENOMEM = -5
HOST_ZEROCOPY = 1
HOST_STABLE_BUFFERS = 2
PLAN_METRO = 0
PLAN_EPLB = 1

MAX_G = 128
MAX_N = 4096


class NativeLibraryError(RuntimeError):
    """The sm_100a routing library is missing, stale or failed a CUDA call."""


_lib: Optional[ctypes.CDLL] = None


def build(verbose: bool = False) -> str:
    """Compile csrc/ with nvcc for sm_100a (works without a GPU)."""
    cmd = ["make", "-C", CSRC] + ([] if verbose else ["-s"])
    subprocess.run(cmd, check=True)
    return LIB_PATH


def lib() -> ctypes.CDLL:
    """Load the library once; raise loudly if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make -C paper_2512_09277_b200/csrc` (no CPU fallback exists)"
        )
    L = ctypes.CDLL(LIB_PATH)
    P, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    sig = {
        "metro_abi_version": ([], ctypes.c_int),
        "metro_strerror": ([ctypes.c_int], ctypes.c_char_p),
        "metro_last_cuda_error": ([], ctypes.c_int),
        "metro_mask_words": ([i32], ctypes.c_int),
        "metro_pack_placement": ([P, i32, i32, P], ctypes.c_int),
        "metro_aggregate_loads_v1": ([P, i64, i32, P, P, i32, P], ctypes.c_int),
        "metro_route_v1": ([P, i64, P, i32, i32, P, P, P, P, P, P, i32, P], ctypes.c_int),
        "metro_route_scores_v1": ([P, i64, i32, P, i32, i32, P, P, P, P, P, P, P, P, i32, P], ctypes.c_int),
        "metro_scores_workspace_bytes": ([i32], ctypes.c_size_t),
        "metro_route_from_loads_v1": ([P, P, i32, i32, P, P, P, P, P], ctypes.c_int),
        "metro_route_ordered_v1": ([P, i32, P, i32, i32, P, P, P, P, P], ctypes.c_int),
        "eplb_route_v1": ([P, i64, P, i32, i32, P, P, P, P, P, P, i32, P], ctypes.c_int),
        "eplb_route_from_loads_v1": ([P, P, i32, i32, P, P, P, P, P], ctypes.c_int),
        "metro_route_plan_create_v1": ([i32, P, i64, P, i32, i32, P, P, P, P, P, P, P, i32, P], ctypes.c_int),
        "metro_route_plan_launch_v1": ([P, P], ctypes.c_int),
        "metro_route_plan_destroy_v1": ([P], ctypes.c_int),
        "metro_host_workspace_bytes": ([i64, i32, i32], ctypes.c_size_t),
        "metro_route_host_v1": ([P, i64, P, i32, i32, P, P, P, i32, i32, P], ctypes.c_int),
        "metro_debug_set_stamps": ([P], None),
        "metro_set_pdl": ([i32], None),
        "metro_server_create_v1": ([P, i32, i32, i64, i32, P], ctypes.c_int),
        "metro_server_route_v1": ([P, P, i64, P, P], ctypes.c_int),
        "metro_server_launches": ([P], ctypes.c_int64),
        "metro_server_destroy_v1": ([P], ctypes.c_int),
        "metro_server_debug_stamps": ([P, P], ctypes.c_int),
        "metro_exchange_bytes": ([i32, i32, i64], ctypes.c_size_t),
        "metro_allgather_route_v1": ([P, i64, i32, i32, P, i64, P, i32, i32, P, P, P, P, P, P, P, P],
                                     ctypes.c_int),
        "metro_allgather_debug_stamps": ([P], None),
        "metro_allgather_route_layout_v1": ([P, i64, i32, i32, P, i64, P, i32, i32, P, P, i32, P, P, P, P, P, P,
                                             P, P, P], ctypes.c_int),
        "metro_exchange_alloc": ([ctypes.c_size_t, P], ctypes.c_int),
        "metro_exchange_free": ([P], ctypes.c_int),
        "metro_ipc_get_handle": ([P, P], ctypes.c_int),
        "metro_ipc_open_handle": ([P, P], ctypes.c_int),
        "metro_ipc_close_handle": ([P], ctypes.c_int),
        "metro_replica_table": ([P, i32, i32, P, P], ctypes.c_int),
        "metro_dispatch_layout_v1": ([P, P, i64, P, P, i32, i32, i32, P, P, P, i32, P], ctypes.c_int),
        "metro_route_layout_v1": ([P, i64, P, i32, i32, P, P, i32, P, P, P, P, P, P, P, P, i32, P], ctypes.c_int),
    }
    for name, (argtypes, restype) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = argtypes
        fn.restype = restype
    if L.metro_abi_version() != ABI_VERSION:
        raise NativeLibraryError(f"ABI mismatch: library {L.metro_abi_version()} != {ABI_VERSION}")
    _lib = L
    return L


HEADERS = ("metro_route.h", "metro_serve.h", "metro_exchange.h", "moe_gemm.h", "dispatch_layout.h")


def exported_symbols() -> list:
    """Names declared in include/*.h (used by the ABI test)."""
    import re

    names = set()
    for h in HEADERS:
        with open(os.path.join(os.path.dirname(_HERE), "include", h)) as f:
            names.update(re.findall(r"METRO_API\s+[\w\s\*]+?\b(\w+)\s*\(", f.read()))
    return sorted(names)


def check_rc(rc: int, what: str) -> None:
    """Map a negative C-ABI return code to an exception."""
    if rc == OK:
        return
    from .core import ValidationError

    L = lib()
    msg = L.metro_strerror(rc).decode()
    if rc == ECUDA:
        raise NativeLibraryError(f"{what}: CUDA error {L.metro_last_cuda_error()} ({msg})")
    raise ValidationError(f"{what}: {msg}")
