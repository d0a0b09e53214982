"""B200-native (sm_100a) METRO token routing for expert-parallel MoE decode.

Drop-in for the routing API of the reference package ``eproute``
(/root/reference/pkg/src/eproute/__init__.py:8-69): the same names with the same
argument meaning, return types and exceptions, executed by hand-written CUDA
kernels behind the C ABI in include/metro_route.h.  No CPU fallback.

Fast path (device tensors, graph-capturable): ``DevicePlacement`` + ``Router``.
Multi-GPU (one process per GPU, NCCL all-gather of top-k ids): ``dist``.
"""

from .core import (
    ClusterSpec,
    ConfigurationError,
    ExpertLoadVector,
    ModelSpec,
    PlacementMap,
    RoutingAssignment,
    Token,
    TokenBatch,
    ValidationError,
    ValidationReport,
    validate_assignment,
)
from .placement import (
    ReplicationPlan,
    eplb_place,
    eplb_replicate,
    gen_zipf_topk,
    gen_zipf_trace,
    make_placement,
    zipf_popularity,
)
from .routing import (
    ROUTER_KINDS,
    aggregate_loads,
    lambda_of,
    route_bruteforce,
    route_eplb,
    route_metro,
    route_metro_parallel,
    route_optimal,
    run_router,
    save_assignment,
)
from .device import DevicePlacement, HostRouter, RoutePlan, RouteResult, Router, ServedRouter, pack_placement
from .dispatch import DispatchLayout, LayoutResult, replica_table
from .io import (
    Trace,
    TraceBatch,
    TraceFormatError,
    load_placement,
    load_trace,
    load_trace_topk,
    save_placement,
    save_trace,
)
from ._native import NativeLibraryError

__all__ = [
    "ClusterSpec", "ConfigurationError", "ExpertLoadVector", "ModelSpec", "PlacementMap",
    "ReplicationPlan", "ROUTER_KINDS", "RoutingAssignment", "Token", "TokenBatch",
    "ValidationError", "ValidationReport", "aggregate_loads", "eplb_place", "eplb_replicate",
    "gen_zipf_topk", "gen_zipf_trace", "lambda_of", "make_placement", "route_bruteforce",
    "route_eplb", "route_metro", "route_metro_parallel", "route_optimal", "run_router",
    "save_assignment", "validate_assignment", "zipf_popularity",
    "DevicePlacement", "HostRouter", "RoutePlan", "RouteResult", "Router", "ServedRouter", "pack_placement",
    "NativeLibraryError", "Trace", "TraceBatch", "TraceFormatError", "load_placement", "load_trace",
    "load_trace_topk", "save_placement", "save_trace", "DispatchLayout", "LayoutResult", "replica_table",
]

__version__ = "0.1.0"
