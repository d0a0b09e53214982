"""CPU oracle for the METRO routing hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this package, and only as the checker.
The product (``paper_2512_09277_b200``) never imports it and has no CPU
fallback.

``metro_oracle.c`` restates the reference functions literally (see the file
header for the file:line map).  Parity of the oracle itself is pinned against
golden vectors produced by the unmodified reference package
(``tests/golden/make_golden.py``); see ``tests/test_oracle_golden.py``.
"""

from .oracle import (  # noqa: F401
    OracleError,
    aggregate_loads,
    build,
    dispatch_layout,
    gate_topk,
    lib,
    metro_layer,
    pair_rank_eplb,
    pair_rank_metro,
    route_eplb,
    route_metro,
    route_metro_order,
)
