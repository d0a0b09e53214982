"""Time-bounded soak in the driver's GPU suite: random instances (N 1..700, G
1..128, k 1..10, B 0..3000, duplicates, reference-generator and random
placements) through every device entry point -- METRO / EPLB from ids at every
cluster size, route_metro(T, A), metro-parallel, fused gating, dispatch layout,
the persistent host router, the fused exchange on virtual ranks -- each compared
bit-exactly with the oracle (tools/soak_parity.py).  METRO_SOAK_SECONDS sets the
budget (default 60 s); the seed changes per run so each driver round sees fresh
instances, and a failure prints its seed."""

import os
import sys
import time

import pytest
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.init()


@pytest.mark.gpu
def test_soak_parity_time_bounded():
    sys.path.insert(0, os.path.join(REPO, "tools"))
    import soak_parity

    seconds = float(os.environ.get("METRO_SOAK_SECONDS", "60"))
    seed = int(os.environ.get("METRO_SOAK_SEED", str(int(time.time()) & 0xFFFFFF)))
    s = soak_parity.run(seconds, seed)
    bad = {k: v for k, v in s["checks"].items() if v["mismatches"]}
    print(f"soak seed {seed}: {s['instances']} instances, checks "
          + ", ".join(f"{k} {v['run']}" for k, v in s["checks"].items()))
    assert s["instances"] > 0
    assert not bad and not s["failures"], (seed, bad, s["failures"][:3])
