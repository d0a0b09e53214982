"""Golden fixture for the routing-quality statistics (reference criterion 3).

Run in the build container (the reference only exists there):

    python tests/golden/make_quality_golden.py

The reference's acceptance test ``test_criterion_3_routing_quality``
(/root/reference/pkg/tests/test_acceptance.py:70-90) routes 500 Zipf(1.2)
batches (model128 x cluster8: 128 experts top-8, 8 ranks, 32 tokens per GPU,
seeds 1000 + s, popularity seed 7) on make_placement(128, 8, 1.25, 7) and
requires mean(lam_metro / lam_optimal) <= 1.15 and mean(lam_eplb / lam_metro)
>= 1.20.  ``route_optimal`` (binary search + max-flow, routing.py:131-190) is
out of this repo's scope, so its lambda per batch is stored here
together with the reference's METRO and EPLB lambdas; the GPU test
(tests/test_quality_gpu.py) regenerates the same batches with the pinned
generator, routes them through the device router and recomputes the two means.

Output: ``quality.npz`` -- lam_opt, lam_metro, lam_eplb [500] int64, and the
first batch's ids (a generator spot check).
"""

from __future__ import annotations

import importlib.util
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_CONFTEST = "/root/reference/pkg/tests/conftest.py"
HERE = os.path.dirname(os.path.abspath(__file__))

sys.path.insert(0, REF_SRC)
from eproute import aggregate_loads, gen_zipf_trace  # noqa: E402
from eproute.routing import route_eplb, route_metro, route_optimal  # noqa: E402

_spec = importlib.util.spec_from_file_location("ref_conftest", REF_CONFTEST)
ref_conftest = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(ref_conftest)

SEEDS = 500


def main() -> None:
    # the conftest fixtures cluster8 / model128 (conftest.py:17-41), as their bodies build them
    from eproute import ClusterSpec, ModelSpec

    cluster8 = ClusterSpec(num_gpus=8, hbm_bandwidth=1.555e12, peak_flops=312e12, link_bandwidth=600e9,
                           collective_launch_overhead=15e-6, link_base_latency=2e-6)
    model128 = ModelSpec(num_experts=128, top_k=8, hidden_dim=2048, dtype_bytes=2,
                         expert_weight_bytes=9437184.0, dense_weight_bytes=2e7,
                         flops_per_token_per_expert=9437184.0, num_moe_layers=48)
    A = ref_conftest.make_placement(128, 8, 1.25, history_seed=7)
    opt, met, epl = [], [], []
    first = None
    for s in range(SEEDS):
        batch = gen_zipf_trace(model128, cluster8, 32, 1.2, 1000 + s, popularity_seed=7)
        if first is None:
            first = np.array([t.expert_ids for t in batch.tokens], np.int32)
        T = aggregate_loads(batch, model128)
        opt.append(route_optimal(T, A).lam)
        met.append(route_metro(T, A).lam)
        epl.append(route_eplb(T, A).lam)
    opt, met, epl = (np.asarray(v, np.int64) for v in (opt, met, epl))
    np.savez_compressed(os.path.join(HERE, "quality.npz"), lam_opt=opt, lam_metro=met, lam_eplb=epl,
                        ids0=first, A=np.asarray(A.matrix, np.int8))
    print(f"metro/opt={np.mean(met / opt):.4f} eplb/metro={np.mean(epl / met):.4f}")


if __name__ == "__main__":
    main()
