"""Routing quality at the reference's statistical scale (reference criterion 3,
/root/reference/pkg/tests/test_acceptance.py:70-90): 500 Zipf(1.2) batches of
model128 x cluster8 (128 experts top-8, 8 ranks, 32 tokens per GPU) on
make_placement(128, 8, 1.25, 7); mean(lam_metro / lam_opt) <= 1.15 and
mean(lam_eplb / lam_metro) >= 1.20.  lam_opt comes from the reference's
route_optimal (out of scope here) via tests/golden/quality.npz
(make_quality_golden.py).

CPU: the pinned generator + oracle reproduce the reference's lambdas of all 500
batches.  GPU (-m gpu): the device routers (METRO and EPLB, metro_route_v1 /
eplb routing, every batch its own launch) reproduce them and the criterion's
two means hold.
"""

import os

import numpy as np
import pytest

import oracle
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def quality():
    z = np.load(os.path.join(HERE, "golden", "quality.npz"))
    return {k: z[k] for k in z.files}


def batches(n=500):
    return [gen_zipf_topk(128, 8, 32 * 8, 1.2, 1000 + s, popularity_seed=7) for s in range(n)]


def test_quality_fixture_reproduced_by_oracle(quality):
    A = make_placement(128, 8, 1.25, 7).matrix
    assert np.array_equal(A, quality["A"])
    bs = batches()
    assert np.array_equal(bs[0], quality["ids0"])
    met, epl = [], []
    for ids in bs:
        T = oracle.aggregate_loads(ids, 128)
        met.append(oracle.route_metro(T, A)[2])
        epl.append(oracle.route_eplb(T, A)[2])
    assert np.array_equal(met, quality["lam_metro"])
    assert np.array_equal(epl, quality["lam_eplb"])
    opt = quality["lam_opt"]
    assert (opt <= quality["lam_metro"]).all() and (quality["lam_metro"] <= quality["lam_eplb"]).all()
    # the reference's own criterion on its own numbers (test_acceptance.py:86-88)
    assert np.mean(quality["lam_metro"] / opt) <= 1.15 and np.mean(quality["lam_eplb"] / quality["lam_metro"]) >= 1.20


@pytest.mark.gpu
def test_quality_criterion3_device(quality):
    import torch

    from paper_2512_09277_b200 import DevicePlacement, Router

    A = make_placement(128, 8, 1.25, 7).matrix
    pl = DevicePlacement(A, torch.device("cuda", 0))
    rm, re = Router(pl, "metro"), Router(pl, "eplb")
    bs = batches()
    ids = torch.from_numpy(np.stack(bs)).cuda()
    om, oe = rm.alloc(bs[0].size, top_k=8), re.alloc(bs[0].size, top_k=8)
    met, epl = [], []
    for s in range(len(bs)):
        met.append(int(rm.route(ids[s], out=om).check().lam.item()))
        epl.append(int(re.route(ids[s], out=oe).check().lam.item()))
    met, epl = np.asarray(met), np.asarray(epl)
    assert np.array_equal(met, quality["lam_metro"]) and np.array_equal(epl, quality["lam_eplb"])
    mo = float(np.mean(met / quality["lam_opt"]))
    em = float(np.mean(epl / met))
    print(f"criterion 3 on device: metro/opt={mo:.4f} eplb/metro={em:.4f} over {len(bs)} batches")
    assert mo <= 1.15 and em >= 1.20
