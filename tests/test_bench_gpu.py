"""bench.py end to end on the GPU (-m gpu), short runs: the driver's JSON contract
at N = 1 and, through --virtual-ranks 2, the N > 1 branch (torchrun environment,
two processes on one GPU, the fused exchange over CUDA IPC) -- so a change that
breaks either branch fails here rather than in the driver's round-end run."""

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks", "lambda")


def _run(args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=REPO)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_single_gpu_short():
    d = _run(["--steps", "100", "--warmup", "3", "--e2e-steps", "20", "--cpu-seconds", "0.2", "--no-moe"])
    for k in KEYS:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] >= 100
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1
    assert d["cpu_baseline"]["parity_vs_gpu"] is True
    assert d["lambda"]["metro_le_eplb_all"] is True and d["lambda"]["batches"] >= 100


def test_bench_virtual_ranks_two():
    d = _run(["--virtual-ranks", "2", "--steps", "20", "--warmup", "3", "--e2e-steps", "10", "--cpu-seconds",
              "0.2", "--no-moe"])
    for k in KEYS:
        assert k in d, k
    assert d["n_gpus"] == 2 and d["virtual_ranks"]["ranks"] == 2
    assert "nccl_allgather_plus_route_us" in d["timing"]
