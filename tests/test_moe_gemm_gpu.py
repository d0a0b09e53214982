"""K3 grouped expert GEMM (tcgen05) numerics vs a plain PyTorch fp32 reference.

bf16 inputs, fp32 accumulation in TMEM, bf16 outputs: tolerance = bf16 output
rounding (2^-8 relative) plus fp32 summation-order noise -> rtol 2e-2, atol 2e-2
on O(1)-magnitude outputs.
"""

import numpy as np
import pytest
import torch

from paper_2512_09277_b200 import moe

pytestmark = pytest.mark.gpu
RTOL = ATOL = 2e-2


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def ref_gemm(W, X, groups):
    Y = torch.zeros((X.shape[0], W.shape[1]), dtype=torch.float32, device=X.device)
    for e, t0, n in groups:
        Y[t0:t0 + n] = X[t0:t0 + n].float() @ W[e].float().t()
    return Y


@pytest.mark.parametrize("E,M,K,sizes", [
    (3, 256, 512, [1, 17, 40, 300]),
    (2, 128, 64, [16, 32, 5]),
    (4, 384, 1024, [256, 255, 257, 64, 129]),
])
def test_grouped_gemm_vs_torch(E, M, K, sizes):
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(E * 1000 + M + K)
    groups, t = [], 0
    for i, n in enumerate(sizes):
        groups.append((i % E, t, n))
        t += n
    W = (torch.randn((E, M, K), generator=g, device=dev) * K ** -0.5).to(torch.bfloat16)
    X = torch.randn((t, K), generator=g, device=dev).to(torch.bfloat16)
    items = torch.from_numpy(moe.build_items(groups, M))
    Y = moe.grouped_gemm(W, X, items)
    torch.cuda.synchronize()
    torch.testing.assert_close(Y.float(), ref_gemm(W, X, groups), rtol=RTOL, atol=ATOL)


def test_grouped_gemm_few_ctas_many_items():
    """More items than CTAs: the persistent loop, TMEM double buffering and the
    smem ring wrap many times."""
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(7)
    E, M, K = 5, 512, 768
    sizes = [3, 70, 200, 33, 256, 12]
    groups, t = [], 0
    for i, n in enumerate(sizes):
        groups.append((i % E, t, n))
        t += n
    W = (torch.randn((E, M, K), generator=g, device=dev) * K ** -0.5).to(torch.bfloat16)
    X = torch.randn((t, K), generator=g, device=dev).to(torch.bfloat16)
    items = torch.from_numpy(moe.build_items(groups, M))
    for ctas in (1, 3, 7):
        Y = moe.grouped_gemm(W, X, items, num_ctas=ctas)
        torch.cuda.synchronize()
        torch.testing.assert_close(Y.float(), ref_gemm(W, X, groups), rtol=RTOL, atol=ATOL)


def test_expert_ffn_vs_torch():
    dev = torch.device("cuda")
    ffn = moe.ExpertFFN(slots=4, hidden=256, inter=128, device=dev, seed=3)
    groups, t = [], 0
    for e, n in [(0, 9), (3, 130), (1, 1)]:
        groups.append((e, t, n))
        t += n
    X = torch.randn((t, 256), device=dev).to(torch.bfloat16)
    wl = moe.RankWorkload(groups, t, len(groups))
    i1, i2 = ffn.plan(wl, dev)
    Y = ffn.forward(X, i1, i2)
    torch.cuda.synchronize()
    ref = torch.zeros((t, 256), device=dev)
    for e, t0, n in groups:
        gu = X[t0:t0 + n].float() @ ffn.W1[e].float().t()
        h = torch.nn.functional.silu(gu[:, :128]) * gu[:, 128:]
        h = h.to(torch.bfloat16).float()
        ref[t0:t0 + n] = h @ ffn.W2[e].float().t()
    torch.testing.assert_close(Y.float(), ref, rtol=5e-2, atol=5e-2)


def test_deepseek_expert_shape():
    """One DeepSeek-V3 expert (D=7168, I=2048) with a ragged token count."""
    dev = torch.device("cuda")
    ffn = moe.ExpertFFN(slots=2, hidden=7168, inter=2048, device=dev, seed=1)
    groups = [(1, 0, 37)]
    X = torch.randn((37, 7168), device=dev).to(torch.bfloat16)
    i1, i2 = ffn.plan(moe.RankWorkload(groups, 37, 1), dev)
    GU = moe.grouped_gemm(ffn.W1, X, i1)
    torch.cuda.synchronize()
    torch.testing.assert_close(GU.float(), X.float() @ ffn.W1[1].float().t(), rtol=RTOL, atol=ATOL)
