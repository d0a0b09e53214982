"""K3 grouped expert GEMM (tcgen05) numerics vs a plain PyTorch fp32 reference.

bf16 inputs, fp32 accumulation in TMEM, bf16 outputs: tolerance = bf16 output
rounding (2^-8 relative) plus fp32 summation-order noise -> rtol 2e-2, atol 2e-2
on O(1)-magnitude outputs.
"""

import numpy as np
import pytest
import torch

from paper_2512_09277_b200 import moe
from paper_2512_09277_b200.core import ValidationError

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


def wide_items(groups, M, chunk=256):
    """Items chunked at up to 256 tokens (the wide tiling), built here independently."""
    out = []
    for e, t0, n in groups:
        for mb in range(M // moe.BM):
            for c0 in range(0, n, chunk):
                out.append((e, mb, t0 + c0, min(chunk, n - c0)))
    return np.asarray(out, dtype=np.int32).reshape(-1, 4)


@pytest.mark.parametrize("chunk", [64, 128, 256])
def test_grouped_gemm_both_tilings(chunk):
    """Narrow (<= item_tokens() per item, 8-stage ring) and wide (<= 256, 4 stages)
    tilings on the same problem; device-resident items without a hint take the
    wide tiling, host items pick by their largest token count."""
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(chunk)
    E, M, K = 3, 384, 1024
    sizes = [1, 63, 64, 65, 200, 256, 300]
    groups, t = [], 0
    for i, n in enumerate(sizes):
        groups.append((i % E, t, n))
        t += n
    W = (torch.randn((E, M, K), generator=g, device=dev) * K ** -0.5).to(torch.bfloat16)
    X = torch.randn((t, K), generator=g, device=dev).to(torch.bfloat16)
    items = wide_items(groups, M, chunk)
    ref = ref_gemm(W, X, groups)
    for it in (items, torch.from_numpy(items).to(dev)):
        Y = moe.grouped_gemm(W, X, it)
        torch.cuda.synchronize()
        torch.testing.assert_close(Y.float(), ref, rtol=RTOL, atol=ATOL)
    assert moe.item_tokens() == 64


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


def _rank_reference(ffn, ids, hidden, pr, A, rank):
    """fp32 torch reference of one rank's FFN over its rows in dispatch-layout order
    (layout from the CPU oracle)."""
    import oracle

    row, off = oracle.dispatch_layout(ids, pr, A)
    rid = np.cumsum((np.asarray(A) != 0).T.reshape(-1)).reshape(A.shape[1], A.shape[0]).T - 1
    sel = np.flatnonzero(pr.reshape(-1) == rank)
    rows = int(sel.size)
    tok = np.empty(rows, np.int64)
    tok[row[sel]] = sel // ids.shape[1]
    X = hidden[torch.from_numpy(tok).to(hidden.device)].float()
    Y = torch.zeros((rows, ffn.hidden), dtype=torch.float32, device=hidden.device)
    slots = np.cumsum(np.asarray(A)[:, rank] != 0) - 1
    ids_f = ids.reshape(-1)
    base = off[rid[np.flatnonzero(np.asarray(A)[:, rank])[0], rank]] if rows else 0
    for e in np.unique(ids_f[sel]):
        r0 = off[rid[e, rank]] - base
        n = off[rid[e, rank] + 1] - off[rid[e, rank]]
        s = int(slots[e])
        gu = X[r0:r0 + n] @ ffn.W1[s].float().t()
        h = torch.nn.functional.silu(gu[:, :ffn.inter]) * gu[:, ffn.inter:]
        h = h.to(torch.bfloat16).float()
        Y[r0:r0 + n] = h @ ffn.W2[s].float().t()
    return Y, rows


@pytest.mark.parametrize("kind", ["metro", "eplb"])
def test_rank_moe_pipeline_on_device(kind):
    """route -> dispatch layout -> items -> gather -> FFN with no host round trip,
    against an fp32 torch reference built from the CPU oracle's layout; and the
    same pipeline replayed from a CUDA graph gives bit-identical outputs."""
    from paper_2512_09277_b200 import DevicePlacement
    from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement

    dev = torch.device("cuda")
    N, k, G, B = 64, 4, 4, 96
    A = make_placement(N, G, 1.5, 7).matrix
    pl = DevicePlacement(A, dev)
    slots = int(np.asarray(A).sum(axis=0).max())
    ffn = moe.ExpertFFN(slots, hidden=256, inter=128, device=dev, seed=11)
    ids = gen_zipf_topk(N, k, B, 1.2, 5, popularity_seed=7)
    hidden = torch.randn((B, 256), device=dev).to(torch.bfloat16)
    it = torch.from_numpy(ids).to(dev)
    for rank in range(G):
        pipe = moe.RankMoE(pl, kind, rank, ffn, max_pairs=B * k, top_k=k)
        Y = pipe(it, hidden)
        torch.cuda.synchronize()
        pipe.route_out.check()
        pipe.layout_out.check()
        pr = pipe.route_out.pair_rank[: ids.size].cpu().numpy().reshape(ids.shape)
        ref, rows = _rank_reference(ffn, ids, hidden, pr, A, rank)
        assert int(pipe.counts[2].item()) == rows
        torch.testing.assert_close(Y[:rows].float(), ref, rtol=RTOL, atol=ATOL)
        y0 = Y[:rows].clone()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            pipe(it, hidden)  # warm on the capture stream
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                pipe(it, hidden, stream=s)
        pipe.Y.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(pipe.Y[:rows], y0)


# ------------------------------------------------------------------ FP8 (E4M3)
@pytest.mark.parametrize("E,M,K,sizes", [
    (3, 256, 512, [1, 17, 40, 300]),
    (2, 384, 1024, [64, 65, 5]),
])
def test_grouped_gemm_fp8_vs_torch(E, M, K, sizes):
    """E4M3 weights (scale per 128-row block) and activations (scale per row):
    the kernel against a torch fp32 GEMM of the same dequantised values."""
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(E * 7 + M + K)
    groups, t = [], 0
    for i, n in enumerate(sizes):
        groups.append((i % E, t, n))
        t += n
    W = (torch.randn((E, M, K), generator=g, device=dev) * K ** -0.5).to(torch.bfloat16)
    X = torch.randn((t, K), generator=g, device=dev).to(torch.bfloat16)
    W8, ws = moe.quantize_weights_fp8(W)
    X8, xs = moe.quantize_rows_fp8(X)
    torch.cuda.synchronize()
    Wd = moe.dequantize_fp8(W8, ws, moe.BM)
    Xd = X8.view(torch.float8_e4m3fn).float() * xs[:, None]
    ref = torch.zeros((t, M), dtype=torch.float32, device=dev)
    for e, t0, n in groups:
        ref[t0:t0 + n] = Xd[t0:t0 + n] @ Wd[e].t()
    for items in (moe.build_items(groups, M), wide_items(groups, M, 256)):
        Y = moe.grouped_gemm_fp8(W8, ws, X8, xs, items)
        torch.cuda.synchronize()
        torch.testing.assert_close(Y.float(), ref, rtol=RTOL, atol=ATOL)
    # the quantisation itself: |x - dequant(x)| within half an E4M3 step (3 mantissa bits)
    err = (Xd - X.float()).abs()
    assert bool((err <= X.float().abs() * 2.0 ** -4 + xs[:, None] * 2.0 ** -9).all())


def test_silu_mul_fp8():
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(5)
    T, I = 37, 512
    GU = torch.randn((T, 2 * I), generator=g, device=dev).to(torch.bfloat16)
    H8, hs = moe.silu_mul_fp8(GU)
    torch.cuda.synchronize()
    gf, uf = GU[:, :I].float(), GU[:, I:].float()
    ref = gf * torch.sigmoid(gf) * uf
    Hd = H8.view(torch.float8_e4m3fn).float() * hs[:, None]
    torch.testing.assert_close(hs, ref.abs().amax(dim=1) / 448.0, rtol=1e-5, atol=1e-7)
    assert bool(((Hd - ref).abs() <= ref.abs() * 2.0 ** -4 + hs[:, None] * 2.0 ** -9 + 1e-6).all())


def test_rank_moe_fp8_matches_host_plan():
    """The device pipeline (route -> layout -> items -> gather -> quantise -> FP8
    GEMMs) equals the same rank's FFN run from host-planned items."""
    from paper_2512_09277_b200 import DevicePlacement
    from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement

    dev = torch.device("cuda")
    N, k, G, B, D, I = 64, 4, 4, 96, 256, 128
    A = make_placement(N, G, 1.5, 7).matrix
    pl = DevicePlacement(A, dev)
    slots = int(A.sum(axis=0).max())
    ids = torch.from_numpy(gen_zipf_topk(N, k, B, 1.2, 3, popularity_seed=7)).to(dev)
    g = torch.Generator(device=dev).manual_seed(11)
    hidden = torch.randn((B, D), generator=g, device=dev).to(torch.bfloat16)
    for rank in range(G):
        ffn = moe.ExpertFFN(slots, D, I, dev, seed=rank, dtype="fp8")
        pipe = moe.RankMoE(pl, "metro", rank, ffn, max_pairs=B * k, top_k=k)
        Y = pipe(ids, hidden)
        torch.cuda.synchronize()
        rows = int(pipe.counts[2].item())
        # host reference of the same rank: its received rows in layout order, host items
        X = pipe.X[:rows].clone()
        lo = pipe.layout_out
        rep_off = lo.rep_off.cpu().numpy()
        sb = pipe.layout.slot_base.cpu().numpy()
        groups = []
        base = rep_off[sb[rank]]
        for sl in range(sb[rank + 1] - sb[rank]):
            n = int(rep_off[sb[rank] + sl + 1] - rep_off[sb[rank] + sl])
            if n:
                groups.append((sl, int(rep_off[sb[rank] + sl] - base), n))
        if not groups:
            assert rows == 0
            continue
        i1 = moe.build_items(groups, 2 * I)
        i2 = moe.build_items(groups, D)
        Yh = ffn.forward(X, torch.from_numpy(i1).to(dev), torch.from_numpy(i2).to(dev))
        torch.cuda.synchronize()
        torch.testing.assert_close(Y[:rows].float(), Yh.float(), rtol=0, atol=0)


def test_grouped_gemm_rejects_items_and_outputs_outside_the_problem():
    """Host items must address existing experts / row blocks / token rows, and a
    caller's Y must be the [T, M] bf16 output (the kernel writes through raw
    pointers; its epilogue also drops stores past T as a guard for device items)."""
    dev = torch.device("cuda")
    E, M, K, T = 2, 256, 128, 40
    W = torch.zeros((E, M, K), dtype=torch.bfloat16, device=dev)
    X = torch.zeros((T, K), dtype=torch.bfloat16, device=dev)
    good = np.array([[0, 1, 0, 40]], dtype=np.int32)
    moe.grouped_gemm(W, X, good)
    for bad in ([[2, 0, 0, 8]], [[0, 2, 0, 8]], [[0, 0, 36, 8]], [[-1, 0, 0, 8]], [[0, 0, -1, 8]]):
        with pytest.raises(ValidationError):
            moe.grouped_gemm(W, X, np.array(bad, dtype=np.int32))
    with pytest.raises(ValidationError):
        moe.grouped_gemm(W, X, good, Y=torch.empty((T - 1, M), dtype=torch.bfloat16, device=dev))
    # device items past T: the stores beyond row T are dropped, nothing else is touched
    big = torch.full((T + 8, M), 7.0, dtype=torch.bfloat16, device=dev)
    moe.grouped_gemm(W, X, torch.tensor([[0, 0, 32, 16]], dtype=torch.int32, device=dev),
                     Y=big[:T], max_item_tokens=64)
    torch.cuda.synchronize()
    assert bool((big[T:] == 7.0).all()) and bool((big[32:T, :128] == 0).all())
