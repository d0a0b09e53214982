"""Trace / placement / assignment JSONL formats interoperate with the reference."""

import numpy as np
import pytest

import paper_2512_09277_b200 as pkg
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement


def _trace():
    tr = pkg.Trace(64, 4, 8)
    for layer in range(3):
        ids = gen_zipf_topk(64, 8, 12, 1.1, 100 + layer)
        tr.batches.append(pkg.TraceBatch(layer, "decode" if layer else "prefill", pkg.TokenBatch.from_topk(ids, 4)))
    return tr


def test_trace_roundtrip(tmp_path):
    tr = _trace()
    p = tmp_path / "t.jsonl"
    pkg.save_trace(tr, p)
    back = pkg.load_trace(p)
    assert (back.num_experts, back.num_gpus, back.top_k) == (64, 4, 8)
    for a, b in zip(tr.batches, back.batches):
        assert a.layer == b.layer and a.phase == b.phase
        assert np.array_equal(a.batch.topk_ids(8), b.batch.topk_ids(8))
    hdr, arrays = pkg.load_trace_topk(p)
    assert hdr == (64, 4, 8) and len(arrays) == 3
    assert np.array_equal(arrays[1][2], tr.batches[1].batch.topk_ids(8))
    pkg.save_trace(back, tmp_path / "again.jsonl")
    assert p.read_text() == (tmp_path / "again.jsonl").read_text()


@pytest.mark.parametrize("bad,msg", [
    ('{"nope": 1}\n', "first record must be the header"),
    ('{"header": {"N": 4, "G": 2}}\n', "header missing field"),
    ('{"header": {"N": 4, "G": 2, "k": 2}}\n{"layer": 0, "phase": "x", "tokens": []}\n', "unknown phase"),
    ('{"header": {"N": 4, "G": 2, "k": 2}}\n{"layer": 0, "phase": "decode", "tokens": [{"src": 0, "experts": [1, 9]}]}\n',
     "out of range"),
    ('{"header": {"N": 4, "G": 2, "k": 2}}\nnot json\n', "invalid JSON"),
])
def test_trace_errors(tmp_path, bad, msg):
    p = tmp_path / "bad.jsonl"
    p.write_text(bad)
    with pytest.raises(pkg.TraceFormatError, match=msg):
        pkg.load_trace(p)


def test_empty_trace(tmp_path):
    p = tmp_path / "e.jsonl"
    p.write_text("")
    t = pkg.load_trace(p)
    assert (t.num_experts, t.num_gpus, t.top_k, len(t.batches)) == (0, 0, 0, 0)


def test_placement_roundtrip(tmp_path):
    A = make_placement(128, 8, 1.5, 7)
    pkg.save_placement(A, tmp_path / "p.jsonl")
    B = pkg.load_placement(tmp_path / "p.jsonl")
    assert np.array_equal(A.matrix, B.matrix) and A.slots_per_gpu == B.slots_per_gpu


def test_formats_interoperate_with_reference(tmp_path, eproute_ref):
    from eproute.core import load_trace as rload, save_trace as rsave
    from eproute.placement import load_placement as rlp, save_placement as rsp

    tr = _trace()
    pkg.save_trace(tr, tmp_path / "ours.jsonl")
    ref_tr = rload(tmp_path / "ours.jsonl")
    rsave(ref_tr, tmp_path / "theirs.jsonl")
    assert (tmp_path / "ours.jsonl").read_text() == (tmp_path / "theirs.jsonl").read_text()
    assert len(pkg.load_trace(tmp_path / "theirs.jsonl").batches) == 3
    A = make_placement(64, 4, 1.25, 3)
    pkg.save_placement(A, tmp_path / "pa.jsonl")
    rA = rlp(tmp_path / "pa.jsonl")
    rsp(rA, tmp_path / "pb.jsonl")
    assert (tmp_path / "pa.jsonl").read_text() == (tmp_path / "pb.jsonl").read_text()
