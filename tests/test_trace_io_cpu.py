"""Detailed-record files (chm_trace_load / chm_record_save):
round trips, equality with the recorded path, and parse errors with byte offsets."""
import json

import numpy as np
import pytest

import oracle as O
from paper_2509_11076_b200 import chm
from workloads import traces as W


def _params(tr):
    return (tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd)


def _tables_equal(a, b):
    ta, tb = a.tables(), b.tables()
    for k in ta:
        assert np.array_equal(ta[k], tb[k]), k
    assert (a.N, a.K, a.L, a.peak0) == (b.N, b.K, b.L, b.peak0)


def _recorded(tr):
    ctx = chm.Context(device=-1)
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    return ctx, ctx.trace_build(*_params(tr), t_iter=tr.t_iter)


@pytest.mark.parametrize("name", ["C1", "C2", "C5"])
def test_save_load_round_trip(name):
    tr = W.CONFIGS[name]()
    ctx, pt = _recorded(tr)
    text = ctx.record_save()
    ctx2 = chm.Context(device=-1)
    pt2 = ctx2.trace_load(text, *_params(tr))
    _tables_equal(pt, pt2)
    assert len(text.splitlines()) == tr.n_ops + 1
    # saving the same record again is byte-identical (determinism of the writer)
    assert ctx.record_save() == text


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_generator_file_equals_recorded_path_and_oracle(name):
    tr = W.CONFIGS[name]()
    ctx, pt = _recorded(tr)
    pt_f = chm.Context(device=-1).trace_load(W.to_jsonl(tr), *_params(tr))
    _tables_equal(pt, pt_f)
    m = O.Model(tr)
    assert np.array_equal(pt_f.tables()["f0"], m.f0())
    assert pt_f.K == m.K


def test_swap_log_and_live_bytes_survive_the_file():
    tr = W.tiny()
    m = O.Model(tr)
    meas = m.f0() - 4096
    lines = W.to_jsonl(tr).decode().splitlines()
    out = [lines[0]]
    for i, ln in enumerate(lines[1:]):
        d = json.loads(ln)
        d["live"] = int(meas[i])
        out.append(json.dumps(d))
    out.append(json.dumps({"swap": [3, 7, 4096]}))
    pt = chm.Context(device=-1).trace_load(("\n".join(out) + "\n").encode(), *_params(tr), f0_source=1)
    exp = meas.copy()
    exp[3:7] += 4096
    assert np.array_equal(pt.tables()["f0"], exp)


def _load_err(text):
    with pytest.raises(chm.ChmError) as ei:
        chm.Context(device=-1).trace_load(text, 1 << 30, 0, 1e9, 1, 1)
    return ei.value


def test_parse_errors_carry_byte_offsets():
    tr = W.tiny()
    text = W.to_jsonl(tr)
    # truncated mid-line: the offset is inside the last (cut) line
    cut = len(text) - 7
    e = _load_err(text[:cut])
    assert e.code == chm.CHM_E_PARSE and text.rfind(b"\n", 0, cut) < e.offset <= cut
    # a corrupted character at a known offset
    k = text.index(b"\n", 200) + 5
    bad = text[:k] + b"#" + text[k + 1:]
    e = _load_err(bad)
    assert e.code == chm.CHM_E_PARSE and text.rfind(b"\n", 0, k) < e.offset < text.index(b"\n", k)  # on that line
    # missing header, bad tensor id, double output, interleaved phases
    assert _load_err(b'{"op":"a","phase":0}\n').code == chm.CHM_E_PARSE
    hdr = b'{"chm_trace":1,"tensors":[[512,0],[512,0]]}\n'
    assert _load_err(hdr + b'{"op":"a","phase":0,"out":[2]}\n').offset == len(hdr)
    assert _load_err(hdr + b'{"op":"a","phase":0,"out":[0]}\n{"op":"b","phase":0,"out":[0]}\n').code == chm.CHM_E_PARSE
    two = hdr + b'{"op":"a","phase":1,"out":[0]}\n'
    assert _load_err(two + b'{"op":"b","phase":0,"in":[0]}\n').offset == len(two)
    # no partial trace: a good file still loads on the same ctx afterwards
    ctx = chm.Context(device=-1)
    with pytest.raises(chm.ChmError):
        ctx.trace_load(text[:cut], *_params(tr))
    assert ctx.trace_load(text, *_params(tr)).N == tr.n_ops


def test_record_save_needs_a_detailed_iteration():
    with pytest.raises(chm.ChmError):
        chm.Context(device=-1).record_save()
