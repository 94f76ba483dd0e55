"""Property-based checks (hypothesis) on CPU: the product's host path -- trace build (a3) through a
host-only ctx, the generator (NEXT-1), the stall models, Detailed-record files -- against the
oracle on random traces with random link speeds, iteration times, layer groupings and budgets.
The oracle itself is pinned elsewhere (tests/test_oracle_pins.py); here hypothesis searches the
input space for a disagreement and shrinks it."""
import numpy as np
import pytest

hypothesis = pytest.importorskip("hypothesis")
from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

import oracle as O  # noqa: E402
from paper_2509_11076_b200 import chm  # noqa: E402
from workloads import traces as W  # noqa: E402

traces = st.builds(
    W.random_trace,
    seed=st.integers(0, 10 ** 6),
    n_layers=st.integers(1, 5),
    ops_per_layer=st.integers(1, 4),
    max_kib=st.sampled_from([1, 8, 64, 512]),
    bw=st.sampled_from([1e6, 3e7, 1e9, 5e10]),
    t_iter=st.sampled_from([1e-5, 1e-3, 0.1]),
)


def _product(tr, omega):
    ctx = chm.Context(device=-1)
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    return ctx, ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter,
                                omega=omega)


@settings(max_examples=60, deadline=None)
@given(tr=traces, omega=st.sampled_from([0.5, 1.0, 1.7]))
def test_trace_build_equals_oracle(tr, omega):
    ctx, pt = _product(tr, omega)
    m = O.Model(tr, omega=omega)
    tb = pt.tables()
    assert (pt.N, pt.K, pt.L) == (m.N, m.K, m.L)
    assert np.array_equal(tb["f0"], m.f0())
    sw = m.swappable()
    assert np.array_equal(tb["tensor"].astype(np.int64), sw["t"])
    for k in ("r", "s", "lin", "lout"):
        assert np.array_equal(tb[k], sw[k]), k
    st_, n, ty, bud = m.layers()
    assert np.array_equal(tb["lay_start"], st_) and np.array_equal(tb["bud"], bud)
    assert np.array_equal(tb["base"], m.base_mask())


@settings(max_examples=40, deadline=None)
@given(tr=traces, cc=st.sampled_from([0.0, 1.0, 3.0]), rr=st.sampled_from([0.5, 1.0, 2.0]))
def test_generator_and_stall_models_equal_oracle(tr, cc, rr):
    ctx, pt = _product(tr, 1.0)
    m = O.Model(tr)
    items, feas = pt.generate_policy(cc, rr)
    ref = O.generate(m, C_coef=cc, rem_scale=rr)
    assert items["t"].tolist() == ref["t"].tolist()
    assert items["r"].tolist() == ref["r"].tolist() and items["s"].tolist() == ref["s"].tolist()
    assert feas == ref["feasible"]
    if len(items):
        t, r, s = items["t"].astype(np.int32), items["r"], items["s"]
        got = pt.stall_models(items)
        assert got.tolist() == [m.stall(t, r, s), m.stall_dir(t, r, s), m.stall_timeline(t, r, s)]


@settings(max_examples=30, deadline=None)
@given(tr=traces)
def test_record_file_round_trip(tr):
    ctx, pt = _product(tr, 1.0)
    pt2 = chm.Context(device=-1).trace_load(ctx.record_save(), tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd,
                                            tr.groups_bwd, t_iter=tr.t_iter)
    a, b = pt.tables(), pt2.tables()
    for k in a:
        assert np.array_equal(a[k], b[k]), k
