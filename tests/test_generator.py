"""NEXT-1: Algo. 2 policy generator.  Oracle pins (SPEC examples, feasibility via the
independent replay) and the product's host implementation against the oracle (identical items)."""
import numpy as np
import pytest

import oracle as O
from tests.helpers import make_trace
from workloads import traces as W

from paper_2509_11076_b200 import chm


def product_trace(ctx, tr):
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    ctx.set_detailed(False)
    return ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter,
                           omega=tr.omega)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C5"])
@pytest.mark.parametrize("C_coef,rem", [(0.0, 1.0), (1.0, 1.0), (4.0, 1.0), (1.0, 3.0)])
def test_product_generator_matches_oracle(name, C_coef, rem):
    tr = W.CONFIGS[name]()
    m = O.Model(tr)
    g = O.generate(m, C_coef=C_coef, rem_scale=rem)
    pt = product_trace(chm.Context(device=-1), tr)
    items, feasible = pt.generate_policy(C_coef, rem)
    assert feasible == g["feasible"]
    assert items["t"].astype(np.int64).tolist() == g["t"].tolist()
    assert items["r"].tolist() == g["r"].tolist() and items["s"].tolist() == g["s"].tolist()
    assert ((items["flags"] & 1) != 0).astype(int).tolist() == g["fallback"].tolist()
    assert ((items["flags"] & 2) != 0).astype(int).tolist() == g["saturated"].tolist()


@pytest.mark.parametrize("seed", range(12))
def test_product_generator_random(seed):
    tr = W.random_trace(300 + seed, n_layers=3 + seed % 3, ops_per_layer=3, bw=[1e5, 1e6, 1e7][seed % 3])
    m = O.Model(tr)
    g = O.generate(m, C_coef=float(seed % 3))
    items, feasible = product_trace(chm.Context(device=-1), tr).generate_policy(float(seed % 3), 1.0)
    assert feasible == g["feasible"]
    assert items["t"].astype(np.int64).tolist() == g["t"].tolist()
    assert items["r"].tolist() == g["r"].tolist() and items["s"].tolist() == g["s"].tolist()


def _ladder(sizes, n_fwd_layers=4, ops_per=2, t_iter=8.0, bw=1.0, static=100, budget=None):
    """FWD layers of `ops_per` ops, each tensor j produced at FWD op 2j, read at the mirrored BWD op."""
    nf = n_fwd_layers * ops_per
    n = 2 * nf
    ins = [[] for _ in range(n)]
    outs = [[] for _ in range(n)]
    frees = [[] for _ in range(n)]
    for j, _ in enumerate(sizes):
        p = 2 * j
        b = n - 1 - p
        outs[p] = [j]
        ins[b] = [j]
        frees[b] = [j]
    ph = [0] * nf + [1] * nf
    total = sum(sizes)
    return make_trace(ph, sizes, ins, outs, frees, static, t_iter, bw,
                      static + total // 2 if budget is None else budget, n_fwd_layers, n_fwd_layers)


def test_generator_under_budget_is_empty_S259():
    tr = _ladder([10, 10, 10, 10], budget=10 ** 9)
    g = O.generate(O.Model(tr))
    assert g["feasible"] and len(g["t"]) == 0


def test_generator_raise_error_when_no_candidate_S260():
    # the only tensor that overlaps the peak is a BWD temporary (not a candidate): Raise Error
    ins = [[], [], [0], []]
    outs = [[], [], [0], []]
    frees = [[], [], [0], []]
    tr = make_trace([0, 0, 1, 1], [50], ins, outs, frees, 100, 4.0, 1.0, 120, 1, 1)
    g = O.generate(O.Model(tr))
    assert not g["feasible"] and len(g["t"]) == 0


def test_generator_clears_mrl_and_replay_confirms_S261():
    # 4 FWD layers, generous bandwidth: the generator's items clear the MRL and the independent
    # event replay of those items is within budget
    # F0 = [140,140,170,170,190,190,200,200,200,200,190,190,170,170,140,140], budget 175: MREs on
    # ops 4..11.  Hand derivation: the 40 B tensor (a=0, b=15) scores highest; T_swap = 0.04 < 2.0
    # in layer 6 (ops 12-13) -> s = 12, crediting ops 1..11 clears the MRL; SetFreeTime: layer 0
    # has 2.0 > 0.04 -> r = 1.  Replay: the peak drops to 170.
    tr = _ladder([40, 30, 20, 10], n_fwd_layers=4, ops_per=2, t_iter=16.0, bw=1000.0, static=100, budget=175)
    m = O.Model(tr)
    assert m.f0().max() == 200
    g = O.generate(m)
    assert g["feasible"]
    assert (g["t"].tolist(), g["r"].tolist(), g["s"].tolist()) == ([0], [1], [12])
    rep = m.replay(g["t"], g["r"], g["s"])
    assert rep["peak"] == 170
    # every item: a_t <= r, r + 1 < s <= b_t
    p, f, a, b = m.tensor_table()
    for t, r, s in zip(g["t"], g["r"], g["s"]):
        assert a[t] <= r and r + 1 < s <= b[t]


def test_generator_fallback_when_nothing_fits_S241():
    # bandwidth so low no layer has T_remaining > T_swap: the highest-score candidate is still
    # scheduled in the layer before its first BWD use, flagged as fallback
    tr = _ladder([40, 30], n_fwd_layers=4, ops_per=2, t_iter=8.0, bw=1e-3, static=100, budget=120)
    g = O.generate(O.Model(tr))
    assert len(g["t"]) >= 1 and g["fallback"][0] == 1
    st, n, ty, bud = O.Model(tr).layers()
    lay = np.repeat(np.arange(len(n)), n)
    p, f, a, b = O.Model(tr).tensor_table()
    t0 = g["t"][0]
    assert g["s"][0] == st[lay[b[t0]] - 1]


def test_explicit_validation_and_install_host():
    tr = W.tiny()
    ctx = chm.Context(device=-1)
    pt = product_trace(ctx, tr)
    items, _ = pt.generate_policy(1.0, 1.0)
    ctx.policy_install_items(pt, items)
    bad = items.copy()
    bad["s"][0] = bad["r"][0] + 1  # empty window
    with pytest.raises(chm.ChmError):
        ctx.policy_install_items(pt, bad)
    # installed explicit items fire at their own r / s
    ev = {"rel": [], "in": []}

    def on(i, act):
        av = chm.actions_view(act)
        ev["rel"] += [(i, it) for it in av["release"]]
        ev["in"] += [(i, it) for it in av["swap_in_item"]]
    chm.record_iteration(ctx, tr, on_actions=on)
    assert sorted(i for i, _ in ev["rel"]) == sorted(items["r"].tolist())
    assert sorted(i for i, _ in ev["in"]) == sorted((items["s"] - 1).tolist())


def test_generator_infeasible_budget_reports_and_keeps_items():
    # budget 150: op 12 still needs 20 after both large tensors are placed and no unselected
    # tensor's span covers it -> Raise Error, items chosen so far are returned
    tr = _ladder([40, 30, 20, 10], n_fwd_layers=4, ops_per=2, t_iter=16.0, bw=1000.0, static=100, budget=150)
    g = O.generate(O.Model(tr))
    assert not g["feasible"]
    assert (g["t"].tolist(), g["r"].tolist(), g["s"].tolist()) == ([0, 1], [1, 3], [12, 10])
