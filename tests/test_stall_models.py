"""Stall-model variants of reading Q11: per-direction layer budgets and the
max-plus serial-stream timeline.  The oracle is pinned against closed forms derived by hand
(one item: the copy time beyond its slack on each side; two items in one FIFO: their summed copy
time beyond the shared slack), against the earliest-start schedule of the model's precedence DAG
derived separately (absolute times, one final subtraction), against invariants (per-direction
<= one shared budget; a slower link never stalls less; an infinitely fast link never stalls),
then the product's host
evaluation (`chm_stall_models`) must equal the oracle bit for bit, and its R-stall entry must
equal the replay kernels' model (the oracle's orc_stall)."""
import numpy as np
import pytest

import oracle as O
from paper_2509_11076_b200 import chm
from tests.helpers import make_trace
from workloads import traces as W

TAU = 1e-3  # op time T_iter / N of the hand traces


def _hand(sizes, r=2, s=6):
    """10 ops, 5 FWD + 5 BWD; every listed tensor is produced by op 0, used by op 1 (a = 1) and
    op 8 (b = 8), freed at op 8; items released after r, swapped in before s"""
    n = 10
    T = len(sizes)
    ins = [[] for _ in range(n)]
    outs = [[] for _ in range(n)]
    frees = [[] for _ in range(n)]
    outs[0] = list(range(T))
    ins[1] = list(range(T))
    ins[8] = list(range(T))
    frees[8] = list(range(T))
    tr = make_trace([0] * 5 + [1] * 5, sizes, ins, outs, frees, 0, TAU * n, 1e9, 1 << 40, 5, 5)
    m = O.Model(tr)
    return tr, m, list(range(T)), [r] * T, [s] * T


def test_timeline_single_item_closed_form():
    # S / B = 2.5 tau: slack (r - a) tau = 1 tau on the way out, (b - s) tau = 2 tau on the way in
    tr, m, t, r, s = _hand([int(2.5 * TAU * 1e9)])
    exp = max(0.0, 2.5 * TAU - (2 - 1) * TAU) + max(0.0, 2.5 * TAU - (8 - 6) * TAU)
    assert m.stall_timeline(t, r, s) == pytest.approx(exp, rel=1e-12)
    # enough slack on both sides: no stall
    tr, m, t, r, s = _hand([int(0.5 * TAU * 1e9)], r=3, s=6)
    assert m.stall_timeline(t, r, s) == 0.0


def test_timeline_fifo_two_items_closed_form():
    # two 1.5 tau copies queue on each direction: (S1 + S2)/B beyond the shared slack
    tr, m, t, r, s = _hand([int(1.5 * TAU * 1e9)] * 2)
    exp = max(0.0, 3.0 * TAU - 1 * TAU) + max(0.0, 3.0 * TAU - 2 * TAU)
    assert m.stall_timeline(t, r, s) == pytest.approx(exp, rel=1e-12)


def _hand_items(sizes_tau, r, s):
    """like _hand, but each item k has its own release op r[k] and swap-in op s[k]; sizes in
    units of tau * B (so S/B = sizes_tau[k] * tau).  10 ops, one op per layer: Bud_l = tau."""
    tr, m, t, _, _ = _hand([int(x * TAU * 1e9) for x in sizes_tau])
    return tr, m, t, list(r), list(s)


def test_stall_dir_one_item_two_layers_closed_form():
    """orc_stall_dir (Q11 per-direction variant, P:333 / P:340): one item released after op 4
    (out charged to layer 4) and swapped in before op 6 (in charged to layer 6),
    S/B = 2.5 tau against Bud = tau in each layer:
    stall = (2.5 - 1) tau [out, layer 4] + (2.5 - 1) tau [in, layer 6] = 3 tau (= R-stall here:
    the two directions never share a layer)"""
    tr, m, t, r, s = _hand_items([2.5], [4], [6])
    assert m.stall_dir(t, r, s) == pytest.approx(3.0 * TAU, rel=1e-12)
    assert m.stall(t, r, s) == pytest.approx(3.0 * TAU, rel=1e-12)
    # under budget on both sides: nothing
    tr, m, t, r, s = _hand_items([0.9], [4], [6])
    assert m.stall_dir(t, r, s) == 0.0


def test_stall_dir_opposite_directions_in_one_layer_closed_form():
    """Three items (sizes in tau * B): A = 2.5 (r 4, s 6), B = 0.5 (r 2, s 4), C = 0.8 (r 3, s 6).
    Layer 4 holds A's swap-out and B's swap-in; layer 6 the swap-ins of A and C.  By hand:
      per direction: out l2 max(0, .5-1)=0, out l3 max(0, .8-1)=0, out l4 2.5-1=1.5,
                     in l4 max(0, .5-1)=0, in l6 (2.5+.8)-1=2.3            -> 3.8 tau
      R-stall (one budget per layer): l4 (2.5+.5)-1=2.0, l6 2.3, l2/l3 0  -> 4.3 tau
    so R-stall - per-direction = 0.5 tau.  Plausible slips give other numbers: one budget of
    2 Bud for both directions (l4 3-2=1, l6 3.3-2=1.3: 2.3 tau); swap-ins charged to lay(r)
    (in l4 A 1.5, out l4 A 1.5: 3.0 tau); the max taken over the sum of both directions' terms
    (l4 1.5-0.5=1.0: 3.3 tau)."""
    tr, m, t, r, s = _hand_items([2.5, 0.5, 0.8], [4, 2, 3], [6, 4, 6])
    d, lay = m.stall_dir(t, r, s), m.stall(t, r, s)
    assert d == pytest.approx(3.8 * TAU, rel=1e-12)
    assert lay == pytest.approx(4.3 * TAU, rel=1e-12)
    assert lay - d == pytest.approx(0.5 * TAU, rel=1e-9)
    # the item order does not matter (sums of integers per layer, then a fixed-order tree)
    perm = [2, 0, 1]
    assert m.stall_dir([t[k] for k in perm], [r[k] for k in perm], [s[k] for k in perm]) == d


def _random_items(m, rng, n_max=None):
    sw = m.swappable()
    if m.K == 0:
        return [], [], []
    k = rng.choice(m.K, size=rng.integers(1, (n_max or m.K) + 1) if m.K > 1 else 1, replace=False)
    return sw["t"][k], sw["r"][k], sw["s"][k]


@pytest.mark.parametrize("seed", range(12))
def test_invariants_on_random_traces(seed):
    rng = np.random.default_rng(seed)
    tr = W.random_trace(seed, bw=rng.uniform(2e8, 2e9), t_iter=rng.uniform(1e-4, 1e-2))
    m = O.Model(tr)
    t, r, s = _random_items(m, rng)
    if len(t) == 0:
        return
    lay, dirs, tl = m.stall(t, r, s), m.stall_dir(t, r, s), m.stall_timeline(t, r, s)
    assert 0.0 <= dirs <= lay + 1e-15  # two budgets per layer never stall more than one
    assert tl >= 0.0
    slow = O.Model(tr, bw=tr.bw / 2)
    assert slow.stall(t, r, s) >= lay and slow.stall_dir(t, r, s) >= dirs
    assert slow.stall_timeline(t, r, s) >= tl
    fast = O.Model(tr, bw=1e30)
    assert fast.stall(t, r, s) == fast.stall_dir(t, r, s) == fast.stall_timeline(t, r, s) == 0.0
    # the timeline never waits longer than the copies themselves take
    assert tl <= 2 * float(tr.nbytes[t].sum()) / tr.bw * (1 + 1e-12)


def _product(tr):
    ctx = chm.Context(device=-1)
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    return ctx, ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter,
                                omega=tr.omega)


@pytest.mark.parametrize("name", ["C1", "C2", "C5"])
def test_product_equals_oracle_on_masks_and_generator_items(name):
    tr = W.CONFIGS[name]()
    m = O.Model(tr)
    ctx, pt = _product(tr)
    sw = m.swappable()
    rng = np.random.default_rng(7)
    for trial in range(6):
        bits = rng.random(pt.K) < (0.1 + 0.15 * trial)
        words = np.zeros(max(pt.W, 1), np.uint64)
        for k in np.nonzero(bits)[0]:
            words[k // 64] |= np.uint64(1 << int(k % 64))
        got = pt.stall_models(pt.mask_items(words[:pt.W]))
        t, r, s = sw["t"][bits], sw["r"][bits], sw["s"][bits]
        exp = [m.stall(t, r, s), m.stall_dir(t, r, s), m.stall_timeline(t, r, s)]
        assert got.tolist() == exp, (trial, got, exp)
    for cc in (0.0, 1.0):
        items, _ = pt.generate_policy(cc, 1.0)
        if len(items) == 0:
            continue
        got = pt.stall_models(items)
        p, f, a, b = m.tensor_table()
        # production rank == trace tensor index for the synthetic traces
        t, r, s = items["t"].astype(np.int32), items["r"], items["s"]
        exp = [m.stall(t, r, s), m.stall_dir(t, r, s), m.stall_timeline(t, r, s)]
        assert got.tolist() == exp


def test_product_validates_items():
    tr = W.tiny()
    ctx, pt = _product(tr)
    bad = np.zeros(1, chm.ITEM_DTYPE)
    bad["t"] = 10 ** 6
    with pytest.raises(chm.ChmError):
        pt.stall_models(bad)
    assert pt.stall_models(np.zeros(0, chm.ITEM_DTYPE)).tolist() == [0.0, 0.0, 0.0]


def test_eval_model_timeline_is_stall_timeline_of_mask_items():
    """orc_eval_model(stall_model = 1) scores each candidate with stall_timeline of its items in
    mask-bit order; peak / swapped / footprint equal those of the R-stall evaluation; the key's
    stall field follows the model"""
    tr = W.tiny()
    m = O.Model(tr)
    n = 3000
    a = m.eval(O.EXHAUSTIVE, 0, n, stall_model=1, footprint=True)
    b = m.eval(O.EXHAUSTIVE, 0, n, footprint=True)
    for c in (0, 1, 2, 17, 1234, n - 1):
        t, r, s = m.mask_items([(c >> k) & 1 for k in range(m.K)])
        assert a["stall"][c] == m.stall_timeline(t, r, s)
    for key in ("peak", "swapped", "footprint"):
        assert np.array_equal(a[key], b[key])
    assert np.count_nonzero(a["stall"] != b["stall"]) > 0
    i = int(a["best"].index)
    exc = np.maximum(a["peak"] - tr.budget, 0)
    order = np.lexsort((np.arange(n), a["swapped"], a["stall"], exc))
    assert order[0] == i


def _dag_timeline(tr, m, t, r, s):
    """The Q11 timeline derived independently as earliest start times of a precedence DAG (ops
    of tau each in sequence; a FIFO per direction; the rules chm_stall_models documents), then
    stall = (time the last op's releases are done) - N tau.  Absolute times and one final
    subtraction, not the oracle's running `now` with stall increments."""
    N = len(tr.phase)
    tau = tr.t_iter / N
    ranks = [int(x) for i in range(N) for x in tr.out_idx[tr.out_ptr[i]:tr.out_ptr[i + 1]]]
    _, _, a, b = m.tensor_table()
    items = list(range(len(t)))
    S = [int(tr.nbytes[ranks[int(t[k])]]) for k in items]
    dur = [S[k] / tr.bw for k in items]
    out_end, in_end = {}, {}
    pre = 0.0  # ready time before op i's swap-in / wait phase
    d2h_free = h2d_free = 0.0
    for i in range(N):
        for k in items:  # swap-ins issued before op i, FIFO in item order
            if s[k] == i:
                st = max(pre, h2d_free, out_end.get(k, 0.0))
                in_end[k] = st + dur[k]
                h2d_free = in_end[k]
        start = max([pre] + [in_end[k] for k in items if b[int(t[k])] == i])  # first-use waits
        end = start + tau
        for k in items:  # swap-outs issued after op i, FIFO in item order
            if a[int(t[k])] == i:
                st = max(end, d2h_free)
                out_end[k] = st + dur[k]
                d2h_free = out_end[k]
        pre = max([end] + [out_end[k] for k in items if r[k] == i])  # releases after op i
    return pre - N * tau


@pytest.mark.parametrize("seed", range(16))
def test_timeline_equals_the_precedence_dag(seed):
    """pin: the oracle's timeline = the longest-path (earliest-start) schedule of the model's
    precedence DAG on random traces and item sets, to rounding (the two sum in different orders)"""
    rng = np.random.default_rng(100 + seed)
    tr = W.random_trace(seed, bw=rng.uniform(2e7, 2e9), t_iter=rng.uniform(1e-4, 1e-2))
    m = O.Model(tr)
    t, r, s = _random_items(m, rng)
    if len(t) == 0:
        return
    got = m.stall_timeline(t, r, s)
    exp = _dag_timeline(tr, m, t, r, s)
    assert got == pytest.approx(exp, rel=1e-9, abs=1e-12 * tr.t_iter)
