"""Host-side steps of the product (a1-a3, a8) through the C-ABI with a host-only ctx (device -1),
against the CPU oracle: trace build tables, Algo. 1, executor trigger positions, tolerance of
minor operator-sequence drift.  Runs without a GPU."""
import numpy as np
import pytest

import oracle as O
from tests.helpers import w1_trace
from workloads import traces as W

from paper_2509_11076_b200 import chm


def host_ctx(**kw):
    return chm.Context(device=-1, **kw)


def product_trace(ctx, tr):
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    ctx.set_detailed(False)
    return ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter,
                           omega=tr.omega)


def check_tables(pt, m):
    tb = pt.tables()
    assert (pt.N, pt.K, pt.L) == (m.N, m.K, m.L)
    assert np.array_equal(tb["f0"], m.f0())
    sw = m.swappable()
    assert np.array_equal(tb["tensor"].astype(np.int64), sw["t"])
    for k in ("r", "s", "lin", "lout"):
        assert np.array_equal(tb[k], sw[k]), k
    st, n, ty, bud = m.layers()
    assert np.array_equal(tb["lay_start"], st) and np.array_equal(tb["lay_count"], n)
    assert np.array_equal(tb["bud"], bud)
    assert np.array_equal(tb["base"], m.base_mask())
    assert pt.peak0 == int(m.f0().max())


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4a", "C4b", "C5"])
def test_trace_build_configs(name):
    tr = W.CONFIGS[name]()
    check_tables(product_trace(host_ctx(), tr), O.Model(tr))


@pytest.mark.parametrize("seed", range(20))
def test_trace_build_random(seed):
    tr = W.random_trace(seed, n_layers=2 + seed % 4, ops_per_layer=1 + seed % 4, bw=[1e5, 1e6, 1e7, 1e8][seed % 4])
    check_tables(product_trace(host_ctx(), tr), O.Model(tr))


@pytest.mark.parametrize("bw", [40.0, 15.0])
def test_trace_build_w1(bw):
    tr, _ = w1_trace(bw)
    check_tables(product_trace(host_ctx(), tr), O.Model(tr))


def test_trace_build_errors():
    ctx = host_ctx()
    with pytest.raises(chm.ChmError) as e:
        ctx.trace_build(0, 0, 1e9, 1, 1)
    assert e.value.code == chm.CHM_E_STATE  # no Detailed iteration yet
    tr = W.tiny()
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    with pytest.raises(chm.ChmError):
        ctx.trace_build(tr.budget, tr.static_bytes, 0.0, 6, 6)  # B must be > 0
    with pytest.raises(chm.ChmError):
        ctx.trace_build(tr.budget, tr.static_bytes, 1e9, 33, 6)  # more groups than FWD ops
    with pytest.raises(chm.ChmError):
        ctx.record_op(1, 1)
        ctx.record_op(1, 0)  # phases interleave
    with pytest.raises(chm.ChmError):
        ctx.record_op(0, 0)  # token 0 is reserved


def test_eval_and_swap_refused_on_host_ctx():
    ctx = host_ctx()
    tr = W.tiny()
    pt = product_trace(ctx, tr)
    with pytest.raises(chm.ChmError) as e:
        ctx.eval_policies(pt, chm.EXHAUSTIVE, 0, 1, best=0x1000)
    assert e.value.code == chm.CHM_E_STATE
    with pytest.raises(chm.ChmError):
        ctx.swap_out([(0x1000, 0, 16)])


def test_candidate_mask_decode():
    tr = W.tiny()
    ctx = host_ctx()
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    for c in (0, 5, 77777, (1 << 24) - 1):
        w = pt.candidate_mask(chm.EXHAUSTIVE, c)
        assert int(w[0]) == c
        w = pt.candidate_mask(chm.SEEDED, c, seed=9, flip_thr=1 << 62)
        bits = [(int(w[k // 64]) >> (k % 64)) & 1 for k in range(m.K)]
        t, r, s = m.mask_items(bits)
        ref = m.eval(O.SEEDED, c, 1, seed=9, flip_thr=1 << 62)
        assert m.replay(t, r, s, footprint=False)["peak"] == ref["peak"][0]
        assert int(sum(tr.nbytes[t])) == ref["swapped"][0]


def test_algo1_parity_and_detect_bytes():
    rng = np.random.default_rng(3)
    base = list(rng.integers(1, 40, size=300))
    for cos_mode in (0, 1):
        sm = O.StageMachine(2, 5, cos_mode=cos_mode)
        ctx = host_ctx(cos_mode=cos_mode)
        for it in range(80):
            seq = list(base)
            r = rng.random()
            if r < 0.12:
                seq += list(rng.integers(1, 40, size=int(rng.integers(10, 60))))
            elif r < 0.24:
                seq = seq[:len(seq) - int(rng.integers(1, 40))]
            elif r < 0.34:
                rng.shuffle(seq)
            for t in seq:
                ctx.record_op(int(t), 0)
            got = ctx.detect_seq_change(0.1)
            exp = sm.step(seq)
            assert (got["stage"], got["len_diff"], got["cos"]) == (exp["stage"], exp["len_diff"], exp["cos"])
    # C4 seq 2048 -> 8192: the 3 extra cross-entropy chunks add 27 ops (len_diff 1.4%).  The
    # positional cosine sees the shift of every later op (cos 0.938 < 0.95: change); the histogram
    # cosine does not (0.99990), so there only the opt-in byte signature (reading Q4) detects it.
    a, b = W.llama2_13b(2048), W.llama2_13b(8192)
    for cos_mode, detect_bytes, expect_change in ((0, 0, True), (1, 0, False), (1, 1, True)):
        ctx = host_ctx(detect_bytes=detect_bytes, cos_mode=cos_mode)
        for tr in (a, a, b):
            chm.record_iteration(ctx, tr)
            got = ctx.detect_seq_change(tr.t_iter)
        assert got["changed"] == expect_change
        assert got["len_diff"] < 0.05


def _install_all(ctx, pt):
    words = np.zeros(pt.W, np.uint64)
    for k in range(pt.K):
        words[k // 64] |= np.uint64(1 << (k % 64))
    ctx.policy_install(pt, words)


@pytest.mark.parametrize("name", ["C1", "C2", "C5"])
def test_executor_trigger_positions(name):
    """Installed policy = every swappable tensor; replaying the same iteration must fire swap-out
    right after a_t, release after r_t, swap-in before s_t and the wait
    before b_t, each exactly once (bijection)."""
    tr = W.CONFIGS[name]()
    m = O.Model(tr)
    ctx = host_ctx()
    pt = product_trace(ctx, tr)
    _install_all(ctx, pt)
    sw = m.swappable()
    p, f, a, b = m.tensor_table()
    ev = {"out": [], "rel": [], "in": []}

    def on(i, act):
        av = chm.actions_view(act)
        ev["out"] += [(i, it) for it in av["swap_out_item"]]
        ev["rel"] += [(i, it) for it in av["release"]]
        ev["in"] += [(i, it) for it in av["swap_in_item"]]
    chm.record_iteration(ctx, tr, on_actions=on)
    ctx.detect_seq_change(tr.t_iter)
    st = ctx.exec_stats()
    assert st["n_items"] == st["n_matched"] == pt.K and st["n_stale"] == 0
    assert sorted(ev["out"]) == sorted((int(a[sw["t"][k]]), k) for k in range(pt.K))
    assert sorted(ev["rel"]) == sorted((int(sw["r"][k]), k) for k in range(pt.K))
    assert sorted(ev["in"]) == sorted((int(sw["s"][k]) - 1, k) for k in range(pt.K))
    # (the waits before b_t need an issued swap-in batch, i.e. a device: tests/test_gpu_swap.py)


@pytest.mark.parametrize("where", ["opt_tail", "validation", "early_fwd"])
def test_executor_tolerates_minor_drift(where):
    """P:472 / S:330: minor sequence changes (skipped optimizer step, an inserted op) are absorbed
    by fuzzy matching: every item still matches."""
    tr = W.gpt2_xl()
    ctx = host_ctx()
    pt = product_trace(ctx, tr)
    _install_all(ctx, pt)
    tok = [ctx.tokenize(nm) for nm in tr.op_names]
    extra = ctx.tokenize("aten::_local_scalar_dense")
    n_fwd = int((tr.phase == 0).sum())
    matched = 0
    for i in range(tr.n_ops):
        if where == "early_fwd" and i == 3:
            ctx.record_op(extra, 0)  # inserted FWD op shifts every later index by one
        if where == "opt_tail" and tr.phase[i] == 2:
            break  # loss-scale overflow: optimizer step skipped
        ins = [(tr.ptr[t], tr.nbytes[t], tr.dtype[t]) for t in tr.ins(i)]
        outs = [(tr.ptr[t], tr.nbytes[t], tr.dtype[t]) for t in tr.outs(i)]
        act = ctx.record_op(tok[i], int(tr.phase[i]), ins, outs, [tr.ptr[t] for t in tr.frees(i)])
        matched += act.n_swap_out
    if where == "validation":
        for _ in range(20):  # on-the-fly validation appends ops
            ctx.record_op(extra, 2)
    assert matched == pt.K
    ctx.detect_seq_change(tr.t_iter)
    assert ctx.exec_stats()["n_stale"] == 0
    assert n_fwd > 0


@pytest.mark.parametrize("name,seed", [("C1", 0), ("C2", 1), ("C2", 2), ("C5", 3), ("C3", 4)])
def test_executor_partial_policy_swaps_exactly_the_selected_tensors(name, seed):
    """A random partial policy: every swap-out names the selected tensor's own storage (ids are
    reused data_ptrs, so resolve them against the live tensor at that op) -- no same-role tensor of
    a neighbouring layer or sibling output is swapped instead."""
    tr = W.CONFIGS[name]()
    m = O.Model(tr)
    ctx = host_ctx()
    pt = product_trace(ctx, tr)
    rng = np.random.default_rng(seed)
    words = np.zeros(pt.W, np.uint64)
    sel = sorted(rng.choice(pt.K, size=max(1, pt.K // 3), replace=False).tolist())
    for k in sel:
        words[k // 64] |= np.uint64(1 << (k % 64))
    ctx.policy_install(pt, words)
    sw = m.swappable()
    p, f, a, b = m.tensor_table()
    got = []

    def on(i, act):
        av = chm.actions_view(act)
        for (dev, off, nb), it in zip(av["swap_out"], av["swap_out_item"]):
            live = [t for t in range(tr.n_tensors) if int(tr.ptr[t]) == dev and p[t] <= i <= f[t] and p[t] >= 0]
            assert len(live) == 1
            got.append((i, it, live[0]))
    chm.record_iteration(ctx, tr, on_actions=on)
    exp = sorted((int(a[sw["t"][k]]), j, int(sw["t"][k])) for j, k in enumerate(sel))
    assert sorted(got) == exp


def test_c4_dynamic_schedule_detection():
    """C4: s 2048 (it 0-29) -> 8192 (30-59) -> 2048 (60-89) through the profiler hook.  Positional
    cosine (default) detects both switches; the stage machine then walks WarmUp (3 iterations) ->
    GenPolicy (6) -> Stable, as Algo. 1 with m = 2, n = 5 prescribes."""
    import json
    import subprocess
    import sys
    out = subprocess.run([sys.executable, "tools/c4_dynamic.py", "--host-only"], capture_output=True, text=True,
                         cwd=__import__("os").path.dirname(__import__("os").path.dirname(__file__)), timeout=300)
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["detections"] == [30, 60]
    st = d["stages"]
    for start in (0, 30, 60):
        off = 0 if start == 0 else 1  # the first call initialises PrevOpSeq (stable with itself)
        warm = 2 if start == 0 else 3
        assert st[start:start + warm] == [0] * warm
        assert st[start + warm:start + warm + 6] == [1] * 6
        assert st[start + warm + 6] == 2
        del off


@pytest.mark.parametrize("name", ["C2", "C3", "C4a", "C4b", "C5"])
def test_auto_groups_find_the_layer_count(name):
    """groups 0: each phase is split into its layer count, found from the token period (P:283-288
    -- the grouping estimate holds up to the model's layer count); equals the configured groups
    of the synthetic transformer traces, and the rest of the trace is the configured one's"""
    tr = W.CONFIGS[name]()
    ctx = host_ctx()
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    auto = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, 0, 0, t_iter=tr.t_iter)
    given = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    a, g = auto.tables(), given.tables()
    for k in a:
        assert np.array_equal(a[k], g[k]), k


def test_auto_groups_on_a_real_model_sequence():
    """the runtime's default (groups 0) on a 4-layer GPT: four FWD logical layers"""
    torch = pytest.importorskip("torch")
    from paper_2509_11076_b200.runtime import Runtime
    from workloads import tiny_gpt as G
    model = G.make(0, n_layer=4)
    opt = torch.optim.SGD(model.parameters(), lr=0.01)
    rt = Runtime(None, hbm_budget=1)
    for x, y in G.batches(6, 2, 16, 64):
        with rt.step():
            model(x, y).backward()
            opt.step()
            opt.zero_grad()
    assert rt.plans and rt.policy is not None
    assert rt.policy[0].L == 4 + 4 + 1  # 4 FWD + 4 BWD logical layers + the optimizer's group


def test_record_tokens_equals_per_op_records():
    """chm_record_tokens (bulk Lightweight mode) drives Algo. 1 exactly like chm_record_op per op"""
    rng = np.random.default_rng(11)
    base = rng.integers(1, 40, size=300).astype(np.int32)
    phases = np.array([0] * 120 + [1] * 170 + [2] * 10, np.uint8)
    a, b = host_ctx(), host_ctx()
    for it in range(14):
        seq = base if it < 8 else np.concatenate([base, base[:40]])  # a change at iteration 8
        ph = phases if it < 8 else np.concatenate([phases[:120], np.zeros(40, np.uint8), phases[120:]])
        for t, p in zip(seq, ph):
            a.record_op(int(t), int(p))
        b.record_tokens(seq, ph)
        assert a.detect_seq_change(1e-3) == b.detect_seq_change(1e-3)
    with pytest.raises(chm.ChmError):
        b.record_tokens([1, 0], [0, 0])  # token 0
    with pytest.raises(chm.ChmError):
        b.record_tokens([1, 2], [1, 0])  # interleaved phases
