"""Pins of the CPU oracle against values fixed by the paper, hand derivations, brute force
and invariants (not against itself).  -m "not gpu"."""
import math

import numpy as np
import pytest

import oracle as O
from tests.helpers import load_golden, make_trace, w1_trace
from workloads import traces as W


# ---------------------------------------------------------------- W1
def test_w1_b40_f0_layers_timing():
    g = load_golden("w1.json")
    tr, ix = w1_trace(40.0)
    m = O.Model(tr)
    assert m.f0().tolist() == g["F0"]
    st, n, ty, bud = m.layers()
    assert n.tolist() == [2] * 6 and ty.tolist() == [0, 0, 0, 1, 1, 1]
    assert bud.tolist() == [2.0] * 6  # Eq. 1: 12 / 12 * 2
    sw = m.swappable()
    exp = g["B40"]["swappable"]
    assert sw["t"].tolist() == [ix[e["tensor"]] for e in exp]
    assert sw["r"].tolist() == [e["r"] for e in exp]
    assert sw["s"].tolist() == [e["s"] for e in exp]


def test_w1_b40_all_masks_and_best():
    g = load_golden("w1.json")["B40"]
    tr, _ = w1_trace(40.0)
    m = O.Model(tr)
    res = m.eval(O.EXHAUSTIVE, 0, 4, footprint=True)
    for mask, e in g["masks"].items():
        c = int(mask)
        assert res["footprint"][c].tolist() == e["F"]
        assert res["peak"][c] == e["peak"]
        assert res["stall"][c] == e["stall"]
        key = (max(0, res["peak"][c] - tr.budget), res["stall"][c], res["swapped"][c], c)
        assert list(key) == e["key"]
    assert res["best"].index == g["best"]


def test_w1_b15_saturated_and_stall():
    g = load_golden("w1.json")["B15"]
    tr, ix = w1_trace(15.0)
    m = O.Model(tr)
    sw = m.swappable()
    assert m.K == 1 and sw["t"][0] == ix["X0"] and sw["r"][0] == 5 and sw["s"][0] == 8
    assert sw["saturated"][0] == 1
    res = m.eval(O.EXHAUSTIVE, 1, 1, footprint=True)
    e = g["masks"]["1"]
    assert res["footprint"][0].tolist() == e["F"]
    assert repr(float(res["stall"][0])) == e["stall_repr"]
    assert res["peak"][0] - tr.budget == e["key_excess"]


# ------------------------------------------------------------- SPEC worked examples
def _phase_trace(n_fwd, n_bwd, n_opt, t_iter, gf, gb, bw=1.0):
    n = n_fwd + n_bwd + n_opt
    ph = [0] * n_fwd + [1] * n_bwd + [2] * n_opt
    return make_trace(ph, [], [[]] * n, [[]] * n, [[]] * n, 0, t_iter, bw, 0, gf, gb)


def test_eq1_example_S222():
    # T_iter = 1000, N_iter = 400, a layer of 40 ops -> 100 (Eq. 1)
    m = O.Model(_phase_trace(400, 0, 0, 1000.0, 10, 1))
    st, n, ty, bud = m.layers()
    assert n.tolist() == [40] * 10 and bud.tolist() == [100.0] * 10


def test_near_even_split_S223():
    # 10 FWD ops into 3 groups -> 4, 3, 3
    m = O.Model(_phase_trace(10, 3, 2, 1.0, 3, 1))
    st, n, ty, bud = m.layers()
    assert n.tolist() == [4, 3, 3, 3, 2] and st.tolist() == [0, 4, 7, 10, 13]
    assert ty.tolist() == [0, 0, 0, 1, 2]


def _one_tensor_trace(size, n_fwd, bw, t_iter, n_bwd=3):
    """tensor produced at op 0 (FWD), first BWD use at the last BWD op."""
    n = n_fwd + n_bwd
    ins = [[] for _ in range(n)]
    outs = [[] for _ in range(n)]
    frees = [[] for _ in range(n)]
    outs[0] = [0]
    ins[n - 1] = [0]
    frees[n - 1] = [0]
    ph = [0] * n_fwd + [1] * n_bwd
    return make_trace(ph, [size], ins, outs, frees, 0, t_iter, bw, 0, 1, n_bwd)


def test_eq3_and_swapout_search_S250():
    # T_swap = S/B = 10 (Eq. 3).  FWD 4 ops in 2 layers, 2.5 per op -> budgets [5, 5]:
    # no layer has T_remaining > T_swap -> completion at the end of the last FWD layer and the
    # item is flagged saturated.  With near-even groups the FWD budgets never
    # increase, so the solo forward search ends in the own layer or saturates.
    tr = _one_tensor_trace(size=10 * 512, n_fwd=4, bw=512.0, t_iter=2.5 * 7)
    m = O.Model(tr, groups=(2, 3))
    st, n, ty, bud = m.layers()
    assert n.tolist()[:2] == [2, 2] and bud.tolist()[:2] == [5.0, 5.0]
    sw = m.swappable()
    assert sw["r"].tolist() == [3] and sw["saturated"].tolist() == [1]


def test_swapout_fits_own_layer_S251():
    # T_swap = 4 smaller than every budget -> completes in the layer of its last FWD use
    tr = _one_tensor_trace(size=4 * 512, n_fwd=4, bw=512.0, t_iter=2.5 * 7)
    sw = O.Model(tr, groups=(2, 3)).swappable()
    assert sw["r"].tolist() == [1] and sw["saturated"].tolist() == [0]


def test_eq3_2gib_16gibps():
    # 2 GiB at 16 GiB/s -> T_swap = 0.125 s.  A layer budget of exactly 0.125 does not
    # fit (strict >, reading Q10); 0.125 + one ulp does.
    G = 1 << 30
    for per_layer, exp_r, sat in ((0.125, 3, 1), (math.nextafter(0.125, 1), 1, 0)):
        tr = _one_tensor_trace(size=2 * G, n_fwd=4, bw=16.0 * G, t_iter=per_layer / 2 * 7)
        m = O.Model(tr, groups=(2, 3))
        assert m.layers()[3][0] == per_layer
        sw = m.swappable()
        assert sw["r"].tolist() == [exp_r] and sw["saturated"].tolist() == [sat]


def test_swapin_placement_previous_layer():
    # s_t = first op of the layer before the layer holding the first BWD use (Q8)
    tr = _one_tensor_trace(size=512, n_fwd=4, bw=512.0, t_iter=40.0)
    sw = O.Model(tr, groups=(2, 3)).swappable()
    # layers: F0={0,1}, F1={2,3}, B0={4}, B1={5}, B2={6}; b = 6 -> layer B2 -> s = start(B1) = 5
    assert sw["s"].tolist() == [5]


def test_mrl_example_S204():
    # usage [90, 110, 105, 95], budget 100 -> MRL {1: 10, 2: 5}; excess = 10
    ins = [[], [], [], []]
    outs = [[], [0], [1], [2]]
    frees = [[], [0], [1], []]
    tr = make_trace([0, 0, 0, 1], [20, 15, 5], ins, outs, frees, 90, 1.0, 1.0, 100, 1, 1)
    m = O.Model(tr)
    f0 = m.f0()
    assert f0.tolist() == [90, 110, 105, 95]
    mrl = {i: int(v - 100) for i, v in enumerate(f0) if v > 100}
    assert mrl == {1: 10, 2: 5}
    assert m.eval(O.EXHAUSTIVE, 0, 1)["best"].excess == 10


def test_reconstruction_S146():
    # measured 50 at op k with a 30 tensor swapped out before k, back after k -> 80
    out = O.reconstruct([50, 50, 50], [30], [0], [2])
    assert out.tolist() == [50, 80, 50]


# ------------------------------------------------- brute force vs an independent closed form
def _closed_form(tr, items):
    """F_P[i] = M_0 + sum_t S_t [p_t <= i <= f_t] - sum_{t in P} S_t [r_t < i < s_t]
    with p_t, f_t read straight from the raw records (SURVEY §8(c).2 closed form)."""
    N, T = tr.n_ops, tr.n_tensors
    p = np.full(T, -1)
    f = np.full(T, N)
    for i in range(N):
        for t in tr.outs(i):
            p[t] = i
        for t in tr.frees(i):
            f[t] = i
    i = np.arange(N)
    F = np.full(N, tr.static_bytes, np.int64)
    for t in range(T):
        if p[t] >= 0:
            F += tr.nbytes[t] * ((p[t] <= i) & (i <= f[t]))
        elif f[t] < N:  # static tensor released during the iteration
            F -= tr.nbytes[t] * (i > f[t])
    for (t, r, s) in items:
        F -= tr.nbytes[t] * ((r < i) & (i < s))
    return F


@pytest.mark.parametrize("seed", range(12))
def test_bruteforce_all_subsets_random_traces(seed):
    tr = W.random_trace(seed, n_layers=3 + seed % 2, ops_per_layer=3, bw=[1e6, 1e7, 1e8][seed % 3])
    m = O.Model(tr)
    K = m.K
    assert K <= 12
    sw = m.swappable()
    res = m.eval(O.EXHAUSTIVE, 0, 1 << K, footprint=True)
    keys = []
    for c in range(1 << K):
        items = [(sw["t"][k], sw["r"][k], sw["s"][k]) for k in range(K) if (c >> k) & 1]
        F = _closed_form(tr, items)
        assert np.array_equal(res["footprint"][c], F), c
        assert res["peak"][c] == F.max()
        assert res["swapped"][c] == sum(tr.nbytes[t] for t, _, _ in items)
        keys.append((max(0, int(F.max()) - tr.budget), float(res["stall"][c]), int(res["swapped"][c]), c))
    assert min(keys)[3] == res["best"].index
    # F_empty == F0
    assert np.array_equal(res["footprint"][0], m.f0())


@pytest.mark.parametrize("seed", range(6))
def test_invariants_additivity_monotonicity_conservation(seed):
    tr = W.random_trace(100 + seed, n_layers=4, ops_per_layer=3)
    m = O.Model(tr)
    K = m.K
    f0 = m.f0()
    sw = m.swappable()
    res = m.eval(O.EXHAUSTIVE, 0, 1 << K, footprint=True)
    F = res["footprint"]
    solo = {k: f0 - F[1 << k] for k in range(K)}
    for c in range(1 << K):
        # additivity: F0 - F_P = sum_{t in P} (F0 - F_{t})
        tot = sum((solo[k] for k in range(K) if (c >> k) & 1), np.zeros_like(f0))
        assert np.array_equal(f0 - F[c], tot)
        # conservation at the last op
        assert F[c][-1] == f0[-1]
        # monotonicity: adding an item never raises the footprint or lowers the stall
        for k in range(K):
            if not (c >> k) & 1:
                d = c | (1 << k)
                assert np.all(F[d] <= F[c])
                assert res["peak"][d] <= res["peak"][c]
                assert res["stall"][d] >= res["stall"][c]
    # live after the last op = M_0 + bytes of tensors that survive the iteration
    p, f, a, b = m.tensor_table()
    surv = sum(int(tr.nbytes[t]) for t in range(tr.n_tensors) if f[t] == tr.n_ops and p[t] >= 0)
    last = f0[-1] - sum(int(tr.nbytes[t]) for t in tr.frees(tr.n_ops - 1))
    assert last == tr.static_bytes + surv
    # Fig. 3 round trip: reconstruct(F_P, swap log) == F0
    for c in (0, (1 << K) - 1, (1 << K) // 3):
        sel = [k for k in range(K) if (c >> k) & 1]
        rec = O.reconstruct(F[c], tr.nbytes[sw["t"][sel]], sw["r"][sel], sw["s"][sel])
        assert np.array_equal(rec, f0)


def test_timing_invariants_on_configs():
    for name in ("C1", "C2", "C5"):
        tr = W.CONFIGS[name]()
        m = O.Model(tr)
        p, f, a, b = m.tensor_table()
        st, n, ty, bud = m.layers()
        lay = np.repeat(np.arange(m.L), n)
        sw = m.swappable()
        last_fwd = max(l for l in range(m.L) if ty[l] == 0)
        for k in range(m.K):
            t, r, s = sw["t"][k], sw["r"][k], sw["s"][k]
            assert p[t] >= 0 and a[t] >= p[t] and b[t] > a[t]
            assert r >= a[t] and r + 1 < s < b[t]
            assert r == st[lay[r]] + n[lay[r]] - 1  # release after the last op of a layer
            assert s == st[lay[b[t]] - 1]  # previous layer of the first BWD use
            tsw = tr.nbytes[t] / tr.bw
            for l in range(lay[a[t]], lay[r]):
                assert not bud[l] > tsw
            if sw["saturated"][k]:
                assert lay[r] == last_fwd and not bud[lay[r]] > tsw
            else:
                assert bud[lay[r]] > tsw
        # mask-bit order: ascending (a_t, t)
        order = [(a[t], t) for t in sw["t"]]
        assert order == sorted(order)


def test_stall_single_item_closed_form():
    tr, ix = w1_trace(15.0)
    m = O.Model(tr)
    sw = m.swappable()
    st, n, ty, bud = m.layers()
    S = 40
    exp = max(0.0, S / 15.0 - bud[4]) + max(0.0, S / 15.0 - bud[2])
    assert m.stall([ix["X0"]], [5], [8]) == exp


# ------------------------------------------------------------------ candidates / argmin
def test_splitmix64_reference_vectors():
    # Vigna's splitmix64 from state 0: outputs mix(0), mix(golden), mix(2*golden) ...
    g = 0x9E3779B97F4A7C15
    assert O.splitmix64(0) == 0xE220A8397B1DCDAF
    assert O.splitmix64(g) == 0x6E789E6AA1B965F4
    assert O.splitmix64((2 * g) % 2 ** 64) == 0x06C45D188009454F


def test_seeded_bits_and_masks_agree():
    tr = W.tiny()
    m = O.Model(tr)
    K, Wd = m.K, m.W
    base = m.base_mask()
    seed, thr = 7, int(0.3 * 2 ** 64)
    res = m.eval(O.SEEDED, 5, 50, seed=seed, flip_thr=thr, words=base)
    masks = np.zeros((50, Wd), np.uint64)
    J = (K + 3) // 4
    for j in range(50):
        c = 5 + j
        for k in range(K):
            w = O.splitmix64(seed ^ ((c * J + k // 4) % 2 ** 64))
            field = (w >> (16 * (k % 4))) & 0xFFFF
            bit = int((int(base[k // 64]) >> (k % 64)) & 1) ^ int(field < (thr >> 48))
            if bit:
                masks[j, k // 64] |= np.uint64(1 << (k % 64))
    res2 = m.eval(O.MASKS, 5, 50, words=masks)
    assert np.array_equal(res["peak"], res2["peak"]) and np.array_equal(res["stall"], res2["stall"])
    assert res["best"].key() == res2["best"].key()


def _mix_np(z):
    # splitmix64's finaliser, vectorised (wrapping uint64), checked against the oracle's below
    z = z + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


@pytest.mark.parametrize("p", [0.02, 0.3])
def test_seeded_flip_statistics(p):
    """reading R-seeded draws one splitmix64 finaliser per 4 items, w = mix(seed ^ (c J + q)):
    over 20,000 candidates x 120 words the 16-bit fields fall below flip_thr >> 48 at rate p
    (within 5 standard errors), and flips of neighbouring fields, words and candidates are
    uncorrelated (|r| < 0.01) -- the counter's structure does not leak through the finaliser"""
    seed, J, n = 0x5EED, 120, 20_000
    with np.errstate(over="ignore"):
        ctr = (np.arange(n, dtype=np.uint64)[:, None] * np.uint64(J) + np.arange(J, dtype=np.uint64)[None, :])
        w = _mix_np(np.uint64(seed) ^ ctr)
    assert all(int(w[c, q]) == O.splitmix64(seed ^ (c * J + q)) for c, q in ((0, 0), (17, 3), (n - 1, J - 1)))
    thr = int(p * 2 ** 16)
    f = np.stack([((w >> np.uint64(16 * e)) & np.uint64(0xFFFF)) < np.uint64(thr) for e in range(4)], axis=-1)
    f = f.reshape(n, 4 * J).astype(np.float64)
    rate, q16 = f.mean(), thr / 2 ** 16
    assert abs(rate - q16) < 5 * np.sqrt(q16 * (1 - q16) / f.size), (rate, q16)
    for a, b in ((f[:, :-1], f[:, 1:]), (f[:, :-4], f[:, 4:]), (f[:-1, :], f[1:, :])):
        r = np.corrcoef(a.ravel(), b.ravel())[0, 1]
        assert abs(r) < 0.01, r


def test_default_base_mask_contains_argmax():
    tr = W.tiny()
    m = O.Model(tr)
    f0 = m.f0()
    imax = int(np.argmax(f0))
    sw = m.swappable()
    base = m.base_mask()
    for k in range(m.K):
        bit = (int(base[k // 64]) >> (k % 64)) & 1
        assert bit == int(sw["r"][k] < imax < sw["s"][k])


# ------------------------------------------------------------------------------ Algo. 1
def test_algo1_derived_sequence_m2_n5():
    sm = O.StageMachine(2, 5)
    seq = [1, 2, 3, 2, 1]
    stages = [sm.step(seq)["stage"] for _ in range(12)]
    assert stages == [0, 0] + [1] * 6 + [2] * 4


def test_algo1_change_resets_to_warmup_S137():
    sm = O.StageMachine(2, 5)
    seq = list(range(1, 101))
    for _ in range(10):
        sm.step(seq)
    r = sm.step(seq + list(range(1, 11)))  # 10% longer
    assert r["stage"] == O.WARMUP and r["stable_step"] == 0 and not r["stable"]


def _algo1_table(stage, step, stable, m, n):
    """Algo. 1 transcribed as a transition table, reading Q3."""
    if not stable:
        return 0, 0
    step += 1
    if stage == 0 and step > m:
        return 1, 0
    if stage == 1 and step > n:
        return 2, step
    return stage, step


def test_algo1_exhaustive_table_S494():
    m, n = 2, 5
    A, B = [1, 2, 3, 4] * 10, [4, 3, 2, 1] * 10  # cos(A, B) = 0.667 -> changed
    for stage in range(3):
        for step in range(n + 3):
            for stable in (True, False):
                sm = O.StageMachine(m, n)
                sm.step(A)  # initialise PrevOpSeq
                sm._st.prev_stage = stage
                sm._st.stable_step = step
                r = sm.step(A if stable else B)
                exp = _algo1_table(stage, step, stable, m, n)
                assert (r["stage"], r["stable_step"]) == exp, (stage, step, stable)
                assert not (stage == 0 and r["stage"] == 2)  # never WarmUp -> Stable


def test_cosine_examples_S127_S129():
    assert O.compare([1, 2, 3], [1, 2, 3]) == (0.0, 1.0)
    ld, cs = O.compare([1, 2, 3], [1, 2, 3, 4])
    assert ld == 0.25 and cs == 14 / math.sqrt(14 * 30)
    ld, cs = O.compare([1, 1, 2, 2], [1, 1, 2], cos_mode=1)
    assert cs == 6 / (math.sqrt(8) * math.sqrt(5))
    with pytest.raises(ValueError):
        O.compare([], [1])


def test_tokenize_first_appearance_S71():
    tok, table = O.tokenize(["matmul", "add", "matmul"])
    assert tok.tolist() == [1, 2, 1]


# ------------------------------------------------------------------------ App. A features
def test_feature_callstack_S311_S313():
    # 40 distinct ops, op k appears (41 - k) times -> rank k; op index = rank + 1
    names = []
    for k in range(40):
        names += [f"op{k}"] * (41 - k)
    tok, table = O.tokenize(names)
    idx, oh = O.feature_tables(tok)
    for k in range(40):
        assert idx[table[f"op{k}"]] == k + 1
        assert oh[table[f"op{k}"]] == ((1 << k) if k < 32 else 0)
    # stack 0 -> 0x2A -> 0x2A11 (ops with index 0x2A = 42 and 0x11 = 17); build a trace
    # whose tensor 0 is used by an op of index 42 then an op of index 17
    tok2 = np.zeros(3, np.int32)
    idx2 = np.zeros(4, np.uint8)
    oh2 = np.zeros(4, np.uint32)
    idx2[1], idx2[2], idx2[3] = 0x2A, 0x11, 0x05
    oh2[2] = 1 << 3  # op token 2 is in the top 32; tokens 1, 3 are not
    tok2[:] = [1, 2, 3]
    tr = make_trace([0, 0, 0], [512], [[], [0], [0]], [[0], [], []], [[], [], [0]], 0, 1.0, 1.0, 0, 1, 1)
    c, tag, stk = O.features_after(tr, tok2, idx2, oh2, 0)
    assert stk[0] == 0x2A and c[0] == 1 and tag[0] == 0  # non-top-32 leaves the tag
    c, tag, stk = O.features_after(tr, tok2, idx2, oh2, 1)
    assert stk[0] == 0x2A11 and c[0] == 2 and tag[0] == 1 << 3
    # 9 uses shift the first entry out of the 64-bit stack
    n = 9
    tr9 = make_trace([0] * n, [512], [[]] + [[0]] * (n - 1), [[0]] + [[]] * (n - 1),
                     [[]] * (n - 1) + [[0]], 0, 1.0, 1.0, 0, 1, 1)
    tok9 = np.arange(1, n + 1, dtype=np.int32)
    idx9 = np.arange(0, n + 1, dtype=np.uint8) + 0x10
    c, tag, stk = O.features_after(tr9, tok9, idx9, np.zeros(n + 1, np.uint32), n - 1)
    exp = 0
    for i in range(n):
        exp = ((exp << 8) + int(idx9[tok9[i]])) % 2 ** 64
    assert int(stk[0]) == exp and c[0] == n
    assert (int(stk[0]) >> 56) == int(idx9[tok9[1]])  # first use (0x11) shifted out


def test_stall_pairwise_within_error_bound_of_exact_sum():
    """R-stall: the stall is the pairwise sum of max(0, load_l/B - Bud_l).  Pin it to the exactly
    rounded sum of those terms (math.fsum) within pairwise summation's error bound
    gamma_{log2 P} * sum|t| (Higham, Accuracy and Stability, §4.2) on traces with many layers."""
    for seed in range(6):
        tr = W.random_trace(200 + seed, n_layers=6, ops_per_layer=4, bw=1e5)
        m = O.Model(tr)
        st, n, ty, bud = m.layers()
        sw = m.swappable()
        lay = np.repeat(np.arange(m.L), n)
        for c in range(1, 1 << min(m.K, 8)):
            sel = [k for k in range(m.K) if (c >> k) & 1]
            t, r, s = sw["t"][sel], sw["r"][sel], sw["s"][sel]
            load = np.zeros(m.L, np.int64)
            for tt, rr, ss in zip(t, r, s):
                load[lay[ss]] += tr.nbytes[tt]
                load[lay[rr]] += tr.nbytes[tt]
            terms = [max(0.0, float(load[l]) / tr.bw - bud[l]) for l in range(m.L)]
            exact = math.fsum(terms)
            got = m.stall(t, r, s)
            P = 1 << (m.L - 1).bit_length()
            u = 2.0 ** -53
            k = P.bit_length() - 1
            bound = k * u / (1 - k * u) * sum(terms)
            assert abs(got - exact) <= bound + 1e-300


def test_seeded_flip_rate():
    """R-seeded: the flip probability is (flip_thr >> 48) / 2^16 per item."""
    tr = W.gpt2_xl()
    m = O.Model(tr)
    base = m.base_mask()
    thr = int(0.02 * 2 ** 64)
    res = m.eval(O.SEEDED, 0, 400, seed=2, flip_thr=thr, words=np.zeros_like(base), nthreads=4)
    p_hat = res["swapped"].sum() / (400 * tr.nbytes[m.swappable()["t"]].sum())
    # swapped-bytes-weighted rate is an unbiased estimate of the flip probability
    assert abs(p_hat - (thr >> 48) / 65536) < 0.004
