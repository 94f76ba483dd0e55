"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, element by element,
on the same seeded inputs.  Bar (BASELINE.json north_star): footprints, peak, swapped bytes and
argmin bit-exact; stall within 1e-6 relative (we also assert bit-equality, which the fixed-order
IEEE evaluation on both sides gives)."""
import numpy as np
import pytest

import oracle as O
from tests.helpers import w1_trace
from workloads import traces as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2509_11076_b200 import chm  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    c = chm.Context(device=0, host_arena_bytes=64 << 20)
    yield c
    c.close()


def product_trace(ctx, tr, budget=None):
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    ctx.set_detailed(False)
    return ctx.trace_build(tr.budget if budget is None else budget, tr.static_bytes, tr.bw, tr.groups_fwd,
                           tr.groups_bwd, t_iter=tr.t_iter, omega=tr.omega)


def check_trace_tables(pt, m):
    tb = pt.tables()
    assert (pt.N, pt.K, pt.L) == (m.N, m.K, m.L)
    assert np.array_equal(tb["f0"], m.f0())
    sw = m.swappable()
    assert np.array_equal(tb["tensor"].astype(np.int64), sw["t"])
    for k in ("r", "s", "lin", "lout"):
        assert np.array_equal(tb[k], sw[k]), k
    st, n, ty, bud = m.layers()
    assert np.array_equal(tb["lay_start"], st) and np.array_equal(tb["lay_count"], n)
    assert np.array_equal(tb["bud"], bud)  # bit-exact doubles (Eq. 1 evaluated in the same order)
    assert np.array_equal(tb["base"], m.base_mask())
    assert pt.peak0 == m.f0().max()


def run_eval(ctx, pt, kind, first, count, footprint=False, **kw):
    dev = torch.device("cuda:0")
    peak = torch.empty(count, dtype=torch.int64, device=dev)
    stall = torch.empty(count, dtype=torch.float64, device=dev)
    swapped = torch.empty(count, dtype=torch.int64, device=dev)
    best = torch.empty(5, dtype=torch.int64, device=dev)
    ld = (pt.N + 1) // 2 * 2
    fp = torch.empty((count, ld), dtype=torch.int64, device=dev) if footprint else None
    ctx.eval_policies(pt, kind, first, count, best=best, peak=peak, stall=stall, swapped=swapped, footprint=fp,
                      ld=ld if footprint else 0, **kw)
    torch.cuda.synchronize()
    b = best.cpu().numpy().view(chm.BEST_DTYPE)[0]
    return dict(peak=peak.cpu().numpy(), stall=stall.cpu().numpy(), swapped=swapped.cpu().numpy(),
                footprint=fp[:, :pt.N].cpu().numpy() if footprint else None, best=b)


def assert_same(res, ref, budget):
    assert np.array_equal(res["peak"], ref["peak"])
    assert np.array_equal(res["swapped"], ref["swapped"])
    np.testing.assert_allclose(res["stall"], ref["stall"], rtol=1e-6, atol=0)
    assert np.array_equal(res["stall"], ref["stall"])  # fixed-order IEEE: bit-identical
    if ref.get("footprint") is not None and res.get("footprint") is not None:
        assert np.array_equal(res["footprint"], ref["footprint"])
    rb, ob = res["best"], ref["best"]
    assert (int(rb["excess"]), float(rb["stall"]), int(rb["swapped_bytes"]), int(rb["index"])) == ob.key()
    assert int(rb["peak"]) == ob.peak


# ------------------------------------------------------------------------ trace build
@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C5"])
def test_trace_build_matches_oracle(ctx, name):
    tr = W.CONFIGS[name]()
    check_trace_tables(product_trace(ctx, tr), O.Model(tr))


@pytest.mark.parametrize("seed", range(8))
def test_trace_build_random(ctx, seed):
    tr = W.random_trace(seed, n_layers=3 + seed % 3, ops_per_layer=2 + seed % 3, bw=[1e6, 1e7, 1e8][seed % 3])
    check_trace_tables(product_trace(ctx, tr), O.Model(tr))


# ---------------------------------------------------------------------------- eval
@pytest.mark.parametrize("bw,scale", [(40.0, 1), (15.0, 1), (40.0, (1 << 28) + 1)])
def test_w1_all_masks(ctx, bw, scale):
    # scale 2^28 + 1: F0 up to 200 * (2^28 + 1) B, not a multiple of 8 -> the kernel's wide
    # (int64) F0 path; scale 1 exercises the narrow path with a 4 B unit
    tr, _ = w1_trace(bw, scale=scale)
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    check_trace_tables(pt, m)
    n = 1 << m.K
    assert_same(run_eval(ctx, pt, chm.EXHAUSTIVE, 0, n, footprint=True),
                m.eval(O.EXHAUSTIVE, 0, n, footprint=True), tr.budget)


@pytest.mark.parametrize("seed", range(6))
def test_random_traces_exhaustive(ctx, seed):
    tr = W.random_trace(50 + seed, n_layers=4, ops_per_layer=3, bw=[1e6, 1e7][seed % 2])
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    n = 1 << m.K
    assert_same(run_eval(ctx, pt, chm.EXHAUSTIVE, 0, n, footprint=True),
                m.eval(O.EXHAUSTIVE, 0, n, footprint=True), tr.budget)


def test_c1_exhaustive_all_subsets(ctx):
    """C1: all 2^K subsets (K = 24), search mode, vs the oracle's brute force."""
    tr = W.tiny()
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    n = 1 << m.K
    res = run_eval(ctx, pt, chm.EXHAUSTIVE, 0, n)
    ref = m.eval(O.EXHAUSTIVE, 0, n, nthreads=16)
    assert_same(res, ref, tr.budget)


def test_c1_exhaustive_footprints_ragged_window(ctx):
    tr = W.tiny()
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    first, count = 9_876_543, 3001  # ragged tail, arbitrary offset
    assert_same(run_eval(ctx, pt, chm.EXHAUSTIVE, first, count, footprint=True),
                m.eval(O.EXHAUSTIVE, first, count, footprint=True), tr.budget)


@pytest.mark.parametrize("name", ["C2", "C5"])
def test_seeded_footprints(ctx, name):
    tr = W.CONFIGS[name]()
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    sd = W.SEEDED[name[:2]]
    res = run_eval(ctx, pt, chm.SEEDED, 17, 1500, footprint=True, seed=sd["seed"], flip_thr=sd["flip_thr"])
    ref = m.eval(O.SEEDED, 17, 1500, seed=sd["seed"], flip_thr=sd["flip_thr"], footprint=True, nthreads=8)
    assert_same(res, ref, tr.budget)


def test_seeded_custom_base_and_masks(ctx):
    tr = W.gpt2_xl()
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    rng = np.random.default_rng(5)
    base = rng.integers(0, 2 ** 63, size=m.W, dtype=np.int64).astype(np.uint64)
    thr = int(0.3 * 2 ** 64)
    res = run_eval(ctx, pt, chm.SEEDED, 0, 700, footprint=True, seed=11, flip_thr=thr, base=base)
    ref = m.eval(O.SEEDED, 0, 700, seed=11, flip_thr=thr, words=base, footprint=True, nthreads=8)
    assert_same(res, ref, tr.budget)
    masks = rng.integers(0, 2 ** 63, size=(500, m.W), dtype=np.int64).astype(np.uint64)
    if m.K % 64:
        masks[:, -1] &= np.uint64((1 << (m.K % 64)) - 1)
    dmask = torch.from_numpy(masks.view(np.int64)).cuda()
    res = run_eval(ctx, pt, chm.MASKS, 1000, 500, footprint=True, masks=dmask)
    ref = m.eval(O.MASKS, 1000, 500, words=masks, footprint=True, nthreads=8)
    assert_same(res, ref, tr.budget)


@pytest.mark.parametrize("name", ["C2", "C3h"])
def test_bench_size_full_compare(ctx, name):
    """The launches bench.py times at full size (10^5 SEEDED candidates: C3h, the headline line's
    workload, and C2, its block), every candidate's peak / stall / swapped and the argmin against
    the oracle; footprints on a sample one by one, then every row element by element."""
    tr = W.CONFIGS[name]()
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    sd = W.SEEDED[name[:2]]
    n = 100_000
    res = run_eval(ctx, pt, chm.SEEDED, 0, n, seed=sd["seed"], flip_thr=sd["flip_thr"])
    ref = m.eval(O.SEEDED, 0, n, seed=sd["seed"], flip_thr=sd["flip_thr"], nthreads=16)
    assert_same(res, ref, tr.budget)
    full = run_eval(ctx, pt, chm.SEEDED, 0, n, footprint=True, seed=sd["seed"], flip_thr=sd["flip_thr"])
    assert np.array_equal(full["peak"], ref["peak"])
    rng = np.random.default_rng(0)
    for c in rng.choice(n, size=64, replace=False):
        one = m.eval(O.SEEDED, int(c), 1, seed=sd["seed"], flip_thr=sd["flip_thr"], footprint=True)
        assert np.array_equal(full["footprint"][c], one["footprint"][0])
    # and every footprint row of the launch (C2 2.1 GB, C3h 1.26 GB), element by element
    ref_full = m.eval(O.SEEDED, 0, n, seed=sd["seed"], flip_thr=sd["flip_thr"], footprint=True, nthreads=16)
    assert np.array_equal(full["footprint"], ref_full["footprint"])


@pytest.mark.parametrize("name", ["C3", "C4a", "C4b", "C5"])
def test_full_size_configs_all_keys_sampled_rows(ctx, name):
    """BASELINE configs C3-C5 at full size: 10^5 SEEDED candidates (the bench's launch), every
    key vs the oracle, footprint rows on a sample computed one by one"""
    tr = W.CONFIGS[name]()
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    sd = W.SEEDED[name[:2]]
    n = 100_000
    full = run_eval(ctx, pt, chm.SEEDED, 0, n, footprint=True, seed=sd["seed"], flip_thr=sd["flip_thr"])
    ref = m.eval(O.SEEDED, 0, n, seed=sd["seed"], flip_thr=sd["flip_thr"], nthreads=16)
    assert_same(dict(full, footprint=None), ref, tr.budget)
    rng = np.random.default_rng(1)
    for c in rng.choice(n, size=24, replace=False):
        one = m.eval(O.SEEDED, int(c), 1, seed=sd["seed"], flip_thr=sd["flip_thr"], footprint=True)
        assert np.array_equal(full["footprint"][c], one["footprint"][0])


@pytest.mark.parametrize("name", ["C1", "C2", "C5"])
def test_flip1_neighbourhood_matches_oracle_masks(ctx, name):
    """FLIP1 (the descent's candidates): candidate g = base with bit g flipped, g = K the base --
    equal to the oracle's MASKS replay of those masks, every key and footprint row"""
    tr = W.CONFIGS[name]()
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    rng = np.random.default_rng(3)
    base = np.zeros(m.W, np.uint64)
    for k in np.nonzero(rng.random(m.K) < 0.4)[0]:
        base[k // 64] |= np.uint64(1 << int(k % 64))
    n = m.K + 1
    res = run_eval(ctx, pt, chm.FLIP1, 0, n, footprint=True, base=base)
    masks = np.repeat(base[None, :], n, axis=0)
    for g in range(m.K):
        masks[g, g // 64] ^= np.uint64(1 << (g % 64))
    ref = m.eval(O.MASKS, 0, n, words=masks, footprint=True, nthreads=8)
    assert_same(res, ref, tr.budget)
    for g in (0, m.K // 2, m.K):
        assert np.array_equal(pt.candidate_mask(chm.FLIP1, g, base=base), masks[g])
    with pytest.raises(chm.ChmError):
        run_eval(ctx, pt, chm.FLIP1, 1, n, base=base)  # past K + 1 candidates


def test_candidate_mask_matches_oracle_decode(ctx):
    tr = W.tiny()
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    sw = m.swappable()
    for c in (0, 1, 12345, 2 ** 24 - 1):
        w = pt.candidate_mask(chm.SEEDED, c, seed=3, flip_thr=2 ** 62)
        bits = [(int(w[k // 64]) >> (k % 64)) & 1 for k in range(m.K)]
        t, r, s = m.mask_items(bits)
        one = m.eval(O.SEEDED, c, 1, seed=3, flip_thr=2 ** 62)
        assert m.replay(t, r, s, footprint=False)["peak"] == one["peak"][0]


# --------------------------------------------------------------------------- Algo. 1
def test_algo1_parity_random_schedule(ctx):
    rng = np.random.default_rng(7)
    base = list(rng.integers(1, 30, size=200))
    sm = O.StageMachine(2, 5)
    c = chm.Context(device=0)
    for it in range(60):
        seq = list(base)
        r = rng.random()
        if r < 0.15:
            seq = seq + list(rng.integers(1, 30, size=int(rng.integers(5, 40))))
        elif r < 0.25:
            seq = seq[: len(seq) - int(rng.integers(1, 30))]
        elif r < 0.35:
            k = int(rng.integers(0, len(seq)))
            seq[k] = int(rng.integers(1, 30))
        for t in seq:
            c.record_op(int(t), 0)
        got = c.detect_seq_change(0.1)
        exp = sm.step(seq)
        assert got["stage"] == exp["stage"], it
        assert got["len_diff"] == exp["len_diff"] and got["cos"] == exp["cos"]
        assert got["changed"] == (not exp["stable"])
    c.close()


# ------------------------------------------------------------------- EXPLICIT (NEXT-1)
def run_explicit(ctx, pt, lists, footprint=True):
    dev = torch.device("cuda:0")
    n = len(lists)
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum([len(x) for x in lists])
    items = np.concatenate([np.asarray(x, chm.ITEM_DTYPE) for x in lists] + [np.zeros(0, chm.ITEM_DTYPE)])
    peak = torch.empty(n, dtype=torch.int64, device=dev)
    stall = torch.empty(n, dtype=torch.float64, device=dev)
    swapped = torch.empty(n, dtype=torch.int64, device=dev)
    best = torch.empty(5, dtype=torch.int64, device=dev)
    ld = (pt.N + 1) // 2 * 2
    fp = torch.empty((n, ld), dtype=torch.int64, device=dev) if footprint else None
    ctx.eval_policies(pt, chm.EXPLICIT, 0, n, best=best, peak=peak, stall=stall, swapped=swapped, footprint=fp,
                      ld=ld if footprint else 0, item_offsets=off, items=items)
    torch.cuda.synchronize()
    return dict(peak=peak.cpu().numpy(), stall=stall.cpu().numpy(), swapped=swapped.cpu().numpy(),
                footprint=fp[:, :pt.N].cpu().numpy() if footprint else None,
                best=best.cpu().numpy().view(chm.BEST_DTYPE)[0])


@pytest.mark.parametrize("name", ["C1", "C2", "C5"])
def test_explicit_generator_policies(ctx, name):
    """best-of-n over Algo. 2 policies for a grid of (C, rem_scale): GPU replay of the
    EXPLICIT item lists vs the oracle's event replay, bit-exact."""
    tr = W.CONFIGS[name]()
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    lists, ref_lists = [], []
    for C_coef in (0.0, 0.5, 1.0, 2.0):
        for rem in (0.5, 1.0, 2.0):
            items, _ = pt.generate_policy(C_coef, rem)
            lists.append(items)
            ref_lists.append((items["t"].astype(np.int32), items["r"], items["s"]))
    res = run_explicit(ctx, pt, lists)
    ref = O.eval_explicit(m, ref_lists, footprint=True)
    assert_same(res, ref, tr.budget)


def test_explicit_random_windows_and_empty(ctx):
    tr = W.gpt2_xl()
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    p, f, a, b = m.tensor_table()
    rng = np.random.default_rng(4)
    acts = [t for t in range(tr.n_produced) if a[t] >= 0 and b[t] >= 0 and b[t] - a[t] >= 3]
    lists, ref_lists = [], []
    for c in range(40):
        sel = rng.choice(acts, size=int(rng.integers(0, 60)), replace=False)
        its = []
        for t in sel:
            r = int(rng.integers(a[t], b[t] - 1))
            s = int(rng.integers(r + 2, b[t] + 1))
            its.append((t, r, s, 0))
        arr = np.array(its, chm.ITEM_DTYPE) if its else np.zeros(0, chm.ITEM_DTYPE)
        lists.append(arr)
        ref_lists.append((arr["t"].astype(np.int32), arr["r"], arr["s"]))
    res = run_explicit(ctx, pt, lists)
    ref = O.eval_explicit(m, ref_lists, footprint=True)
    assert_same(res, ref, tr.budget)


def test_explicit_validation_error_index(ctx):
    tr = W.tiny()
    pt = product_trace(ctx, tr)
    items, _ = pt.generate_policy(1.0, 1.0)
    bad = items.copy()
    bad["r"][1] = bad["s"][1]  # r + 1 < s violated on item 1
    with pytest.raises(chm.ChmError) as e:
        run_explicit(ctx, pt, [items, bad])
    assert e.value.code == chm.CHM_E_INVAL and e.value.index == len(items) + 1
