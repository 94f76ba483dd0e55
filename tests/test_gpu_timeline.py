"""GPU parity of the timeline stall model in the search (chm_eval_out.stall_model =
CHM_STALL_TIMELINE, csrc/timeline.cu) against the oracle's orc_eval_model(stall_model = 1), which
scores each candidate's items with orc_stall_timeline (reading Q11's max-plus serial-stream
variant, pinned in tests/test_stall_models.py).  Bar: peak, swapped, footprints and the argmin
bit-exact; the stall within 1e-6 relative (asserted bit-identical: same IEEE operations in the
same order on both sides)."""
import numpy as np
import pytest

import oracle as O
from workloads import traces as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2509_11076_b200 import chm  # noqa: E402
from tests.test_gpu_parity import assert_same, product_trace, run_eval  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    c = chm.Context(device=0)
    yield c
    c.close()


def tl(ctx, pt, kind, first, count, **kw):
    return run_eval(ctx, pt, kind, first, count, stall_model=chm.STALL_TIMELINE, **kw)


def test_c1_exhaustive_all_subsets_prefix(ctx):
    tr = W.tiny()
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    n = 1 << 16
    res = tl(ctx, pt, chm.EXHAUSTIVE, 0, n, footprint=True)
    ref = m.eval(O.EXHAUSTIVE, 0, n, footprint=True, nthreads=8, stall_model=1)
    assert_same(res, ref, tr.budget)
    assert np.count_nonzero(ref["stall"]) > n // 10  # the model is exercised, not all zeros
    # the layer model's outputs other than the stall are unchanged
    lay = run_eval(ctx, pt, chm.EXHAUSTIVE, 0, n, footprint=True)
    assert np.array_equal(lay["peak"], res["peak"]) and np.array_equal(lay["footprint"], res["footprint"])


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C5"])
def test_seeded(ctx, name):
    tr = W.CONFIGS[name]()
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    sd = W.SEEDED[name[:2]]
    res = tl(ctx, pt, chm.SEEDED, 29, 1200, seed=sd["seed"], flip_thr=sd["flip_thr"])
    ref = m.eval(O.SEEDED, 29, 1200, seed=sd["seed"], flip_thr=sd["flip_thr"], nthreads=16, stall_model=1)
    assert_same(res, ref, tr.budget)


def test_masks_and_flip1_dense(ctx):
    """random dense masks (many items in flight: the slot colouring under load) and FLIP1"""
    tr = W.gpt2_xl()
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    rng = np.random.default_rng(8)
    for density in (0.1, 0.5, 0.95):
        masks = np.zeros((300, m.W), np.uint64)
        for i in range(300):
            for k in np.nonzero(rng.random(m.K) < density)[0]:
                masks[i, k // 64] |= np.uint64(1 << int(k % 64))
        dmask = torch.from_numpy(masks.view(np.int64)).cuda()
        res = tl(ctx, pt, chm.MASKS, 7, 300, masks=dmask)
        ref = m.eval(O.MASKS, 7, 300, words=masks, nthreads=16, stall_model=1)
        assert_same(res, ref, tr.budget)
    base = masks[0]
    n = m.K + 1
    res = tl(ctx, pt, chm.FLIP1, 0, n, base=base)
    fm = np.repeat(base[None, :], n, axis=0)
    for g in range(m.K):
        fm[g, g // 64] ^= np.uint64(1 << (g % 64))
    ref = m.eval(O.MASKS, 0, n, words=fm, nthreads=16, stall_model=1)
    assert_same(res, ref, tr.budget)


@pytest.mark.parametrize("name", ["C2", "C5"])
def test_bench_size_every_candidate(ctx, name):
    """the bench's launch size (10^5 SEEDED candidates, full mode) on C2 and on C5 (the per-rank
    trace of the 8-GPU config): every stall and the argmin"""
    tr = W.CONFIGS[name]()
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    sd = W.SEEDED[name]
    n = 100_000
    res = tl(ctx, pt, chm.SEEDED, 0, n, footprint=True, seed=sd["seed"], flip_thr=sd["flip_thr"])
    ref = m.eval(O.SEEDED, 0, n, seed=sd["seed"], flip_thr=sd["flip_thr"], nthreads=16, stall_model=1)
    res["footprint"] = None
    assert_same(res, ref, tr.budget)


def test_outputs_optional_and_errors(ctx):
    """peak / swapped / stall may be omitted (internal scratch); EXPLICIT and unknown models fail"""
    tr = W.tiny()
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    best = torch.empty(5, dtype=torch.int64, device="cuda")
    ctx.eval_policies(pt, chm.EXHAUSTIVE, 100, 5000, best=best, stall_model=chm.STALL_TIMELINE)
    torch.cuda.synchronize()
    b = best.cpu().numpy().view(chm.BEST_DTYPE)[0]
    ref = m.eval(O.EXHAUSTIVE, 100, 5000, nthreads=8, stall_model=1)["best"]
    assert (int(b["excess"]), float(b["stall"]), int(b["swapped_bytes"]), int(b["index"])) == ref.key()
    with pytest.raises(chm.ChmError):
        ctx.eval_policies(pt, chm.EXPLICIT, 0, 1, best=best, item_offsets=np.array([0, 0], np.uint64),
                          items=np.zeros(0, chm.ITEM_DTYPE), stall_model=chm.STALL_TIMELINE)
    with pytest.raises(chm.ChmError):
        ctx.eval_policies(pt, chm.EXHAUSTIVE, 0, 4, best=best, stall_model=2)


@pytest.mark.parametrize("path,cpt", [("0", "1"), ("0", "2"), ("1", "1")])
def test_both_slot_paths(ctx, path, cpt, monkeypatch):
    """global-memory slots (one or two candidates per thread) and shared-memory slots (one warp
    per CTA), forced either way on the same launch (3001 candidates: a ragged last pair), all
    bit-identical to the oracle"""
    monkeypatch.setenv("CHM_TL_SMEM", path)
    monkeypatch.setenv("CHM_TL_CPT", cpt)
    tr = W.CONFIGS["C5"]()
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    sd = W.SEEDED["C5"]
    res = tl(ctx, pt, chm.SEEDED, 5, 3001, seed=sd["seed"], flip_thr=sd["flip_thr"])
    ref = m.eval(O.SEEDED, 5, 3001, seed=sd["seed"], flip_thr=sd["flip_thr"], nthreads=16, stall_model=1)
    assert_same(res, ref, tr.budget)


def test_long_op_gaps_between_events():
    """40,000 ops with the events of two activations far apart: gaps of more than 16,383 ops
    between consecutive events take the program's tick-only NOP events"""
    from tests.helpers import make_trace
    n = 40_000
    half = n // 2
    ins = [[] for _ in range(n)]
    outs = [[] for _ in range(n)]
    frees = [[] for _ in range(n)]
    outs[0] = [0, 1]
    ins[1] = [0, 1]
    outs[2] = [2]  # a transient that makes the forward peak sit after the activations' last use
    frees[3] = [2]
    ins[n - 2] = [0, 1]
    frees[n - 2] = [0, 1]
    tr = make_trace([0] * half + [1] * half, [64 << 20, 32 << 20, 16 << 20], ins, outs, frees, 0, 1.0, 1e7,
                    (70 << 20), 4, 4)
    ctx = chm.Context(device=0)
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    assert pt.N == n and pt.K >= 1
    res = tl(ctx, pt, chm.EXHAUSTIVE, 0, 1 << pt.K)
    ref = m.eval(O.EXHAUSTIVE, 0, 1 << pt.K, stall_model=1)
    assert_same(res, ref, tr.budget)
    assert ref["stall"].max() > 0.0
    ctx.close()


def test_release_scratch_between_launches(ctx):
    """chm_release_scratch frees the evaluation scratch; the next launches (layer and timeline
    models) allocate it again and give the same results"""
    tr = W.CONFIGS["C5"]()
    pt = product_trace(ctx, tr)
    sd = W.SEEDED["C5"]
    kw = dict(seed=sd["seed"], flip_thr=sd["flip_thr"])
    a = tl(ctx, pt, chm.SEEDED, 0, 20_000, **kw)
    b = run_eval(ctx, pt, chm.SEEDED, 0, 20_000, footprint=True, **kw)
    for _ in range(2):
        ctx.release_scratch()
        a2 = tl(ctx, pt, chm.SEEDED, 0, 20_000, **kw)
        ctx.release_scratch()
        b2 = run_eval(ctx, pt, chm.SEEDED, 0, 20_000, footprint=True, **kw)
        for x, y in ((a, a2), (b, b2)):
            assert np.array_equal(x["stall"], y["stall"]) and np.array_equal(x["peak"], y["peak"])
            assert x["best"].tobytes() == y["best"].tobytes()
        assert np.array_equal(b["footprint"], b2["footprint"])
