"""Edge cases of the CUDA path vs the oracle: no swappable tensors, FWD-only and single-op
traces, one candidate, candidate ranges at the 2^K boundary, padded footprint rows, argument
errors, repeated launches reusing the scratch counters, MASKS with several words."""
import numpy as np
import pytest

import oracle as O
from tests.helpers import make_trace
from workloads import traces as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2509_11076_b200 import chm  # noqa: E402
from tests.test_gpu_parity import assert_same, product_trace, run_eval  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    c = chm.Context(device=0, host_arena_bytes=16 << 20)
    yield c
    c.close()


def test_no_swappable_tensors(ctx):
    # activations are freed before backward: K = 0, every candidate is F0
    n = 6
    ins = [[], [0], [1], [], [], []]
    outs = [[0], [1], [2], [3], [], []]
    frees = [[], [0], [1, 2], [3], [], []]
    tr = make_trace([0, 0, 0, 1, 1, 1], [512, 1024, 2048, 4096], ins, outs, frees, 512, 1.0, 1e9, 2048, 2, 2)
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    assert pt.K == 0 and m.K == 0
    for kind in (chm.SEEDED, chm.EXHAUSTIVE):
        res = run_eval(ctx, pt, kind, 0, 1, footprint=True, seed=1, flip_thr=1 << 63)
        ref = m.eval(O.SEEDED if kind == chm.SEEDED else O.EXHAUSTIVE, 0, 1, seed=1, flip_thr=1 << 63, footprint=True)
        assert_same(res, ref, tr.budget)
        assert np.array_equal(res["footprint"][0], m.f0())


def test_single_op_and_fwd_only(ctx):
    tr = make_trace([0], [512], [[]], [[0]], [[0]], 0, 1.0, 1e9, 0, 1, 1)
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    assert pt.N == 1 and pt.L == 1
    assert_same(run_eval(ctx, pt, chm.EXHAUSTIVE, 0, 1, footprint=True),
                m.eval(O.EXHAUSTIVE, 0, 1, footprint=True), tr.budget)


def test_exhaustive_range_limits(ctx):
    tr = W.tiny()
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    last = (1 << m.K) - 1
    assert_same(run_eval(ctx, pt, chm.EXHAUSTIVE, last, 1, footprint=True),
                m.eval(O.EXHAUSTIVE, last, 1, footprint=True), tr.budget)
    with pytest.raises(chm.ChmError):
        run_eval(ctx, pt, chm.EXHAUSTIVE, last, 2)  # past 2^K


def test_padded_rows_and_bad_ld(ctx):
    tr = W.tiny()
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    dev = torch.device("cuda:0")
    ld = pt.N + 10
    fp = torch.full((50, ld), -7, dtype=torch.int64, device=dev)
    best = torch.empty(5, dtype=torch.int64, device=dev)
    ctx.eval_policies(pt, chm.EXHAUSTIVE, 100, 50, best=best, footprint=fp, ld=ld)
    torch.cuda.synchronize()
    ref = m.eval(O.EXHAUSTIVE, 100, 50, footprint=True)
    assert np.array_equal(fp[:, :pt.N].cpu().numpy(), ref["footprint"])
    assert bool((fp[:, pt.N + 2:] == -7).all())  # nothing written past the padded row
    for bad_ld in (pt.N - 1, pt.N + 1 if pt.N % 2 == 0 else pt.N):  # too short / odd
        with pytest.raises(chm.ChmError):
            ctx.eval_policies(pt, chm.EXHAUSTIVE, 0, 4, best=best, footprint=fp, ld=bad_ld)
    with pytest.raises(chm.ChmError):
        ctx.eval_policies(pt, chm.EXHAUSTIVE, 0, 0, best=best)  # empty range
    with pytest.raises(chm.ChmError):
        ctx.eval_policies(pt, chm.EXHAUSTIVE, 0, 4, best=None)  # best required


def test_repeated_launches_reuse_counters(ctx):
    """the work counter / ticket are reset by the last CTA: back-to-back launches on one stream
    (different sizes) must all be exact"""
    tr = W.gpt2_xl()
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    sd = W.SEEDED["C2"]
    for first, count in ((0, 1), (5, 37), (1000, 4096), (7, 1), (123, 20000)):
        res = run_eval(ctx, pt, chm.SEEDED, first, count, seed=sd["seed"], flip_thr=sd["flip_thr"])
        ref = m.eval(O.SEEDED, first, count, seed=sd["seed"], flip_thr=sd["flip_thr"], nthreads=8)
        assert_same(res, ref, tr.budget)


def test_search_and_full_agree_on_many_candidates(ctx):
    tr = W.llama2_7b_rank()
    pt = product_trace(ctx, tr)
    sd = W.SEEDED["C5"]
    a = run_eval(ctx, pt, chm.SEEDED, 0, 50000, seed=sd["seed"], flip_thr=sd["flip_thr"])
    b = run_eval(ctx, pt, chm.SEEDED, 0, 50000, footprint=True, seed=sd["seed"], flip_thr=sd["flip_thr"])
    assert np.array_equal(a["peak"], b["peak"]) and np.array_equal(a["stall"], b["stall"])
    assert np.array_equal(b["footprint"].max(axis=1), b["peak"])  # peak = max of the row


@pytest.mark.parametrize("gf,gb", [(100, 100), (40, 20), (1, 1)])
def test_layer_counts_across_lane_blockings(ctx, gf, gb):
    """L from 3 to 201 logical layers: each lane of the replay warp owns E = P/32 layers
    (P the next power of two >= L), E = 1 .. 8 -- keys and rows vs the oracle"""
    import dataclasses
    tr = W.random_trace(77, n_layers=50, ops_per_layer=3, bw=1e8, t_iter=1e-3)
    tr = dataclasses.replace(tr, groups_fwd=gf, groups_bwd=gb)
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    assert pt.L == m.L
    for first, count in ((0, 3000), (12345, 777)):
        res = run_eval(ctx, pt, chm.SEEDED, first, count, footprint=True, seed=9, flip_thr=int(0.1 * 2 ** 64))
        ref = m.eval(O.SEEDED, first, count, seed=9, flip_thr=int(0.1 * 2 ** 64), footprint=True, nthreads=8)
        assert_same(res, ref, tr.budget)
