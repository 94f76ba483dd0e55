"""The CUDA path at its size limits, element by element against the oracle: L = 256 logical
layers (the trace build's bound; E = 8 layers per lane, the widest padded slot layout), K = 4094
swappable tensors (64 mask words, the SEEDED / FLIP1 bound) with N = 9,360 ops in full mode, and
K = 4,129 (65 words): SEEDED / FLIP1 refuse it with CHM_E_INVAL while MASKS candidates and the
device descent (no word bound) still match the oracle."""
import dataclasses

import numpy as np
import pytest

import oracle as O
from workloads import traces as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2509_11076_b200 import chm  # noqa: E402
from tests.test_gpu_parity import assert_same, check_trace_tables, product_trace, run_eval  # noqa: E402

DEV = "cuda:0"


@pytest.fixture(scope="module")
def ctx():
    c = chm.Context(device=0, host_arena_bytes=1 << 20)
    yield c
    c.close()


def _trace(seed, nl, opl, gf, gb):
    tr = W.random_trace(seed, n_layers=nl, ops_per_layer=opl, bw=1e9, t_iter=1e-2)
    return dataclasses.replace(tr, groups_fwd=gf, groups_bwd=gb)


def _descend(ctx, pt, words, max_rounds):
    st = torch.from_numpy(np.asarray(words, np.uint64).view(np.int64).reshape(1, -1).copy()).to(DEV)
    keys = torch.empty((1, 5), dtype=torch.int64, device=DEV)
    rounds = torch.empty(1, dtype=torch.int32, device=DEV)
    ctx.descend(pt, st, 1, ends=st, keys=keys, rounds=rounds, max_rounds=max_rounds)
    k = keys.cpu().numpy().view(chm.BEST_DTYPE).reshape(-1)[0]
    return (st.cpu().numpy().view(np.uint64)[0], (int(k["excess"]), float(k["stall"]), int(k["swapped_bytes"])),
            int(rounds.cpu()[0]))


def test_256_layers(ctx):
    tr = _trace(5, 128, 8, 128, 127)
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    assert pt.L == 256 and pt.K > 900
    check_trace_tables(pt, m)
    sd = dict(seed=9, flip_thr=int(0.05 * 2 ** 64))
    assert_same(run_eval(ctx, pt, chm.SEEDED, 0, 3000, footprint=True, **sd),
                m.eval(O.SEEDED, 0, 3000, footprint=True, nthreads=16, **sd), tr.budget)
    base = np.asarray(pt.candidate_mask(chm.FLIP1, pt.K), np.uint64)
    nb = np.repeat(base[None, :], pt.K + 1, axis=0)
    for k in range(pt.K):
        nb[k, k // 64] ^= np.uint64(1 << (k % 64))
    assert_same(run_eval(ctx, pt, chm.FLIP1, 0, pt.K + 1, footprint=True, base=base),
                m.eval(O.MASKS, 0, pt.K + 1, words=nb.reshape(-1), footprint=True, nthreads=16), tr.budget)
    e, key, r = _descend(ctx, pt, base, 25)
    oe, okey, orr = O.descend(m, base, max_rounds=25)
    assert np.array_equal(e, oe) and key == okey and r == orr


def test_4094_swappables_full_mode(ctx):
    tr = _trace(11, 8, 585, 8, 8)
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    assert pt.K == 4094 and pt.W == 64 and pt.N > 9000
    check_trace_tables(pt, m)
    sd = dict(seed=3, flip_thr=int(0.01 * 2 ** 64))
    assert_same(run_eval(ctx, pt, chm.SEEDED, 0, 1500, footprint=True, **sd),
                m.eval(O.SEEDED, 0, 1500, footprint=True, nthreads=16, **sd), tr.budget)
    base = np.asarray(pt.candidate_mask(chm.FLIP1, pt.K), np.uint64)
    e, key, r = _descend(ctx, pt, base, 6)
    oe, okey, orr = O.descend(m, base, max_rounds=6)
    assert np.array_equal(e, oe) and key == okey and r == orr


def test_past_the_seeded_word_bound(ctx):
    tr = _trace(11, 8, 590, 8, 8)
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    assert pt.K == 4129 and pt.W == 65
    with pytest.raises(chm.ChmError):
        run_eval(ctx, pt, chm.SEEDED, 0, 10, seed=1, flip_thr=1 << 60)
    with pytest.raises(chm.ChmError):
        run_eval(ctx, pt, chm.FLIP1, 0, 10, base=np.zeros(pt.W, np.uint64))
    rng = np.random.default_rng(4)
    masks = rng.integers(0, 2 ** 63, size=(64, pt.W), dtype=np.int64).view(np.uint64)
    masks[:, -1] &= np.uint64((1 << (pt.K - 64 * (pt.W - 1))) - 1)  # bits >= K zero
    dm = torch.from_numpy(masks.view(np.int64).copy()).to(DEV)
    assert_same(run_eval(ctx, pt, chm.MASKS, 0, 64, footprint=True, masks=dm),
                m.eval(O.MASKS, 0, 64, words=masks.reshape(-1), footprint=True, nthreads=16), tr.budget)
    e, key, r = _descend(ctx, pt, masks[0], 3)
    oe, okey, orr = O.descend(m, masks[0], max_rounds=3)
    assert np.array_equal(e, oe) and key == okey and r == orr
