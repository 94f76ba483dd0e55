"""Property-based device parity (hypothesis): random traces, random candidate kinds and ranges,
search and full mode -- the replay kernels against the oracle, every key and footprint row."""
import numpy as np
import pytest

hypothesis = pytest.importorskip("hypothesis")
from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

import oracle as O  # noqa: E402
from workloads import traces as W  # noqa: E402

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2509_11076_b200 import chm  # noqa: E402
from tests.test_gpu_parity import assert_same, product_trace, run_eval  # noqa: E402

traces = st.builds(W.random_trace, seed=st.integers(0, 10 ** 6), n_layers=st.integers(1, 6),
                   ops_per_layer=st.integers(1, 4), max_kib=st.sampled_from([1, 64, 4096]),
                   bw=st.sampled_from([1e6, 1e8, 5e10]), t_iter=st.sampled_from([1e-5, 1e-3]))


@pytest.fixture(scope="module")
def ctx():
    c = chm.Context(device=0, host_arena_bytes=1 << 20)
    yield c
    c.close()


@settings(max_examples=150, deadline=None)
@given(tr=traces, kind=st.sampled_from(["exhaustive", "seeded", "masks", "explicit"]), first=st.integers(0, 5000),
       count=st.integers(1, 700), full=st.booleans(), seed=st.integers(0, 2 ** 32), flip=st.floats(0.0, 0.9))
def test_replay_matches_oracle(ctx, tr, kind, first, count, full, seed, flip):
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    thr = int(flip * 2 ** 64) & ((1 << 64) - 1)
    if kind == "exhaustive":
        first = min(first, (1 << m.K) - 1)
        count = min(count, (1 << m.K) - first)
        res = run_eval(ctx, pt, chm.EXHAUSTIVE, first, count, footprint=full)
        ref = m.eval(O.EXHAUSTIVE, first, count, footprint=full)
    elif kind == "seeded":
        res = run_eval(ctx, pt, chm.SEEDED, first, count, footprint=full, seed=seed, flip_thr=thr)
        ref = m.eval(O.SEEDED, first, count, seed=seed, flip_thr=thr, footprint=full)
    elif kind == "masks":
        rng = np.random.default_rng(seed)
        W_ = max(m.W, 1)
        masks = rng.integers(0, 2 ** 63, size=(count, W_), dtype=np.int64).astype(np.uint64)
        if m.K % 64:
            masks[:, -1] &= np.uint64((1 << (m.K % 64)) - 1)
        if m.K == 0:
            masks[:] = 0
        res = run_eval(ctx, pt, chm.MASKS, first, count, footprint=full,
                       masks=torch.from_numpy(masks[:, :m.W].copy().view(np.int64)).cuda() if m.W else
                       torch.zeros((count, 1), dtype=torch.int64, device="cuda"))
        ref = m.eval(O.MASKS, first, count, words=masks[:, :m.W] if m.W else np.zeros((count, 1), np.uint64),
                     footprint=full)
    else:
        rng = np.random.default_rng(seed)
        sw = m.swappable()
        lists = []
        for _ in range(min(count, 40)):
            k = rng.random(m.K) < 0.5
            lists.append((sw["t"][k], sw["r"][k], sw["s"][k]))
        off = np.zeros(len(lists) + 1, np.uint64)
        off[1:] = np.cumsum([len(x[0]) for x in lists])
        items = np.zeros(int(off[-1]), chm.ITEM_DTYPE)
        if len(items):
            items["t"] = np.concatenate([x[0] for x in lists])
            items["r"] = np.concatenate([x[1] for x in lists])
            items["s"] = np.concatenate([x[2] for x in lists])
        res = run_eval(ctx, pt, chm.EXPLICIT, first, len(lists), footprint=full, item_offsets=off, items=items)
        ref = O.eval_explicit(m, lists, first_index=first, footprint=full)
    assert_same(res, ref, tr.budget)


@settings(max_examples=120, deadline=None)
@given(tr=traces, kind=st.sampled_from(["exhaustive", "seeded", "masks", "flip1"]), first=st.integers(0, 5000),
       count=st.integers(1, 700), seed=st.integers(0, 2 ** 32), flip=st.floats(0.0, 0.9),
       path=st.sampled_from(["0", "1", "auto"]))
def test_timeline_matches_oracle(ctx, tr, kind, first, count, seed, flip, path):
    """the timeline stall model in the search (CHM_STALL_TIMELINE) on random traces and candidate
    ranges, on either slot path, against the oracle's orc_eval_model(stall_model = 1)"""
    import os
    old = os.environ.pop("CHM_TL_SMEM", None)
    if path != "auto":
        os.environ["CHM_TL_SMEM"] = path
    try:
        pt = product_trace(ctx, tr)
        m = O.Model(tr)
        thr = int(flip * 2 ** 64) & ((1 << 64) - 1)
        rng = np.random.default_rng(seed)
        W_ = max(m.W, 1)
        if kind == "exhaustive":
            first = min(first, (1 << m.K) - 1)
            count = min(count, (1 << m.K) - first)
            res = run_eval(ctx, pt, chm.EXHAUSTIVE, first, count, stall_model=chm.STALL_TIMELINE)
            ref = m.eval(O.EXHAUSTIVE, first, count, stall_model=1)
        elif kind == "seeded":
            res = run_eval(ctx, pt, chm.SEEDED, first, count, seed=seed, flip_thr=thr, stall_model=chm.STALL_TIMELINE)
            ref = m.eval(O.SEEDED, first, count, seed=seed, flip_thr=thr, stall_model=1)
        else:
            if kind == "flip1":  # the one-bit neighbourhood of a random base, as MASKS for the oracle
                base = rng.integers(0, 2 ** 63, size=W_, dtype=np.int64).astype(np.uint64)
                if m.K % 64:
                    base[-1] &= np.uint64((1 << (m.K % 64)) - 1)
                if m.K == 0:
                    base[:] = 0
                first, count = 0, m.K + 1
                masks = np.repeat(base[None, :], count, axis=0)
                for g in range(m.K):
                    masks[g, g // 64] ^= np.uint64(1 << (g % 64))
                res = run_eval(ctx, pt, chm.FLIP1, 0, count, base=base[:m.W], stall_model=chm.STALL_TIMELINE)
            else:
                masks = rng.integers(0, 2 ** 63, size=(count, W_), dtype=np.int64).astype(np.uint64)
                if m.K % 64:
                    masks[:, -1] &= np.uint64((1 << (m.K % 64)) - 1)
                if m.K == 0:
                    masks[:] = 0
                res = run_eval(ctx, pt, chm.MASKS, first, count, stall_model=chm.STALL_TIMELINE,
                               masks=torch.from_numpy(masks[:, :m.W].copy().view(np.int64)).cuda() if m.W else
                               torch.zeros((count, 1), dtype=torch.int64, device="cuda"))
            ref = m.eval(O.MASKS, first, count, words=masks[:, :m.W] if m.W else np.zeros((count, 1), np.uint64),
                         stall_model=1)
        assert_same(res, ref, tr.budget)
    finally:
        os.environ.pop("CHM_TL_SMEM", None)
        if old is not None:
            os.environ["CHM_TL_SMEM"] = old


@settings(max_examples=60, deadline=None)
@given(tr=traces, seed=st.integers(0, 2 ** 32), n_starts=st.integers(1, 6), max_rounds=st.sampled_from([0, 1, 3, 4096]))
def test_descend_matches_oracle(ctx, tr, seed, n_starts, max_rounds):
    """chm_descend from random start masks (any K, including K = 0) = the oracle's descend"""
    pt = product_trace(ctx, tr)
    m = O.Model(tr)
    if m.L < 1:
        return
    W_ = max(m.W, 1)
    rng = np.random.default_rng(seed)
    starts = rng.integers(0, 2 ** 63, size=(n_starts, W_), dtype=np.int64).astype(np.uint64)
    if m.K % 64:
        starts[:, -1] &= np.uint64((1 << (m.K % 64)) - 1)
    if m.K == 0:
        starts[:] = 0
    st_ = torch.from_numpy(starts.view(np.int64).copy()).cuda()
    keys = torch.empty((n_starts, 5), dtype=torch.int64, device="cuda")
    rounds = torch.empty(n_starts, dtype=torch.int32, device="cuda")
    ctx.descend(pt, st_, n_starts, ends=st_, keys=keys, rounds=rounds, max_rounds=max_rounds)
    ends = st_.cpu().numpy().view(np.uint64)
    ks = keys.cpu().numpy().view(chm.BEST_DTYPE).reshape(-1)
    for i in range(n_starts):
        oe, okey, orr = O.descend(m, starts[i, :m.W] if m.W else np.zeros(0, np.uint64), max_rounds=max_rounds,
                                  nthreads=2)
        assert np.array_equal(ends[i, :m.W], oe[:m.W]) and int(rounds.cpu()[i]) == orr
        assert (int(ks[i]["excess"]), float(ks[i]["stall"]), int(ks[i]["swapped_bytes"])) == okey
