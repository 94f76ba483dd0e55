"""chm_descend (the device descent, reading R-search) against the oracle's descend
(tests/test_descend_cpu.py pins it) and against the host loop of FLIP1 launches it replaces
(runtime.descend): the same end masks, keys (stall bit-equal) and round counts, from several
starts per launch; max_rounds = 0 scores the starts; in-place ends; the best key."""
import numpy as np
import pytest

import oracle as O
from workloads import traces as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2509_11076_b200 import chm  # noqa: E402
from paper_2509_11076_b200.runtime import descend as host_descend  # noqa: E402

DEV = "cuda:0"


def _build(tr):
    ctx = chm.Context(device=0)
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    return ctx, pt


def _starts(pt, n_seeded, seed=7, thr=0.05):
    W_ = pt.W
    out = [np.zeros(W_, np.uint64), np.array(pt.candidate_mask(chm.FLIP1, pt.K), np.uint64)]
    full = np.zeros(W_, np.uint64)
    for k in range(pt.K):
        full[k // 64] |= np.uint64(1 << (k % 64))
    out.append(full)
    for i in range(n_seeded):
        out.append(np.array(pt.candidate_mask(chm.SEEDED, 1000 + 37 * i, seed=seed, flip_thr=int(thr * 2 ** 64)),
                            np.uint64))
    return np.stack(out)


def _run(ctx, pt, starts, max_rounds=4096, in_place=False):
    n = len(starts)
    st = torch.from_numpy(starts.view(np.int64).copy()).to(DEV)
    ends = st if in_place else torch.empty_like(st)
    keys = torch.empty((n, 5), dtype=torch.int64, device=DEV)
    rounds = torch.empty(n, dtype=torch.int32, device=DEV)
    best = torch.empty(5, dtype=torch.int64, device=DEV)
    ctx.descend(pt, st, n, ends=ends, keys=keys, max_rounds=max_rounds, rounds=rounds, best=best)
    torch.cuda.synchronize()
    k = keys.cpu().numpy().view(chm.BEST_DTYPE).reshape(n)
    return (ends.cpu().numpy().view(np.uint64).reshape(n, pt.W), k, rounds.cpu().numpy(),
            best.cpu().numpy().view(chm.BEST_DTYPE)[0])


def _key3(k):
    return (int(k["excess"]), float(k["stall"]), int(k["swapped_bytes"]))


@pytest.mark.parametrize("name", ["C1", "C5"])
def test_descend_equals_the_oracle(name):
    tr = W.CONFIGS[name]()
    ctx, pt = _build(tr)
    m = O.Model(tr)
    starts = _starts(pt, 3)
    ends, keys, rounds, best = _run(ctx, pt, starts)
    for i, s in enumerate(starts):
        oe, okey, orounds = O.descend(m, s)
        assert np.array_equal(ends[i], oe), (name, i)
        assert _key3(keys[i]) == okey, (name, i, _key3(keys[i]), okey)
        assert int(rounds[i]) == orounds and int(keys[i]["index"]) == i
    j = min(range(len(starts)), key=lambda i: _key3(keys[i]) + (i,))
    assert _key3(best) == _key3(keys[j]) and int(best["index"]) == j
    ctx.close()


@pytest.mark.parametrize("seed", [101, 102, 104, 205, 310])
def test_descend_equals_the_oracle_on_random_traces(seed):
    tr = W.random_trace(seed, n_layers=6 + seed % 5, ops_per_layer=3 + seed % 3, bw=[3e7, 1e8, 1e6][seed % 3],
                        t_iter=1e-3)
    ctx, pt = _build(tr)
    if pt.K == 0:
        pytest.skip("no swappable tensor")
    m = O.Model(tr)
    starts = _starts(pt, 4, thr=0.3)
    ends, keys, rounds, _ = _run(ctx, pt, starts)
    for i, s in enumerate(starts):
        oe, okey, orounds = O.descend(m, s, nthreads=4)
        assert np.array_equal(ends[i], oe) and _key3(keys[i]) == okey and int(rounds[i]) == orounds, (seed, i)
    ctx.close()


@pytest.mark.parametrize("name", ["C3h", "C2"])
def test_descend_equals_the_host_flip1_loop(name):
    """the device descent retraces runtime.descend (one FLIP1 launch + host argmin per round)"""
    tr = W.CONFIGS[name]()
    ctx, pt = _build(tr)
    sd = W.SEEDED[name[:2]]
    best = torch.empty(5, dtype=torch.int64, device=DEV)
    ctx.eval_policies(pt, chm.SEEDED, 0, 20_000, best=best, seed=sd["seed"], flip_thr=sd["flip_thr"])
    sk = best.cpu().numpy().view(chm.BEST_DTYPE)[0]
    w = np.array(pt.candidate_mask(chm.SEEDED, int(sk["index"]), seed=sd["seed"], flip_thr=sd["flip_thr"]),
                 np.uint64)
    hk, hw, hr = host_descend(ctx, pt, sk, w, torch.device(DEV))
    starts = np.stack([w, np.array(pt.candidate_mask(chm.FLIP1, pt.K), np.uint64)])
    ends, keys, rounds, _ = _run(ctx, pt, starts)
    assert np.array_equal(ends[0], np.asarray(hw, np.uint64))
    assert _key3(keys[0]) == _key3(hk) and int(rounds[0]) == hr
    assert hr > 10
    ctx.close()


def test_descend_zero_rounds_scores_the_starts_and_runs_in_place():
    tr = W.CONFIGS["C5"]()
    ctx, pt = _build(tr)
    starts = _starts(pt, 5)
    n = len(starts)
    ends, keys, rounds, _ = _run(ctx, pt, starts, max_rounds=0)
    assert np.array_equal(ends, starts) and not rounds.any()
    masks = torch.from_numpy(starts.view(np.int64).copy()).to(DEV)
    pk = torch.empty(n, dtype=torch.int64, device=DEV)
    stl = torch.empty(n, dtype=torch.float64, device=DEV)
    sw = torch.empty(n, dtype=torch.int64, device=DEV)
    b = torch.empty(5, dtype=torch.int64, device=DEV)
    ctx.eval_policies(pt, chm.MASKS, 0, n, best=b, masks=masks, peak=pk, stall=stl, swapped=sw)
    pk, stl, sw = pk.cpu().numpy(), stl.cpu().numpy(), sw.cpu().numpy()
    for i in range(n):
        assert _key3(keys[i]) == (max(0, int(pk[i]) - pt.budget), float(stl[i]), int(sw[i]))
        assert int(keys[i]["peak"]) == int(pk[i])
    e1, k1, r1, _ = _run(ctx, pt, starts)
    e2, k2, r2, _ = _run(ctx, pt, starts, in_place=True)
    assert np.array_equal(e1, e2) and np.array_equal(r1, r2)
    assert all(_key3(k1[i]) == _key3(k2[i]) for i in range(n))
    ctx.close()


@pytest.mark.parametrize("max_rounds", [1, 7, 40])
def test_descend_stops_after_max_rounds_like_the_oracle(max_rounds):
    """a bounded descent ends where the oracle's bounded descent ends (C5, from the argmax-window
    base and two SEEDED starts)"""
    tr = W.CONFIGS["C5"]()
    ctx, pt = _build(tr)
    m = O.Model(tr)
    starts = _starts(pt, 2)[1:]
    ends, keys, rounds, _ = _run(ctx, pt, starts, max_rounds=max_rounds)
    for i, s in enumerate(starts):
        oe, okey, orounds = O.descend(m, s, max_rounds=max_rounds)
        assert np.array_equal(ends[i], oe) and _key3(keys[i]) == okey and int(rounds[i]) == orounds
        assert orounds <= max_rounds
    ctx.close()


@pytest.mark.parametrize("model", [chm.STALL_TIMELINE, chm.STALL_LAYER])
def test_lockstep_descents_equal_one_by_one(model):
    """runtime.descend_many (all starts' neighbourhoods in one MASKS launch per round) follows
    each start's descend() trajectory exactly, under either stall model"""
    from paper_2509_11076_b200.runtime import descend_many
    tr = W.CONFIGS["C5"]()
    ctx, pt = _build(tr)
    starts = _starts(pt, 2)[1:]
    best = torch.empty(5, dtype=torch.int64, device=DEV)
    sk = []
    for w in starts:
        ctx.eval_policies(pt, chm.FLIP1, pt.K, 1, best=best, base=w, stall_model=model)
        sk.append((best.cpu().numpy().view(chm.BEST_DTYPE)[0].copy(), w))
    many = descend_many(ctx, pt, sk, torch.device(DEV), 4096, model)
    for (k0, w0), (k, w, r) in zip(sk, many):
        hk, hw, hr = host_descend(ctx, pt, k0, w0, torch.device(DEV), 4096, model)
        assert np.array_equal(np.asarray(hw, np.uint64), w) and r == hr and _key3(hk) == _key3(k)
        assert int(hk["index"]) == int(k["index"]) and int(hk["peak"]) == int(k["peak"])
    ctx.close()



def test_device_descend_without_swappables():
    """K = 0: runtime.device_descend returns each start's (empty) mask and the no-swap key"""
    from paper_2509_11076_b200.runtime import device_descend
    from tests.helpers import make_trace
    ins = [[], [0], [1], [], [], []]
    outs = [[0], [1], [2], [3], [], []]
    frees = [[], [0], [1, 2], [3], [], []]
    tr = make_trace([0, 0, 0, 1, 1, 1], [512, 1024, 2048, 4096], ins, outs, frees, 512, 1.0, 1e9, 2048, 2, 2)
    ctx, pt = _build(tr)
    assert pt.K == 0 and pt.W == 0
    (k, w, r), = device_descend(ctx, pt, [np.zeros(0, np.uint64)], torch.device(DEV))
    assert r == 0 and w.size == 0
    m = O.Model(tr)
    ok = m.eval(O.MASKS, 0, 1, words=np.zeros(1, np.uint64))["best"]
    assert _key3(k) == (int(ok.excess), float(ok.stall), int(ok.swapped))
    ctx.close()
