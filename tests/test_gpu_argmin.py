"""Cross-rank argmin on the device (§8(a) a7; P:421 best-of-n): a 10^5-candidate
launch split into P in {2, 4, 8} contiguous shards with bench.py's shard rule
(paper_2509_11076_b200.dist.shard), the P per-shard keys stacked in one device buffer as the NCCL
all-gather leaves them, reduced by chm_best_reduce_device -- must equal the single launch's key
and the oracle's argmin over all candidates.  A forced tie on (excess, stall, swapped) across two
shards (the same mask at two global indices) exercises the index tie-break."""
import numpy as np
import pytest

import oracle as O
from workloads import traces as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2509_11076_b200 import chm  # noqa: E402
from paper_2509_11076_b200.dist import shard  # noqa: E402

C = 100_000


@pytest.fixture(scope="module")
def ctx():
    c = chm.Context(device=0, host_arena_bytes=1 << 20)
    yield c
    c.close()


def _trace(ctx, tr):
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    ctx.set_detailed(False)
    return ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter,
                           omega=tr.omega)


def _key(t):
    b = t.cpu().numpy().view(chm.BEST_DTYPE)[0]
    return (int(b["excess"]), float(b["stall"]), int(b["swapped_bytes"]), int(b["index"]), int(b["peak"]))


def _sharded(ctx, pt, P, count, reverse=False, **kw):
    dev = torch.device("cuda:0")
    keys = torch.empty((P, 5), dtype=torch.int64, device=dev)
    for r in range(P):
        lo, cnt = shard(count, P, r)
        masks = kw.get("masks")  # MASKS: row c of the shard's array is global candidate lo + c
        ctx.eval_policies(pt, kw["kind"], lo, cnt, best=keys[r], seed=kw.get("seed", 0),
                          flip_thr=kw.get("flip_thr", 0), masks=masks[lo:lo + cnt] if masks is not None else None)
    if reverse:  # the min must not depend on the keys' order in the buffer
        keys = keys.flip(0).contiguous()
    out = torch.empty(5, dtype=torch.int64, device=dev)
    ctx.best_reduce_device(keys, P, out)
    torch.cuda.synchronize()
    return _key(out)


@pytest.mark.parametrize("name", ["C2", "C5"])
def test_sharded_seeded_argmin(ctx, name):
    tr = W.CONFIGS[name]()
    pt = _trace(ctx, tr)
    sd = W.SEEDED[name[:2]]
    dev = torch.device("cuda:0")
    single = torch.empty(5, dtype=torch.int64, device=dev)
    ctx.eval_policies(pt, chm.SEEDED, 0, C, best=single, seed=sd["seed"], flip_thr=sd["flip_thr"])
    torch.cuda.synchronize()
    ref = O.Model(tr).eval(O.SEEDED, 0, C, seed=sd["seed"], flip_thr=sd["flip_thr"], nthreads=16)["best"]
    exp = (ref.excess, ref.stall, ref.swapped, ref.index, ref.peak)
    assert _key(single) == exp
    for P in (2, 4, 8):
        for rev in (False, True):
            got = _sharded(ctx, pt, P, C, reverse=rev, kind=chm.SEEDED, seed=sd["seed"], flip_thr=sd["flip_thr"])
            assert got == exp, (P, rev, got, exp)


def test_sharded_argmin_tie_break_across_shards(ctx):
    """MASKS on C5: the best of 4096 random masks also placed at a later global index in the
    last of 8 shards -> both copies tie on (excess, stall, swapped); the lower index must win,
    whatever the keys' order; moving the earlier copy away makes the later one win."""
    tr = W.CONFIGS["C5"]()
    pt = _trace(ctx, tr)
    m = O.Model(tr)
    rng = np.random.default_rng(11)
    n = 4096
    bits = rng.random((n, pt.K)) < rng.uniform(0.3, 0.9, size=(n, 1))
    words = np.zeros((n, pt.W), np.uint64)
    for k in range(pt.K):
        words[:, k // 64] |= bits[:, k].astype(np.uint64) << np.uint64(k % 64)
    dev = torch.device("cuda:0")
    best = torch.empty(5, dtype=torch.int64, device=dev)
    ctx.eval_policies(pt, chm.MASKS, 0, n, best=best, masks=torch.from_numpy(words.view(np.int64)).to(dev))
    torch.cuda.synchronize()
    j = _key(best)[3]
    if j >= n - n // 8:  # move the best out of the last shard
        words[[j, 5]] = words[[5, j]]
        j = 5
    j2 = n - 3  # inside shard 7 of 8
    words[j2] = words[j]
    masks = torch.from_numpy(words.view(np.int64)).to(dev)
    ref = m.eval(O.MASKS, 0, n, words=words, nthreads=16)["best"]
    assert ref.index == j
    exp = (ref.excess, ref.stall, ref.swapped, ref.index, ref.peak)
    for P in (2, 4, 8):
        for rev in (False, True):
            assert _sharded(ctx, pt, P, n, reverse=rev, kind=chm.MASKS, masks=masks) == exp
    # the two copies do tie: their keys differ only in the index
    r2 = m.eval(O.MASKS, j2, 1, words=words[j2:j2 + 1], nthreads=1)
    assert (int(np.maximum(r2["peak"][0] - tr.budget, 0)), float(r2["stall"][0]), int(r2["swapped"][0])) == \
        (ref.excess, ref.stall, ref.swapped)
    # drop the first copy (swap in the all-zero mask): now the later copy is the unique best
    # unless another mask ties it; the oracle decides
    words[j] = 0
    masks = torch.from_numpy(words.view(np.int64)).to(dev)
    ref2 = m.eval(O.MASKS, 0, n, words=words, nthreads=16)["best"]
    exp2 = (ref2.excess, ref2.stall, ref2.swapped, ref2.index, ref2.peak)
    assert _sharded(ctx, pt, 8, n, reverse=True, kind=chm.MASKS, masks=masks) == exp2
