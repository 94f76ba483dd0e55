"""Plan quality of the descent (reading R-search): from the best of 2,000 SEEDED candidates,
steepest descent over FLIP1 rounds reaches the exhaustive optimum's (excess, stall) on small
random traces, where all 2^K swap sets can be replayed."""
import pytest

from workloads import traces as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2509_11076_b200 import chm  # noqa: E402
from paper_2509_11076_b200.runtime import descend  # noqa: E402


@pytest.mark.parametrize("seed", range(100, 106))
def test_descent_reaches_the_exhaustive_optimum(seed):
    tr = W.random_trace(seed, n_layers=5, ops_per_layer=4, bw=3e7, t_iter=1e-3)
    ctx = chm.Context(device=0)
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    assert 0 < pt.K <= 24
    best = torch.empty(5, dtype=torch.int64, device="cuda")
    ctx.eval_policies(pt, chm.EXHAUSTIVE, 0, 1 << pt.K, best=best)
    ex = best.cpu().numpy().view(chm.BEST_DTYPE)[0]
    thr = int(0.02 * 2 ** 64)
    ctx.eval_policies(pt, chm.SEEDED, 0, 2000, best=best, seed=1, flip_thr=thr)
    sk = best.cpu().numpy().view(chm.BEST_DTYPE)[0]
    w = pt.candidate_mask(chm.SEEDED, int(sk["index"]), seed=1, flip_thr=thr)
    dk, dw, rounds = descend(ctx, pt, sk, w, torch.device("cuda:0"))
    key = lambda k: (int(k["excess"]), float(k["stall"]), int(k["swapped_bytes"]))  # noqa: E731
    assert key(dk) <= key(sk)
    assert key(dk) == key(ex), (key(dk), key(ex), rounds)
    ctx.close()


@pytest.mark.parametrize("seed", range(100, 103))
@pytest.mark.parametrize("model", [chm.STALL_LAYER, chm.STALL_TIMELINE])
def test_batched_descent_ends_in_a_single_flip_local_optimum(seed, model):
    """descend(batch=8): each round moves to the best of the single best flip and the best 2..8
    improving flips applied together; it ends where no single flip improves the key (the same
    stopping rule as batch=1), never above its start"""
    tr = W.random_trace(seed, n_layers=5, ops_per_layer=4, bw=3e7, t_iter=1e-3)
    ctx = chm.Context(device=0)
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    best = torch.empty(5, dtype=torch.int64, device="cuda")
    thr = int(0.02 * 2 ** 64)
    ctx.eval_policies(pt, chm.SEEDED, 0, 2000, best=best, seed=1, flip_thr=thr, stall_model=model)
    sk = best.cpu().numpy().view(chm.BEST_DTYPE)[0]
    w = pt.candidate_mask(chm.SEEDED, int(sk["index"]), seed=1, flip_thr=thr)
    dk, dw, rounds = descend(ctx, pt, sk, w, torch.device("cuda:0"), 4096, model, 8)
    key = lambda k: (int(k["excess"]), float(k["stall"]), int(k["swapped_bytes"]))  # noqa: E731
    assert key(dk) <= key(sk)
    ctx.eval_policies(pt, chm.FLIP1, 0, pt.K + 1, best=best, base=dw, stall_model=model)
    nb = best.cpu().numpy().view(chm.BEST_DTYPE)[0]
    assert not key(nb) < key(dk)  # no improving single flip left
    ctx.eval_policies(pt, chm.FLIP1, pt.K, 1, best=best, base=dw, stall_model=model)
    assert key(best.cpu().numpy().view(chm.BEST_DTYPE)[0]) == key(dk)  # the reported key is the mask's
    ctx.close()


def test_multibase_seeded_finds_the_empty_plan_when_nothing_needs_swapping():
    """C4a (Llama-2 13B at s = 2048) fits its 80 GiB budget with nothing swapped: the single-base
    SEEDED search (centred on the no-swap peak's window) still swaps GBs; around several bases
    (reading R-bases: the empty mask is one, scored as it is) the best key is the empty plan
    (0, 0.0, 0).  The argmin is checked against the per-base keys it reports."""
    import numpy as np

    from paper_2509_11076_b200.runtime import default_bases, seeded_multibase
    tr = W.CONFIGS["C4a"]()
    sd = W.SEEDED["C4"]
    ctx = chm.Context(device=0)
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    assert pt.peak0 <= pt.budget and pt.K > 0
    dev = torch.device("cuda:0")
    best = torch.empty(5, dtype=torch.int64, device=dev)
    ctx.eval_policies(pt, chm.SEEDED, 0, 100_000, best=best, seed=sd["seed"], flip_thr=sd["flip_thr"])
    single = best.cpu().numpy().view(chm.BEST_DTYPE)[0]
    assert int(single["swapped_bytes"]) > 0  # r01's search never reaches the empty plan
    k, w, name, per = seeded_multibase(ctx, pt, default_bases(pt), 100_000, sd["seed"], sd["flip_thr"], dev)
    assert (int(k["excess"]), float(k["stall"]), int(k["swapped_bytes"])) == (0, 0.0, 0)
    assert name == "empty" and not np.any(w)
    key = lambda x: (int(x["excess"]), float(x["stall"]), int(x["swapped_bytes"]))  # noqa: E731
    assert key(k) == min(key(x) for x, _ in per.values())
    ctx.close()
