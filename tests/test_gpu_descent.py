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
