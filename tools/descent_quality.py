"""Plan quality of the descent (reading R-search) on traces small enough for EXHAUSTIVE: the
best of 2,000 SEEDED candidates, its descent, and the exhaustive optimum, per trace (C1 and
six random traces).  Prints one line per trace."""
import numpy as np, torch, sys
sys.path.insert(0, "/root/repo")
from paper_2509_11076_b200 import chm
from paper_2509_11076_b200.runtime import descend
from workloads import traces as W
for name in ["C1"] + [f"rand{s}" for s in range(6)]:
    tr = W.tiny() if name == "C1" else W.random_trace(int(name[4:]) + 100, n_layers=5, ops_per_layer=4, bw=3e7, t_iter=1e-3)
    ctx = chm.Context(device=0)
    ctx.set_detailed(True); chm.record_iteration(ctx, tr); ctx.detect_seq_change(tr.t_iter)
    pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    if pt.K > 26 or pt.K == 0: continue
    best = torch.empty(5, dtype=torch.int64, device="cuda")
    ctx.eval_policies(pt, chm.EXHAUSTIVE, 0, 1 << pt.K, best=best)
    ex = best.cpu().numpy().view(chm.BEST_DTYPE)[0]
    ctx.eval_policies(pt, chm.SEEDED, 0, 2000, best=best, seed=1, flip_thr=int(0.02 * 2**64))
    sk = best.cpu().numpy().view(chm.BEST_DTYPE)[0]
    w = pt.candidate_mask(chm.SEEDED, int(sk["index"]), seed=1, flip_thr=int(0.02 * 2**64))
    dk, dw, r = descend(ctx, pt, sk, w, torch.device("cuda:0"))
    f = lambda k: (int(k["excess"]), round(float(k["stall"]), 6), int(k["swapped_bytes"]))
    print(name, "K", pt.K, "exhaustive", f(ex), "seeded", f(sk), "descent", f(dk), "rounds", r, "optimal" if f(dk) == f(ex) else "")
