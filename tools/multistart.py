"""Does starting the descent (R-search) from more than the best SEEDED candidate help?  For the
C2-C5 traces: the key after descending from the best, and the best key over descents from the
top-8 distinct SEEDED candidates.  Prints one line per config."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200 import chm  # noqa: E402
from paper_2509_11076_b200.runtime import descend  # noqa: E402
from workloads import traces as W  # noqa: E402


def key(k):
    return (int(k["excess"]) >> 20, round(float(k["stall"]), 4), int(k["swapped_bytes"]) >> 20)


for name in ("C2", "C3", "C4b", "C5"):
    tr = W.CONFIGS[name]()
    ctx = chm.Context(device=0)
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    sd = W.SEEDED[name[:2]]
    n = 100_000
    dev = torch.device("cuda:0")
    peak = torch.empty(n, dtype=torch.int64, device=dev)
    stall = torch.empty(n, dtype=torch.float64, device=dev)
    sw = torch.empty(n, dtype=torch.int64, device=dev)
    best = torch.empty(5, dtype=torch.int64, device=dev)
    ctx.eval_policies(pt, chm.SEEDED, 0, n, best=best, seed=sd["seed"], flip_thr=sd["flip_thr"], peak=peak, stall=stall,
                      swapped=sw)
    ex = np.maximum(peak.cpu().numpy() - pt.budget, 0)
    order = np.lexsort((sw.cpu().numpy(), stall.cpu().numpy(), ex))[:8]
    results = []
    for i in order:
        w = pt.candidate_mask(chm.SEEDED, int(i), seed=sd["seed"], flip_thr=sd["flip_thr"])
        k0 = np.zeros(1, chm.BEST_DTYPE)[0]
        k0["excess"], k0["stall"], k0["swapped_bytes"] = ex[i], stall[i].item(), sw[i].item()
        dk, _, r = descend(ctx, pt, k0, w, dev)
        results.append((key(dk), r))
    print(name, "K", pt.K, "from best:", results[0], " best of 8 starts:", min(results))
    ctx.close()
