"""ncu driver: 3 timeline-mode launches over 10^5 SEEDED C2 candidates (search mode)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200 import chm  # noqa: E402
from workloads import traces as W  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    tr = W.CONFIGS[name]()
    sd = W.SEEDED[name]
    ctx = chm.Context(device=0)
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    n = 100_000
    dev = torch.device("cuda:0")
    peak = torch.empty(n, dtype=torch.int64, device=dev)
    stall = torch.empty(n, dtype=torch.float64, device=dev)
    best = torch.empty(5, dtype=torch.int64, device=dev)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for it in range(3):
        s.record()
        ctx.eval_policies(pt, chm.SEEDED, 0, n, best=best, seed=sd["seed"], flip_thr=sd["flip_thr"], peak=peak,
                          stall=stall, stall_model=chm.STALL_TIMELINE)
        e.record()
        torch.cuda.synchronize()
        print(f"timeline eval {it}: {s.elapsed_time(e):.3f} ms")


if __name__ == "__main__":
    main()
