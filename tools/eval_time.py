"""Device time of one full-mode (per-op footprints) or search-mode chm_eval_policies launch over
10^5 SEEDED candidates of a config, the bench's way (a short device-side wait, then CUDA events
around the launch), median and min of 15 after 3 warm-ups.

    python tools/eval_time.py [C2] [--search]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200 import chm  # noqa: E402
from workloads import traces as W  # noqa: E402


def main():
    name = next((a for a in sys.argv[1:] if not a.startswith("--")), "C2")
    full = "--search" not in sys.argv
    tr = W.CONFIGS[name]()
    sd = W.SEEDED[name[:2]]
    ctx = chm.Context(device=0, eval_ctas_per_sm=int(os.environ.get("EVAL_CTAS_PER_SM", "0")))
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    n, ld = int(os.environ.get("EVAL_N", "100000")), (pt.N + 1) // 2 * 2
    dev = torch.device("cuda:0")
    peak = torch.empty(n, dtype=torch.int64, device=dev)
    stall = torch.empty(n, dtype=torch.float64, device=dev)
    fp = torch.empty((n, ld), dtype=torch.int64, device=dev) if full else None
    best = torch.empty(5, dtype=torch.int64, device=dev)
    ts = []
    for it in range(18):
        torch.cuda.synchronize()
        torch.cuda._sleep(1_000_000)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        ctx.eval_policies(pt, chm.SEEDED, 0, n, best=best, seed=sd["seed"], flip_thr=sd["flip_thr"], peak=peak,
                          stall=stall, footprint=fp, ld=ld if full else 0)
        e.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(s.elapsed_time(e))
    byt = (8 * ld + 16) * n if full else 16 * n
    med = float(np.median(ts))
    print(f"ctas/SM {os.environ.get('EVAL_CTAS_PER_SM', 'auto')} {name} {'full' if full else 'search'}: median {med:.4f} ms "
          f"min {min(ts):.4f} ms  {byt / (med * 1e-3) / 1e9:.0f} GB/s")


if __name__ == "__main__":
    main()
