"""Batched descent (runtime.descend(batch=...)): the best 2 .. batch improving flips of a FLIP1
round tried together in one MASKS launch.  For C2 / C3 / C4b / C5 and both stall models: the key
after descending from the best of 10^5 SEEDED candidates, the rounds and the wall time, for
batch = 1 (single flip per round) and 4 / 8 / 16.

    python tools/descent_batch.py  ->  gpurun_out/descent_batch.json"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200 import chm  # noqa: E402
from paper_2509_11076_b200.runtime import descend  # noqa: E402
from workloads import traces as W  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    out = []
    for name in ("C2", "C3", "C4b", "C5"):
        tr = W.CONFIGS[name]()
        sd = W.SEEDED[name[:2]]
        ctx = chm.Context(device=0)
        ctx.set_detailed(True)
        chm.record_iteration(ctx, tr)
        ctx.detect_seq_change(tr.t_iter)
        pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
        for model, mname in ((chm.STALL_LAYER, "layer"), (chm.STALL_TIMELINE, "timeline")):
            best = torch.empty(5, dtype=torch.int64, device=dev)
            ctx.eval_policies(pt, chm.SEEDED, 0, 100_000, best=best, seed=sd["seed"], flip_thr=sd["flip_thr"],
                              stall_model=model)
            k0 = best.cpu().numpy().view(chm.BEST_DTYPE)[0]
            w0 = pt.candidate_mask(chm.SEEDED, int(k0["index"]), seed=sd["seed"], flip_thr=sd["flip_thr"])
            for b in (1, 4, 8, 16):
                descend(ctx, pt, k0, w0, dev, 3, model, b)  # warm-up
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                k, w, r = descend(ctx, pt, k0, w0, dev, 4096, model, b)
                dt = time.perf_counter() - t0
                row = dict(config=name, model=mname, batch=b, rounds=r, ms=round(dt * 1e3, 2),
                           excess=int(k["excess"]), stall=float(k["stall"]), swapped=int(k["swapped_bytes"]))
                print(json.dumps(row), flush=True)
                out.append(row)
        ctx.close()
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/descent_batch.json", "w"), indent=1)


if __name__ == "__main__":
    main()
