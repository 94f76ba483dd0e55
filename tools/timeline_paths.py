"""Timeline kernel paths by launch size: shared-memory slots (one warp per CTA) vs global-memory
slots (256-thread CTAs), forced with CHM_TL_SMEM, for FLIP1 neighbourhoods (a descent round) and
SEEDED launches of 1k-100k candidates on C2 / C5.  Device time per launch, median of 10.

    python tools/timeline_paths.py  ->  gpurun_out/timeline_paths.json"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200 import chm  # noqa: E402
from workloads import traces as W  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    out = []
    for name in ("C2", "C5"):
        tr = W.CONFIGS[name]()
        sd = W.SEEDED[name]
        ctx = chm.Context(device=0)
        ctx.set_detailed(True)
        chm.record_iteration(ctx, tr)
        ctx.detect_seq_change(tr.t_iter)
        pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
        best = torch.empty(5, dtype=torch.int64, device=dev)
        stall = torch.empty(100_000, dtype=torch.float64, device=dev)
        cases = [("FLIP1", pt.K + 1)] + [("SEEDED", n) for n in (1024, 4736, 18944, 100_000)]
        for kind, n in cases:
            row = dict(config=name, kind=kind, n=n)
            ref = None
            for path in ("0", "1"):
                os.environ["CHM_TL_SMEM"] = path
                ts = []
                for it in range(13):
                    torch.cuda.synchronize()
                    torch.cuda._sleep(200_000)
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record()
                    if kind == "FLIP1":
                        ctx.eval_policies(pt, chm.FLIP1, 0, n, best=best, stall=stall, base=pt.tables()["base"],
                                          stall_model=chm.STALL_TIMELINE)
                    else:
                        ctx.eval_policies(pt, chm.SEEDED, 0, n, best=best, stall=stall, seed=sd["seed"],
                                          flip_thr=sd["flip_thr"], stall_model=chm.STALL_TIMELINE)
                    e.record()
                    torch.cuda.synchronize()
                    if it >= 3:
                        ts.append(s.elapsed_time(e))
                got = stall[:n].cpu().numpy().copy()
                if ref is None:
                    ref = got
                row["same_stalls"] = bool(np.array_equal(ref, got))
                row["smem_ms" if path == "1" else "global_ms"] = float(np.median(ts))
            print(json.dumps(row), flush=True)
            out.append(row)
        os.environ.pop("CHM_TL_SMEM", None)
        ctx.close()
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/timeline_paths.json", "w"), indent=1)


if __name__ == "__main__":
    main()
