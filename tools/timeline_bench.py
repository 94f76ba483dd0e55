"""Timeline stall model in the search (csrc/timeline.cu) vs the layer model (R-stall): device
time of one chm_eval_policies launch over 10^5 SEEDED candidates (search mode) on C2 / C3 / C5,
CUDA events on the launching stream, median of 20 after 3 warm-ups; and how different the two
winners are (the timeline stall of the R-stall winner vs the timeline winner).

    python tools/timeline_bench.py   ->  gpurun_out/timeline_bench.json"""
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
    out = {}
    for name in ("C2", "C3", "C5"):
        tr = W.CONFIGS[name]()
        sd = W.SEEDED[name]
        ctx = chm.Context(device=0)
        ctx.set_detailed(True)
        chm.record_iteration(ctx, tr)
        ctx.detect_seq_change(tr.t_iter)
        ctx.set_detailed(False)
        pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
        n = 100_000
        peak = torch.empty(n, dtype=torch.int64, device=dev)
        stall = torch.empty(n, dtype=torch.float64, device=dev)
        swapped = torch.empty(n, dtype=torch.int64, device=dev)
        best = torch.empty(5, dtype=torch.int64, device=dev)
        row = {"ops": pt.N, "K": pt.K, "L": pt.L}
        stalls = {}
        for model, nm in ((chm.STALL_LAYER, "layer"), (chm.STALL_TIMELINE, "timeline")):
            def run():
                ctx.eval_policies(pt, chm.SEEDED, 0, n, best=best, seed=sd["seed"], flip_thr=sd["flip_thr"],
                                  peak=peak, stall=stall, swapped=swapped, stall_model=model)
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            ts = []
            for _ in range(20):
                torch.cuda._sleep(1_000_000)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            b = best.cpu().numpy().view(chm.BEST_DTYPE)[0]
            stalls[nm] = stall.cpu().numpy().copy()
            row[nm] = {"ms": float(np.median(ts)), "candidates_per_s": n / (np.median(ts) * 1e-3),
                       "best_index": int(b["index"]), "best_excess": int(b["excess"]),
                       "best_stall_s": float(b["stall"])}
        il = row["layer"]["best_index"]
        row["timeline_stall_of_layer_winner_s"] = float(stalls["timeline"][il])
        row["rank_corr_note"] = "Spearman rho of the two stalls over all candidates"
        ra = np.argsort(np.argsort(stalls["layer"]))
        rb = np.argsort(np.argsort(stalls["timeline"]))
        row["spearman"] = float(np.corrcoef(ra, rb)[0, 1])
        out[name] = row
        print(name, json.dumps(row), flush=True)
        ctx.close()
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/timeline_bench.json", "w"), indent=1)


if __name__ == "__main__":
    main()
