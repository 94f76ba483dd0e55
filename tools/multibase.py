"""SEEDED search around several bases (reading R-bases): for C2, C3h, C4a,
C4b and C5, 10^5 SEEDED candidates around the trace's argmax-window base alone (r01) against the
same 10^5 split over the empty mask, the argmax-window base and Algo. 2's best plan (each base
also scored as it is), then the steepest descent (FLIP1 rounds) from each search's best -- keys,
launch times, rounds.  R-stall ranking (STALL_LAYER).  Prints one JSON line per config.

    python tools/multibase.py [C2 C3h ...]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200 import chm  # noqa: E402
from paper_2509_11076_b200.runtime import _generate_all, default_bases, descend, seeded_multibase  # noqa: E402
from workloads import traces as W  # noqa: E402


def key(k):
    return {"excess_gib": int(k["excess"]) / 2 ** 30, "stall_s": float(k["stall"]),
            "swapped_gb": int(k["swapped_bytes"]) / 1e9}


def main():
    names = [a for a in sys.argv[1:]] or ["C2", "C3h", "C4a", "C4b", "C5"]
    dev = torch.device("cuda:0")
    n = 100_000
    for name in names:
        tr = W.CONFIGS[name]()
        sd = W.SEEDED[name[:2]]
        ctx = chm.Context(device=0, host_arena_bytes=1 << 20)
        ctx.set_detailed(True)
        chm.record_iteration(ctx, tr)
        ctx.detect_seq_change(tr.t_iter)
        pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
        best = torch.empty(5, dtype=torch.int64, device=dev)
        out = {"config": name, "K": pt.K, "peak0_gib": pt.peak0 / 2 ** 30, "budget_gib": pt.budget / 2 ** 30}
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.eval_policies(pt, chm.SEEDED, 0, n, best=best, seed=sd["seed"], flip_thr=sd["flip_thr"])
        k1 = best.cpu().numpy().view(chm.BEST_DTYPE)[0].copy()
        out["single_base"] = dict(key(k1), ms=(time.perf_counter() - t0) * 1e3)
        w1 = pt.candidate_mask(chm.SEEDED, int(k1["index"]), seed=sd["seed"], flip_thr=sd["flip_thr"])
        t0 = time.perf_counter()
        gen = _generate_all(pt)
        gkeys = []
        for g in gen:
            off = np.array([0, len(g)], np.uint64)
            ctx.eval_policies(pt, chm.EXPLICIT, 0, 1, best=best, item_offsets=off, items=g)
            gkeys.append(best.cpu().numpy().view(chm.BEST_DTYPE)[0].copy())
        t_gen = (time.perf_counter() - t0) * 1e3
        t0 = time.perf_counter()
        km, wm, bname, per = seeded_multibase(ctx, pt, default_bases(pt, gen, gkeys), n, sd["seed"], sd["flip_thr"],
                                              dev)
        out["multi_base"] = dict(key(km), ms=(time.perf_counter() - t0) * 1e3, generator_ms=t_gen, base=bname,
                                 per_base={nm: key(x) for nm, (x, _) in per.items()})
        for label, k0, w0 in (("descent_from_single", k1, w1), ("descent_from_multi", km, wm)):
            t0 = time.perf_counter()
            kd, _, r = descend(ctx, pt, k0, w0, dev)
            out[label] = dict(key(kd), rounds=r, ms=(time.perf_counter() - t0) * 1e3)
        # the runtime's planner: a descent from each base's best, the best end point kept
        t0 = time.perf_counter()
        ends = [descend(ctx, pt, kx, wx, dev) for kx, wx in per.values()]
        kb_, _, _ = min(ends, key=lambda e: (int(e[0]["excess"]), float(e[0]["stall"]), int(e[0]["swapped_bytes"])))
        out["descent_from_each_base"] = dict(key(kb_), rounds=sum(e[2] for e in ends),
                                             ms=(time.perf_counter() - t0) * 1e3)
        d = out["descent_from_single"]["stall_s"]
        out["multi_vs_descent_stall"] = (out["multi_base"]["stall_s"] / d) if d > 0 else None
        print(json.dumps(out), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
