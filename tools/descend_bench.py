"""Device descent (chm_descend) against the runtime's host-driven descent (one FLIP1 launch and a
host argmin per round), R-stall ranking, per config:
  host:    SEEDED 10^5 around the R-bases (empty / argmax-window / Algo. 2), then runtime.descend
           from each base's best, the best end kept (the runtime's planner; tools/multibase.py);
  device3: one chm_descend launch from the same 3 starts;
  deviceM: device3's starts plus the best distinct SEEDED candidates around the R-bases (per-
           candidate keys of the same 10^5), M = 2 x SMs starts in one chm_descend launch
           (multi-start descent; never worse than device3).
Times are host wall clock around each whole search (synchronised), medians of 3.  Prints one JSON
line per config.

    python tools/descend_bench.py [C2 C3h ...]"""
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

DEV = torch.device("cuda:0")


def key(k):
    return {"excess_gib": int(k["excess"]) / 2 ** 30, "stall_s": float(k["stall"]),
            "swapped_gb": int(k["swapped_bytes"]) / 1e9}


def k3(k):
    return (int(k["excess"]), float(k["stall"]), int(k["swapped_bytes"]))


def dev_descend(ctx, pt, starts):
    n = len(starts)
    st = torch.from_numpy(np.ascontiguousarray(starts).view(np.int64)).to(DEV)
    ends = torch.empty_like(st)
    keys = torch.empty((n, 5), dtype=torch.int64, device=DEV)
    rounds = torch.empty(n, dtype=torch.int32, device=DEV)
    best = torch.empty(5, dtype=torch.int64, device=DEV)
    ctx.descend(pt, st, n, ends=ends, keys=keys, rounds=rounds, best=best)
    b = best.cpu().numpy().view(chm.BEST_DTYPE)[0].copy()
    return b, rounds.cpu().numpy()


def main():
    names = [a for a in sys.argv[1:]] or ["C2", "C3h", "C4a", "C4b", "C5"]
    n = 100_000
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    M = 2 * sms
    for name in names:
        tr = W.CONFIGS[name]()
        sd = W.SEEDED[name[:2]]
        ctx = chm.Context(device=0, host_arena_bytes=1 << 20)
        ctx.set_detailed(True)
        chm.record_iteration(ctx, tr)
        ctx.detect_seq_change(tr.t_iter)
        pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
        out = {"config": name, "K": pt.K, "L": pt.L}
        gen = _generate_all(pt)
        gkeys = []
        best = torch.empty(5, dtype=torch.int64, device=DEV)
        for g in gen:
            ctx.eval_policies(pt, chm.EXPLICIT, 0, 1, best=best, item_offsets=np.array([0, len(g)], np.uint64), items=g)
            gkeys.append(best.cpu().numpy().view(chm.BEST_DTYPE)[0].copy())
        bases = default_bases(pt, gen, gkeys)
        res = {}
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, _, _, per = seeded_multibase(ctx, pt, bases, n, sd["seed"], sd["flip_thr"], DEV)
            t_seeded = time.perf_counter() - t0
            ends = [descend(ctx, pt, kx, wx, DEV) for kx, wx in per.values()]
            kh = min((e[0] for e in ends), key=k3)
            t_host = time.perf_counter() - t0
            res.setdefault("host", []).append((t_host, kh, sum(e[2] for e in ends)))
            # the same 3 starts, one device launch
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            kd3, r3 = dev_descend(ctx, pt, np.stack([wx for _, wx in per.values()]))
            res.setdefault("device3", []).append((t_seeded + time.perf_counter() - t0, kd3, int(r3.sum())))
            # multi-start: the M best distinct SEEDED candidates around the bases
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            pk = torch.empty(n, dtype=torch.int64, device=DEV)
            stl = torch.empty(n, dtype=torch.float64, device=DEV)
            sw = torch.empty(n, dtype=torch.int64, device=DEV)
            starts = [np.ascontiguousarray(wx, np.uint64) for _, wx in per.values()]  # device3's starts
            seen = {x.tobytes() for x in starts}
            nb = len(bases)
            cand = []
            for j, (bn, w) in enumerate(bases):
                lo, hi = j * n // nb, (j + 1) * n // nb
                ctx.eval_policies(pt, chm.SEEDED, lo, hi - lo, best=best, seed=sd["seed"], flip_thr=sd["flip_thr"],
                                  base=w, peak=pk[:hi - lo], stall=stl[:hi - lo], swapped=sw[:hi - lo])
                ex = np.maximum(pk[:hi - lo].cpu().numpy() - pt.budget, 0)
                s_, w_ = stl[:hi - lo].cpu().numpy(), sw[:hi - lo].cpu().numpy()
                order = np.lexsort((np.arange(hi - lo), w_, s_, ex))[:M]
                cand += [((int(ex[i]), float(s_[i]), int(w_[i])), j, lo + int(i)) for i in order]
            cand.sort()
            for _, j, g in cand:
                if len(starts) >= M:
                    break
                m = pt.candidate_mask(chm.SEEDED, g, seed=sd["seed"], flip_thr=sd["flip_thr"], base=bases[j][1])
                t = m.tobytes()
                if t not in seen:
                    seen.add(t)
                    starts.append(m)
            kdm, rm = dev_descend(ctx, pt, np.stack(starts))
            res.setdefault("deviceM", []).append((t_seeded + time.perf_counter() - t0, kdm, int(rm.sum())))
        for label, runs in res.items():
            t = float(np.median([r[0] for r in runs]))
            out[label] = dict(key(runs[-1][1]), ms=t * 1e3, rounds=runs[-1][2])
        out["M"] = M
        out["device3_equals_host"] = k3(res["device3"][-1][1]) == k3(res["host"][-1][1])
        print(json.dumps(out), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
