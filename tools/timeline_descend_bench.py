"""The runtime's default planner search (timeline stall ranking): the descents from each R-base's
best SEEDED mask one after the other (runtime.descend, one FLIP1 launch per round and start)
against the same descents in lockstep (runtime.descend_many, one MASKS launch per round for all
still-moving starts).  Same end keys; wall clock (synchronised), median of 3.  One JSON line per
config.

    python tools/timeline_descend_bench.py [C2 C3h ...]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200 import chm  # noqa: E402
from paper_2509_11076_b200.runtime import (_generate_all, _key3, default_bases, descend, descend_many,  # noqa: E402
                                           device_descend, seeded_multibase)
from workloads import traces as W  # noqa: E402

DEV = torch.device("cuda:0")
TL = chm.STALL_TIMELINE


def main():
    names = [a for a in sys.argv[1:]] or ["C2", "C3h", "C4b", "C5"]
    for name in names:
        tr = W.CONFIGS[name]()
        sd = W.SEEDED[name[:2]]
        ctx = chm.Context(device=0, host_arena_bytes=1 << 20)
        ctx.set_detailed(True)
        chm.record_iteration(ctx, tr)
        ctx.detect_seq_change(tr.t_iter)
        pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
        gen = _generate_all(pt)
        best = torch.empty(5, dtype=torch.int64, device=DEV)
        gkeys = []
        for g in gen:
            ctx.eval_policies(pt, chm.EXPLICIT, 0, 1, best=best, item_offsets=np.array([0, len(g)], np.uint64), items=g)
            gkeys.append(best.cpu().numpy().view(chm.BEST_DTYPE)[0].copy())
        _, _, _, per = seeded_multibase(ctx, pt, default_bases(pt, gen, gkeys), 100_000, sd["seed"], sd["flip_thr"],
                                        DEV, TL)
        starts = [(k.copy(), np.array(w, np.uint64)) for k, w in per.values()]
        seq_t, lock_t = [], []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            seq = [descend(ctx, pt, k, w, DEV, 4096, TL) for k, w in starts]
            seq_t.append(time.perf_counter() - t0)
            t0 = time.perf_counter()
            lock = descend_many(ctx, pt, starts, DEV, 4096, TL)
            lock_t.append(time.perf_counter() - t0)
        same = all(_key3(a[0]) == _key3(b[0]) and a[2] == b[2] for a, b in zip(seq, lock))
        kb = min((e[0] for e in lock), key=_key3)
        # extra starts: the R-stall descents' end points (chm_descend), scored under the timeline
        ext_t = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rs = device_descend(ctx, pt, [w for _, w in starts], DEV)
            extra = []
            for _, w, _ in rs:
                ctx.eval_policies(pt, chm.FLIP1, pt.K, 1, best=best, base=w, stall_model=TL)
                extra.append((best.cpu().numpy().view(chm.BEST_DTYPE)[0].copy(), np.array(w, np.uint64)))
            lock2 = descend_many(ctx, pt, starts + extra, DEV, 4096, TL)
            ext_t.append(time.perf_counter() - t0)
        kb2 = min((e[0] for e in lock2), key=_key3)
        print(json.dumps({"config": name, "K": pt.K, "starts": len(starts), "rounds": [e[2] for e in lock],
                          "sequential_ms": float(np.median(seq_t)) * 1e3, "lockstep_ms": float(np.median(lock_t)) * 1e3,
                          "same_ends": same, "best_stall_s": float(kb["stall"]),
                          "best_excess_gib": int(kb["excess"]) / 2 ** 30,
                          "with_rstall_starts": {"ms": float(np.median(ext_t)) * 1e3, "rounds": [e[2] for e in lock2],
                                                 "best_stall_s": float(kb2["stall"]),
                                                 "best_excess_gib": int(kb2["excess"]) / 2 ** 30,
                                                 "best_swapped_gb": int(kb2["swapped_bytes"]) / 1e9},
                          "best_swapped_gb": int(kb["swapped_bytes"]) / 1e9}), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
