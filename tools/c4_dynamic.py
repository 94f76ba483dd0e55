"""C4 (BASELINE.json configs[3]): Llama-2 13B, sequence length switching 2048 -> 8192 -> 2048
mid-run; change detection (Algo. 1) + re-plan through the C ABI.

Schedule: iterations 0-29 at s = 2048, 30-59 at 8192, 60-89 at 2048.  Every iteration goes
through chm_record_op (the profiler hook; Detailed mode whenever the stage machine is in
GenPolicy) and chm_detect_seq_change.  On the first GenPolicy iteration after a change the tool
re-plans: chm_trace_build (host + table upload), chm_eval_policies over 10^5 SEEDED candidates
(GPU), Algo. 2 best-of-n (host + GPU EXPLICIT replay), read-back of the best key -- timed.  It
also replays the stale policy (planned for the previous sequence length) on the new trace: the
"undersized swap" failure of P:126.  Prints one JSON line.

    python tools/c4_dynamic.py [--detect-bytes] [--cos-mode 0|1] [--host-only]
"""
import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200 import chm  # noqa: E402
from paper_2509_11076_b200.runtime import descend  # noqa: E402
from workloads import traces as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--detect-bytes", action="store_true")
    ap.add_argument("--cos-mode", type=int, default=0)
    ap.add_argument("--host-only", action="store_true")
    ap.add_argument("--candidates", type=int, default=100_000)
    args = ap.parse_args()
    short, long_ = W.llama2_13b(2048), W.llama2_13b(8192)
    dev = -1 if args.host_only else 0
    ctx = chm.Context(device=dev, cos_mode=args.cos_mode, detect_bytes=1 if args.detect_bytes else 0)
    L = chm.load()
    preps = {}
    for tr in (short, long_):
        toks = [ctx.tokenize(nm) for nm in tr.op_names]
        ids = np.array([(1 << 60) + int(p) for p in tr.ptr], np.uint64)
        preps[tr.name] = chm.PreparedIteration(tr, ids, toks)
    act = chm.Actions()
    schedule = [short] * 30 + [long_] * 30 + [short] * 30
    log, replans = [], []
    policies = {}
    if not args.host_only:
        import torch
        dev_t = torch.device("cuda:0")
    stage_before = chm.WARMUP
    for it, tr in enumerate(schedule):
        t0 = time.perf_counter()
        for r in preps[tr.name].recs:
            chm._check(L.chm_record_op(ctx.h, ctypes.byref(r), ctypes.byref(act)))
        t_rec = time.perf_counter() - t0
        d = ctx.detect_seq_change(tr.t_iter)
        log.append(dict(it=it, seq=int(tr.meta["shape"]["seq"]), stage=d["stage"], changed=d["changed"],
                        len_diff=round(d["len_diff"], 5), cos=round(d["cos"], 5), record_ms=round(t_rec * 1e3, 2)))
        # this iteration ran in GenPolicy, i.e. was recorded in Detailed mode: re-plan once per phase
        phase = it // 30
        detailed = stage_before == chm.GENPOLICY
        stage_before = d["stage"]
        if detailed and not any(rp["phase"] == phase for rp in replans) and not args.host_only:
            rp = dict(phase=phase, iteration=it, seq=int(tr.meta["shape"]["seq"]))
            t0 = time.perf_counter()
            pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
            rp["trace_build_ms"] = (time.perf_counter() - t0) * 1e3
            sd = W.SEEDED["C4"]
            best = torch.empty(5, dtype=torch.int64, device=dev_t)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ctx.eval_policies(pt, chm.SEEDED, 0, args.candidates, best=best, seed=sd["seed"], flip_thr=sd["flip_thr"])
            bk = best.cpu().numpy().view(chm.BEST_DTYPE)[0]
            rp["eval_ms"] = (time.perf_counter() - t0) * 1e3
            t0 = time.perf_counter()
            gen = [pt.generate_policy(cc, rr)[0] for cc in (0.0, 1.0, 2.0) for rr in (0.5, 1.0, 2.0)]
            off = np.zeros(len(gen) + 1, np.uint64)
            off[1:] = np.cumsum([len(x) for x in gen])
            gbest = torch.empty(5, dtype=torch.int64, device=dev_t)
            ctx.eval_policies(pt, chm.EXPLICIT, 0, len(gen), best=gbest, item_offsets=off, items=np.concatenate(gen))
            gk = gbest.cpu().numpy().view(chm.BEST_DTYPE)[0]
            rp["generator_ms"] = (time.perf_counter() - t0) * 1e3
            rp["replan_ms"] = rp["trace_build_ms"] + rp["eval_ms"] + rp["generator_ms"]
            rp.update(peak0_gib=pt.peak0 / 2 ** 30, budget_gib=pt.budget / 2 ** 30,
                      seeded_best=dict(excess_gib=int(bk["excess"]) / 2 ** 30, stall_s=float(bk["stall"]),
                                       swapped_gib=int(bk["swapped_bytes"]) / 2 ** 30),
                      generator_best=dict(excess_gib=int(gk["excess"]) / 2 ** 30, stall_s=float(gk["stall"]),
                                          swapped_gib=int(gk["swapped_bytes"]) / 2 ** 30))
            words = pt.candidate_mask(chm.SEEDED, int(bk["index"]), seed=sd["seed"], flip_thr=sd["flip_thr"])
            t0 = time.perf_counter()
            dk, words, rounds = descend(ctx, pt, bk, words, dev_t)  # the runtime's refinement
            rp["descent_ms"] = (time.perf_counter() - t0) * 1e3
            rp["replan_with_descent_ms"] = rp["replan_ms"] + rp["descent_ms"]
            rp["descent_best"] = dict(rounds=rounds, excess_gib=int(dk["excess"]) / 2 ** 30, stall_s=float(dk["stall"]),
                                      swapped_gib=int(dk["swapped_bytes"]) / 2 ** 30)
            policies[int(tr.meta["shape"]["seq"])] = (pt, words)
            replans.append(rp)
    out = dict(config=W.CONFIGS["C4a"]().meta["config"], detect_bytes=args.detect_bytes, cos_mode=args.cos_mode,
               detections=[e["it"] for e in log if e["changed"] and e["it"] > 0],
               stages=[e["stage"] for e in log], replans=replans,
               record_ms_per_iteration=float(np.median([e["record_ms"] for e in log])))
    # stale policy: the s=2048 plan (empty: it fits) on the s=8192 trace -> the peak it leaves
    if 8192 in policies and 2048 in policies:
        pt8, _ = policies[8192]
        out["stale_policy_on_8192"] = dict(peak_gib=pt8.peak0 / 2 ** 30, budget_gib=pt8.budget / 2 ** 30,
                                           excess_gib=max(0, pt8.peak0 - pt8.budget) / 2 ** 30,
                                           note="s=2048 fits without swapping (Algo. 2 plans nothing); kept "
                                                "on s=8192 that plan leaves the no-swap peak above the budget: "
                                                "the undersized-swap failure of P:126 that re-planning avoids")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
