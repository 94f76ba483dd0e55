"""NEXT-4 evidence: one GPT-2 XL (s=512, b=1) iteration under a cap on the produced bytes, Algo. 3
handling every overflow (tools/oom_driver.py), for several caps; per cap: passive swaps, demand
restores, early releases, wall time of the iteration, and whether the Fig. 3 reconstruction
(f0_source = 1: measured bytes + swap log) equals the F0 from the recorded events (f0_source =
0).  (The oracle comparison of both: tests/test_gpu_oom.py.)  Prints one JSON line.

    python tools/oom_warmup.py
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200 import chm  # noqa: E402
from tools.oom_driver import run_capped  # noqa: E402
from workloads import traces as W  # noqa: E402


def main():
    tr = W.gpt2_xl(seq=512, batch=1)
    h = chm.Context(device=-1)
    h.set_detailed(True)
    chm.record_iteration(h, tr)
    h.detect_seq_change(tr.t_iter)
    pt = h.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    act_peak = int(pt.peak0 - tr.static_bytes)
    out = dict(trace=tr.name, ops=tr.n_ops, no_swap_activation_peak=act_peak, runs=[])
    for frac in (1.0, 0.85, 0.7, 0.6, 0.5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        measured, f0_log, f0_ev, st = run_capped(tr, int(act_peak * frac), arena_extra=act_peak)
        dt = time.perf_counter() - t0
        out["runs"].append(dict(mode="warmup", cap_frac=frac, wall_s=round(dt, 3), peak=st["peak"],
                                passive=st["passive"], restored=st["restored"], dropped=st["dropped"],
                                reconstruction_equals_events=bool(np.array_equal(f0_log, f0_ev))))
    sd = W.SEEDED["C2"]
    policy_peak = None
    for frac in (1.0, 0.9, 0.8):
        # cap relative to the SEEDED best policy's own activation peak (first run: uncapped)
        cap = 1 << 62 if policy_peak is None else int(policy_peak * frac)
        t0 = time.perf_counter()
        measured, f0_log, f0_ev, st = run_capped(tr, cap, seeded=(sd["seed"], sd["flip_thr"], 2000),
                                                 arena_extra=act_peak)
        dt = time.perf_counter() - t0
        if policy_peak is None:
            policy_peak = st["peak"]
        out["runs"].append(dict(mode="policy", cap_frac_of_policy_peak=frac, wall_s=round(dt, 3), peak=st["peak"],
                                items=st["items"], early_released=st["early"], passive=st["passive"],
                                restored=st["restored"], swapped_in_checked=st["checked"] - st["restored"],
                                reconstruction_equals_events=bool(np.array_equal(f0_log, f0_ev))))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
