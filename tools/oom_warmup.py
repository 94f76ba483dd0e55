"""NEXT-4 evidence: one GPT-2 XL (s=512, b=1) iteration under a cap on the produced bytes, Algo. 3
handling every overflow (tests/test_gpu_oom.py's driver), for several caps; per cap: passive
swaps, demand restores, early releases, bytes moved, wall time of the iteration and whether the
Fig. 3 reconstruction equals the oracle F0.  Prints one JSON line.

    python tools/oom_warmup.py
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402  (reference F0 and the policy choice; not on the measured path)
from tests.test_gpu_executor_memory import _policy  # noqa: E402
from tests.test_gpu_oom import run_capped  # noqa: E402
from workloads import traces as W  # noqa: E402


def main():
    tr = W.gpt2_xl(seq=512, batch=1)
    act_peak = int(O.Model(tr).f0().max() - tr.static_bytes)
    out = dict(trace=tr.name, ops=tr.n_ops, no_swap_activation_peak=act_peak, runs=[])
    for frac in (1.0, 0.85, 0.7, 0.6, 0.5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m, measured, f0_log, f0_ev, st = run_capped(tr, int(act_peak * frac), arena_extra=act_peak)
        dt = time.perf_counter() - t0
        out["runs"].append(dict(mode="warmup", cap_frac=frac, wall_s=round(dt, 3), peak=st["peak"],
                                passive=st["passive"], restored=st["restored"], dropped=st["dropped"],
                                reconstruction_exact=bool(np.array_equal(f0_log, m.f0())),
                                events_exact=bool(np.array_equal(f0_ev, m.f0()))))
    m0 = O.Model(tr)
    sel = _policy("C2b1", tr, m0)
    sw = m0.swappable()
    fp = m0.replay(sw["t"][sel], sw["r"][sel], sw["s"][sel])["footprint"]
    pol_peak = int(fp.max() - tr.static_bytes)
    for frac in (1.0, 0.9, 0.8):
        t0 = time.perf_counter()
        m, measured, f0_log, f0_ev, st = run_capped(tr, int(pol_peak * frac), sel=sel, arena_extra=act_peak)
        dt = time.perf_counter() - t0
        out["runs"].append(dict(mode="policy", cap_frac_of_policy_peak=frac, wall_s=round(dt, 3), peak=st["peak"],
                                early_released=st["early"], passive=st["passive"], restored=st["restored"],
                                swapped_in_checked=st["checked"] - st["restored"],
                                reconstruction_exact=bool(np.array_equal(f0_log, m.f0())),
                                events_exact=bool(np.array_equal(f0_ev, m.f0()))))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
