"""Host cost of the runtime in its Stable stage (a policy installed: per-op matching, swap issue,
releases, swap-ins) on a host-bound and on a device-bound model, against the plain step and
against the Lightweight (no policy) step; with the C++ dispatch hook (csrc/hook.cpp) and with
the Python TorchDispatchMode.  Step time (to the final synchronize: includes the device waiting on
swap-ins over the host link) and host time (until the step is enqueued: the hook, the matching,
the swap issue).  Prints one JSON line.

    python tools/stable_cost.py  ->  stdout"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200.runtime import Runtime  # noqa: E402
from workloads import tiny_gpt as G  # noqa: E402


def run(cfg, batch, frac, native=True):
    dev = torch.device("cuda:0")
    m = G.make(0, dev, **cfg)
    opt = torch.optim.SGD(m.parameters(), lr=0.01)
    x, y = G.batches(1, batch, cfg["seq"], cfg["vocab"], seed=1, device=dev)[0]

    host = []  # host time to enqueue the step (hook, matching, swap issue), before the sync

    def step(cm=None):
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        base = torch.cuda.memory_allocated()
        t0 = time.perf_counter()
        if cm is not None:
            cm.__enter__()
        loss = m(x, y)
        loss.backward()
        opt.step()
        opt.zero_grad(set_to_none=True)
        if cm is not None:
            cm.__exit__(None, None, None)
        host.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
        return time.perf_counter() - t0, torch.cuda.max_memory_allocated() - base

    for _ in range(3):
        step()
    host.clear()
    plain = sorted(step()[0] for _ in range(7))[3]
    plain_host = sorted(host)[3]
    peak = max(step()[1] for _ in range(2))
    light_rt = Runtime(0, hbm_budget=1 << 62, bw=50e9, native_hook=native)
    host.clear()
    light = sorted(step(light_rt.step())[0] for _ in range(5))[2]
    light_host = sorted(host)[2]
    ops = light_rt.last_step["ops"]
    own_light = None
    if native:
        light_rt.host_timing = True
        costs = []
        for _ in range(5):
            step(light_rt.step())
            costs.append(light_rt.host_cost)
        c = sorted(costs, key=lambda x: x["total_s"])[2]
        own_light = dict(c, us_per_op=c["total_s"] / c["ops"] * 1e6)
    light_rt.close()
    rt = Runtime(0, hbm_budget=torch.cuda.memory_allocated() + int(frac * peak), groups_fwd=cfg["n_layer"],
                 groups_bwd=cfg["n_layer"], trials=1, native_hook=native)
    for _ in range(12):  # WarmUp -> GenPolicy (plan) -> Stable
        step(rt.step())
    host.clear()
    stable = sorted(step(rt.step())[0] for _ in range(7))[3]
    stable_host = sorted(host)[3]
    own = None
    if native:  # the runtime's own host time in a Stable step: hook + matching + actions + pack / unpack
        rt.host_timing = True
        costs = []
        for _ in range(5):
            step(rt.step())
            costs.append(rt.host_cost)
        rt.host_timing = False
        c = sorted(costs, key=lambda x: x["total_s"])[2]
        own = dict(c, us_per_op=c["total_s"] / c["ops"] * 1e6)
    st = rt.stats
    rt.close()
    return dict(hook="C++ dispatch fallback" if native else "Python TorchDispatchMode", ops=ops,
                plain_ms=plain * 1e3, lightweight_ms=light * 1e3, stable_ms=stable * 1e3,
                stable_over_plain=stable / plain - 1, us_per_op_stable=(stable - plain) / ops * 1e6,
                us_per_op_lightweight=(light - plain) / ops * 1e6, lightweight_over_plain=light / plain - 1,
                host_ms={"plain": plain_host * 1e3, "lightweight": light_host * 1e3, "stable": stable_host * 1e3},
                host_us_per_op={"lightweight": (light_host - plain_host) / ops * 1e6,
                                "stable": (stable_host - plain_host) / ops * 1e6},
                stable_swap_bytes_per_step=st["released_bytes"] / max(1, st["steps"]),
                stable_runtime_host_cost=own, lightweight_runtime_host_cost=own_light,
                swap_out_per_step=st["swap_out"] / max(1, st["steps"]), budget_frac=frac)


def main():
    out = {}
    for native in (True, False):
        tag = "native" if native else "python"
        out[f"host_bound_tiny_gpt_{tag}"] = run(dict(vocab=512, d=256, n_layer=6, n_head=8, seq=256), 16, 0.55, native)
        out[f"device_bound_gpt_d1024_{tag}"] = run(dict(vocab=8192, d=1024, n_layer=12, n_head=16, seq=1024), 16,
                                                   0.55, native)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
