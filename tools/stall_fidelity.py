"""The one unpinned part of the method, measured: the stall model (R-stall, per-layer overflow of
load / B over the Eq. 1 budget) against the real slowdown of a Llama-2 7B training step (bf16,
workloads/llama.py) whose saved activations the runtime swaps with the swap kernels, overlapped
with compute, on one B200.

For each HBM budget (M0 + frac x no-swap activation peak) the runtime re-plans on a Detailed step
and then runs `--steps` policy steps.  Per budget: the plan's predicted peak and stall, the
measured peak allocated and the measured step time minus the no-swap step time.  Prints one JSON
line.

    python tools/stall_fidelity.py [--batch 4] [--seq 4096] [--fracs 0.4,0.5,...] [--steps 3]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200 import chm  # noqa: E402
from paper_2509_11076_b200.runtime import Runtime  # noqa: E402
from workloads import llama as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--seq", type=int, default=4096)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--fracs", default="0.9,0.8,0.7,0.6,0.5,0.4,0.3")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--arena-gib", type=float, default=80.0)
    ap.add_argument("--swap-ctas", type=int, default=0, help="swap kernel CTAs (0: the library default, 8)")
    ap.add_argument("--flags", default="auto", choices=["kernel", "ce", "auto"])
    ap.add_argument("--model", default="llama", choices=["llama", "gpt2xl"],
                    help="gpt2xl: GPT-2 XL shape (48 layers, d 1600, 25 heads), fp32, attention written "
                         "out (scores materialised), workloads/tiny_gpt.py; use --seq 1024 --batch 4")
    ap.add_argument("--stall-model", default="layer", choices=["layer", "timeline"],
                    help="the stall that ranks the runtime's plans (R-stall or the timeline)")
    args = ap.parse_args()
    if args.model == "llama":
        cfg = dict(L.LLAMA2_7B, n_layer=args.layers)
        model = L.make(cfg, max_seq=args.seq)
        x, y = L.batch(args.batch, args.seq, cfg["vocab"])
    else:
        from workloads import tiny_gpt as G
        args.layers = 48
        model = G.make(0, "cuda", vocab=50304, d=1600, n_layer=48, n_head=25, seq=args.seq)
        x, y = G.batches(1, args.batch, args.seq, 50304, seed=1, device="cuda")[0]
    opt = torch.optim.SGD(model.parameters(), lr=1e-5)

    def one(rt=None):
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        base = torch.cuda.memory_allocated()
        t0 = time.perf_counter()
        cm = rt.step() if rt is not None else None
        if cm is not None:
            cm.__enter__()
        loss = model(x, y)
        loss.backward()
        opt.step()
        opt.zero_grad(set_to_none=True)
        if cm is not None:
            cm.__exit__(None, None, None)
        torch.cuda.synchronize()
        return time.perf_counter() - t0, torch.cuda.max_memory_allocated() - base

    plain = [one() for _ in range(3)][1:]
    t_plain = min(t for t, _ in plain)
    act_peak = max(p for _, p in plain)
    m0 = torch.cuda.memory_allocated()
    flags = dict(kernel=chm.SWAP_KERNEL, ce=chm.SWAP_CE, auto=chm.SWAP_AUTO)[args.flags]
    rt = Runtime(0, hbm_budget=m0 + act_peak, groups_fwd=args.layers, groups_bwd=args.layers,
                 host_arena_bytes=int(args.arena_gib * 2 ** 30), swap_ctas=args.swap_ctas, swap_flags=flags,
                 trials=1,  # one plan per budget
                 stall_model=chm.STALL_TIMELINE if args.stall_model == "timeline" else chm.STALL_LAYER)
    for _ in range(4):  # WarmUp -> GenPolicy; the first plan fits (no policy)
        one(rt)
    rows = []
    for frac in [float(f) for f in args.fracs.split(",")]:
        rt.uninstall()
        t_np, _ = one(rt)  # a step without policy: T_iter for Eq. 1
        rt.request_replan(m0 + int(frac * act_peak))
        one(rt)
        plan = rt.plans[-1]
        models = rt.policy[0].stall_models(rt.policy_items) if rt.policy is not None else np.zeros(3)
        meas = [one(rt) for _ in range(args.steps)]
        t_pol = sorted(t for t, _ in meas)[len(meas) // 2]
        peak = max(p for _, p in meas) + m0
        rows.append(dict(frac=frac, budget_gib=round((m0 + frac * act_peak) / 2 ** 30, 3), kind=plan.get("kind"),
                         swapped_gib=round(plan.get("swapped", 0) / 2 ** 30, 3), items=plan.get("items", 0),
                         predicted_peak_gib=round(plan.get("peak", plan["peak0"]) / 2 ** 30, 3),
                         measured_peak_gib=round(peak / 2 ** 30, 3), excess_gib=round(plan.get("excess", 0) / 2 ** 30, 3),
                         predicted_stall_s=round(plan.get("stall", 0.0), 4), t_iter_s=round(plan["t_iter"], 4),
                         stall_layer_s=round(float(models[0]), 4), stall_per_direction_s=round(float(models[1]), 4),
                         stall_timeline_s=round(float(models[2]), 4),
                         step_s=round(t_pol, 4), measured_overhead_s=round(t_pol - t_np, 4), plan_ms=round(plan["plan_ms"], 1)))
    out = dict(flags=args.flags, swap_ctas=args.swap_ctas or 8, stall_model=args.stall_model,
               model=("gpt2-xl-fp32" if args.model == "gpt2xl" else
                      "llama2-7b" if args.layers == 32 else f"llama2-7b-{args.layers}L"), dtype="fp32" if args.model == "gpt2xl" else "bf16", batch=args.batch,
               seq=args.seq, m0_gib=round(m0 / 2 ** 30, 3), no_swap_peak_gib=round((m0 + act_peak) / 2 ** 30, 3),
               plain_step_s=round(t_plain, 4), bw_GBps=round(rt.bw / 1e9, 2), rows=rows, exec=rt.ctx.exec_stats(),
               demand_swap_in=rt.stats["demand_swap_in"])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
