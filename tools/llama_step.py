"""NEXT-2 end goal: a real Llama-2 7B training step (config C3's model, bf16,
seq 4096, workloads/llama.py) under the runtime, on one B200.  The planner's HBM budget is set
below the step's no-swap peak (the oversubscription of C3, scaled to the batch that fits the
box's host RAM for the pinned arena); the runtime profiles, plans after its Detailed step and
swaps the saved activations of every later step with the swap kernels, overlapped with compute.

Per step: wall time (CUDA-synchronised), peak allocated bytes above the step's start, bytes
released / swapped in, stage.  The plain run (no runtime) gives the no-swap peak and step time.
Prints one JSON line.

    python tools/llama_step.py [--batch 4] [--seq 4096] [--layers 32] [--budget-frac 0.6] [--steps 9]
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200.runtime import Runtime  # noqa: E402
from workloads import llama as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--seq", type=int, default=4096)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--budget-frac", type=float, default=0.6, help="budget = M0 + frac x no-swap activation peak")
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--plain-steps", type=int, default=2)
    ap.add_argument("--candidates", type=int, default=1 << 16)
    ap.add_argument("--search-rounds", type=int, default=4096)
    ap.add_argument("--arena-gib", type=float, default=0.0, help="pinned arena reserved at runtime init")
    args = ap.parse_args()
    cfg = dict(L.LLAMA2_7B, n_layer=args.layers)
    model = L.make(cfg, max_seq=args.seq)
    opt = torch.optim.SGD(model.parameters(), lr=1e-5)
    x, y = L.batch(args.batch, args.seq, cfg["vocab"])
    torch.cuda.synchronize()
    out = dict(model="llama2-7b" if args.layers == 32 else f"llama2-7b-{args.layers}L", dtype="bf16", batch=args.batch,
               seq=args.seq, params=sum(p.numel() for p in model.parameters()))

    def one(rt=None):
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        base = torch.cuda.memory_allocated()
        t0 = time.perf_counter()
        ctx = rt.step() if rt is not None else None
        if ctx is not None:
            ctx.__enter__()
        loss = model(x, y)
        loss.backward()
        opt.step()
        opt.zero_grad(set_to_none=True)
        if ctx is not None:
            ctx.__exit__(None, None, None)
        torch.cuda.synchronize()
        return dict(s=round(time.perf_counter() - t0, 4), peak_gib=round((torch.cuda.max_memory_allocated() - base) / 2 ** 30, 3),
                    loss=float(loss.detach()))

    plain = [one() for _ in range(args.plain_steps)]
    out["plain"] = plain
    m0 = torch.cuda.memory_allocated()
    act_peak = int(max(p["peak_gib"] for p in plain) * 2 ** 30)
    budget = m0 + int(args.budget_frac * act_peak)
    out.update(m0_gib=round(m0 / 2 ** 30, 3), budget_gib=round(budget / 2 ** 30, 3))
    t0 = time.perf_counter()
    rt = Runtime(0, hbm_budget=budget, groups_fwd=args.layers, groups_bwd=args.layers, candidates=args.candidates,
                 search_rounds=args.search_rounds, host_arena_bytes=int(args.arena_gib * 2 ** 30))
    out["runtime_init_s"] = round(time.perf_counter() - t0, 3)
    out["bw_measured_GBps"] = round(rt.bw / 1e9, 2)
    steps = []
    for i in range(args.steps):
        before = dict(rt.stats)
        r = one(rt)
        r.update(stage=rt.last_step["stage"], ops=rt.last_step["ops"],
                 released_gib=round((rt.stats["released_bytes"] - before["released_bytes"]) / 2 ** 30, 3),
                 swap_in=rt.stats["swap_in"] - before["swap_in"], demand=rt.stats["demand_swap_in"] - before["demand_swap_in"])
        steps.append(r)
    out["runtime"] = steps
    out["plans"] = [{k: (round(v / 2 ** 30, 3) if k in ("peak0", "budget", "peak", "excess", "swapped") else v)
                     for k, v in p.items() if k != "tensors"} for p in rt.plans]
    out["stats"] = rt.stats
    out["exec"] = rt.ctx.exec_stats()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
