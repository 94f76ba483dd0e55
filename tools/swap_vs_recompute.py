"""Context for the paper's claim that swapping beats recomputation (Ascend 910B):
the same Llama-2 7B bf16 step (seq 4096, batch 4, workloads/llama.py) on one B200 with
PyTorch's activation checkpointing (torch.utils.checkpoint, non-reentrant) on every k-th layer,
next to the runtime's swapping at budgets chosen to match each checkpointing peak.  Per
configuration: step time (median of 3 after warm-up) and peak allocated bytes.  Prints one JSON
line.

    python tools/swap_vs_recompute.py
"""
import json
import os
import sys
import time

import torch
import torch.utils.checkpoint as ckpt

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200.runtime import Runtime  # noqa: E402
from workloads import llama as L  # noqa: E402


def main():
    cfg = dict(L.LLAMA2_7B)
    model = L.make(cfg, max_seq=4096)
    opt = torch.optim.SGD(model.parameters(), lr=1e-5)
    x, y = L.batch(4, 4096, cfg["vocab"])
    every = {"k": 0}
    orig_forward = L.Layer.forward

    def layer_forward(self, h, cos, sin):
        if every["k"] and self.idx % every["k"] == 0:
            return ckpt.checkpoint(orig_forward, self, h, cos, sin, use_reentrant=False)
        return orig_forward(self, h, cos, sin)
    for i, layer in enumerate(model.layers):
        layer.idx = i
    L.Layer.forward = layer_forward

    def one(rt=None):
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        t0 = time.perf_counter()
        cm = rt.step() if rt is not None else None
        if cm is not None:
            cm.__enter__()
        model(x, y).backward()
        opt.step()
        opt.zero_grad(set_to_none=True)
        if cm is not None:
            cm.__exit__(None, None, None)
        torch.cuda.synchronize()
        return time.perf_counter() - t0, torch.cuda.max_memory_allocated()

    def med(rt=None, n=3):
        r = [one(rt) for _ in range(n)]
        return sorted(t for t, _ in r)[n // 2], max(p for _, p in r)

    gib = 2 ** 30
    out = dict(model="llama2-7b", batch=4, seq=4096, dtype="bf16", rows=[])
    one()
    t, p = med()
    out["plain"] = dict(step_s=round(t, 4), peak_gib=round(p / gib, 3))
    for k in (4, 2, 1):
        every["k"] = k
        one()
        t, p = med()
        out["rows"].append(dict(mode=f"checkpoint every {k} layer(s)", step_s=round(t, 4), peak_gib=round(p / gib, 3)))
    every["k"] = 0
    for row in list(out["rows"]):
        budget = int(row["peak_gib"] * gib)
        rt = Runtime(0, hbm_budget=budget, groups_fwd=32, groups_bwd=32, host_arena_bytes=int(64 * gib), trials=1)
        for _ in range(4):  # WarmUp -> GenPolicy (plan)
            one(rt)
        t, p = med(rt)
        plan = rt.plans[-1] if rt.plans else {}
        out["rows"].append(dict(mode=f"swap at {row['mode']}'s peak", budget_gib=row["peak_gib"], step_s=round(t, 4),
                                peak_gib=round(p / gib, 3), swapped_gib=round(plan.get("swapped", 0) / gib, 3),
                                predicted_stall_s=round(plan.get("stall", 0.0), 4)))
        rt.close()
        del rt
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
