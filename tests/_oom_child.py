"""Child process of tests/test_gpu_runtime_oom.py (a per-process memory cap must not leak into the
other tests): trains the GPT-style model uncapped, then under a cap below its no-swap peak with
and without the runtime's Algo. 3 handling; prints one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200.runtime import Runtime  # noqa: E402
from workloads import tiny_gpt as G  # noqa: E402

CFG = dict(vocab=512, d=256, n_layer=6, n_head=8, seq=256)


def train(rt=None, steps=10):
    dev = torch.device("cuda:0")
    model = G.make(0, dev, **CFG)
    opt = torch.optim.SGD(model.parameters(), lr=0.05)
    data = G.batches(steps, 16, CFG["seq"], CFG["vocab"], seed=1, device=dev)
    losses = []
    for x, y in data:
        if rt is None:
            loss = model(x, y)
            loss.backward()
        else:
            with rt.step():
                loss = model(x, y)
                loss.backward()
                opt.step()
                opt.zero_grad(set_to_none=True)
        if rt is None:
            opt.step()
            opt.zero_grad(set_to_none=True)
        losses.append(float(loss.detach()))
    params = torch.cat([p.detach().flatten() for p in model.parameters()]).cpu()
    return losses, params


def main():
    frac = float(sys.argv[1])
    budget_frac = float(sys.argv[2]) if len(sys.argv) > 2 else None  # plan a policy for this budget
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    ref_losses, ref_params = train()
    peak = torch.cuda.max_memory_allocated() - base
    torch.cuda.empty_cache()
    total = torch.cuda.get_device_properties(0).total_memory
    budget = (1 << 62) if budget_frac is None else torch.cuda.memory_allocated() + int(budget_frac * peak)
    hook = os.environ.get("CHM_OOM_HOOK")  # "native" / "python": force the hook (default: the runtime's choice)
    rt = Runtime(0, hbm_budget=budget, groups_fwd=6, groups_bwd=6, oom_host_bytes=1 << 30, trials=1,
                 native_hook=None if hook is None else hook == "native",
                 defrag=os.environ.get("CHM_OOM_DEFRAG") == "1")
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    cap = torch.cuda.memory_reserved() + int(frac * peak)
    torch.cuda.set_per_process_memory_fraction(cap / total)
    out = dict(peak=int(peak), cap=int(cap))
    try:
        train()
        out["plain_under_cap"] = "ok"
    except torch.OutOfMemoryError:
        out["plain_under_cap"] = "oom"
    import gc
    gc.collect()
    torch.cuda.empty_cache()
    try:
        losses, params = train(rt)
    except torch.OutOfMemoryError as e:
        print(json.dumps(dict(out, error=str(e)[:300], oom_log=list(rt.oom_log), stats=rt.stats)))
        raise
    out.update(losses_equal=losses == ref_losses, params_equal=bool(torch.equal(params, ref_params)),
               stats=rt.stats, stages=rt.stage, plans=[{k: v for k, v in p.items() if k != "tensors"} for p in rt.plans])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
