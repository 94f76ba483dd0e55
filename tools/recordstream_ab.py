"""NEXT-3: PyTorch's recordStream vs the custom recordStream of P:391-393, on
B200 with real allocations (PyTorch's stream-ordered caching allocator), real swaps and stand-in
compute per op (a GPU spin of T_iter / N, so the host dispatches ahead of the device).

  custom: the swap-out's block is released after op r_t (the op during which the simulator says
          the copy completes) with an event record/wait between swap and compute streams; no host
          polling
  naive:  Tensor.record_stream(swap_stream) when the swap-out is issued and the reference dropped
          at once; the allocator reuses the block only after it has queried the swap stream's
          event as complete, at a later allocation

Per variant: peak allocated / reserved bytes, bytes x ops the swapped blocks stay allocated
beyond the custom release (mean extra residency in ops per swapped byte), host dispatch time per
op.  (Byte-exactness of the custom path: tests/test_gpu_executor_memory.py.)  Prints one JSON line.

    python tools/recordstream_ab.py [--batch 1] [--op-us 40]
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
from workloads import traces as W  # noqa: E402


def run(tr, sel, variant, op_us, cycles_per_us):
    dev = torch.device("cuda:0")
    m_bytes = int(sum((int(tr.nbytes[t]) + 511) // 512 * 512 for t in sel.values()))
    ctx = chm.Context(device=0, host_arena_bytes=max(m_bytes, 1 << 20))
    tok = [ctx.tokenize(nm) for nm in tr.op_names]
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr, tokens=tok)
    ctx.detect_seq_change(tr.t_iter)
    ctx.set_detailed(False)
    t_iter = tr.n_ops * op_us * 1e-6  # Eq. 1's T_iter = the stand-in compute of the iteration
    pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=t_iter)
    words = np.zeros(max(pt.W, 1), np.uint64)
    for k in sel:
        words[k // 64] |= np.uint64(1 << (k % 64))
    ctx.policy_install(pt, words[:pt.W])
    comp = torch.cuda.current_stream()
    s_out, s_in = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    static = {t: torch.empty(int(tr.nbytes[t]), dtype=torch.uint8, device=dev) for t in range(tr.n_produced, tr.n_tensors)}
    base = torch.cuda.memory_allocated()
    storage, item_tensor = {}, {}
    alloc = np.zeros(tr.n_ops, np.int64)
    spin = int(op_us * cycles_per_us)
    t_host = 0.0
    for i in range(tr.n_ops):
        t0 = time.perf_counter()
        for t in tr.outs(i):
            storage[t] = torch.empty(int(tr.nbytes[t]), dtype=torch.uint8, device=dev)
        torch.cuda._sleep(spin)  # the op's compute
        alloc[i] = torch.cuda.memory_allocated() - base
        ref_of = lambda t: ((storage[t] if t < tr.n_produced else static[t]).data_ptr(), int(tr.nbytes[t]),  # noqa: E731
                            int(tr.dtype[t]))
        act = ctx.record_op(tok[i], int(tr.phase[i]), [ref_of(t) for t in tr.ins(i)],
                            [ref_of(t) for t in tr.outs(i)], [ref_of(t)[0] for t in tr.frees(i)])
        av = chm.actions_view(act)
        for t in tr.frees(i):
            storage.pop(t, None)
        if av["swap_out"]:
            for (d, off, nb), it in zip(av["swap_out"], av["swap_out_item"]):
                t = next(t for t, b in storage.items() if b is not None and b.data_ptr() == d)
                item_tensor[it] = t
            ctx.issue_swap_out(comp, s_out)
            if variant == "naive":
                for it in av["swap_out_item"]:
                    t = item_tensor[it]
                    storage[t].record_stream(s_out)  # PyTorch recordStream
                    storage[t] = None
        for it in av["release"]:
            if variant == "custom":
                ctx.item_wait(it, False, comp)  # event pair, stream-ordered reclaim
                storage[item_tensor[it]] = None
        if av["swap_in"]:
            ptrs = []
            for (d, off, nb), it in zip(av["swap_in"], av["swap_in_item"]):
                storage[item_tensor[it]] = torch.empty(int(nb), dtype=torch.uint8, device=dev)
                ptrs.append(storage[item_tensor[it]].data_ptr())
            ctx.issue_swap_in(ptrs, comp, s_in)
        for it in av["wait"]:
            ctx.item_wait(it, True, comp)
        t_host += time.perf_counter() - t0
    ctx.detect_seq_change(tr.t_iter)
    torch.cuda.synchronize()
    out = dict(peak_allocated=int(torch.cuda.max_memory_allocated() - base),
               peak_reserved=int(torch.cuda.max_memory_reserved()),
               host_us_per_op=t_host / tr.n_ops * 1e6, exec_stats=ctx.exec_stats())
    storage.clear()
    static.clear()
    ctx.close()
    return out, alloc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--op-us", type=float, default=1000.0)
    ap.add_argument("--policy-candidates", type=int, default=2000)
    args = ap.parse_args()
    tr = W.gpt2_xl(batch=args.batch)
    # policy: the best of the SEEDED candidates, evaluated by the product on the GPU
    t_iter = tr.n_ops * args.op_us * 1e-6
    pc = chm.Context(device=0)
    pc.set_detailed(True)
    chm.record_iteration(pc, tr)
    pc.detect_seq_change(tr.t_iter)
    ptp = pc.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=t_iter)
    sd = W.SEEDED["C2"]
    best = torch.empty(5, dtype=torch.int64, device="cuda:0")
    pc.eval_policies(ptp, chm.SEEDED, 0, args.policy_candidates, best=best, seed=sd["seed"], flip_thr=sd["flip_thr"])
    bk = best.cpu().numpy().view(chm.BEST_DTYPE)[0]
    words = ptp.candidate_mask(chm.SEEDED, int(bk["index"]), seed=sd["seed"], flip_thr=sd["flip_thr"])
    tens = ptp.tables()["tensor"]
    sel = {k: int(tens[k]) for k in range(ptp.K) if (int(words[k // 64]) >> (k % 64)) & 1}
    no_swap_peak, policy_peak = int(ptp.peak0 - tr.static_bytes), int(int(bk["peak"]) - tr.static_bytes)
    pc.close()
    # cycles per microsecond of torch.cuda._sleep
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(1000)
    s.record()
    torch.cuda._sleep(10_000_000)
    e.record()
    torch.cuda.synchronize()
    cycles_per_us = 10_000_000 / (s.elapsed_time(e) * 1e3)
    res = {}
    allocs = {}
    for variant in ("custom", "naive"):
        res[variant], allocs[variant] = run(tr, sel, variant, args.op_us, cycles_per_us)
        res[variant]["reserved_over_policy_peak"] = None
    swapped = sum(int(tr.nbytes[t]) for t in sel.values())
    extra = np.maximum(allocs["naive"] - allocs["custom"], 0)
    res["naive_extra_residency_ops_per_swapped_byte"] = float(extra.sum() / max(swapped, 1))
    res["naive_peak_extra_bytes"] = int(extra.max())
    res["config"] = dict(trace=tr.name, batch=args.batch, ops=tr.n_ops, swapped_items=len(sel), swapped_bytes=swapped,
                         op_us=args.op_us, t_iter_s=tr.n_ops * args.op_us * 1e-6,
                         no_swap_peak_bytes=no_swap_peak, policy_peak_bytes=policy_peak)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
