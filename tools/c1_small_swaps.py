"""C1's execution measurement: the 24 activations of the tiny trace (4 KiB - 4 MiB,
log-uniform) swapped out and back in as one batch per direction, 1000 repetitions, through the
swap kernel (one launch per direction) vs one cudaMemcpyAsync per tensor on the copy engines
(and AUTO).  The small-tensor regime, where per-call overhead decides.  Prints one JSON line.

    python tools/c1_small_swaps.py [--reps 1000]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200 import chm  # noqa: E402
from workloads import traces as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=1000)
    args = ap.parse_args()
    tr = W.tiny()
    h = chm.Context(device=-1)
    h.set_detailed(True)
    chm.record_iteration(h, tr)
    h.detect_seq_change(tr.t_iter)
    pt = h.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    sizes = [int(x) for x in pt.tables()["nbytes"]]
    total = sum(sizes)
    ctx = chm.Context(device=0, host_arena_bytes=total + 4096 * len(sizes))
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(1)
    src = [torch.randint(0, 256, (n,), dtype=torch.uint8, device=dev, generator=g) for n in sizes]
    dst = [torch.empty_like(x) for x in src]
    offs = np.concatenate([[0], np.cumsum([(n + 511) // 512 * 512 for n in sizes])[:-1]]).astype(np.uint64)
    d_out = [(x.data_ptr(), int(o), x.numel()) for x, o in zip(src, offs)]
    d_in = [(x.data_ptr(), int(o), x.numel()) for x, o in zip(dst, offs)]
    comp, s = torch.cuda.current_stream(), torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = dict(tensors=len(sizes), bytes=total, min_bytes=min(sizes), max_bytes=max(sizes), reps=args.reps, modes={})
    for name, flags in (("kernel", chm.SWAP_KERNEL), ("copy_engines", chm.SWAP_CE), ("auto", chm.SWAP_AUTO)):
        for rep in range(args.reps + 20):
            if rep == 20:
                torch.cuda.synchronize()
                e0.record(comp)
            b = ctx.swap_out(d_out, comp, s, flags)
            ctx.batch_wait(b, comp)
            b = ctx.swap_in(d_in, comp, s, flags)
            ctx.batch_wait(b, comp)
        e1.record(comp)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        ok = all(torch.equal(a, c) for a, c in zip(src, dst))
        for x in dst:
            x.zero_()
        out["modes"][name] = dict(us_per_round_trip=round(ms * 1e3, 2), GBps=round(2 * total / (ms * 1e-3) / 1e9, 2),
                                  per_direction=("1 kernel launch" if flags == chm.SWAP_KERNEL else
                                                 f"{len(sizes)} cudaMemcpyAsync" if flags == chm.SWAP_CE else
                                                 f"{sum(n >= 4 << 20 for n in sizes)} cudaMemcpyAsync + "
                                                 f"{1 if any(n < 4 << 20 for n in sizes) else 0} kernel launch"),
                                  byte_exact=ok)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
