"""Why the replay launch is slower inside the bench step than back to back: the C3h 10^5-candidate
full-mode launch timed (CUDA events, median of 5) right after (a) another eval launch, (b) an idle
GPU, (c) ~1.3 s of back-to-back bf16 GEMMs (power cap, dirty L2), (d) a 16 GiB device memset
(TLB / L2 churn over other pages), (e) 8 GiB swapped out and back in through the kernel.

    python tools/eval_after.py"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200 import chm  # noqa: E402
from workloads import traces as W  # noqa: E402


def main():
    tr = W.CONFIGS["C3h"]()
    sd = W.SEEDED["C3"]
    ctx = chm.Context(device=0, host_arena_bytes=8 << 30, time_batches=True)
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    n, ld = 100_000, (pt.N + 1) // 2 * 2
    dev = torch.device("cuda:0")
    fp = torch.empty((n, ld), dtype=torch.int64, device=dev)
    best = torch.empty(5, dtype=torch.int64, device=dev)
    comp = torch.cuda.current_stream()
    s_sw = torch.cuda.Stream()
    A = torch.randn(8192, 8192, dtype=torch.bfloat16, device=dev)
    B = torch.randn(8192, 8192, dtype=torch.bfloat16, device=dev)
    Cm = torch.empty(8192, 8192, dtype=torch.bfloat16, device=dev)
    big = torch.empty(16 << 30, dtype=torch.uint8, device=dev)
    swp = torch.empty(8 << 30, dtype=torch.uint8, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def ev():
        e0.record(comp)
        ctx.eval_policies(pt, chm.SEEDED, 0, n, best=best, seed=sd["seed"], flip_thr=sd["flip_thr"], footprint=fp,
                          ld=ld, stream=comp)
        e1.record(comp)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    pre = {
        "after_eval": lambda: ev(),
        "idle_50ms": lambda: time.sleep(0.05),
        "after_gemms_1.3s": lambda: [torch.matmul(A, B, out=Cm) for _ in range(1900)],
        "after_memset_16GiB": lambda: big.fill_(1),
        "after_swap_8GiB_out_in": lambda: [ctx.batch_wait(ctx.swap_out([(swp.data_ptr(), 0, swp.numel())], comp, s_sw),
                                                          comp),
                                           ctx.batch_wait(ctx.swap_in([(swp.data_ptr(), 0, swp.numel())], comp, s_sw),
                                                          comp)],
    }
    for _ in range(3):
        ev()
    out = {}
    for name, f in pre.items():
        ts = []
        for _ in range(5):
            f()
            torch.cuda.synchronize()
            torch.cuda._sleep(1_000_000)
            ts.append(ev())
        out[name] = round(float(np.median(ts)), 4)
        print(name, out[name], flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
