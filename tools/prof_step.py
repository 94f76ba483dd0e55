"""Short driver for ncu: the C2 hot-path kernels at bench sizes, without the 97 GB policy.

  eval: chm_eval_policies, 10^5 SEEDED candidates, full mode (per-op footprints), 3 launches
  swap: one 1 GiB batch of 64 descriptors out and back in (kernel path), 2 round trips
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200 import chm  # noqa: E402
from workloads import traces as W  # noqa: E402


def main():
    full = "--search" not in sys.argv
    tr = W.gpt2_xl()
    sd = W.SEEDED["C2"]
    ctx = chm.Context(device=0, host_arena_bytes=1 << 30, swap_ctas=int(os.environ.get("SWAP_CTAS", "32")))
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    n = 100_000
    ld = (pt.N + 1) // 2 * 2
    dev = torch.device("cuda:0")
    peak = torch.empty(n, dtype=torch.int64, device=dev)
    stall = torch.empty(n, dtype=torch.float64, device=dev)
    fp = torch.empty((n, ld), dtype=torch.int64, device=dev) if full else None
    best = torch.empty(5, dtype=torch.int64, device=dev)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for it in range(3):
        s.record()
        ctx.eval_policies(pt, chm.SEEDED, 0, n, best=best, seed=sd["seed"], flip_thr=sd["flip_thr"], peak=peak,
                          stall=stall, footprint=fp, ld=ld if full else 0)
        e.record()
        torch.cuda.synchronize()
        print(f"eval {it}: {s.elapsed_time(e):.3f} ms  ({n / s.elapsed_time(e) * 1e3 / 1e6:.1f} M cand/s)")
    nb = (1 << 30) // 64
    bufs = [torch.empty(nb, dtype=torch.uint8, device=dev) for _ in range(64)]
    descs = [(b.data_ptr(), j * nb, nb) for j, b in enumerate(bufs)]
    comp, sw = torch.cuda.current_stream(), torch.cuda.Stream()
    for it in range(2):
        s.record(sw)
        ctx.swap_out(descs, comp, sw)
        e.record(sw)
        torch.cuda.synchronize()
        t_out = s.elapsed_time(e)
        s.record(sw)
        ctx.swap_in(descs, comp, sw)
        e.record(sw)
        torch.cuda.synchronize()
        print(f"swap {it}: out {(1 << 30) / t_out / 1e6:.1f} GB/s  in {(1 << 30) / s.elapsed_time(e) / 1e6:.1f} GB/s")


if __name__ == "__main__":
    main()
