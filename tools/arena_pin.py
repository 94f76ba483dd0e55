"""Host arena allocation: cudaHostAlloc (first touch, driver-pinned 4 KiB pages) vs mmap + mbind
to the GPU's NUMA node + THP + parallel pre-fault + cudaHostRegister (chm_config.arena_mode).
For each mode and size: seconds to allocate + pin, then swap bandwidth through that arena
(kernel and copy engines, 1 GiB batch of 64 x 16 MiB) and a byte-exact round trip.

    python tools/arena_pin.py [--sizes-gib 8,32,94] [--threads 8,16,32]

Writes gpurun_out/arena_pin.json."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200 import chm  # noqa: E402


def meminfo(key):
    for line in open("/proc/meminfo"):
        if line.startswith(key + ":"):
            return int(line.split()[1]) * 1024
    return 0


def rd(p):
    try:
        return open(p).read().strip()
    except OSError:
        return None


def bw(ctx, descs, flags, reps=3):
    comp, sw = torch.cuda.current_stream(), torch.cuda.Stream()
    out, inn = [], []
    for _ in range(reps + 1):
        b = ctx.swap_out(descs, comp, sw, flags)
        ctx.batch_wait(b, comp)
        b2 = ctx.swap_in(descs, comp, sw, flags)
        ctx.batch_wait(b2, comp)
        torch.cuda.synchronize()
        out.append(ctx.batch_elapsed_ms(b))
        inn.append(ctx.batch_elapsed_ms(b2))
    n = sum(d[2] for d in descs)
    return n / (np.median(out[1:]) * 1e-3) / 1e9, n / (np.median(inn[1:]) * 1e-3) / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-gib", default="8,32,94")
    ap.add_argument("--threads", default="0")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(0)
    nb = 16 << 20
    bufs = [torch.randint(0, 256, (nb,), dtype=torch.uint8, device=dev, generator=g) for _ in range(64)]
    ref = [b.clone() for b in bufs]
    avail = meminfo("MemAvailable")
    res = {"thp_enabled": rd("/sys/kernel/mm/transparent_hugepage/enabled"),
           "thp_defrag": rd("/sys/kernel/mm/transparent_hugepage/defrag"),
           "numa_online": rd("/sys/devices/system/node/online"), "mem_available": avail,
           "cores": os.cpu_count(), "runs": []}
    for gib in [int(x) for x in a.sizes_gib.split(",")]:
        size = gib << 30
        if size > 0.6 * avail:
            res["runs"].append({"gib": gib, "skipped": f"> 60% of MemAvailable ({avail >> 30} GiB)"})
            continue
        modes = [(chm.ARENA_HOSTALLOC, 0)] + [(chm.ARENA_REGISTER, int(t)) for t in a.threads.split(",")]
        for mode, thr in modes:
            ctx = chm.Context(device=0, time_batches=True, arena_mode=mode, arena_threads=thr)
            huge0 = meminfo("AnonHugePages")
            ctx.arena_reserve(size)
            pl = ctx.arena_placement()
            huge = meminfo("AnonHugePages") - huge0
            # place the batch at the end of the arena (pages touched last by the pre-fault)
            base = size - 64 * nb
            descs = [(b.data_ptr(), base + j * nb, nb) for j, b in enumerate(bufs)]
            k = bw(ctx, descs, chm.SWAP_KERNEL)
            e = bw(ctx, descs, chm.SWAP_CE)
            for b in bufs:
                b.zero_()
            comp, sw = torch.cuda.current_stream(), torch.cuda.Stream()
            ctx.batch_wait(ctx.swap_out([(r.data_ptr(), base + j * nb, nb) for j, r in enumerate(ref)], comp, sw), comp)
            ctx.batch_wait(ctx.swap_in(descs, comp, sw), comp)
            torch.cuda.synchronize()
            exact = all(torch.equal(b, r) for b, r in zip(bufs, ref))
            row = {"gib": gib, "mode": "hostalloc" if mode == chm.ARENA_HOSTALLOC else "register", "threads": thr,
                   "pin_s": pl["pin_s"], "pin_GBps": size / pl["pin_s"] / 1e9, "numa_node": pl["numa_node"],
                   "anon_huge_gib": huge / 2**30, "kernel_d2h": k[0], "kernel_h2d": k[1], "ce_d2h": e[0],
                   "ce_h2d": e[1], "exact": exact}
            res["runs"].append(row)
            print(json.dumps(row), flush=True)
            ctx.close()
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(res, open("gpurun_out/arena_pin.json", "w"), indent=1)


if __name__ == "__main__":
    main()
