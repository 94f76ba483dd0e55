"""Run-to-run D2H variance ("find the cause of the 49.2-51.9 GB/s spread"): pin an
arena of --arena-gib, then for --seconds alternate a 4 GiB swap-out through the kernel and
through the copy engines (and the swap-ins back), recording GB/s per direction over time next to
host-side counters (/proc/vmstat compaction / THP / page-zeroing activity, /proc/loadavg, CPU
time of the host).  A slowdown that decays after the pin points at the host's post-pin work; one
that comes and goes with no local cause points outside the process.

    python tools/d2h_timeline.py [--arena-gib 100] [--seconds 60]"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200 import chm  # noqa: E402

KEYS = ("thp_fault_alloc", "thp_collapse_alloc", "compact_stall", "compact_migrate_scanned", "pgfault", "numa_hit",
        "nr_free_pages", "pgmigrate_success")


def vmstat():
    out = {}
    try:
        for ln in open("/proc/vmstat"):
            k, v = ln.split()
            if k in KEYS:
                out[k] = int(v)
    except OSError:
        pass
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--arena-gib", type=float, default=100.0)
    ap.add_argument("--seconds", type=float, default=60.0)
    args = ap.parse_args()
    nb = 4 << 30
    t_pin0 = time.perf_counter()
    ctx = chm.Context(device=0, host_arena_bytes=int(args.arena_gib * 2 ** 30), swap_ctas=8, time_batches=True)
    t_pin = time.perf_counter() - t_pin0
    dev = torch.device("cuda:0")
    buf = torch.empty(nb, dtype=torch.uint8, device=dev)
    buf.random_(0, 255)
    comp, s = torch.cuda.current_stream(), torch.cuda.Stream()
    hb, hn = ctx.host_arena()
    offs = [0, hn // 2 - nb, hn - nb]  # start, middle, end of the arena
    rows = []
    t0 = time.perf_counter()
    v0 = vmstat()
    i = 0
    while time.perf_counter() - t0 < args.seconds:
        off = offs[i % len(offs)]
        for name, flags in (("kernel", chm.SWAP_KERNEL), ("copy_engines", chm.SWAP_CE)):
            bo = ctx.swap_out([(buf.data_ptr(), off, nb)], comp, s, flags)
            ctx.batch_wait(bo, comp)
            bi = ctx.swap_in([(buf.data_ptr(), off, nb)], comp, s, flags)
            ctx.batch_wait(bi, comp)
            torch.cuda.synchronize()
            v = vmstat()
            rows.append({"t": round(time.perf_counter() - t0, 2), "path": name, "arena_off_gib": round(off / 2 ** 30, 1),
                         "d2h": round(nb / (ctx.batch_elapsed_ms(bo) * 1e-3) / 1e9, 2),
                         "h2d": round(nb / (ctx.batch_elapsed_ms(bi) * 1e-3) / 1e9, 2),
                         "load1": float(open("/proc/loadavg").read().split()[0]),
                         "vmstat_delta": {k: v.get(k, 0) - v0.get(k, 0) for k in KEYS}})
        i += 1
        time.sleep(0.5)
    out = {"arena_gib": args.arena_gib, "pin_s": t_pin, "rows": rows}
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/d2h_timeline.json", "w"))
    for r in rows:
        print(r["t"], r["path"], r["arena_off_gib"], r["d2h"], r["h2d"], r["load1"],
              r["vmstat_delta"].get("compact_migrate_scanned"), r["vmstat_delta"].get("thp_collapse_alloc"), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
