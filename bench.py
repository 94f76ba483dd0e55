#!/usr/bin/env python
"""bench.py -- the Chameleon swap hot path on B200 (BASELINE.json metric and configs).

One step = one pass of the whole hot path over the workload's iteration:
  policy evaluation: chm_eval_policies over this rank's shard of the 10^5 SEEDED candidates
  (full mode: every candidate's per-op footprint written), NCCL all-gather + device argmin of
  the per-rank keys (N > 1); policy execution: the installed best policy replayed through the
  profiler hook (chm_record_op per op: App. A matching + trigger tables), swap-outs after a_t,
  stream-ordered releases at r_t, swap-ins before s_t and waits before b_t on real HBM buffers
  and the pinned mapped host arena.
Inputs (activations, trace tables) are resident in HBM when the timed region starts.

value = swap bytes moved by all ranks (D2H + H2D) / step time (device events, max over ranks);
candidates/s of the evaluation is reported beside it.  `e2e` repeats the step through the public
API from host-side records: Detailed recording, trace build + table upload, evaluation, best-key
read-back, policy install, swap execution on the public API's default copy path (CHM_SWAP_AUTO,
what the runtime uses: tensors >= 4 MiB on the copy engines, smaller ones in the kernel); `value`
times the hand-written kernel path alone.

    python bench.py [--gpus N --steps K --warmup W]        # this implementation
    python bench.py --impl reference ...                    # the CPU oracle (reference arm)
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import traces as W  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
PCIE_GEN5_X16_GBPS = 32 * 16 * 128 / 130 / 8  # 63.0 GB/s per direction (nominal)
FAKE_ID_BASE = 1 << 60  # ids of tensors the policy does not swap (never dereferenced)


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:  # noqa: BLE001
        return {"hbm_gbs": 6650.0, "_fallback": True}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="chm", choices=["chm", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--candidates", type=int, default=100_000)
    ap.add_argument("--search-mode", action="store_true", help="no footprint rows (peak/stall/argmin only)")
    ap.add_argument("--swap-ctas", type=int, default=8)
    ap.add_argument("--host-frac", type=float, default=0.6, help="max fraction of host RAM pinned per node")
    ap.add_argument("--ce-steps", type=int, default=1, help="steps of the copy-engine baseline")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--force-dist", action="store_true", help="NCCL argmin path even at N = 1 (one-rank group)")
    return ap.parse_args()


def mem_available():
    for line in open("/proc/meminfo"):
        if line.startswith("MemAvailable:"):
            return int(line.split()[1]) * 1024
    return 0


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    def __init__(self, index: int, enabled: bool = True):
        self.enabled = enabled
        self.index = index
        self.proc = None

    def __enter__(self):
        if self.enabled:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            try:
                self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                              "--format=csv,noheader,nounits", "-lms", "200"],
                                             stdout=self.f, stderr=subprocess.DEVNULL)
            except Exception:  # noqa: BLE001
                self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if self.proc is None:
            return None
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            if len(r) < 9:
                continue
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


# ------------------------------------------------------------------------------- reference arm
def run_reference(args, rank: int):
    """The CPU oracle as it stands, on this box's host cores, on a bounded proportional sample of
    the same workload: evaluate f*C of the candidates and execute f of the best policy's swap
    bytes (out and back) with the oracle's swap-execution definition (memcpy)."""
    if rank != 0:
        return
    import oracle as O
    tr = W.CONFIGS[args.config]()
    sd = W.SEEDED[args.config[:2]]
    m = O.Model(tr)
    cores = os.cpu_count() or 1
    C = args.candidates
    full = m.eval(O.SEEDED, 0, C, seed=sd["seed"], flip_thr=sd["flip_thr"], nthreads=cores)  # setup (untimed)
    best = full["best"]
    bytes_pol = int(best.swapped)
    f = 1.0 / 64
    n_c = max(1, int(C * f))
    n_b = max(1 << 20, int(bytes_pol * f))
    src = np.random.default_rng(0).integers(0, 256, size=n_b, dtype=np.uint8)
    arena = np.empty(n_b, np.uint8)
    back = np.empty(n_b, np.uint8)
    times = []
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        first = (step * n_c) % max(1, C - n_c)
        m.eval(O.SEEDED, first, n_c, seed=sd["seed"], flip_thr=sd["flip_thr"], nthreads=cores,
               footprint=not args.search_mode)
        O.swap_execute([arena.ctypes.data], [src.ctypes.data], [n_b])   # swap-out
        O.swap_execute([back.ctypes.data], [arena.ctypes.data], [n_b])  # swap-in
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
    assert np.array_equal(back, src)
    t = float(np.mean(times))
    value = 2 * n_b / t / 1e9
    sample = (f"per step 1/64 of the workload: {n_c} of {C} SEEDED candidates "
              f"({'search' if args.search_mode else 'full'} mode) + {n_b} of {bytes_pol} policy bytes "
              f"swapped out and back (memcpy, the oracle's swap definition)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": tr.meta["config"], "candidates": C, "candidate_kind": "SEEDED"},
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": sample,
                             "candidates_per_s": n_c / t},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(args, tr, best_swapped: int):
    """The oracle timed on this box's host cores (rank 0, N = 1): a bounded sample, extrapolated
    to the full step (eval of C candidates + swap of the policy bytes out and in)."""
    import oracle as O
    sd = W.SEEDED[args.config[:2]]
    m = O.Model(tr)
    cores = os.cpu_count() or 1
    budget_s = args.cpu_seconds
    n = 2000
    t0 = time.perf_counter()
    m.eval(O.SEEDED, 0, n, seed=sd["seed"], flip_thr=sd["flip_thr"], nthreads=cores, footprint=not args.search_mode)
    dt = time.perf_counter() - t0
    n2 = int(min(args.candidates, max(n, n * (0.5 * budget_s) / max(dt, 1e-6))))
    t0 = time.perf_counter()
    m.eval(O.SEEDED, 0, n2, seed=sd["seed"], flip_thr=sd["flip_thr"], nthreads=cores, footprint=not args.search_mode)
    t_eval = time.perf_counter() - t0
    rate_c = n2 / t_eval
    nb = 1 << 30
    src = np.ones(nb, np.uint8)
    dst = np.empty(nb, np.uint8)
    O.swap_execute([dst.ctypes.data], [src.ctypes.data], [nb])
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        O.swap_execute([dst.ctypes.data], [src.ctypes.data], [nb])
    rate_b = reps * nb / (time.perf_counter() - t0)
    t_step = args.candidates / rate_c + 2 * best_swapped / rate_b
    return {"value": 2 * best_swapped / t_step / 1e9, "unit": "GB/s", "cores": cores, "kind": "oracle",
            "sample": (f"{n2} SEEDED candidates on {cores} threads ({rate_c:.0f} cand/s, "
                       f"{'search' if args.search_mode else 'full'} mode) + 3 x 1 GiB memcpy swap "
                       f"({rate_b / 1e9:.1f} GB/s), extrapolated to the full step"),
            "candidates_per_s": rate_c}


# ----------------------------------------------------------------------------- this repo
def _replan_c4(chm, dev, comp):
    """C4 (Llama-2 13B, s = 8192 after a switch): record one Detailed iteration through
    chm_record_op, build the trace, evaluate 10^5 SEEDED candidates, run Algo. 2's grid (replayed
    as EXPLICIT candidates), refine by steepest descent (MASKS), install -- each step timed"""
    import torch
    from paper_2509_11076_b200.runtime import _generate_all, descend
    tr = W.llama2_13b(8192)
    ctx = chm.Context(device=dev.index, host_arena_bytes=1 << 20)
    ids = np.array([(1 << 60) + int(p) for p in tr.ptr], np.uint64)
    prep = chm.PreparedIteration(tr, ids, [ctx.tokenize(nm) for nm in tr.op_names])
    act = chm.Actions()
    L = chm.load()
    out = {"workload": tr.meta["config"], "ops": tr.n_ops}
    ctx.set_detailed(True)
    t0 = time.perf_counter()
    for r in prep.recs:
        chm._check(L.chm_record_op(ctx.h, ctypes.byref(r), ctypes.byref(act)))
    ctx.detect_seq_change(tr.t_iter)
    out["record_ms"] = (time.perf_counter() - t0) * 1e3
    out["record_ns_per_op"] = out["record_ms"] * 1e6 / tr.n_ops  # host step a1 (+ a2 below)
    t0 = time.perf_counter()
    pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    out["trace_build_ms"] = (time.perf_counter() - t0) * 1e3
    sd = W.SEEDED["C4"]
    best = torch.empty(5, dtype=torch.int64, device=dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.eval_policies(pt, chm.SEEDED, 0, 100_000, best=best, seed=sd["seed"], flip_thr=sd["flip_thr"], stream=comp)
    bk = best.cpu().numpy().view(chm.BEST_DTYPE)[0]
    out["eval_1e5_ms"] = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    gen = _generate_all(pt)
    off = np.zeros(len(gen) + 1, np.uint64)
    off[1:] = np.cumsum([len(x) for x in gen])
    gbest = torch.empty(5, dtype=torch.int64, device=dev)
    ctx.eval_policies(pt, chm.EXPLICIT, 0, len(gen), best=gbest, item_offsets=off, items=np.concatenate(gen))
    gk = gbest.cpu().numpy().view(chm.BEST_DTYPE)[0]
    out["generator_ms"] = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    words = pt.candidate_mask(chm.SEEDED, int(bk["index"]), seed=sd["seed"], flip_thr=sd["flip_thr"])
    dk, words, rounds = descend(ctx, pt, bk, words, dev)
    out["descent_ms"] = (time.perf_counter() - t0) * 1e3
    hctx = chm.Context(device=-1)  # the trigger tables; the arena is reserved ahead in a real run
    t0 = time.perf_counter()
    hctx.policy_install(pt, words)
    out["install_ms"] = (time.perf_counter() - t0) * 1e3
    hctx.close()
    out["replan_ms"] = sum(out[k] for k in ("trace_build_ms", "eval_1e5_ms", "generator_ms", "descent_ms", "install_ms"))
    gib = 2 ** 30
    out.update(peak0_gib=pt.peak0 / gib, budget_gib=pt.budget / gib, descent_rounds=rounds,
               plan={"excess_gib": int(dk["excess"]) / gib, "stall_s": float(dk["stall"]),
                     "swapped_gib": int(dk["swapped_bytes"]) / gib},
               seeded_best={"excess_gib": int(bk["excess"]) / gib, "stall_s": float(bk["stall"])},
               generator_best={"excess_gib": int(gk["excess"]) / gib, "stall_s": float(gk["stall"])})
    # the runtime's default ranking (the timeline stall, csrc/timeline.cu): the same eval and
    # descent under it, single-flip and batched (search_batch = 16)
    tl = {}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.eval_policies(pt, chm.SEEDED, 0, 100_000, best=best, seed=sd["seed"], flip_thr=sd["flip_thr"], stream=comp,
                      stall_model=chm.STALL_TIMELINE)
    tk = best.cpu().numpy().view(chm.BEST_DTYPE)[0]
    tl["eval_1e5_ms"] = (time.perf_counter() - t0) * 1e3
    w0 = pt.candidate_mask(chm.SEEDED, int(tk["index"]), seed=sd["seed"], flip_thr=sd["flip_thr"])
    for b in (1, 16):
        t0 = time.perf_counter()
        k, _, r = descend(ctx, pt, tk, w0, dev, 4096, chm.STALL_TIMELINE, b)
        tl[f"descent_batch{b}"] = {"ms": (time.perf_counter() - t0) * 1e3, "rounds": r,
                                   "excess_gib": int(k["excess"]) / gib, "timeline_stall_s": float(k["stall"])}
    out["timeline_ranking"] = tl
    ctx.close()
    return out


def _traffic(kernel: str, algorithmic_bytes: float):
    """DRAM bytes per launch: the ncu-measured traffic / algorithmic ratio of `kernel`
    (profiles/r01_ncu_traffic.json) times this run's algorithmic bytes per launch; None if absent"""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01_ncu_traffic.json")
    try:
        with open(path) as f:
            return float(json.load(f)[kernel]["ratio"]) * float(algorithmic_bytes)
    except (OSError, KeyError, ValueError):
        return None


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    import torch
    import torch.distributed as dist
    from paper_2509_11076_b200 import chm
    # collectives run whenever a process group is up: N > 1, or --force-dist at N = 1 (the NCCL
    # argmin path exercised on one GPU: a one-rank all-gather)
    use_dist = world > 1 or args.force_dist
    if use_dist:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    P = world

    def barrier():
        if use_dist:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if not use_dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if not use_dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        return float(t.item())

    tr = W.CONFIGS[args.config]()
    sd = W.SEEDED[args.config[:2]]
    ctx = chm.Context(device=local, time_batches=True, swap_ctas=args.swap_ctas)
    tokens = [ctx.tokenize(nm) for nm in tr.op_names]
    # ---- setup (untimed): profile one Detailed iteration, build the trace
    sim_ids = np.array([FAKE_ID_BASE + int(p) for p in tr.ptr], dtype=np.uint64)
    ctx.set_detailed(True)
    rec = chm.PreparedIteration(tr, sim_ids, tokens)
    L = chm.load()
    act = chm.Actions()
    for r in rec.recs:
        chm._check(L.chm_record_op(ctx.h, ctypes.byref(r), ctypes.byref(act)))
    ctx.detect_seq_change(tr.t_iter)
    ctx.set_detailed(False)
    pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    C = args.candidates
    lo, hi = rank * C // P, (rank + 1) * C // P
    cnt = hi - lo
    full = not args.search_mode
    ld = (pt.N + 1) // 2 * 2
    peak = torch.empty(cnt, dtype=torch.int64, device=dev)
    stall = torch.empty(cnt, dtype=torch.float64, device=dev)
    fp = torch.empty((cnt, ld), dtype=torch.int64, device=dev) if full else None
    best_local = torch.empty(5, dtype=torch.int64, device=dev)
    gathered = torch.empty(5 * P, dtype=torch.int64, device=dev)
    best_global = torch.empty(5, dtype=torch.int64, device=dev)
    comp = torch.cuda.current_stream(dev)

    def evaluate(ev_kernel=None):
        ctx.eval_policies(pt, chm.SEEDED, lo, cnt, best=best_local, seed=sd["seed"], flip_thr=sd["flip_thr"],
                          peak=peak, stall=stall, footprint=fp, ld=ld if full else 0, stream=comp)
        if ev_kernel is not None:
            ev_kernel.record(comp)  # replay kernel done; the rest is the argmin exchange
        if use_dist:
            dist.all_gather_into_tensor(gathered, best_local)
            ctx.best_reduce_device(gathered, P, best_global, comp)
        else:
            best_global.copy_(best_local)

    evaluate()
    torch.cuda.synchronize()
    bk = best_global.cpu().numpy().view(chm.BEST_DTYPE)[0]
    words = pt.candidate_mask(chm.SEEDED, int(bk["index"]), seed=sd["seed"], flip_thr=sd["flip_thr"])
    tb = pt.tables()
    sel = [k for k in range(pt.K) if (int(words[k // 64]) >> (k % 64)) & 1]
    # host-RAM guard: the arena is pinned; with many ranks per node keep only a prefix of the
    # policy (mask-bit order) and say so in the JSON line
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(P)))
    budget_pin = int(args.host_frac * mem_available() / max(1, local_world))
    need, keep = 0, []
    for k in sel:
        nb = (int(tb["nbytes"][k]) + 511) // 512 * 512
        if need + nb > budget_pin:
            break
        keep.append(k)
        need += nb
    truncated = len(keep) < len(sel)
    words_exec = np.zeros(pt.W, np.uint64)
    for k in keep:
        words_exec[k // 64] |= np.uint64(1 << (k % 64))
    t0 = time.perf_counter()
    ctx.arena_reserve(max(need, 1 << 20))
    t_pin = time.perf_counter() - t0
    ctx.policy_install(pt, words_exec)
    # real HBM storage for the swapped tensors; their data_ptr becomes the op records' ids
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    storage = {}
    ids = sim_ids.copy()
    for k in keep:
        t = int(tb["tensor"][k])
        buf = torch.empty(int(tr.nbytes[t]) // 8, dtype=torch.int64, device=dev)
        buf.random_(generator=gen)
        storage[t] = buf
        ids[t] = buf.data_ptr()
    item_dev = [storage[int(tb["tensor"][k])].data_ptr() for k in keep]  # swap-in destinations
    real_ids = set(item_dev)
    check_t = [int(tb["tensor"][k]) for k in keep[:: max(1, len(keep) // 8)]]
    check_sum = {t: int(storage[t].sum().item()) for t in check_t}
    run = chm.PreparedIteration(tr, ids, tokens)
    s_out = torch.cuda.Stream(dev)
    s_in = torch.cuda.Stream(dev)
    bytes_swap = sum(int(tb["nbytes"][k]) for k in keep)

    def execute(flags, detailed=False):
        """one iteration of policy execution through the profiler hook; returns launches"""
        if detailed:
            ctx.set_detailed(True)
        launches = 0
        outs, ins = [], []
        h = ctx.h
        for r in run.recs:
            chm._check(L.chm_record_op(h, ctypes.byref(r), ctypes.byref(act)))
            if act.n_swap_out:
                n = act.n_swap_out
                for j in range(n):
                    if act.swap_out[j].dev not in real_ids:
                        raise RuntimeError(f"executor matched a tensor outside the policy at op {len(outs)}")
                outs.append(ctx.issue_swap_out(comp, s_out, flags))
                launches += (n + 63) // 64 if flags == chm.SWAP_KERNEL else 0
            for j in range(act.n_release):
                ctx.item_wait(act.release_item[j], False, comp)
            if act.n_swap_in:
                n = act.n_swap_in
                devs = [item_dev[act.swap_in_item[j]] for j in range(n)]
                ins.append(ctx.issue_swap_in(devs, comp, s_in, flags))
                launches += (n + 63) // 64 if flags == chm.SWAP_KERNEL else 0
            for j in range(act.n_wait):
                ctx.item_wait(act.wait_item[j], True, comp)
        ctx.detect_seq_change(tr.t_iter)
        if detailed:
            ctx.set_detailed(False)
        return launches, outs, ins

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    spin_cycles = 1_000_000  # ~0.5 ms at 1.9 GHz
    # ---- warm-up + timed steps (device loop)
    step_ms, eval_ms, d2h_ms, h2d_ms, argmin_ms = [], [], [], [], []
    ev_k = torch.cuda.Event(enable_timing=True)
    launches = launches_swap = 0
    for step in range(args.warmup):
        evaluate()
        execute(chm.SWAP_KERNEL)
    torch.cuda.synchronize()
    with ClockSampler(local, enabled=not args.no_clocks) as clk:
        for step in range(args.steps):
            barrier()
            torch.cuda.synchronize()
            # a short device-side wait first, so the events bracket the replay kernel itself and
            # not the host's launch latency after an idle GPU
            torch.cuda._sleep(spin_cycles)
            ev[0].record(comp)
            ev[1].record(comp)
            evaluate(ev_k)
            ev[2].record(comp)
            n_l, outs, ins = execute(chm.SWAP_KERNEL)
            ev[3].record(comp)
            torch.cuda.synchronize()
            barrier()
            launches += n_l + 1 + (1 if use_dist else 0)
            launches_swap = n_l
            step_ms.append(ev[0].elapsed_time(ev[3]))
            eval_ms.append(ev[1].elapsed_time(ev_k))
            argmin_ms.append(ev_k.elapsed_time(ev[2]))
            d2h_ms.append(sum(ctx.batch_elapsed_ms(b) for b in outs))
            h2d_ms.append(sum(ctx.batch_elapsed_ms(b) for b in ins))
    clocks = clk.summary()
    st = ctx.exec_stats()
    ok = all(int(storage[t].sum().item()) == check_sum[t] for t in check_t)
    # ---- copy-engine baseline (per-tensor cudaMemcpyAsync on the same batches)
    ce_ms, ce_d2h, ce_h2d = [], [], []
    for step in range(args.ce_steps):
        torch.cuda.synchronize()
        ev[0].record(comp)
        _, outs, ins = execute(chm.SWAP_CE)
        ev[3].record(comp)
        torch.cuda.synchronize()
        ce_ms.append(ev[0].elapsed_time(ev[3]))
        ce_d2h.append(sum(ctx.batch_elapsed_ms(b) for b in outs))
        ce_h2d.append(sum(ctx.batch_elapsed_ms(b) for b in ins))
    ok = ok and all(int(storage[t].sum().item()) == check_sum[t] for t in check_t)
    # ---- AUTO engine selection (tensors >= 4 MiB on the copy engines, the rest in the kernel)
    auto_ms = []
    for step in range(args.ce_steps):
        torch.cuda.synchronize()
        ev[0].record(comp)
        execute(chm.SWAP_AUTO)
        ev[3].record(comp)
        torch.cuda.synchronize()
        auto_ms.append(ev[0].elapsed_time(ev[3]))
    ok = ok and all(int(storage[t].sum().item()) == check_sum[t] for t in check_t)
    # ---- e2e: the GenPolicy loop through the public API from host records
    e2e_ms = []
    table_bytes = 8 * pt.N + 28 * pt.K + 8 * pt.L + 8 * pt.W
    for step in range(args.e2e_steps):
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev[0].record(comp)
        # executes the policy (the public API's default copy path, AUTO: what Runtime uses) and
        # records the iteration
        execute(chm.SWAP_AUTO, detailed=True)
        pt2 = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
        ctx.eval_policies(pt2, chm.SEEDED, lo, cnt, best=best_local, seed=sd["seed"], flip_thr=sd["flip_thr"],
                          peak=peak, stall=stall, footprint=fp, ld=ld if full else 0, stream=comp)
        if use_dist:
            dist.all_gather_into_tensor(gathered, best_local)
            ctx.best_reduce_device(gathered, P, best_global, comp)
        else:
            best_global.copy_(best_local)
        bk2 = best_global.cpu().numpy().view(chm.BEST_DTYPE)[0]  # the step's result, D2H
        w2 = pt2.candidate_mask(chm.SEEDED, int(bk2["index"]), seed=sd["seed"], flip_thr=sd["flip_thr"])
        assert truncated or np.array_equal(w2, words), "re-planned policy differs on an unchanged trace"
        ctx.policy_install(pt2, words_exec if truncated else w2)
        ev[3].record(comp)
        torch.cuda.synchronize()
        e2e_ms.append(max(ev[0].elapsed_time(ev[3]), (time.perf_counter() - t0) * 1e3))
        pt2.free()
    ok = ok and all(int(storage[t].sum().item()) == check_sum[t] for t in check_t)

    # ---- re-plan with the paper's generator (NEXT-1): Algo. 2 for a grid of (C, rem_scale) on the
    # host, then the best of n by a GPU replay of the EXPLICIT item lists
    t0 = time.perf_counter()
    gen_lists = [pt.generate_policy(cc, rr)[0] for cc in (0.0, 0.5, 1.0, 2.0) for rr in (0.5, 1.0, 2.0)]
    t_gen = time.perf_counter() - t0
    off = np.zeros(len(gen_lists) + 1, np.uint64)
    off[1:] = np.cumsum([len(x) for x in gen_lists])
    g_items = np.concatenate(gen_lists)
    g_peak = torch.empty(len(gen_lists), dtype=torch.int64, device=dev)
    g_stall = torch.empty(len(gen_lists), dtype=torch.float64, device=dev)
    g_best = torch.empty(5, dtype=torch.int64, device=dev)
    torch.cuda.synchronize()
    ev[0].record(comp)
    ctx.eval_policies(pt, chm.EXPLICIT, 0, len(gen_lists), best=g_best, peak=g_peak, stall=g_stall,
                      item_offsets=off, items=g_items, stream=comp)
    ev[3].record(comp)
    torch.cuda.synchronize()
    gb = g_best.cpu().numpy().view(chm.BEST_DTYPE)[0]
    generator = {"policies": len(gen_lists), "host_generate_ms": t_gen * 1e3,
                 "gpu_eval_ms": ev[0].elapsed_time(ev[3]), "best_index": int(gb["index"]),
                 "best_peak": int(gb["peak"]), "best_excess": int(gb["excess"]), "best_stall_s": float(gb["stall"]),
                 "seeded_best_excess": int(bk["excess"]), "seeded_best_stall_s": float(bk["stall"])}
    # ---- the same candidates ranked by the timeline stall (csrc/timeline.cu, reading Q11), the
    # runtime's default ranking: device time of one launch (this rank's shard, search mode)
    tl_ms = []
    tl_best = torch.empty(5, dtype=torch.int64, device=dev)
    for it in range(4):
        torch.cuda.synchronize()
        torch.cuda._sleep(spin_cycles)
        ev[0].record(comp)
        ctx.eval_policies(pt, chm.SEEDED, lo, cnt, best=tl_best, seed=sd["seed"], flip_thr=sd["flip_thr"],
                          stall_model=chm.STALL_TIMELINE, stream=comp)
        ev[3].record(comp)
        torch.cuda.synchronize()
        if it:
            tl_ms.append(ev[0].elapsed_time(ev[3]))
    tb_ = tl_best.cpu().numpy().view(chm.BEST_DTYPE)[0]
    eval_timeline = {"ms_per_launch": float(np.mean(tl_ms)), "candidates_per_s": cnt / (np.mean(tl_ms) * 1e-3),
                     "mode": "search (peak / swapped by the replay kernel, then the timeline kernel)",
                     "best_index": int(tb_["index"]), "best_stall_s": float(tb_["stall"]),
                     "layer_best_index": int(bk["index"])}
    # ---- re-plan latency on C4 (BASELINE configs[3]): the sequence switched to s = 8192; from the
    # Detailed iteration's records to an installed policy, through the public API (rank 0 work,
    # reported beside the line; not part of `value`)
    replan = _replan_c4(chm, dev, comp) if rank == 0 else None
    # ---- aggregate (max over ranks of time, sum of work)
    t_step = max_over_ranks(float(np.mean(step_ms)))
    t_eval = max_over_ranks(float(np.mean(eval_ms)))
    t_argmin = max_over_ranks(float(np.mean(argmin_ms)))
    t_d2h = max_over_ranks(float(np.mean(d2h_ms)))
    t_h2d = max_over_ranks(float(np.mean(h2d_ms)))
    tot_bytes = sum_over_ranks(2.0 * bytes_swap)
    value = tot_bytes / (t_step * 1e-3) / 1e9
    fp_bytes = (8 * ld * cnt if full else 0) + 16 * cnt
    hbm_peak = measured_peaks().get("hbm_gbs", 6650.0)
    per_dir = [bytes_swap / (t_d2h * 1e-3) / 1e9 if t_d2h > 0 else 0.0,
               bytes_swap / (t_h2d * 1e-3) / 1e9 if t_h2d > 0 else 0.0]
    ce_dir = ([bytes_swap / (np.mean(ce_d2h) * 1e-3) / 1e9, bytes_swap / (np.mean(ce_h2d) * 1e-3) / 1e9]
              if ce_d2h and ce_h2d else None)
    achieved_swap = 2 * bytes_swap / ((t_d2h + t_h2d) * 1e-3) / 1e9
    e2e_t = max_over_ranks(float(np.mean(e2e_ms))) if e2e_ms else None
    if rank != 0:
        ctx.close()
        if use_dist:
            dist.destroy_process_group()
        return
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "GB/s",
        "n_gpus": P,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic",
        "config": {
            "workload": tr.meta["config"],
            "trace": {"ops": pt.N, "swappable": pt.K, "layers": pt.L, "peak0": pt.peak0, "budget": pt.budget},
            "candidates": C, "candidate_kind": "SEEDED", "candidates_per_rank": cnt,
            "eval_mode": "search" if args.search_mode else "full (per-op footprints written)",
            "policy": {"index": int(bk["index"]), "items": len(sel), "executed_items": len(keep),
                       "truncated_for_host_ram": truncated, "swap_bytes_per_direction": bytes_swap},
            "parallelism": f"dp{P}: per-rank swapping, candidates sharded, NCCL argmin all-gather",
            "l2": "inputs larger than L2 (swap set and footprint rows are GBs per step)",
            "swap_ctas": args.swap_ctas, "arena_pin_s": round(t_pin, 2),
            "arena": ctx.arena_placement(),  # mode 2 = mmap + mbind(GPU's node) + THP + cudaHostRegister
        },
        "roofline": {
            "bound": "pcie", "kernel": "swap_copy_kernel (D2H + H2D)", "achieved": achieved_swap,
            "peak": PCIE_GEN5_X16_GBPS, "unit": "GB/s", "frac": achieved_swap / PCIE_GEN5_X16_GBPS,
            "traffic": _traffic("swap_copy_kernel", 2 * bytes_swap / max(1, launches_swap)),
            "traffic_source": "ncu dram bytes / algorithmic bytes (profiles/r01_ncu_traffic.json) x this run's "
                              "algorithmic bytes per swap launch",
            "peak_source": "nominal PCIe Gen5 x16 per direction (no measured host-link peak in MEASURED_PEAKS.json; "
                           "the box's copy engines reach 57.3 D2H / 55.6 H2D GB/s, tools/probe_box.py)",
            "d2h_GBps": per_dir[0], "h2d_GBps": per_dir[1],
            "frac_of_copy_engines": ({"d2h": per_dir[0] / ce_dir[0], "h2d": per_dir[1] / ce_dir[1],
                                      "what": "vs the same batches on the copy engines (best pinned large-block "
                                              "cudaMemcpyAsync path), this run"} if ce_dir else None),
        },
        "roofline_replay": {
            "bound": "hbm", "kernel": "replay_kernel<%s>" % ("true" if full else "false"),
            "achieved": fp_bytes / (t_eval * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
            "frac": fp_bytes / (t_eval * 1e-3) / 1e9 / hbm_peak,
            "traffic": _traffic("replay_kernel_full", fp_bytes) if full else None,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst)",
            "algorithmic_bytes_per_launch": fp_bytes,
            "frac_of_spec_8TBps": fp_bytes / (t_eval * 1e-3) / 1e9 / 8000.0,
        },
        "argmin_exchange_us": t_argmin * 1e3 if use_dist else None,
        "eval": {"candidates_per_s": C / (t_eval * 1e-3), "ms_per_launch": t_eval, "unit": "candidates/s"},
        "eval_timeline": eval_timeline,
        "ce_baseline": {
            "what": "same batches, one cudaMemcpyAsync per tensor on the copy engines",
            "ms_per_step": float(np.mean(ce_ms)) if ce_ms else None,
            "d2h_GBps": bytes_swap / (np.mean(ce_d2h) * 1e-3) / 1e9 if ce_d2h else None,
            "h2d_GBps": bytes_swap / (np.mean(ce_h2d) * 1e-3) / 1e9 if ce_h2d else None,
            "GBps": 2 * bytes_swap / (np.mean(ce_ms) * 1e-3) / 1e9 if ce_ms else None,
        },
        "auto_mode": {
            "what": "CHM_SWAP_AUTO: tensors >= 4 MiB on the copy engines, the rest in the kernel",
            "ms_per_step": float(np.mean(auto_ms)) if auto_ms else None,
            "GBps": 2 * bytes_swap / (np.mean(auto_ms) * 1e-3) / 1e9 if auto_ms else None,
        },
        "generator": generator,
        "replan_c4": replan,
        "e2e": {"value": tot_bytes / (e2e_t * 1e-3) / 1e9 if e2e_t else None, "unit": "GB/s",
                "copy_path": "CHM_SWAP_AUTO (the runtime's default: >= 4 MiB on the copy engines, smaller in the kernel)",
                "h2d_bytes_per_step": bytes_swap + table_bytes, "d2h_bytes_per_step": bytes_swap + 40,
                "ms_per_step": e2e_t},
        "gpu_launches": launches,
        "gpu_launches_per_step": launches // max(1, args.steps),
        "byte_exact_sample": ok,
        "exec_stats": st,
        "clocks": clocks,
    }
    if P == 1:
        line["cpu_baseline"] = cpu_baseline(args, tr, bytes_swap)
    print(json.dumps(line), flush=True)
    ctx.close()
    if use_dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
