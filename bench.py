#!/usr/bin/env python
"""bench.py -- the Chameleon swap hot path on B200 (BASELINE.json metric and configs).

One step = one pass of the whole hot path over one training iteration of the
workload:
  policy evaluation: chm_eval_policies over this rank's shard of the 10^5 SEEDED candidates
  (full mode: every candidate's per-op footprint written), NCCL all-gather + device argmin of
  the per-rank keys (N > 1);
  policy execution: the best policy replayed through the profiler hook (chm_record_op per op:
  App. A matching + trigger tables), swap-outs after a_t, stream-ordered releases at r_t,
  swap-ins before s_t and waits before b_t on real HBM buffers and the pinned mapped host
  arena, while each op's compute runs on the compute stream (a bf16 GEMM calibrated to the
  trace's per-op time T_iter / N: the swaps overlap compute as in P:389 / P:428).
Inputs (activations, trace tables) are resident in HBM when the timed region starts.

Workload (default C3h): Llama-2 7B bf16, seq 4096, HBM budget = half the no-swap peak (2x
oversubscription), batch 6 so the whole policy (~106 GB each way) fits the box's pinnable host
RAM (C3 at b = 18 would need ~300 GB pinned).  C2 (GPT-2 1.5B) runs beside it as a
block of its own at N = 1, as do C1's small-tensor swaps and the C4 re-plan.

value = swap bytes moved per GPU (D2H + H2D) / step time (device events, max over ranks);
`value_aggregate` = the sum over ranks / the same time.  Candidates/s of the evaluation, the
swap GB/s per direction during overlap, GEMM TFLOP/s alone / with copy-engine swaps / with the
kernel, and measured vs estimated stall are reported beside it.  `e2e` repeats the step through
the public API from host records (Detailed recording, trace build + table upload, evaluation,
best-key read-back, policy install, execution on the API's default copy path CHM_SWAP_AUTO).

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
GEMM_N = 8192  # stand-in compute: C[M, N] = A[M, N] @ B[N, N], bf16, M calibrated per trace


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:  # noqa: BLE001
        return {"hbm_gbs": 6650.0, "_fallback": True}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="chm", choices=["chm", "reference"])
    ap.add_argument("--config", default="C3h", help="C3h (default), C2, C3, C5, ... (workloads/traces.py)")
    ap.add_argument("--batch", type=int, default=6, help="C3h batch (sized to the box's host RAM)")
    ap.add_argument("--candidates", type=int, default=100_000)
    ap.add_argument("--search-mode", action="store_true", help="no footprint rows (peak/stall/argmin only)")
    ap.add_argument("--swap-ctas", type=int, default=8)
    ap.add_argument("--host-frac", type=float, default=0.6, help="max fraction of host RAM pinned per node")
    ap.add_argument("--no-compute", action="store_true", help="no stand-in GEMMs (swap-only steps)")
    ap.add_argument("--alone-steps", type=int, default=2, help="steps of compute alone (no swaps)")
    ap.add_argument("--ce-steps", type=int, default=1, help="steps of the copy-engine baseline")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--c2-steps", type=int, default=3, help="C2 block steps at N = 1 (0: skip)")
    ap.add_argument("--c1-reps", type=int, default=1000, help="C1 small-tensor block repetitions (0: skip)")
    ap.add_argument("--no-extras", action="store_true", help="skip generator / timeline / C4 re-plan blocks")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--force-dist", action="store_true", help="NCCL argmin path even at N = 1 (one-rank group)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: collectives on host tensors (a functional check of the N > 1 path, not a measurement)")
    ap.add_argument("--same-device", action="store_true",
                    help="every rank on cuda:0 (with --dist-backend gloo: the N > 1 path on one GPU, functional only)")
    return ap.parse_args(argv)


# the paper's own figures (Ascend 910B), context only: it publishes no swap GB/s or candidates/s,
# so vs_baseline stays null
PAPER_CONTEXT = {
    "hardware": "Ascend 910B (PAPER.md P:441-457)",
    "profiler_overhead_pct": {"lightweight": 0.9, "detailed": 34.6},
    "largest_model_vs_device_memory": "up to 4x (P:107)",
    "swap_vs_full_recompute_gain_pct": [18.78, 16.69, 19.32],
    "recordstream_reuse": "custom recordStream reuses blocks 3-4x sooner (P:490)",
    "note": "no published number for either hot-path metric",
}


def workload(args):
    if args.config == "C3h":
        return W.llama2_7b_2x(args.batch)
    return W.CONFIGS[args.config]()


def workload_desc(args, tr):
    d = {"workload": tr.meta["config"], "trace_name": tr.name}
    if args.config == "C3h":
        d["sizing"] = (f"batch {args.batch} (the SEEDED best policy fits 0.6 x the box's ~206 GB host RAM; b = 18 "
                       f"would need ~300 GB pinned); HBM budget = half the no-swap peak (2x oversubscription)")
    return d


def mem_available():
    for line in open("/proc/meminfo"):
        if line.startswith("MemAvailable:"):
            return int(line.split()[1]) * 1024
    return 0


def anon_huge_bytes():
    for line in open("/proc/meminfo"):
        if line.startswith("AnonHugePages:"):
            return int(line.split()[1]) * 1024
    return 0


def thp_mode():
    try:
        t = open("/sys/kernel/mm/transparent_hugepage/enabled").read()
        return t[t.index("[") + 1:t.index("]")]
    except (OSError, ValueError):
        return None


def host_info():
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count() or 1, "cpu_model": model, "mem_available_bytes": mem_available()}


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
    tr = workload(args)
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
              f"swapped out and back (memcpy, the oracle's swap definition); no stand-in compute")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": dict(workload_desc(args, tr), candidates=C, candidate_kind="SEEDED"),
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": sample,
                             "candidates_per_s": n_c / t, **host_info()},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(args, tr, best_swapped: int):
    """The oracle timed on this box's host cores (rank 0): a bounded sample on all cores and on one
    thread, extrapolated to the full step (eval of C candidates + swap of the policy bytes out and
    in), plus C1's 2^24-subset brute force (SURVEY §8(d) "Oracle timed beside it")."""
    import oracle as O
    sd = W.SEEDED[args.config[:2]]
    m = O.Model(tr)
    cores = os.cpu_count() or 1
    budget_s = args.cpu_seconds
    fpm = not args.search_mode

    def rate(nthreads, share):
        n = 500 * nthreads
        t0 = time.perf_counter()
        m.eval(O.SEEDED, 0, n, seed=sd["seed"], flip_thr=sd["flip_thr"], nthreads=nthreads, footprint=fpm)
        dt = time.perf_counter() - t0
        n2 = int(min(args.candidates, max(n, n * (share * budget_s) / max(dt, 1e-6))))
        t0 = time.perf_counter()
        m.eval(O.SEEDED, 0, n2, seed=sd["seed"], flip_thr=sd["flip_thr"], nthreads=nthreads, footprint=fpm)
        return n2, n2 / (time.perf_counter() - t0)

    n_all, rate_c = rate(cores, 0.4)
    n_one, rate_1 = rate(1, 0.2)
    nb = 1 << 30
    src = np.ones(nb, np.uint8)
    dst = np.empty(nb, np.uint8)
    O.swap_execute([dst.ctypes.data], [src.ctypes.data], [nb])
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        O.swap_execute([dst.ctypes.data], [src.ctypes.data], [nb])
    rate_b = reps * nb / (time.perf_counter() - t0)
    # C1: all 2^K subsets (K = 24), search mode, all cores
    c1 = O.Model(W.tiny())
    t0 = time.perf_counter()
    c1.eval(O.EXHAUSTIVE, 0, 1 << c1.K, nthreads=cores)
    t_c1 = time.perf_counter() - t0
    t_step = args.candidates / rate_c + 2 * best_swapped / rate_b
    return {"value": 2 * best_swapped / t_step / 1e9, "unit": "GB/s", "cores": cores, "kind": "oracle",
            "sample": (f"{n_all} SEEDED candidates on {cores} threads ({rate_c:.0f} cand/s) and {n_one} on 1 thread "
                       f"({rate_1:.0f} cand/s), {'full' if fpm else 'search'} mode; 3 x 1 GiB memcpy swap "
                       f"({rate_b / 1e9:.1f} GB/s); extrapolated to the full step (no stand-in compute)"),
            "candidates_per_s": rate_c, "candidates_per_s_1thread": rate_1,
            "c1_bruteforce": {"subsets": 1 << c1.K, "seconds": t_c1, "threads": cores},
            **host_info()}


# ----------------------------------------------------------------------------- this repo
class Compute:
    """Stand-in for the model's operators on the compute stream: one bf16 GEMM per traced op,
    [M, 8192] x [8192, 8192], M calibrated so one GEMM takes the trace's per-op time T_iter / N
    (the tau of Eq. 1's budgets and of the timeline stall model).  Each GEMM is bracketed by CUDA
    events so its duration is measured alone and under the swaps."""

    def __init__(self, dev, tau_s: float, n_ops: int):
        import torch
        self.torch = torch
        n = GEMM_N
        g = torch.Generator(device=dev).manual_seed(7)
        self.B = torch.randn(n, n, dtype=torch.bfloat16, device=dev, generator=g)
        self.A = torch.randn(2 * n, n, dtype=torch.bfloat16, device=dev, generator=g)
        self.C = torch.empty(2 * n, n, dtype=torch.bfloat16, device=dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(3):
            torch.matmul(self.A[:n], self.B, out=self.C[:n])
        torch.cuda.synchronize()
        e0.record()
        reps = 20
        for _ in range(reps):
            torch.matmul(self.A[:n], self.B, out=self.C[:n])
        e1.record()
        torch.cuda.synchronize()
        rate = reps * 2.0 * n ** 3 / (e0.elapsed_time(e1) * 1e-3)
        self.tau = tau_s
        self.n_ops = n_ops
        self._set_m(tau_s * rate / (2.0 * n * n))
        self.rate_burst = rate
        self.ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_ops)]

    def _set_m(self, m: float):
        n = GEMM_N
        self.M = int(min(2 * n, max(128, round(m / 128) * 128)))
        self.flops = 2.0 * self.M * n * n

    def recalibrate(self, stream, passes: int = 2):
        """a back-to-back GEMM iteration runs at the sustained (power-capped) rate, not the
        burst rate of the first calibration: rescale M until one iteration of compute alone
        takes N x tau (once or twice, whole iterations)"""
        torch = self.torch
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        hist = []
        for _ in range(passes):
            torch.cuda.synchronize()
            e0.record(stream)
            for i in range(self.n_ops):
                torch.matmul(self.A[:self.M], self.B, out=self.C[:self.M])
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            hist.append({"M": self.M, "iteration_ms": ms})
            self._set_m(self.M * (self.n_ops * self.tau * 1e3) / ms)
        return hist

    def op(self, i: int, stream):
        e0, e1 = self.ev[i]
        e0.record(stream)
        self.torch.matmul(self.A[:self.M], self.B, out=self.C[:self.M])
        e1.record(stream)

    def gemm_ms(self) -> float:
        """summed GEMM durations of the last iteration (call after a synchronize)"""
        return float(sum(a.elapsed_time(b) for a, b in self.ev))


def _k3(k):
    return (int(k["excess"]), float(k["stall"]), int(k["swapped_bytes"]))


def _replan_c4(chm, dev, comp):
    """C4 (Llama-2 13B, s = 8192 after a switch): record one Detailed iteration through
    chm_record_op, build the trace, evaluate 10^5 SEEDED candidates, run Algo. 2's grid (replayed
    as EXPLICIT candidates), refine by steepest descent (chm_descend), install -- each step timed"""
    import torch
    from paper_2509_11076_b200.runtime import _generate_all, descend, device_descend
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
    w0 = pt.candidate_mask(chm.SEEDED, int(bk["index"]), seed=sd["seed"], flip_thr=sd["flip_thr"])
    device_descend(ctx, pt, [w0], dev, max_rounds=0)  # warm (first-call setup), as the eval above is
    t0 = time.perf_counter()
    dk, words, rounds = device_descend(ctx, pt, [w0], dev)[0]  # one chm_descend launch
    out["descent_ms"] = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    hk, _, _ = descend(ctx, pt, bk, w0, dev)  # the same walk as a host loop of FLIP1 launches
    out["descent_host_loop_ms"] = (time.perf_counter() - t0) * 1e3
    out["descent_host_loop_same_key"] = bool(_k3(hk) == _k3(dk))
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
    ctx.close()
    return out


def _traffic(kernel: str, algorithmic_bytes: float):
    """DRAM bytes per launch: the ncu-measured traffic / algorithmic ratio of `kernel`
    (profiles/*_ncu_traffic.json, newest round first) times this run's algorithmic bytes per
    launch; None if absent"""
    for rnd in ("r02", "r01"):
        path = os.path.join(ROOT, "profiles", f"{rnd}_ncu_traffic.json")
        try:
            with open(path) as f:
                return float(json.load(f)[kernel]["ratio"]) * float(algorithmic_bytes)
        except (OSError, KeyError, ValueError):
            continue
    return None


class PolicyRun:
    """The installed policy's execution through the profiler hook on real HBM buffers (setup
    untimed): storage for every swapped tensor, pre-marshalled op records, the op loop."""

    def __init__(self, chm, ctx, tr, pt, words, keep, dev, seed):
        import torch
        self.chm, self.ctx, self.tr = chm, ctx, tr
        tb = pt.tables()
        gen = torch.Generator(device=dev).manual_seed(seed)
        self.storage = {}
        ids = np.array([FAKE_ID_BASE + int(p) for p in tr.ptr], dtype=np.uint64)
        for k in keep:
            t = int(tb["tensor"][k])
            buf = torch.empty(int(tr.nbytes[t]) // 8, dtype=torch.int64, device=dev)
            buf.random_(generator=gen)
            self.storage[t] = buf
            ids[t] = buf.data_ptr()
        self.item_dev = [self.storage[int(tb["tensor"][k])].data_ptr() for k in keep]  # swap-in destinations
        self.real_ids = set(self.item_dev)
        self.check_t = [int(tb["tensor"][k]) for k in keep[:: max(1, len(keep) // 8)]]
        self.check_sum = {t: int(self.storage[t].sum().item()) for t in self.check_t}
        tokens = [ctx.tokenize(nm) for nm in tr.op_names]
        self.run = chm.PreparedIteration(tr, ids, tokens)
        self.s_out = torch.cuda.Stream(dev)
        self.s_in = torch.cuda.Stream(dev)
        self.act = chm.Actions()
        self.L = chm.load()
        self.bytes_swap = sum(int(tb["nbytes"][k]) for k in keep)

    def intact(self) -> bool:
        return all(int(self.storage[t].sum().item()) == self.check_sum[t] for t in self.check_t)

    def execute(self, comp, flags, compute=None, detailed=False):
        """one iteration: per op, its compute (if any), then chm_record_op and the actions after
        it.  flags None: compute alone (no hook, no swaps).  Returns (kernel launches, out
        batches, in batches)."""
        chm, ctx = self.chm, self.ctx
        if detailed:
            ctx.set_detailed(True)
        launches = 0
        outs, ins = [], []
        h, act, L = ctx.h, self.act, self.L
        for i, r in enumerate(self.run.recs):
            if compute is not None:
                compute.op(i, comp)
            if flags is None:
                continue
            chm._check(L.chm_record_op(h, ctypes.byref(r), ctypes.byref(act)))
            if act.n_swap_out:
                n = act.n_swap_out
                for j in range(n):
                    if act.swap_out[j].dev not in self.real_ids:
                        raise RuntimeError(f"executor matched a tensor outside the policy at op {i}")
                outs.append(ctx.issue_swap_out(comp, self.s_out, flags))
                launches += (n + 63) // 64 if flags == chm.SWAP_KERNEL else 0
            for j in range(act.n_release):
                ctx.item_wait(act.release_item[j], False, comp)
            if act.n_swap_in:
                n = act.n_swap_in
                devs = [self.item_dev[act.swap_in_item[j]] for j in range(n)]
                ins.append(ctx.issue_swap_in(devs, comp, self.s_in, flags))
                launches += (n + 63) // 64 if flags == chm.SWAP_KERNEL else 0
            for j in range(act.n_wait):
                ctx.item_wait(act.wait_item[j], True, comp)
        if flags is not None:
            ctx.detect_seq_change(self.tr.t_iter)
        if detailed:
            ctx.set_detailed(False)
        return launches, outs, ins

    def close(self):
        self.storage.clear()


def _exchange(D, ctx, bl, ga, bg, P, stream, backend):
    """the argmin exchange: NCCL on device keys (all_gather_into_tensor + chm_best_reduce_device
    on `stream`), or gloo on host copies (all-gather + chm_best_reduce; functional runs)"""
    if backend == "nccl":
        D.argmin_exchange(ctx, bl, ga, bg, P, stream=stream)
        return
    import torch
    stream.synchronize()
    gh = torch.empty(5 * P, dtype=torch.int64)
    bh = torch.empty(5, dtype=torch.int64)
    D.argmin_exchange(None, bl.cpu(), gh, bh, P)
    bg.copy_(bh)


def _eval_strong_block(chm, D, dev, comp, rank, P, use_dist, barrier, max_over_ranks, total=10_000_000,
                       backend="nccl"):
    """the evaluation's strong scaling: C5's trace, `total` SEEDED candidates (search mode)
    sharded over the P ranks, the per-rank launch + the argmin exchange timed with CUDA events,
    the slowest rank's time"""
    import torch
    tr = W.CONFIGS["C5"]()
    sd = W.SEEDED["C5"]
    ctx = chm.Context(device=dev.index)
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    lo, cnt = D.shard(total, P, rank)
    bl = torch.empty(5, dtype=torch.int64, device=dev)
    ga = torch.empty(5 * P, dtype=torch.int64, device=dev)
    bg = torch.empty(5, dtype=torch.int64, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for it in range(5):
        barrier()
        torch.cuda.synchronize()
        torch.cuda._sleep(1_000_000)
        e0.record(comp)
        ctx.eval_policies(pt, chm.SEEDED, lo, cnt, best=bl, seed=sd["seed"], flip_thr=sd["flip_thr"], stream=comp)
        if use_dist:
            _exchange(D, ctx, bl, ga, bg, P, comp, backend)
        else:
            bg.copy_(bl)
        e1.record(comp)
        torch.cuda.synchronize()
        if it:
            ts.append(e0.elapsed_time(e1))
    t = max_over_ranks(float(np.median(ts)))
    b = bg.cpu().numpy().view(chm.BEST_DTYPE)[0]
    ctx.release_scratch()
    pt.free()
    ctx.close()
    return {"workload": tr.meta["config"], "candidates_total": total, "candidates_per_rank": cnt,
            "mode": "search", "ms": t, "candidates_per_s": total / (t * 1e-3), "scaling": "strong",
            "best_index": int(b["index"]), "includes": "each rank's launch + NCCL all-gather + device argmin (N > 1)"}


def _c1_block(chm, dev, reps):
    """C1's execution measurement: the 24 activations of the tiny trace (4 KiB -
    4 MiB) out and back in as one batch per direction, `reps` times: the swap kernel (one launch
    per direction) vs one cudaMemcpyAsync per tensor (the copy engines)"""
    import torch
    tr = W.tiny()
    h = chm.Context(device=-1)
    h.set_detailed(True)
    chm.record_iteration(h, tr)
    h.detect_seq_change(tr.t_iter)
    pt = h.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    sizes = [int(x) for x in pt.tables()["nbytes"]]
    h.close()
    total = sum(sizes)
    ctx = chm.Context(device=dev.index, host_arena_bytes=total + 4096 * len(sizes))
    g = torch.Generator(device=dev).manual_seed(1)
    src = [torch.randint(0, 256, (n,), dtype=torch.uint8, device=dev, generator=g) for n in sizes]
    dst = [torch.empty_like(x) for x in src]
    offs = np.concatenate([[0], np.cumsum([(n + 511) // 512 * 512 for n in sizes])[:-1]]).astype(np.uint64)
    d_out = [(x.data_ptr(), int(o), x.numel()) for x, o in zip(src, offs)]
    d_in = [(x.data_ptr(), int(o), x.numel()) for x, o in zip(dst, offs)]
    comp, s = torch.cuda.current_stream(dev), torch.cuda.Stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = {"tensors": len(sizes), "bytes": total, "min_bytes": min(sizes), "max_bytes": max(sizes), "reps": reps}
    for name, flags in (("kernel", chm.SWAP_KERNEL), ("copy_engines", chm.SWAP_CE)):
        for rep in range(reps + 20):
            if rep == 20:
                torch.cuda.synchronize()
                e0.record(comp)
            b = ctx.swap_out(d_out, comp, s, flags)
            ctx.batch_wait(b, comp)
            b = ctx.swap_in(d_in, comp, s, flags)
            ctx.batch_wait(b, comp)
        e1.record(comp)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        ok = all(torch.equal(a, c) for a, c in zip(src, dst))
        for x in dst:
            x.zero_()
        res[name] = {"us_per_round_trip": ms * 1e3, "GBps": 2 * total / (ms * 1e-3) / 1e9, "byte_exact": ok,
                     "calls_per_direction": 1 if flags == chm.SWAP_KERNEL else len(sizes)}
    # C1's evaluation measurement: all 2^K subsets in search mode, and full mode
    # (64-op footprint rows) in a batch of 2^20 -- the oracle's brute force is in cpu_baseline
    res["kernel_speedup"] = res["copy_engines"]["us_per_round_trip"] / res["kernel"]["us_per_round_trip"]
    ctx.close()
    ev_ctx = chm.Context(device=dev.index)
    ev_ctx.set_detailed(True)
    chm.record_iteration(ev_ctx, tr)
    ev_ctx.detect_seq_change(tr.t_iter)
    ptd = ev_ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    best = torch.empty(5, dtype=torch.int64, device=dev)
    n_all = 1 << ptd.K
    ld = (ptd.N + 1) // 2 * 2
    fpb = torch.empty((1 << 20, ld), dtype=torch.int64, device=dev)
    tm = {}
    for name, cnt, fp_ in (("search_all_subsets", n_all, None), ("full_2^20", 1 << 20, fpb)):
        ts = []
        for it in range(4):
            torch.cuda.synchronize()
            e0.record(comp)
            ev_ctx.eval_policies(ptd, chm.EXHAUSTIVE, 0, cnt, best=best, footprint=fp_, ld=ld if fp_ is not None else 0,
                                 stream=comp)
            e1.record(comp)
            torch.cuda.synchronize()
            if it:
                ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        tm[name] = {"candidates": cnt, "ms": ms, "candidates_per_s": cnt / (ms * 1e-3)}
    bk = best.cpu().numpy().view(chm.BEST_DTYPE)[0]
    res["eval"] = dict(tm, K=ptd.K, best_index=int(bk["index"]), best_excess=int(bk["excess"]))
    ptd.free()
    ev_ctx.close()
    return res


def _runtime_plan_block(chm, ctx, tr, pt, sd, C, dev, comp, compute, alone_ms, budget_pin):
    """the runtime's planner on the step's trace (Algo. 2's grid, SEEDED around the empty mask,
    the argmax-window base and Algo. 2's best, descent from each base's best; R-stall), then two
    executed iterations of its plan under the step's compute"""
    import torch
    from paper_2509_11076_b200.runtime import _generate_all, _key3, default_bases, device_descend, seeded_multibase
    t0 = time.perf_counter()
    gen = _generate_all(pt)
    best = torch.empty(5, dtype=torch.int64, device=dev)
    gkeys = []
    for g in gen:
        ctx.eval_policies(pt, chm.EXPLICIT, 0, 1, best=best, item_offsets=np.array([0, len(g)], np.uint64), items=g)
        gkeys.append(best.cpu().numpy().view(chm.BEST_DTYPE)[0].copy())
    k, w, name, per = seeded_multibase(ctx, pt, default_bases(pt, gen, gkeys), C, sd["seed"], sd["flip_thr"], dev)
    ends = device_descend(ctx, pt, [wx for _, wx in per.values()], dev)  # one chm_descend launch
    kd, wd, _ = min(ends, key=lambda e: _key3(e[0]))
    plan_ms = (time.perf_counter() - t0) * 1e3
    tb = pt.tables()
    keep = [j for j in range(pt.K) if (int(wd[j // 64]) >> (j % 64)) & 1]
    need = sum((int(tb["nbytes"][j]) + 511) // 512 * 512 for j in keep)
    out = {"what": "the runtime's planner (SEEDED around 3 bases + descent from each in one chm_descend launch, "
                   "R-stall) on the step's trace, "
                   "executed for 2 iterations under the same compute",
           "plan_ms": plan_ms, "items": len(keep), "swap_bytes_per_direction": int(kd["swapped_bytes"]),
           "excess": int(kd["excess"]), "predicted_stall_s": float(kd["stall"]),
           "seeded_best": {"base": name, "stall_s": float(k["stall"]), "swapped": int(k["swapped_bytes"])}}
    if need > budget_pin:
        out["executed"] = f"skipped: the plan needs {need} B pinned"
        return out
    ctx.arena_reserve(max(need, 1 << 20))
    ctx.policy_install(pt, wd)
    pr = PolicyRun(chm, ctx, tr, pt, wd, keep, dev, 77)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pr.execute(comp, chm.SWAP_KERNEL, compute)  # warm-up
    ms, d2h, h2d = [], [], []
    for _ in range(2):
        torch.cuda.synchronize()
        ev0.record(comp)
        _, outs, ins = pr.execute(comp, chm.SWAP_KERNEL, compute)
        ev1.record(comp)
        torch.cuda.synchronize()
        ms.append(ev0.elapsed_time(ev1))
        d2h.append(sum(ctx.batch_elapsed_ms(b) for b in outs))
        h2d.append(sum(ctx.batch_elapsed_ms(b) for b in ins))
    bsw = pr.bytes_swap
    rate = 2 * bsw / ((np.mean(d2h) + np.mean(h2d)) * 1e-3) if bsw else 0.0
    items = pt.mask_items(wd)
    ptm = ctx.trace_build(tr.budget, tr.static_bytes, rate if rate else tr.bw, tr.groups_fwd, tr.groups_bwd,
                          t_iter=tr.t_iter)
    out.update(exec_ms=float(np.mean(ms)), measured_stall_s=(float(np.mean(ms)) - alone_ms) * 1e-3,
               estimated_at_measured_B=dict(zip(("r_stall", "per_direction", "timeline"),
                                                ptm.stall_models(items).tolist())),
               swap_GBps={"d2h": bsw / (np.mean(d2h) * 1e-3) / 1e9 if bsw else None,
                          "h2d": bsw / (np.mean(h2d) * 1e-3) / 1e9 if bsw else None},
               byte_exact_sample=pr.intact())
    ptm.free()
    pr.close()
    return out


def _swap_only_block(chm, args, dev, name, steps):
    """A config's policy executed without compute (swap-bound steps), kernel and copy engines:
    the r01 headline kept as a block (C2) beside the C3h line"""
    import torch
    tr = W.CONFIGS[name]()
    sd = W.SEEDED[name[:2]]
    ctx = chm.Context(device=dev.index, time_batches=True, swap_ctas=args.swap_ctas)
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr, [ctx.tokenize(nm) for nm in tr.op_names])
    ctx.detect_seq_change(tr.t_iter)
    ctx.set_detailed(False)
    pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    best = torch.empty(5, dtype=torch.int64, device=dev)
    ctx.eval_policies(pt, chm.SEEDED, 0, args.candidates, best=best, seed=sd["seed"], flip_thr=sd["flip_thr"])
    bk = best.cpu().numpy().view(chm.BEST_DTYPE)[0]
    words = pt.candidate_mask(chm.SEEDED, int(bk["index"]), seed=sd["seed"], flip_thr=sd["flip_thr"])
    tb = pt.tables()
    keep = [k for k in range(pt.K) if (int(words[k // 64]) >> (k % 64)) & 1]
    need = sum((int(tb["nbytes"][k]) + 511) // 512 * 512 for k in keep)
    if need > args.host_frac * mem_available():
        ctx.close()
        return {"workload": tr.meta["config"], "skipped": f"policy needs {need} B pinned, host RAM too small"}
    ctx.arena_reserve(need)
    ctx.policy_install(pt, words)
    pr = PolicyRun(chm, ctx, tr, pt, words, keep, dev, 4321)
    comp = torch.cuda.current_stream(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = {"workload": tr.meta["config"], "items": len(keep), "swap_bytes_per_direction": pr.bytes_swap}
    for mode, flags, n in (("kernel", chm.SWAP_KERNEL, steps), ("copy_engines", chm.SWAP_CE, 1)):
        pr.execute(comp, flags)  # warm-up
        ms, d2h, h2d = [], [], []
        for _ in range(n):
            torch.cuda.synchronize()
            ev0.record(comp)
            _, outs, ins = pr.execute(comp, flags)
            ev1.record(comp)
            torch.cuda.synchronize()
            ms.append(ev0.elapsed_time(ev1))
            d2h.append(sum(ctx.batch_elapsed_ms(b) for b in outs))
            h2d.append(sum(ctx.batch_elapsed_ms(b) for b in ins))
        res[mode] = {"ms_per_step": float(np.mean(ms)), "GBps": 2 * pr.bytes_swap / (np.mean(ms) * 1e-3) / 1e9,
                     "d2h_GBps": pr.bytes_swap / (np.mean(d2h) * 1e-3) / 1e9,
                     "h2d_GBps": pr.bytes_swap / (np.mean(h2d) * 1e-3) / 1e9, "steps": n}
    res["byte_exact_sample"] = pr.intact()
    pr.close()
    ctx.close()
    return res


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if args.same_device else int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    import torch
    import torch.distributed as dist
    from paper_2509_11076_b200 import chm
    from paper_2509_11076_b200 import dist as D
    # collectives run whenever a process group is up: N > 1, or --force-dist at N = 1 (the NCCL
    # argmin path exercised on one GPU: a one-rank all-gather)
    use_dist = world > 1 or args.force_dist
    if use_dist:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        else:  # communicator lines (nranks, rings / NVLS) visible in the log
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local)
        if args.dist_backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    host_coll = use_dist and args.dist_backend == "gloo"  # collectives on host tensors
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    P = world
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(P)))

    def barrier():
        if use_dist:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if not use_dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if host_coll else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if not use_dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if host_coll else dev)
        dist.all_reduce(t)
        return float(t.item())

    tr = workload(args)
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
    digest = D.check_same_trace(pt, device=None if host_coll else dev) if use_dist else pt.digest()  # one trace
    C = args.candidates
    lo, cnt = D.shard(C, P, rank)
    full = not args.search_mode
    ld = (pt.N + 1) // 2 * 2
    peak = torch.empty(cnt, dtype=torch.int64, device=dev)
    stall = torch.empty(cnt, dtype=torch.float64, device=dev)
    fp = torch.empty((cnt, ld), dtype=torch.int64, device=dev) if full else None
    best_local = torch.empty(5, dtype=torch.int64, device=dev)
    gathered = torch.empty(5 * P, dtype=torch.int64, device=dev)
    best_global = torch.empty(5, dtype=torch.int64, device=dev)
    comp = torch.cuda.current_stream(dev)

    def evaluate(ev_kernel=None, trace=pt):
        ctx.eval_policies(trace, chm.SEEDED, lo, cnt, best=best_local, seed=sd["seed"], flip_thr=sd["flip_thr"],
                          peak=peak, stall=stall, footprint=fp, ld=ld if full else 0, stream=comp)
        if ev_kernel is not None:
            ev_kernel.record(comp)  # replay kernel done; the rest is the argmin exchange
        if use_dist:
            _exchange(D, ctx, best_local, gathered, best_global, P, comp, args.dist_backend)
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
    huge0 = anon_huge_bytes()
    t0 = time.perf_counter()
    # concurrent cudaHostRegister calls of tens of GB serialise in the driver: two ranks at a time
    D.staggered(local, local_world, lambda: ctx.arena_reserve(max(need, 1 << 20)), 2, barrier if use_dist else None)
    t_pin = time.perf_counter() - t0
    arena_pages = {"thp": thp_mode(), "anon_huge_bytes_gained": anon_huge_bytes() - huge0,
                   "arena_bytes": need, "base_page_bytes": os.sysconf("SC_PAGE_SIZE")}
    ctx.policy_install(pt, words_exec)
    pr = PolicyRun(chm, ctx, tr, pt, words_exec, keep, dev, 1234 + rank)
    bytes_swap = pr.bytes_swap
    compute = None if args.no_compute else Compute(dev, tr.t_iter / pt.N, pt.N)
    calib = compute.recalibrate(comp) if compute is not None else None

    spin_cycles = 1_000_000  # ~0.5 ms at 1.9 GHz
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev_k = torch.cuda.Event(enable_timing=True)
    # ---- warm-up + timed steps (device loop)
    step_ms, eval_ms, exec_ms, d2h_ms, h2d_ms, argmin_ms, gemm_ms = [], [], [], [], [], [], []
    launches = launches_swap = 0
    for step in range(args.warmup):
        evaluate()
        pr.execute(comp, chm.SWAP_KERNEL, compute)
    torch.cuda.synchronize()
    barrier()
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
            n_l, outs, ins = pr.execute(comp, chm.SWAP_KERNEL, compute)
            ev[3].record(comp)
            torch.cuda.synchronize()
            barrier()
            launches += n_l + 1 + (1 if use_dist else 0)
            launches_swap = n_l
            step_ms.append(ev[0].elapsed_time(ev[3]))
            eval_ms.append(ev[1].elapsed_time(ev_k))
            argmin_ms.append(ev_k.elapsed_time(ev[2]))
            exec_ms.append(ev[2].elapsed_time(ev[3]))
            d2h_ms.append(sum(ctx.batch_elapsed_ms(b) for b in outs))
            h2d_ms.append(sum(ctx.batch_elapsed_ms(b) for b in ins))
            if compute is not None:
                gemm_ms.append(compute.gemm_ms())
    clocks = clk.summary()
    st = ctx.exec_stats()
    ok = pr.intact()

    def run_mode(flags, n):
        """n untimed-by-the-headline steps of execution only: (exec ms, d2h ms, h2d ms, gemm ms)"""
        res = ([], [], [], [])
        for _ in range(n):
            torch.cuda.synchronize()
            ev[2].record(comp)
            _, outs_, ins_ = pr.execute(comp, flags, compute)
            ev[3].record(comp)
            torch.cuda.synchronize()
            res[0].append(ev[2].elapsed_time(ev[3]))
            res[1].append(sum(ctx.batch_elapsed_ms(b) for b in outs_))
            res[2].append(sum(ctx.batch_elapsed_ms(b) for b in ins_))
            if compute is not None:
                res[3].append(compute.gemm_ms())
        return [float(np.mean(x)) if x else None for x in res]

    # ---- the replay launch of the step, back to back (warm TLB / L2 state, no step around it):
    # in the step it follows 106 GB of swap traffic and a GEMM phase at the power cap
    iso = []
    for it in range(6):
        torch.cuda.synchronize()
        torch.cuda._sleep(spin_cycles)
        ev[0].record(comp)
        ctx.eval_policies(pt, chm.SEEDED, lo, cnt, best=best_local, seed=sd["seed"], flip_thr=sd["flip_thr"],
                          peak=peak, stall=stall, footprint=fp, ld=ld if full else 0, stream=comp)
        ev[3].record(comp)
        torch.cuda.synchronize()
        if it >= 2:
            iso.append(ev[0].elapsed_time(ev[3]))
    t_eval_iso = float(np.median(iso))
    # ---- compute alone (the same GEMM sequence, no hook, no swaps)
    with ClockSampler(local, enabled=not args.no_clocks and compute is not None) as clk_alone:
        alone = run_mode(None, args.alone_steps) if compute is not None else [None] * 4
    # ---- copy-engine baseline (per-tensor cudaMemcpyAsync on the same batches, same compute)
    with ClockSampler(local, enabled=not args.no_clocks) as clk_ce:
        ce = run_mode(chm.SWAP_CE, args.ce_steps)
    ok = ok and pr.intact()
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
        pr.execute(comp, chm.SWAP_AUTO, compute, detailed=True)
        pt2 = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
        evaluate(trace=pt2)
        bk2 = best_global.cpu().numpy().view(chm.BEST_DTYPE)[0]  # the step's result, D2H
        w2 = pt2.candidate_mask(chm.SEEDED, int(bk2["index"]), seed=sd["seed"], flip_thr=sd["flip_thr"])
        assert truncated or np.array_equal(w2, words), "re-planned policy differs on an unchanged trace"
        ctx.policy_install(pt2, words_exec if truncated else w2)
        ev[3].record(comp)
        torch.cuda.synchronize()
        e2e_ms.append(max(ev[0].elapsed_time(ev[3]), (time.perf_counter() - t0) * 1e3))
        pt2.free()
    ok = ok and pr.intact()
    # ---- the box's best pinned large-block copy-engine rate ("the fraction of the
    # box's best pinned large-block cudaMemcpyAsync"): one 2 GiB copy per direction, best of 3
    ce_big = {"d2h": 0.0, "h2d": 0.0}
    if ctx.host_arena()[1] >= (2 << 30):
        big = torch.empty(2 << 30, dtype=torch.uint8, device=dev)
        s_big = torch.cuda.Stream(dev)
        for _ in range(3):
            for d, fn in (("d2h", ctx.swap_out), ("h2d", ctx.swap_in)):
                b = fn([(big.data_ptr(), 0, big.numel())], comp, s_big, chm.SWAP_CE)
                ctx.batch_wait(b, comp)
                torch.cuda.synchronize()
                ce_big[d] = max(ce_big[d], big.numel() / (ctx.batch_elapsed_ms(b) * 1e-3) / 1e9)
        del big

    # ---- the policy's estimated stall (the models chm_stall_models evaluates), at the trace's B
    # and at the B this run's kernel measured, against the measured one: step with swaps minus
    # the same step's compute alone
    items = pt.mask_items(words_exec)
    t_d2h = max_over_ranks(float(np.mean(d2h_ms)))
    t_h2d = max_over_ranks(float(np.mean(h2d_ms)))
    achieved_swap = 2 * bytes_swap / ((t_d2h + t_h2d) * 1e-3) / 1e9
    est = {"B_trace_GBps": tr.bw / 1e9, "at_trace_B": dict(zip(("r_stall", "per_direction", "timeline"),
                                                             pt.stall_models(items).tolist()))}
    ptm = ctx.trace_build(tr.budget, tr.static_bytes, achieved_swap * 1e9, tr.groups_fwd, tr.groups_bwd,
                          t_iter=tr.t_iter)
    est["B_measured_GBps"] = achieved_swap  # the per-direction mean the kernel reached in the step
    est["at_measured_B"] = dict(zip(("r_stall", "per_direction", "timeline"), ptm.stall_models(items).tolist()))
    ptm.free()

    # ---- candidate policies evaluated / s at this N (the metric's second half):
    # C5's per-rank trace, 10^7 SEEDED candidates in search mode split over the ranks
    # (strong scaling), each rank's shard + the NCCL argmin, max over ranks
    strong = _eval_strong_block(chm, D, dev, comp, rank, P, use_dist, barrier, max_over_ranks,
                                backend=args.dist_backend)
    # ---- rank-0 blocks beside the line: Algo. 2's grid, the timeline ranking, the C4 re-plan,
    # C1's small tensors, C2 (N = 1: host RAM)
    extras = {}
    if rank == 0 and not args.no_extras:
        t0 = time.perf_counter()
        gen_lists = [pt.generate_policy(cc, rr)[0] for cc in (0.0, 0.5, 1.0, 2.0) for rr in (0.5, 1.0, 2.0)]
        t_gen = time.perf_counter() - t0
        off = np.zeros(len(gen_lists) + 1, np.uint64)
        off[1:] = np.cumsum([len(x) for x in gen_lists])
        g_best = torch.empty(5, dtype=torch.int64, device=dev)
        torch.cuda.synchronize()
        ev[0].record(comp)
        ctx.eval_policies(pt, chm.EXPLICIT, 0, len(gen_lists), best=g_best, item_offsets=off,
                          items=np.concatenate(gen_lists), stream=comp)
        ev[3].record(comp)
        torch.cuda.synchronize()
        gb = g_best.cpu().numpy().view(chm.BEST_DTYPE)[0]
        extras["generator"] = {"policies": len(gen_lists), "host_generate_ms": t_gen * 1e3,
                               "gpu_eval_ms": ev[0].elapsed_time(ev[3]), "best_index": int(gb["index"]),
                               "best_peak": int(gb["peak"]), "best_excess": int(gb["excess"]),
                               "best_stall_s": float(gb["stall"]), "seeded_best_excess": int(bk["excess"]),
                               "seeded_best_stall_s": float(bk["stall"])}
        tl_ms = []
        tl_best = torch.empty(5, dtype=torch.int64, device=dev)
        for it in range(4):
            torch.cuda.synchronize()
            torch.cuda._sleep(spin_cycles)
            ev[0].record(comp)
            ctx.eval_policies(pt, chm.SEEDED, 0, C, best=tl_best, seed=sd["seed"], flip_thr=sd["flip_thr"],
                              stall_model=chm.STALL_TIMELINE, stream=comp)
            ev[3].record(comp)
            torch.cuda.synchronize()
            if it:
                tl_ms.append(ev[0].elapsed_time(ev[3]))
        tb_ = tl_best.cpu().numpy().view(chm.BEST_DTYPE)[0]
        extras["eval_timeline"] = {"ms_per_launch": float(np.mean(tl_ms)), "candidates_per_s": C / (np.mean(tl_ms) * 1e-3),
                                   "mode": "search (peak / swapped by the replay kernel, then the timeline kernel)",
                                   "best_index": int(tb_["index"]), "best_stall_s": float(tb_["stall"]),
                                   "layer_best_index": int(bk["index"])}
        ctx.release_scratch()
        extras["replan_c4"] = _replan_c4(chm, dev, comp)
        if args.c1_reps:
            extras["c1_small_swaps"] = _c1_block(chm, dev, args.c1_reps)
    # ---- aggregate (max over ranks of time, sum of work)
    t_step = max_over_ranks(float(np.mean(step_ms)))
    t_eval = max_over_ranks(float(np.mean(eval_ms)))
    t_argmin = max_over_ranks(float(np.mean(argmin_ms)))
    t_exec = max_over_ranks(float(np.mean(exec_ms)))
    tot_bytes = sum_over_ranks(2.0 * bytes_swap)
    e2e_t = max_over_ranks(float(np.mean(e2e_ms))) if e2e_ms else None
    value = 2.0 * bytes_swap / (t_step * 1e-3) / 1e9  # per GPU (this rank's bytes, the slowest rank's time)
    fp_bytes = (8 * ld * cnt if full else 0) + 16 * cnt
    hbm_peak = measured_peaks().get("hbm_gbs", 6650.0)
    per_dir = [bytes_swap / (t_d2h * 1e-3) / 1e9 if t_d2h > 0 else 0.0,
               bytes_swap / (t_h2d * 1e-3) / 1e9 if t_h2d > 0 else 0.0]
    ce_dir = ([bytes_swap / (ce[1] * 1e-3) / 1e9, bytes_swap / (ce[2] * 1e-3) / 1e9] if ce[1] and ce[2] else None)
    # release this run's HBM storage and pinned arena before the C2 block pins its own
    pr.close()
    arena_info = ctx.arena_placement()
    # ---- the plan the runtime would install on this trace (reading R-bases + R-search: SEEDED
    # around three bases, steepest descent from each base's best, R-stall ranking), executed
    # under the same compute: its measured stall against its estimate (rank 0, N = 1)
    if rank == 0 and P == 1 and not args.no_extras and compute is not None:
        extras["runtime_plan"] = _runtime_plan_block(chm, ctx, tr, pt, sd, C, dev, comp, compute, alone[0],
                                                     budget_pin)
    ctx.close()
    del fp, peak, stall
    torch.cuda.empty_cache()
    if rank == 0 and P == 1 and args.c2_steps and args.config != "C2":
        extras["c2"] = _swap_only_block(chm, args, dev, "C2", args.c2_steps)
    if rank != 0:
        barrier()
        if use_dist:
            dist.destroy_process_group()
        return
    gflop = compute.flops * pt.N / 1e9 if compute is not None else None

    def tflops(ms):
        return gflop / ms if (gflop and ms) else None  # GFLOP / ms = TFLOP/s

    kernel_gemm_ms = float(np.mean(gemm_ms)) if gemm_ms else None
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "GB/s",
        "value_aggregate": tot_bytes / (t_step * 1e-3) / 1e9,
        "value_what": "per GPU: this rank's swap bytes (D2H + H2D) / step time (max over ranks); value_aggregate: "
                      "all ranks' bytes / the same time",
        "n_gpus": P,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "paper_context": PAPER_CONTEXT,
        "dtype": "u8",
        "data": "synthetic",
        "config": {
            **workload_desc(args, tr),
            "trace": {"ops": pt.N, "swappable": pt.K, "layers": pt.L, "peak0": pt.peak0, "budget": pt.budget,
                      "t_iter_s": tr.t_iter, "digest": f"{digest:016x}"},
            "candidates": C, "candidate_kind": "SEEDED", "candidates_per_rank": cnt,
            "eval_mode": "search" if args.search_mode else "full (per-op footprints written)",
            "policy": {"index": int(bk["index"]), "items": len(sel), "executed_items": len(keep),
                       "truncated_for_host_ram": truncated, "swap_bytes_per_direction": bytes_swap},
            "compute": (None if compute is None else
                        {"what": f"one bf16 GEMM [{compute.M}, {GEMM_N}] x [{GEMM_N}, {GEMM_N}] per op on the compute "
                                 f"stream, calibrated to T_iter / N = {tr.t_iter / pt.N * 1e3:.3f} ms",
                         "gflop_per_step": gflop}),
            "parallelism": f"dp{P}: per-rank swapping, candidates sharded, "
                           + ("NCCL argmin all-gather" if args.dist_backend == "nccl" else
                              "gloo argmin all-gather on host copies" + (", every rank on cuda:0 -- a functional "
                                                                         "check, not a measurement" if args.same_device else "")),
            "l2": "inputs larger than L2 (swap set and footprint rows are GBs per step)",
            "swap_ctas": args.swap_ctas, "arena_pin_s": round(t_pin, 2), "arena": dict(arena_info, **arena_pages),
            "host": host_info(),
        },
        "roofline": {
            "bound": "pcie", "kernel": "swap_copy_kernel (D2H + H2D)", "achieved": achieved_swap,
            "peak": PCIE_GEN5_X16_GBPS, "unit": "GB/s", "frac": achieved_swap / PCIE_GEN5_X16_GBPS,
            "traffic": _traffic("swap_copy_kernel", 2 * bytes_swap / max(1, launches_swap)),
            "traffic_source": "ncu dram bytes / algorithmic bytes (profiles/*_ncu_traffic.json) x this run's "
                              "algorithmic bytes per swap launch",
            "peak_source": "nominal PCIe Gen5 x16 per direction (no measured host-link peak in MEASURED_PEAKS.json)",
            "d2h_GBps": per_dir[0], "h2d_GBps": per_dir[1],
            "what": "swap-stream busy time of the kernel's batches during the overlapped step",
            "per_step_GBps": {"d2h": [round(bytes_swap / (x * 1e-3) / 1e9, 2) for x in d2h_ms],
                              "h2d": [round(bytes_swap / (x * 1e-3) / 1e9, 2) for x in h2d_ms]},
            "frac_of_copy_engines": ({"d2h": per_dir[0] / ce_dir[0], "h2d": per_dir[1] / ce_dir[1],
                                      "what": "vs the same batches on the copy engines (one cudaMemcpyAsync per "
                                              "tensor) under the same compute, this run"} if ce_dir else None),
            "copy_engine_large_block_GBps": ce_big if ce_big["d2h"] else None,
            "frac_of_copy_engine_large_block": ({"d2h": per_dir[0] / ce_big["d2h"], "h2d": per_dir[1] / ce_big["h2d"],
                                                 "what": "vs one 2 GiB pinned cudaMemcpyAsync per direction (best of 3), "
                                                         "the box's large-block copy-engine rate"}
                                                if ce_big["d2h"] else None),
        },
        "roofline_replay": {
            "bound": "hbm", "kernel": "replay_kernel<%s>" % ("true" if full else "false"),
            "achieved": fp_bytes / (t_eval * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
            "frac": fp_bytes / (t_eval * 1e-3) / 1e9 / hbm_peak,
            "traffic": _traffic("replay_kernel_full", fp_bytes) if full else None,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst)",
            "algorithmic_bytes_per_launch": fp_bytes,
            "frac_of_spec_8TBps": fp_bytes / (t_eval * 1e-3) / 1e9 / 8000.0,
            "what": "the launch inside the timed step: it follows the previous step's GEMM phase, whose power-capped "
                    "clock it partly inherits (tools/eval_after.py: 0.316 ms right after 1.3 s of GEMMs, 0.223 ms idle)",
            "back_to_back": {"ms_per_launch": t_eval_iso, "achieved": fp_bytes / (t_eval_iso * 1e-3) / 1e9,
                             "frac": fp_bytes / (t_eval_iso * 1e-3) / 1e9 / hbm_peak},
        },
        "argmin_exchange_us": t_argmin * 1e3 if use_dist else None,
        "eval": {"candidates_per_s": C / (t_eval * 1e-3), "ms_per_launch": t_eval, "unit": "candidates/s"},
        "eval_strong": strong,
        "overlap": {
            "exec_ms": {"kernel": t_exec, "copy_engines": ce[0], "compute_alone": alone[0]},
            "swap_GBps_during_overlap": {"kernel": {"d2h": per_dir[0], "h2d": per_dir[1]},
                                         "copy_engines": ({"d2h": ce_dir[0], "h2d": ce_dir[1]} if ce_dir else None)},
            "gemm_tflops": {"alone": tflops(alone[3]), "with_copy_engines": tflops(ce[3]),
                            "with_kernel": tflops(kernel_gemm_ms),
                            "what": "GEMM FLOPs / summed GEMM durations (CUDA events around each GEMM); compute "
                                    "alone runs back to back and meets the power cap (see clocks), the swap steps "
                                    "leave gaps at releases and waits"},
            "clocks": {"kernel": clocks, "copy_engines": clk_ce.summary(), "compute_alone": clk_alone.summary()},
            "compute_calibration": calib,
            "stall_s": {"measured_kernel": (t_exec - alone[0]) * 1e-3 if alone[0] else None,
                        "measured_copy_engines": (ce[0] - alone[0]) * 1e-3 if (alone[0] and ce[0]) else None,
                        "estimated": est},
        },
        "ce_baseline": {
            "what": "same batches and compute, one cudaMemcpyAsync per tensor on the copy engines",
            "ms_per_step": ce[0], "d2h_GBps": ce_dir[0] if ce_dir else None, "h2d_GBps": ce_dir[1] if ce_dir else None,
            "GBps": 2 * bytes_swap / (ce[0] * 1e-3) / 1e9 if ce[0] else None,
        },
        **extras,
        "e2e": {"value": 2.0 * bytes_swap / (e2e_t * 1e-3) / 1e9 if e2e_t else None, "unit": "GB/s",
                "copy_path": "CHM_SWAP_AUTO (the runtime's default: >= 4 MiB on the copy engines, smaller in the kernel)",
                "h2d_bytes_per_step": bytes_swap + table_bytes, "d2h_bytes_per_step": bytes_swap + 40,
                "ms_per_step": e2e_t},
        "gpu_launches": launches,
        "gpu_launches_per_step": launches // max(1, args.steps),
        "byte_exact_sample": ok,
        "exec_stats": st,
        "clocks": clocks,
    }
    line["cpu_baseline"] = cpu_baseline(args, tr, bytes_swap)
    print(json.dumps(line), flush=True)
    if use_dist:
        barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
