"""Multi-rank host logic on CPU (gloo, world size 2): contiguous candidate shards, all-gather of
one 40 B key per rank, lexicographic min with the product's chm_best_reduce -- the winner must
equal the single-process argmin over the whole candidate set.  Each rank's shard
key comes from the oracle here (the device evaluation itself is covered by the GPU parity tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, C, out, budget_skew=0):
    """bench.py's distributed evaluation steps with the product's helpers
    (paper_2509_11076_b200.dist): trace built per rank through the ABI, digests all-gathered and
    compared, contiguous shard, one key per rank all-gathered and reduced on the host
    (chm_best_reduce, the gloo path of argmin_exchange)"""
    import sys
    sys.path.insert(0, ROOT)
    import oracle as O
    from paper_2509_11076_b200 import chm
    from paper_2509_11076_b200 import dist as D
    from workloads import traces as W
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tr = W.gpt2_xl()
    sd = W.SEEDED["C2"]
    ctx = chm.Context(device=-1)
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    pt = ctx.trace_build(tr.budget + (512 * rank if budget_skew else 0), tr.static_bytes, tr.bw, tr.groups_fwd,
                         tr.groups_bwd, t_iter=tr.t_iter, omega=tr.omega)
    try:
        digest = D.check_same_trace(pt)
    except RuntimeError as e:
        out[rank] = ("mismatch", str(e))
        dist.destroy_process_group()
        return
    lo, cnt = D.shard(C, world, rank)  # bench.py's shard rule
    m = O.Model(tr)
    b = m.eval(O.SEEDED, lo, cnt, seed=sd["seed"], flip_thr=sd["flip_thr"], nthreads=2)["best"]
    key = np.array([(b.excess, b.stall, b.swapped, b.index, b.peak)], dtype=chm.BEST_DTYPE)
    best_local = torch.from_numpy(key.view(np.int64).copy())
    gathered = torch.empty(world * 5, dtype=torch.int64)
    best_global = torch.empty(5, dtype=torch.int64)
    D.argmin_exchange(None, best_local, gathered, best_global, world)
    g = best_global.numpy().view(chm.BEST_DTYPE)[0]
    out[rank] = (int(g["index"]), int(g["excess"]), float(g["stall"]), int(g["swapped_bytes"]), digest)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_argmin_equals_global(world):
    import oracle as O
    from workloads import traces as W
    C = 3000
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), C, out), nprocs=world, join=True)
    tr = W.gpt2_xl()
    sd = W.SEEDED["C2"]
    ref = O.Model(tr).eval(O.SEEDED, 0, C, seed=sd["seed"], flip_thr=sd["flip_thr"], nthreads=4)["best"]
    for r in range(world):
        assert out[r][:4] == (ref.index, ref.excess, ref.stall, ref.swapped)
    assert out[0][4] == out[1][4]


def test_trace_mismatch_fails_loudly():
    """ranks whose traces differ (here: the budget) must refuse to shard one candidate set"""
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), 100, out, 1), nprocs=2, join=True)
    for r in range(2):
        assert out[r][0] == "mismatch" and "digest differs" in out[r][1], out[r]


def test_shard_rule_covers_every_candidate_once():
    from paper_2509_11076_b200.dist import shard
    for C in (0, 1, 7, 100_000, 10_000_001):
        for P in (1, 2, 3, 4, 8):
            parts = [shard(C, P, r) for r in range(P)]
            assert parts[0][0] == 0 and sum(c for _, c in parts) == C
            assert all(parts[r][0] + parts[r][1] == parts[r + 1][0] for r in range(P - 1))
            assert max(c for _, c in parts) - min(c for _, c in parts) <= 1
    with pytest.raises(ValueError):
        shard(10, 2, 2)


def _ddp_worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    from torch.nn.parallel import DistributedDataParallel as DDP

    from paper_2509_11076_b200 import chm
    from paper_2509_11076_b200.runtime import Runtime
    from workloads import tiny_gpt as G
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    model = DDP(G.make(0))
    opt = torch.optim.SGD(model.parameters(), lr=0.01)
    rt = Runtime(None, hbm_budget=1, groups_fwd=4, groups_bwd=4)
    matched, stages = [], []
    for x, y in G.batches(10, 2, 16, 64, seed=rank):  # each rank its own data shard
        with rt.step():
            loss = model(x, y)
            loss.backward()  # DDP's gradient all-reduce runs inside the step
            opt.step()
            opt.zero_grad()
        matched.append(rt.ctx.exec_stats()["n_matched"])
        stages.append(rt.stage)
    params = torch.cat([p.detach().flatten() for p in model.parameters()])
    gathered = [torch.empty_like(params) for _ in range(world)]
    dist.all_gather(gathered, params)
    out[rank] = dict(plans=len(rt.plans), items=rt.plans[0]["items"] if rt.plans else 0, matched=matched,
                     stages=stages, stale=rt.ctx.exec_stats()["n_stale"], unheld=rt.stats["unheld"],
                     replicas_equal=all(torch.equal(gathered[0], g) for g in gathered))
    dist.destroy_process_group()


def test_runtime_under_ddp_two_ranks():
    """one runtime per rank (host-only ctx) under DistributedDataParallel: the all-reduce inside
    backward does not disturb the profile -- each rank plans once and matches every planned
    tensor in every later step; the replicas stay identical"""
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_ddp_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for r in range(2):
        o = out[r]
        assert o["plans"] == 1 and o["items"] > 0 and o["stale"] == 0 and o["unheld"] == 0, o
        per_step = np.diff([0] + o["matched"])
        assert set(per_step.tolist()) <= {0, o["items"]} and per_step[-1] == o["items"], o
        assert o["replicas_equal"]


def _stagger_worker(rank, world, port, out):
    import sys
    import time
    sys.path.insert(0, ROOT)
    from paper_2509_11076_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def pin():  # stands in for the arena reservation: records when this rank ran
        t0 = time.monotonic()
        time.sleep(0.2)
        return (t0, time.monotonic())
    out[rank] = D.staggered(rank, world, pin, 2, dist.barrier)
    dist.destroy_process_group()


def test_staggered_pins_two_ranks_at_a_time():
    """bench.py pins the arenas of a node's ranks two at a time (concurrent cudaHostRegister calls
    of tens of GB serialise in the driver): with 4 ranks, ranks {0,1} run before {2,3}"""
    world = 4
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_stagger_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    first_end = max(out[0][1], out[1][1])
    second_start = min(out[2][0], out[3][0])
    assert second_start >= first_end - 1e-3, dict(out)
