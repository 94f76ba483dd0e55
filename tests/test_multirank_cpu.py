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


def _worker(rank, world, port, C, out):
    import sys
    sys.path.insert(0, ROOT)
    import oracle as O
    from paper_2509_11076_b200 import chm
    from workloads import traces as W
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tr = W.gpt2_xl()
    sd = W.SEEDED["C2"]
    m = O.Model(tr)
    lo, hi = rank * C // world, (rank + 1) * C // world  # bench.py's shard rule
    b = m.eval(O.SEEDED, lo, hi - lo, seed=sd["seed"], flip_thr=sd["flip_thr"], nthreads=2)["best"]
    key = np.array([(b.excess, b.stall, b.swapped, b.index, b.peak)], dtype=chm.BEST_DTYPE)
    t = torch.from_numpy(key.view(np.int64).copy())
    gathered = torch.empty(world * 5, dtype=torch.int64)
    dist.all_gather_into_tensor(gathered, t)
    best = chm.best_reduce(gathered.numpy().view(chm.BEST_DTYPE))
    out[rank] = (int(best.index), int(best.excess), float(best.stall), int(best.swapped_bytes))
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
        assert out[r] == (ref.index, ref.excess, ref.stall, ref.swapped)


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
