"""The NCCL half of the cross-rank argmin on one B200: a one-rank NCCL process
group runs paper_2509_11076_b200.dist's device path -- all_gather_into_tensor of the 40 B key
straight from device memory, chm_best_reduce_device, and the trace-digest all-gather -- the code
bench.py runs at N > 1 (its multi-rank host logic is covered on CPU by test_multirank_cpu.py)."""
import os
import socket

import pytest

import oracle as O
from workloads import traces as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2509_11076_b200 import chm  # noqa: E402
from paper_2509_11076_b200 import dist as D  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_nccl_one_rank_argmin_exchange_and_digest():
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dev = torch.device("cuda:0")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        tr = W.CONFIGS["C5"]()
        sd = W.SEEDED["C5"]
        ctx = chm.Context(device=0, host_arena_bytes=1 << 20)
        ctx.set_detailed(True)
        chm.record_iteration(ctx, tr)
        ctx.detect_seq_change(tr.t_iter)
        pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
        assert D.check_same_trace(pt, device=dev) == pt.digest()
        C = 100_000
        lo, cnt = D.shard(C, 1, 0)
        best_local = torch.empty(5, dtype=torch.int64, device=dev)
        gathered = torch.empty(5, dtype=torch.int64, device=dev)
        best_global = torch.full((5,), -1, dtype=torch.int64, device=dev)
        comp = torch.cuda.current_stream(dev)
        ctx.eval_policies(pt, chm.SEEDED, lo, cnt, best=best_local, seed=sd["seed"], flip_thr=sd["flip_thr"],
                          stream=comp)
        D.argmin_exchange(ctx, best_local, gathered, best_global, 1, stream=comp)
        torch.cuda.synchronize()
        assert torch.equal(best_global, best_local)
        ref = O.Model(tr).eval(O.SEEDED, 0, C, seed=sd["seed"], flip_thr=sd["flip_thr"], nthreads=16)["best"]
        b = best_global.cpu().numpy().view(chm.BEST_DTYPE)[0]
        assert (int(b["excess"]), float(b["stall"]), int(b["swapped_bytes"]), int(b["index"])) == ref.key()
        ctx.close()
    finally:
        dist.destroy_process_group()
