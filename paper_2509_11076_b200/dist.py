"""Multi-GPU plumbing of policy evaluation ("generates five
different policies and selects the one with the best runtime performance" -> best-of-n over a
sharded candidate set).

Policy execution needs no collective (each rank swaps its own activations over its own host
link).  Evaluation has one exchange step: candidate ids are split contiguously across ranks,
every rank evaluates its shard of the same trace, the 40 B per-rank keys are all-gathered and
every rank takes the lexicographic min.  The key carries the global candidate index, so the
winner is the same for any sharding (§8(c).6).

Argument marshalling and torch.distributed calls only: the min itself is chm_best_reduce_device
(NCCL path, device keys) or chm_best_reduce (host keys, e.g. gloo on CPU).
"""
from __future__ import annotations

from typing import Optional, Tuple

import numpy as np

from . import chm

KEY_WORDS = 5  # chm_best = 5 x 8 B


def shard(count: int, world: int, rank: int) -> Tuple[int, int]:
    """contiguous shard [floor(rank C / P), floor((rank+1) C / P)) -> (first, count)"""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"shard: rank {rank} outside world {world}")
    lo, hi = rank * count // world, (rank + 1) * count // world
    return lo, hi - lo


def _key_tensor(best: chm.Best, like):
    import torch
    k = np.array([(best.excess, best.stall, best.swapped_bytes, best.index, best.peak)], chm.BEST_DTYPE)
    return torch.from_numpy(k.view(np.int64).copy()).to(like.device)


def argmin_exchange(ctx: Optional[chm.Context], best_local, gathered, best_global, world: int,
                    stream=None, group=None) -> None:
    """all-gather one key per rank into `gathered` [world * 5] int64 and reduce it into
    `best_global` [5].  CUDA tensors: NCCL all_gather_into_tensor + chm_best_reduce_device on
    `stream` (no host round trip); CPU tensors (gloo): all-gather + chm_best_reduce on the host."""
    import torch.distributed as dist
    if best_local.numel() != KEY_WORDS or gathered.numel() != KEY_WORDS * world:
        raise ValueError("argmin_exchange: key buffers must hold 5 and 5 * world int64 words")
    dist.all_gather_into_tensor(gathered, best_local, group=group)
    if gathered.is_cuda:
        if ctx is None:
            raise ValueError("argmin_exchange: device keys need a ctx for chm_best_reduce_device")
        ctx.best_reduce_device(gathered, world, best_global, stream)
    else:
        b = chm.best_reduce(gathered.numpy().view(chm.BEST_DTYPE))
        best_global.copy_(_key_tensor(b, best_global))


def check_same_trace(pt: chm.Trace, device=None, group=None) -> int:
    """all-gathers every rank's chm_trace_digest and raises on a mismatch: ranks that shard one
    candidate set must evaluate the same trace (DP ranks share the op sequence and shapes)."""
    import torch
    import torch.distributed as dist
    d = pt.digest()
    mine = torch.tensor([np.int64(np.uint64(d).view(np.int64))], dtype=torch.int64, device=device)
    world = dist.get_world_size(group)
    allk = torch.empty(world, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(allk, mine, group=group)
    got = [int(np.int64(x).view(np.uint64)) for x in allk.cpu().tolist()]
    if any(x != d for x in got):
        raise RuntimeError("trace digest differs across ranks (rank -> digest): " +
                           ", ".join(f"{r}: {x:016x}" for r, x in enumerate(got)))
    return d


def staggered(local_rank: int, local_world: int, fn, group_size: int = 2, barrier=None):
    """runs fn() on the ranks of one node `group_size` at a time (barrier between groups):
    concurrent cudaHostRegister calls of tens of GB each serialise in the driver and hold every
    rank, and concurrent pre-faults contend for the node's free pages."""
    out = None
    for g0 in range(0, max(1, local_world), max(1, group_size)):
        if g0 <= local_rank < g0 + group_size:
            out = fn()
        if barrier is not None:
            barrier()
    return out
