"""Robustness of the ABI's device-side plumbing: a failed arena grow keeps an arena
of the previous size (installed plans still fit it); ABI calls give the caller's current CUDA
device back (libchm links its own runtime; both share the driver's current context)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2509_11076_b200 import chm  # noqa: E402
from workloads import traces as W  # noqa: E402


def _mem_available():
    for ln in open("/proc/meminfo"):
        if ln.startswith("MemAvailable:"):
            return int(ln.split()[1]) * 1024
    return 0


def test_failed_arena_grow_keeps_previous_arena():
    ctx = chm.Context(device=0, host_arena_bytes=64 << 20)
    base, n = ctx.host_arena()
    assert n == 64 << 20
    with pytest.raises(chm.ChmError) as e:
        ctx.arena_reserve(2 * _mem_available() + (1 << 30))  # refused: beyond 90% of MemAvailable
    assert e.value.code == chm.CHM_E_NOMEM and "re-pinned" in str(e.value)
    base2, n2 = ctx.host_arena()
    assert base2 and n2 == 64 << 20
    # and it still works as a swap target
    dev = torch.device("cuda:0")
    src = torch.randint(0, 256, (1 << 20,), dtype=torch.uint8, device=dev)
    dst = torch.empty_like(src)
    comp, s = torch.cuda.current_stream(), torch.cuda.Stream()
    ctx.batch_wait(ctx.swap_out([(src.data_ptr(), 0, src.numel())], comp, s), comp)
    ctx.batch_wait(ctx.swap_in([(dst.data_ptr(), 0, src.numel())], comp, s), comp)
    torch.cuda.synchronize()
    assert torch.equal(src, dst)
    ctx.close()


def test_abi_calls_keep_the_callers_current_device():
    torch.cuda.set_device(0)
    ctx = chm.Context(device=0, host_arena_bytes=1 << 20)
    tr = W.tiny()
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    best = torch.empty(5, dtype=torch.int64, device="cuda:0")
    ctx.eval_policies(pt, chm.EXHAUSTIVE, 0, 1024, best=best)
    ctx.arena_reserve(4 << 20)
    ctx.release_scratch()
    torch.cuda.synchronize()
    assert torch.cuda.current_device() == 0
    pt.free()
    ctx.close()
    assert torch.cuda.current_device() == 0
