"""NEXT-4: WarmUp OOM handling, Algo. 3, and Fig. 3's
reconstruction on the device.

One iteration of a trace runs with real allocations and a hard cap on the produced bytes held
(the "HBM" of the test).  Every allocation that would cross the cap goes through the Algo. 3
hook: chm_oom_release (release the blocks whose swap-out is already issued, behind an event
pair), then chm_passive_swap (the resident tensor closest in size) -- until it fits.  Before an
op reads a passively swapped tensor it is brought back by chm_passive_restore (demand
swap-in); a tensor that dies while out is dropped.  The iteration is recorded in Detailed mode
with the measured bytes per op.

Checked: the cap holds at every op; every tensor that comes back (passive restore or policy
swap-in) is byte-exact; the no-swap F0 rebuilt from the measured bytes and the swap log
(f0_source = 1) and the one from the recorded events (f0_source = 0, ids reused by the
allocator while tensors were out) both equal the oracle's F0 at every op."""
import numpy as np
import pytest

import oracle as O
from workloads import traces as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tests.test_gpu_executor_memory import _policy  # noqa: E402
from tools.oom_driver import run_capped  # noqa: E402


def _assert_reconstruction(m, f0_log, f0_ev):
    f0 = m.f0()
    bad = np.nonzero(f0_log != f0)[0]
    assert bad.size == 0, [(int(i), int(f0_log[i]), int(f0[i])) for i in bad[:8]]
    assert np.array_equal(f0_ev, f0)


@pytest.mark.parametrize("frac", [0.6, 0.85])
def test_warmup_oom_passive_swaps(frac):
    """WarmUp stage, no policy: every overflow is handled by passive swaps (step (iv))"""
    tr = W.gpt2_xl(seq=512, batch=1)
    act_peak = int(O.Model(tr).f0().max() - tr.static_bytes)
    cap = int(act_peak * frac)
    m = O.Model(tr)
    measured, f0_log, f0_ev, st = run_capped(tr, cap, arena_extra=act_peak)
    assert st["peak"] <= cap and st["passive"] > 0 and st["restored"] > 0
    assert st["checked"] == st["restored"]
    _assert_reconstruction(m, f0_log, f0_ev)


def test_policy_undershoot_releases_early_then_passive():
    """a policy whose plan does not fit the cap: marked blocks are released early (steps
    (i)-(ii)) before any passive swap; swap-ins still byte-exact"""
    tr = W.gpt2_xl(seq=512, batch=1)
    m0 = O.Model(tr)
    sel = _policy("C2b1", tr, m0)
    sw = m0.swappable()
    fp = m0.replay(sw["t"][sel], sw["r"][sel], sw["s"][sel])["footprint"]
    act_peak = int(fp.max() - tr.static_bytes)
    cap = int(act_peak * 0.8)
    m = m0
    measured, f0_log, f0_ev, st = run_capped(tr, cap, sel=sel, arena_extra=act_peak)
    assert st["peak"] <= cap
    assert st["early"] > 0, st
    assert st["exec"]["n_matched"] == len(sel)
    _assert_reconstruction(m, f0_log, f0_ev)
