"""Fig. 3 reconstruction through the product's swap log, on a host-only ctx: an
iteration recorded while a policy runs reports the MEASURED footprint (the policy's footprint
F_P, from the oracle's event replay); chm_trace_build(f0_source=1) must rebuild the no-swap F0
from it plus the swap log the executor kept (releases after r_t, swap-ins before s_t) -- equal
to the oracle's F0 from the alloc/free events at every op.  (The device path with real OOMs,
passive swaps and demand swap-ins: tests/test_gpu_oom.py.)"""
import numpy as np
import pytest

import oracle as O
from paper_2509_11076_b200 import chm
from workloads import traces as W


def _prep(tr):
    ctx = chm.Context(device=-1)
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter,
                         omega=tr.omega)
    return ctx, pt


def _record_measured(ctx, tr, measured):
    tok = [ctx.tokenize(nm) for nm in tr.op_names]
    for i in range(tr.n_ops):
        ins = [(tr.ptr[t], tr.nbytes[t], tr.dtype[t]) for t in tr.ins(i)]
        outs = [(tr.ptr[t], tr.nbytes[t], tr.dtype[t]) for t in tr.outs(i)]
        ctx.record_op(tok[i], int(tr.phase[i]), ins, outs, [tr.ptr[t] for t in tr.frees(i)],
                      live_bytes=int(measured[i]))
    ctx.detect_seq_change(tr.t_iter)


def _rebuild(ctx, tr):
    return ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter,
                           omega=tr.omega, f0_source=1)


@pytest.mark.parametrize("name,seed", [("C1", 0), ("C2", 1), ("C5", 2), ("C2", 3)])
def test_reconstruction_from_swap_log_equals_event_f0(name, seed):
    tr = W.CONFIGS[name]()
    m = O.Model(tr)
    ctx, pt = _prep(tr)
    rng = np.random.default_rng(seed)
    bits = np.zeros(pt.K, np.int64)
    bits[rng.choice(pt.K, size=max(1, pt.K // 2), replace=False)] = 1
    words = np.zeros(pt.W, np.uint64)
    for k in np.nonzero(bits)[0]:
        words[k // 64] |= np.uint64(1 << int(k % 64))
    ctx.policy_install(pt, words)
    t, r, s = m.mask_items(bits)
    measured = m.replay(t, r, s)["footprint"]  # what the allocator reports under the policy
    assert (measured < m.f0()).any()  # the policy does lower the footprint somewhere
    ctx.set_detailed(True)
    _record_measured(ctx, tr, measured)
    f0 = _rebuild(ctx, tr).tables()["f0"]
    assert np.array_equal(f0, m.f0())
    # the oracle's own Fig. 3 routine agrees on the same log
    sw = m.swappable()
    sel = np.nonzero(bits)[0]
    nb = np.array([tr.nbytes[sw["t"][k]] for k in sel], np.int64)
    assert np.array_equal(O.reconstruct(measured, nb, sw["r"][sel], sw["s"][sel]), m.f0())


def test_reconstruction_without_swaps_is_the_measurement():
    tr = W.tiny()
    m = O.Model(tr)
    ctx, _ = _prep(tr)
    ctx.set_detailed(True)
    meas = m.f0() - 4096
    _record_measured(ctx, tr, meas)
    assert np.array_equal(_rebuild(ctx, tr).tables()["f0"], meas)


def test_reconstruction_errors():
    tr = W.tiny()
    ctx, _ = _prep(tr)  # recorded without live bytes (-1)
    with pytest.raises(chm.ChmError):
        _rebuild(ctx, tr)
    with pytest.raises(chm.ChmError):
        ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, f0_source=2)


def test_oom_entry_points_need_a_device():
    ctx = chm.Context(device=-1)
    with pytest.raises(chm.ChmError):
        ctx.oom_release()
    with pytest.raises(chm.ChmError):
        ctx.passive_swap(1 << 20)
    with pytest.raises(chm.ChmError):
        ctx.passive_restore(1, 1 << 40)
