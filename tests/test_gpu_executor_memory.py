"""Evaluation against execution: replay a trace on the device with real allocations
(PyTorch's stream-ordered caching allocator) and real swaps driven by the executor (chm_record_op
actions -> chm_issue_swap_out / item_wait + free / allocate + chm_issue_swap_in / item_wait).
At every op, after its swap-ins and outputs are allocated and before its frees, the requested
bytes (torch.cuda.memory_stats requested_bytes; sizes are 512 B multiples) must equal the oracle's event-replay footprint F_P[i] (relative to the static bytes), and
every swapped tensor must be back byte-exact when its first backward use waits for it."""
import numpy as np
import pytest

import oracle as O
from workloads import traces as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2509_11076_b200 import chm  # noqa: E402


def _policy(name, tr, m):
    if name == "C1":
        best = m.eval(O.EXHAUSTIVE, 0, 1 << m.K, nthreads=16)["best"]
        return [k for k in range(m.K) if (best.index >> k) & 1]
    sd = W.SEEDED["C2"]
    best = m.eval(O.SEEDED, 0, 2000, seed=sd["seed"], flip_thr=sd["flip_thr"], nthreads=16)["best"]
    J = (m.K + 3) // 4
    base = m.base_mask()
    sel = []
    for k in range(m.K):
        w = O.splitmix64(sd["seed"] ^ ((best.index * J + k // 4) % 2 ** 64))
        bit = ((int(base[k // 64]) >> (k % 64)) & 1) ^ int(((w >> (16 * (k % 4))) & 0xFFFF) < (sd["flip_thr"] >> 48))
        if bit:
            sel.append(k)
    return sel


@pytest.mark.parametrize("name", ["C1", "C2b1"])
def test_allocated_bytes_equal_replay_footprint(name):
    tr = W.tiny() if name == "C1" else W.gpt2_xl(batch=1)
    m = O.Model(tr)
    sel = _policy(name, tr, m)
    sw = m.swappable()
    F = m.replay(sw["t"][sel], sw["r"][sel], sw["s"][sel])["footprint"]
    need = int(sum((int(tr.nbytes[sw["t"][k]]) + 511) // 512 * 512 for k in sel))
    ctx = chm.Context(device=0, host_arena_bytes=max(need, 1 << 20))
    tok = [ctx.tokenize(nm) for nm in tr.op_names]
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr, tokens=tok)
    ctx.detect_seq_change(tr.t_iter)
    ctx.set_detailed(False)
    pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    words = np.zeros(max(pt.W, 1), np.uint64)
    for k in sel:
        words[k // 64] |= np.uint64(1 << (k % 64))
    ctx.policy_install(pt, words[:pt.W])
    dev = torch.device("cuda:0")
    comp = torch.cuda.current_stream()
    s_out, s_in = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    storage = {}
    static = {t: torch.empty(int(tr.nbytes[t]), dtype=torch.uint8, device=dev)
              for t in range(tr.n_produced, tr.n_tensors)}
    def allocated():  # bytes the program requested (the caching allocator may hand out larger blocks)
        return torch.cuda.memory_stats()["requested_bytes.all.current"]

    base0 = allocated()
    gen = torch.Generator(device=dev).manual_seed(3)
    item_tensor, ref = {}, {}

    def ref_of(t):
        buf = storage[t] if t < tr.n_produced else static[t]
        return (buf.data_ptr(), int(tr.nbytes[t]), int(tr.dtype[t]))

    measured = np.zeros(tr.n_ops, np.int64)
    for i in range(tr.n_ops):
        for t in tr.outs(i):
            storage[t] = torch.randint(0, 256, (int(tr.nbytes[t]),), dtype=torch.uint8, device=dev, generator=gen)
        measured[i] = allocated() - base0
        ins = [ref_of(t) for t in tr.ins(i)]
        outs = [ref_of(t) for t in tr.outs(i)]
        freed = [ref_of(t)[0] for t in tr.frees(i)]
        act = ctx.record_op(tok[i], int(tr.phase[i]), ins, outs, freed)
        av = chm.actions_view(act)
        for t in tr.frees(i):  # refcount releases
            storage.pop(t, None)
        if av["swap_out"]:
            for (d, off, nb), it in zip(av["swap_out"], av["swap_out_item"]):
                t = next(t for t, b in storage.items() if b is not None and b.data_ptr() == d)
                item_tensor[it] = t
                ref[t] = storage[t].clone()  # (test-side copy, freed before the check below)
            ctx.issue_swap_out(comp, s_out)
        for it in av["release"]:  # custom recordStream: stream-ordered reclaim after r_t
            ctx.item_wait(it, False, comp)
            storage[item_tensor[it]] = None
        if av["swap_in"]:  # blocks for op i+1's swap-ins
            dev_ptrs = []
            for (d, off, nb), it in zip(av["swap_in"], av["swap_in_item"]):
                storage[item_tensor[it]] = torch.empty(int(nb), dtype=torch.uint8, device=dev)
                dev_ptrs.append(storage[item_tensor[it]].data_ptr())
            ctx.issue_swap_in(dev_ptrs, comp, s_in)
        for it in av["wait"]:
            ctx.item_wait(it, True, comp)
            t = item_tensor[it]
            assert torch.equal(storage[t], ref[t]), f"tensor {t} not restored before op {i + 1}"
    ctx.detect_seq_change(tr.t_iter)
    torch.cuda.synchronize()
    # the test-side reference copies were allocated too: subtract them where they were live
    ref_bytes = np.zeros(tr.n_ops + 1, np.int64)
    p, f, a, b = m.tensor_table()
    for t in ref:
        ref_bytes[a[t] + 1:] += int(tr.nbytes[t])
    got, exp = measured - ref_bytes[:tr.n_ops], F - tr.static_bytes
    bad = np.nonzero(got != exp)[0]
    assert bad.size == 0, [(int(i), int(got[i]), int(exp[i]), int(got[i] - exp[i])) for i in bad[:8]]
    st = ctx.exec_stats()
    assert st["n_matched"] == len(sel) and st["bytes_out"] == st["bytes_in"]
    ctx.close()
