"""Driver for NEXT-4 (Algo. 3 OOM handling + Fig. 3 reconstruction): one iteration of a
synthetic trace with real allocations under a hard cap on the produced bytes held, every
overflow handled through chm_oom_release / chm_passive_swap, passively swapped tensors restored
(chm_passive_restore) before use, policy actions executed when a policy is installed.  Used by
tests/test_gpu_oom.py (which checks the results against the oracle) and tools/oom_warmup.py.
Product calls only."""
import numpy as np
import torch

from paper_2509_11076_b200 import chm


def _pattern(t, n, dev):
    g = torch.Generator(device=dev).manual_seed(1000 + int(t))
    return torch.randint(0, 256, (n,), dtype=torch.uint8, device=dev, generator=g)


def run_capped(tr, cap, sel=None, arena_extra=1 << 30, seeded=None):
    """one Detailed iteration of `tr` under a cap of `cap` produced bytes.  Policy (planned on an
    uncapped Detailed iteration first): sel = swappable indices, or seeded = (seed, flip_thr,
    count): the best of `count` SEEDED candidates evaluated on the GPU."""
    dev = torch.device("cuda:0")
    ctx = chm.Context(device=0, host_arena_bytes=arena_extra)
    tok = [ctx.tokenize(nm) for nm in tr.op_names]
    static_id = {t: (1 << 60) + t for t in range(tr.n_produced, tr.n_tensors)}
    if sel or seeded:
        ctx.set_detailed(True)
        ids = np.array([(1 << 59) + int(p) for p in tr.ptr], np.uint64)  # planning pass: any ids
        freed = set(int(t) for i in range(tr.n_ops) for t in tr.frees(i))
        survivors = [t for t in range(tr.n_produced) if t not in freed]
        for i in range(tr.n_ops):
            fr = [ids[t] for t in tr.frees(i)] + ([ids[t] for t in survivors] if i == tr.n_ops - 1 else [])
            # (survivors freed at the last op: F0 and the tables are unchanged, and no planning-pass
            # id stays resident as a passive-swap candidate of the capped iteration)
            ctx.record_op(tok[i], int(tr.phase[i]), [(ids[t], tr.nbytes[t], tr.dtype[t]) for t in tr.ins(i)],
                          [(ids[t], tr.nbytes[t], tr.dtype[t]) for t in tr.outs(i)], fr)
        ctx.detect_seq_change(tr.t_iter)
        pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
        if seeded:
            seed, flip_thr, count = seeded
            best = torch.empty(5, dtype=torch.int64, device=dev)
            ctx.eval_policies(pt, chm.SEEDED, 0, count, best=best, seed=seed, flip_thr=flip_thr)
            idx = int(best.cpu().numpy().view(chm.BEST_DTYPE)[0]["index"])
            words = pt.candidate_mask(chm.SEEDED, idx, seed=seed, flip_thr=flip_thr)
            sel = [k for k in range(pt.K) if (int(words[k // 64]) >> (k % 64)) & 1]
        words = np.zeros(max(pt.W, 1), np.uint64)
        for k in sel:
            words[k // 64] |= np.uint64(1 << (k % 64))
        nb = pt.tables()["nbytes"]
        ctx.arena_reserve(int(sum((int(nb[k]) + 511) // 512 * 512 for k in sel)) + arena_extra)
        ctx.policy_install(pt, words[:pt.W])
    ctx.set_detailed(True)
    comp = torch.cuda.current_stream()
    s_out, s_in, s_passive = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    storage, owner, handles, item_tensor = {}, {}, {}, {}
    st = dict(live=0, peak=0, passive=0, restored=0, dropped=0, early=0, checked=0)

    def hold(t, buf):
        storage[t] = buf
        owner[buf.data_ptr()] = t
        st["live"] += int(tr.nbytes[t])

    def drop(t):
        buf = storage.pop(t)
        owner.pop(buf.data_ptr())
        st["live"] -= int(tr.nbytes[t])

    def check(t):
        assert torch.equal(storage[t], _pattern(t, int(tr.nbytes[t]), dev)), f"tensor {t} corrupted"
        st["checked"] += 1

    def alloc(t, nb, exclude):
        """the allocator hook: Algo. 3 until the request fits under the cap"""
        while st["live"] + nb > cap:
            rel = ctx.oom_release(comp)  # (i)-(ii)
            if rel:
                for it in rel:
                    drop(item_tensor[it])
                st["early"] += len(rel)
                continue
            ex = [storage[u].data_ptr() for u in exclude if u in storage]
            p = ctx.passive_swap(nb, ex, comp, s_passive)  # (iv)
            u = owner[p["id"]]
            assert p["nbytes"] == int(tr.nbytes[u])
            handles[u] = p["handle"]
            drop(u)
            st["passive"] += 1
        hold(t, torch.empty(nb, dtype=torch.uint8, device=dev))
        return storage[t]

    def ref(t):
        return (storage[t].data_ptr() if t < tr.n_produced else static_id[t], int(tr.nbytes[t]), int(tr.dtype[t]))

    measured = np.zeros(tr.n_ops, np.int64)
    for i in range(tr.n_ops):
        busy = [t for t in tr.ins(i) if t < tr.n_produced] + list(tr.outs(i))
        for t in tr.ins(i):  # demand swap-in before the op reads it (reading Q20)
            if t in handles:
                buf = alloc(t, int(tr.nbytes[t]), busy)
                ctx.passive_restore(handles.pop(t), buf.data_ptr(), comp, s_passive)
                check(t)
                st["restored"] += 1
        for t in tr.outs(i):
            alloc(t, int(tr.nbytes[t]), busy).copy_(_pattern(t, int(tr.nbytes[t]), dev))  # the op's compute
        measured[i] = st["live"] + tr.static_bytes
        st["peak"] = max(st["peak"], st["live"])
        dead_out = [t for t in tr.frees(i) if t in handles]
        act = ctx.record_op(tok[i], int(tr.phase[i]), [ref(t) for t in tr.ins(i)], [ref(t) for t in tr.outs(i)],
                            [ref(t)[0] for t in tr.frees(i) if t not in handles], live_bytes=int(measured[i]))
        av = chm.actions_view(act)
        for t in dead_out:  # died while passively out
            ctx.passive_restore(handles.pop(t), 0)
            st["dropped"] += 1
        for t in tr.frees(i):
            if t in storage:
                drop(t)
        if av["swap_out"]:
            for (d, off, nb), it in zip(av["swap_out"], av["swap_out_item"]):
                item_tensor[it] = owner[d]
            ctx.issue_swap_out(comp, s_out)
        for it in av["release"]:  # custom recordStream
            ctx.item_wait(it, False, comp)
            drop(item_tensor[it])
        if av["swap_in"]:
            ptrs = []
            for (d, off, nb), it in zip(av["swap_in"], av["swap_in_item"]):
                ptrs.append(alloc(item_tensor[it], int(nb), busy).data_ptr())
            ctx.issue_swap_in(ptrs, comp, s_in)
        for it in av["wait"]:
            ctx.item_wait(it, True, comp)
            check(item_tensor[it])
    ctx.detect_seq_change(tr.t_iter)
    torch.cuda.synchronize()
    f0_log = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter,
                             f0_source=1).tables()["f0"]
    f0_ev = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd,
                            t_iter=tr.t_iter).tables()["f0"]
    st["exec"] = ctx.exec_stats()
    st["items"] = len(sel) if sel else 0
    storage.clear()
    ctx.close()
    return measured, f0_log, f0_ev, st


