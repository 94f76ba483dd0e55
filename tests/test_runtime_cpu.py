"""NEXT-2 on CPU: the PyTorch runtime (paper_2509_11076_b200/runtime.py) on a real eager training
loop (workloads/tiny_gpt.py), host-only ctx (no copies).  Checks the stage machine over real
steps, one plan per stable phase, App. A matching of every planned tensor in every
later step, and matching under sequence drift -- an op inserted mid-forward shifts
every later op index -- against a Capuchin-style fixed (op index, argument) matcher, which picks
the wrong tensors."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2509_11076_b200 import chm  # noqa: E402
from paper_2509_11076_b200.runtime import Runtime  # noqa: E402
from workloads import tiny_gpt as G  # noqa: E402


def _setup(n_batches=12, **algo1):
    model = G.make(0)
    opt = torch.optim.SGD(model.parameters(), lr=0.01)
    data = G.batches(n_batches, 2, 16, 64)
    rt = Runtime(None, hbm_budget=1, groups_fwd=4, groups_bwd=4, **algo1)
    return model, opt, data, rt


def _step(rt, model, opt, x, y, forwards=1):
    with rt.step():
        loss = sum(model(x, y) for _ in range(forwards))
        loss.backward()
        opt.step()
        opt.zero_grad()


@pytest.mark.parametrize("native", [True, False])
def test_stages_plan_and_matching_every_step(native):
    """the C++ dispatch hook (default) and the Python TorchDispatchMode: same stage machine,
    one plan, every planned tensor matched in every later step"""
    model, opt, data, rt = _setup(native_hook=native)
    stages, matched = [], []
    for x, y in data:
        _step(rt, model, opt, x, y)
        stages.append(rt.stage)
        matched.append(rt.ctx.exec_stats()["n_matched"])
    # WarmUp until m = 2 stable comparisons, then GenPolicy (Detailed), then Stable after n = 5
    assert stages[:2] == [chm.WARMUP, chm.WARMUP] and chm.GENPOLICY in stages and stages[-1] == chm.STABLE
    assert len(rt.plans) == 1 and rt.plans[0]["items"] > 0
    n_items = rt.plans[0]["items"]
    first = stages.index(chm.GENPOLICY) + 1  # the Detailed step; its end installs the policy
    per_step = np.diff([0] + matched)
    assert all(v == 0 for v in per_step[:first + 1])
    assert all(v == n_items for v in per_step[first + 1:]), per_step
    st = rt.ctx.exec_stats()
    assert st["n_stale"] == 0 and st["n_collisions"] == 0
    assert rt.stats["unheld"] == 0  # every released tensor was one autograd saved
    assert rt.stats["release"] == rt.stats["swap_out"] == rt.stats["swap_in"] == n_items * (len(data) - first - 1)


def _identity(log):
    """production rank -> (op, out slot); a_t and the argument position there (fixed-index key)"""
    where, cur = [], {}
    a, key = {}, {}
    for e in log:
        for j, p in enumerate(e["outs"]):
            cur[p] = len(where)
            where.append((e["op"], j))
    cur = {}
    for e in log:
        for j, p in enumerate(e["ins"]):
            r = cur.get(p)
            if r is not None and e["phase"] == chm.FWD:
                a[r] = e["op"]
                key[r] = ("in", j)
        for j, p in enumerate(e["outs"]):
            r = sum(len(x["outs"]) for x in log[:e["op"]]) + j
            cur[p] = r
            if e["phase"] == chm.FWD:
                a[r] = e["op"]
                key[r] = ("out", j)
    return where, a, key


def test_matching_under_drift_vs_fixed_index_matcher():
    # histogram cosine (cos_mode 1): an inserted op is a minor change, not a new sequence
    # (positional cosine compares every later op with its shifted neighbour)
    model, opt, data, rt = _setup(14, cos_mode=1, native_hook=False)  # record_log: the Python hook
    rt.record_log = True
    logs = []
    for i, (x, y) in enumerate(data[:10]):
        _step(rt, model, opt, x, y)
        logs.append(rt.log)
    assert rt.policy is not None
    plan = rt.plans[0]
    # the Detailed step is the one whose end planned: the last one before actions appear
    det = max(i for i, lg in enumerate(logs) if all(e["actions"] is None for e in lg))
    base_log = logs[det]
    where, a_t, key = _identity(base_log)
    ranks = plan["tensors"]
    # one step with an op inserted before block 2 (a logging read of a weight)
    model.drift_layer = 2
    x, y = data[10]
    m0 = rt.ctx.exec_stats()["n_matched"]
    _step(rt, model, opt, x, y)
    model.drift_layer = -1
    drift = rt.log
    assert rt.last_step["changed"] is False  # minor drift: Algo. 1 keeps the policy
    tb = [e["token"] for e in base_log]
    td = [e["token"] for e in drift]
    ins_at = next(i for i in range(len(tb)) if tb[i] != td[i])
    d = len(td) - len(tb)
    assert d >= 1

    def shift(i):
        return i if i < ins_at else i + d
    truth = sorted(drift[shift(where[r][0])]["outs"][where[r][1]] for r in ranks)
    ours = sorted(p for e in drift if e["actions"] for (p, _, _) in e["actions"]["swap_out"])
    assert rt.ctx.exec_stats()["n_matched"] - m0 == len(ranks)
    assert ours == truth  # every planned tensor found, none confused with a neighbour
    # Capuchin-style key (op index a_t, argument slot) recorded on the base step
    fixed = []
    for r in ranks:
        e = drift[a_t[r]]
        side, j = key[r]
        lst = e["ins"] if side == "in" else e["outs"]
        fixed.append(lst[j] if j < len(lst) else None)
    wrong = sum(1 for f, t in zip(sorted(fixed, key=lambda v: -1 if v is None else v), truth) if f != t)
    assert wrong > 0 and sorted(x for x in fixed if x is not None) != truth


def test_sequence_change_uninstalls_and_replans():
    model, opt, data, rt = _setup(22)
    for x, y in data[:8]:
        _step(rt, model, opt, x, y)
    assert rt.policy is not None and len(rt.plans) == 1
    x, y = data[8]
    _step(rt, model, opt, x, y, forwards=2)  # e.g. two micro-batches: the op sequence doubles
    assert rt.last_step["changed"] and rt.policy is None and rt.stage == chm.WARMUP
    for x, y in data[9:]:
        _step(rt, model, opt, x, y, forwards=2)
    assert len(rt.plans) == 2 and rt.policy is not None
    assert rt.plans[1]["n_ops"] > 1.8 * rt.plans[0]["n_ops"]  # both passes recorded (OPT ops once)


def test_interleaved_microbatches_and_a_failed_step():
    """two (forward, backward) pairs per step: the second forward is recorded in the later phase
    (FWD* BWD* OPT* is kept), the plan covers the first micro-batch and matches every step; a step
    that raises closes its partial iteration, the policy is dropped and re-planned later"""
    model, opt, data, rt = _setup(24)

    def step2(x, y):
        with rt.step():
            model(x, y).backward()
            model(x, y).backward()
            opt.step()
            opt.zero_grad()
    for x, y in data[:8]:
        step2(x, y)
    assert rt.policy is not None and rt.plans[0]["items"] > 0
    m0 = rt.ctx.exec_stats()["n_matched"]
    step2(*data[8])
    assert rt.ctx.exec_stats()["n_matched"] - m0 == rt.plans[0]["items"]
    with pytest.raises(ValueError):
        with rt.step():
            model(*data[9]).backward()
            raise ValueError("user error mid-step")
    assert rt.policy is None and rt.stats["aborted"] == 1
    for x, y in data[10:]:
        step2(x, y)
    assert len(rt.plans) == 2 and rt.policy is not None


def test_runtime_on_a_conv_net():
    """not only transformers: a small CNN (conv / batch-norm / relu / pool / linear) profiles,
    plans and matches every planned tensor each step"""
    import torch.nn as nn
    torch.manual_seed(0)
    net = nn.Sequential(
        nn.Conv2d(3, 16, 3, padding=1), nn.BatchNorm2d(16), nn.ReLU(),
        nn.Conv2d(16, 16, 3, padding=1), nn.BatchNorm2d(16), nn.ReLU(), nn.MaxPool2d(2),
        nn.Conv2d(16, 32, 3, padding=1), nn.BatchNorm2d(32), nn.ReLU(),
        nn.Conv2d(32, 32, 3, padding=1), nn.BatchNorm2d(32), nn.ReLU(), nn.AdaptiveAvgPool2d(1),
        nn.Flatten(), nn.Linear(32, 10))
    opt = torch.optim.SGD(net.parameters(), lr=0.01, momentum=0.9)
    rt = Runtime(None, hbm_budget=1)
    g = torch.Generator().manual_seed(1)
    matched = []
    for _ in range(10):
        x = torch.randn(4, 3, 32, 32, generator=g)
        y = torch.randint(0, 10, (4,), generator=g)
        with rt.step():
            torch.nn.functional.cross_entropy(net(x), y).backward()
            opt.step()
            opt.zero_grad()
        matched.append(rt.ctx.exec_stats()["n_matched"])
    assert len(rt.plans) == 1 and rt.plans[0]["items"] > 0
    per = np.diff([0] + matched)
    assert per[-1] == rt.plans[0]["items"] and rt.ctx.exec_stats()["n_stale"] == 0


def test_planner_error_is_recorded_and_training_continues():
    """a plan that raises (here: the trace build) must not escape rt.step() nor re-raise in every
    later step: it is recorded in rt.plans, the runtime runs without a policy until the next
    sequence change or request_replan"""
    model, opt, data, rt = _setup()
    real = rt.ctx.trace_build
    calls = []

    def broken(*a, **k):
        calls.append(1)
        raise chm.ChmError(chm.CHM_E_INVAL, "injected planner failure")

    rt.ctx.trace_build = broken
    for x, y in data:
        _step(rt, model, opt, x, y)
    assert len(calls) == 1  # planned once, failed once
    assert rt.plans and rt.plans[-1]["kind"] == "error" and "injected" in rt.plans[-1]["error"]
    assert rt.policy is None and rt.stats["plan_errors"] == 1 and rt.stats["release"] == 0
    # a forced re-plan with a working trace build installs a policy again
    rt.ctx.trace_build = real
    rt.request_replan()
    for x, y in G.batches(3, 2, 16, 64):
        _step(rt, model, opt, x, y)
    assert rt.plans[-1]["kind"] != "error" and rt.plans[-1]["items"] > 0


def test_native_hook_is_scoped_to_steps():
    """the C++ hook records only inside rt.step(): the mode key is in the thread's dispatch key
    set for the step only; ops outside steps are not recorded, and a second runtime's steps get
    their own tokens (the hook is attached per step)"""
    from paper_2509_11076_b200.runtime import native_hook
    nh = native_hook()
    model, opt, data, rt = _setup(4)
    x, y = data[0]
    _step(rt, model, opt, x, y)
    n1 = rt.last_step["ops"]
    assert n1 > 100 and not nh.enabled()
    for _ in range(3):
        model(x, y).backward()  # outside any step: not recorded
    _step(rt, model, opt, x, y)
    assert rt.last_step["ops"] == n1 and not rt.last_step["changed"]
    rt2 = Runtime(None, hbm_budget=1, groups_fwd=4, groups_bwd=4)
    with rt2.step():
        model(x, y).backward()
    assert rt2.last_step["ops"] > 0 and not nh.enabled()
    with pytest.raises(RuntimeError):
        with rt.step():
            with rt2.step():  # two runtimes' steps at once in one process
                pass
    rt.close()
    rt2.close()
