"""cProfile of 10 Stable-stage steps of the runtime on a host-bound toy GPT (policy installed):
where the executor's per-op host time goes.  python tools/prof_stable.py"""
import cProfile, pstats, sys, time, torch, os
sys.path.insert(0, os.getcwd())
from paper_2509_11076_b200.runtime import Runtime
from workloads import tiny_gpt as G
dev = torch.device("cuda:0")
cfg = dict(vocab=512, d=256, n_layer=6, n_head=8, seq=256)
m = G.make(0, dev, **cfg); opt = torch.optim.SGD(m.parameters(), lr=0.01)
x, y = G.batches(1, 16, 256, 512, seed=1, device=dev)[0]
def step(cm=None):
    torch.cuda.synchronize(); torch.cuda.reset_peak_memory_stats(); base = torch.cuda.memory_allocated()
    if cm is not None: cm.__enter__()
    l = m(x, y); l.backward(); opt.step(); opt.zero_grad(set_to_none=True)
    if cm is not None: cm.__exit__(None, None, None)
    torch.cuda.synchronize(); return torch.cuda.max_memory_allocated() - base
for _ in range(3): step()
peak = step()
rt = Runtime(0, hbm_budget=torch.cuda.memory_allocated() + int(0.55 * peak), groups_fwd=6, groups_bwd=6, trials=1)
for _ in range(12): step(rt.step())
pr = cProfile.Profile(); pr.enable()
for _ in range(10): step(rt.step())
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
