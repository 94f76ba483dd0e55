"""Where the runtime hook's per-op cost goes on a host-bound model: step time without a hook,
with an empty TorchDispatchMode, and under the runtime in Lightweight steps.  Prints one line."""
import time, torch
from torch.utils._python_dispatch import TorchDispatchMode
import sys; sys.path.insert(0, "/root/repo")
from workloads import tiny_gpt as G
from paper_2509_11076_b200.runtime import Runtime
dev = torch.device("cuda:0")
m = G.make(0, dev, vocab=512, d=256, n_layer=6, n_head=8, seq=256)
opt = torch.optim.SGD(m.parameters(), lr=0.01)
x, y = G.batches(1, 16, 256, 512, seed=1, device=dev)[0]
class Empty(TorchDispatchMode):
    def __torch_dispatch__(self, func, types, args=(), kwargs=None):
        return func(*args, **(kwargs or {}))
def step(ctx=None):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    if ctx is not None: ctx.__enter__()
    l = m(x, y); l.backward(); opt.step(); opt.zero_grad(set_to_none=True)
    if ctx is not None: ctx.__exit__(None, None, None)
    torch.cuda.synchronize(); return time.perf_counter() - t0
for _ in range(5): step()
plain = sorted(step() for _ in range(9))[4]
empty = sorted(step(Empty()) for _ in range(9))[4]
rt = Runtime(0, hbm_budget=1 << 62, bw=50e9)
ts = []
for i in range(3): ts.append(step(rt.step()))
light = sorted(ts)[1]
ops = rt.last_step["ops"]
print(f"ops {ops} plain {plain*1e3:.2f} ms empty-mode {empty*1e3:.2f} ms runtime-light {light*1e3:.2f} ms; per op: mode {(empty-plain)/ops*1e6:.2f} us, runtime code {(light-empty)/ops*1e6:.2f} us")
