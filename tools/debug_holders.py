"""debug: saved-tensor boxes (holders) seen by the runtime after the forward of a WarmUp step with
OOM handling on, C++ hook vs Python hook (tiny GPT on cuda:0)."""
import collections
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200.runtime import Runtime  # noqa: E402
from workloads import tiny_gpt as G  # noqa: E402

CFG = dict(vocab=512, d=256, n_layer=6, n_head=8, seq=256)
dev = torch.device("cuda:0")
for native in (True, False):
    m = G.make(0, dev, **CFG)
    opt = torch.optim.SGD(m.parameters(), lr=0.05)
    x, y = G.batches(1, 16, CFG["seq"], CFG["vocab"], seed=1, device=dev)[0]
    rt = Runtime(0, hbm_budget=1 << 62, groups_fwd=6, groups_bwd=6, oom_host_bytes=1 << 30, trials=1,
                 native_hook=native)
    with rt.step():
        loss = m(x, y)
        sizes = collections.Counter(h.nbytes for h in rt.holders.values())
        loss.backward()
        opt.step()
        opt.zero_grad(set_to_none=True)
    print("native" if native else "python", sorted(sizes.items()), rt.last_step["ops"], flush=True)
    rt.close()
