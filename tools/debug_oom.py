"""debug: Algo. 3 decisions under a memory cap, C++ hook vs Python hook (tests/_oom_child.py's
model and cap)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200.runtime import Runtime  # noqa: E402
from tests._oom_child import CFG, train  # noqa: E402

torch.cuda.reset_peak_memory_stats()
base = torch.cuda.memory_allocated()
train(steps=2)
peak = torch.cuda.max_memory_allocated() - base
torch.cuda.empty_cache()
total = torch.cuda.get_device_properties(0).total_memory
native = sys.argv[1] == "native"
rt = Runtime(0, hbm_budget=1 << 62, groups_fwd=6, groups_bwd=6, oom_host_bytes=1 << 30, trials=1, native_hook=native)
torch.cuda.synchronize()
torch.cuda.empty_cache()
cap = torch.cuda.memory_reserved() + int(0.6 * peak)
torch.cuda.set_per_process_memory_fraction(cap / total)
try:
    train(rt, steps=3)
    ok = True
except torch.OutOfMemoryError:
    ok = False
log = list(rt.oom_log)
print(json.dumps(dict(mode=sys.argv[1], ok=ok, stats=rt.stats, first=[x for x in log if x[0] != "freed"][:60])))
