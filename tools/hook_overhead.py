"""The profiler hook's cost (the paper's Table 1: Lightweight +0.9%, Detailed +34.6% per
iteration on their stack): step time of a training step without the runtime, under
the runtime in Lightweight mode (WarmUp stage, no policy: every op recorded as a token), and the
Detailed step (tensors, frees, allocator bytes).  Two models: a GPT-style model small enough
that the host is the bottleneck (every microsecond of hook shows), and 4 layers of Llama-2 7B
(the device is the bottleneck).  Prints one JSON line.

    python tools/hook_overhead.py
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200 import chm  # noqa: E402
from paper_2509_11076_b200.runtime import Runtime  # noqa: E402
from workloads import llama as L  # noqa: E402
from workloads import tiny_gpt as G  # noqa: E402


def measure(model, opt, x, y, steps=8):
    def one(rt=None):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if rt is not None:
            cm = rt.step()
            cm.__enter__()
        loss = model(x, y)
        loss.backward()
        opt.step()
        opt.zero_grad(set_to_none=True)
        if rt is not None:
            cm.__exit__(None, None, None)
        torch.cuda.synchronize()
        return time.perf_counter() - t0

    for _ in range(3):
        one()
    plain = sorted(one() for _ in range(steps))[steps // 2]
    rt = Runtime(0, hbm_budget=1 << 62, groups_fwd=4, groups_bwd=4, bw=50e9)
    light = []
    for _ in range(3):  # WarmUp: Lightweight
        light.append(one(rt))
        assert rt.stage == chm.WARMUP or len(light) == 3
    detailed = None
    for _ in range(steps):
        detailing = rt.stage == chm.GENPOLICY and rt.need_plan
        t = one(rt)
        if detailing:
            detailed = t
        elif rt.policy is None:
            light.append(t)
    ops = rt.last_step["ops"]
    lw = sorted(light)[len(light) // 2]
    rt.close()
    return dict(ops=ops, plain_s=round(plain, 5), lightweight_s=round(lw, 5), detailed_s=round(detailed or 0, 5),
                lightweight_overhead=round(lw / plain - 1, 4),
                detailed_overhead=round((detailed or 0) / plain - 1, 4),
                hook_us_per_op=round((lw - plain) / ops * 1e6, 2))


def main():
    dev = torch.device("cuda:0")
    out = {}
    m = G.make(0, dev, vocab=512, d=256, n_layer=6, n_head=8, seq=256)
    x, y = G.batches(1, 16, 256, 512, seed=1, device=dev)[0]
    out["tiny_gpt_host_bound"] = measure(m, torch.optim.SGD(m.parameters(), lr=0.01), x, y)
    del m
    cfg = dict(L.LLAMA2_7B, n_layer=4)
    m = L.make(cfg, max_seq=4096)
    x, y = L.batch(4, 4096, cfg["vocab"])
    out["llama2_7b_4L_b4_s4096"] = measure(m, torch.optim.SGD(m.parameters(), lr=1e-5), x, y)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
