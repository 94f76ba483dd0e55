"""Swap throughput of misaligned views: a 64 MiB batch of 16 x 4 MiB
descriptors out and back in, device and host addresses offset by (dev_mis, host_mis) bytes mod
16 -- aligned, the same misalignment, different misalignments -- through the swap kernel and
the copy engines.  Prints one JSON line (GB/s per direction, byte-exact check).

    python tools/swap_misaligned.py"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200 import chm  # noqa: E402


def main():
    n_desc, each = 16, 4 << 20
    ctx = chm.Context(device=0, host_arena_bytes=n_desc * (each + 4096), swap_ctas=8, time_batches=True)
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(3)
    bufs = [torch.randint(0, 256, (each + 64,), dtype=torch.uint8, device=dev, generator=g) for _ in range(n_desc)]
    outs = [torch.zeros(each + 64, dtype=torch.uint8, device=dev) for _ in range(n_desc)]
    comp, s = torch.cuda.current_stream(), torch.cuda.Stream()
    res = {"batch_bytes": n_desc * each, "descriptors": n_desc, "cases": []}
    for dev_mis, host_mis in ((0, 0), (5, 5), (8, 8), (0, 3), (3, 0), (1, 2), (7, 12), (15, 1)):
        d_out = [(b[dev_mis:].data_ptr(), j * (each + 4096) + host_mis, each) for j, b in enumerate(bufs)]
        d_in = [(o[dev_mis:].data_ptr(), j * (each + 4096) + host_mis, each) for j, o in enumerate(outs)]
        case = {"dev_mis": dev_mis, "host_mis": host_mis}
        for name, flags in (("kernel", chm.SWAP_KERNEL), ("copy_engines", chm.SWAP_CE)):
            t_o, t_i = [], []
            for it in range(6):
                bo = ctx.swap_out(d_out, comp, s, flags)
                ctx.batch_wait(bo, comp)
                bi = ctx.swap_in(d_in, comp, s, flags)
                ctx.batch_wait(bi, comp)
                torch.cuda.synchronize()
                if it >= 2:
                    t_o.append(ctx.batch_elapsed_ms(bo))
                    t_i.append(ctx.batch_elapsed_ms(bi))
            ok = all(torch.equal(o[dev_mis:dev_mis + each], b[dev_mis:dev_mis + each]) for o, b in zip(outs, bufs))
            for o in outs:
                o.zero_()
            case[name] = {"d2h_GBps": n_desc * each / (np.median(t_o) * 1e-3) / 1e9,
                          "h2d_GBps": n_desc * each / (np.median(t_i) * 1e-3) / 1e9, "byte_exact": ok}
        res["cases"].append(case)
        print(json.dumps(case), flush=True)
    ctx.close()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
