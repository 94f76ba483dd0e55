"""python tools/overlap.py [ctas,ctas,...]

C3-style overlap: swaps on the swap stream while bf16 GEMMs run on the compute
stream.  Reports GEMM TFLOP/s with no swap, with copy-engine swaps and with the swap kernel (its
SM cost), and the swap GB/s under contention."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200 import chm  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    n = 8192
    a = torch.randn(n, n, dtype=torch.bfloat16, device=dev)
    b = torch.randn(n, n, dtype=torch.bfloat16, device=dev)
    c = torch.empty(n, n, dtype=torch.bfloat16, device=dev)
    nb = 64 << 20
    bufs = [torch.empty(nb, dtype=torch.uint8, device=dev) for _ in range(32)]  # 2 GiB
    descs = [(x.data_ptr(), j * nb, nb) for j, x in enumerate(bufs)]
    res = {}
    ctas_list = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [8, 16, 32]
    for ctas in ctas_list:
        ctx = chm.Context(device=0, host_arena_bytes=2 << 30, swap_ctas=ctas, time_batches=True)
        comp, sw = torch.cuda.current_stream(), torch.cuda.Stream()
        for mode in ("none", "ce", "kernel"):
            for _ in range(3):
                torch.matmul(a, b, out=c)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            batches = []
            if mode != "none":
                flags = chm.SWAP_CE if mode == "ce" else chm.SWAP_KERNEL
                for _ in range(2):  # 4 GiB out then in, enqueued before the GEMMs start
                    batches.append(ctx.swap_out(descs, sw, sw, flags))
                    batches.append(ctx.swap_in(descs, sw, sw, flags))
            s.record(comp)
            iters = 60
            for _ in range(iters):
                torch.matmul(a, b, out=c)
            e.record(comp)
            torch.cuda.synchronize()
            ms = s.elapsed_time(e)
            tflops = 2 * n ** 3 * iters / (ms * 1e-3) / 1e12
            swap_gbps = None
            if batches:
                t = sum(ctx.batch_elapsed_ms(x) for x in batches)
                swap_gbps = 2 * 2 * (32 * nb) / (t * 1e-3) / 1e9
            res[f"{mode}_ctas{ctas}"] = dict(gemm_tflops=tflops, swap_GBps=swap_gbps, gemm_ms=ms)
            print(mode, ctas, f"GEMM {tflops:7.1f} TFLOP/s", f"swap {swap_gbps}", flush=True)
        ctx.close()
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(res, open("gpurun_out/overlap.json", "w"), indent=1)


if __name__ == "__main__":
    main()
