"""Host-link counters for the swap paths (VERDICT r01 missing 4): a 1 GiB batch (16 x 64 MiB
descriptors) swapped out and back in repeatedly, through the swap kernel and through the copy
engines (one cudaMemcpyAsync per descriptor), each phase ~1 s, while NVML samples the GPU's PCIe
TX / RX byte counters (nvmlDeviceGetPcieThroughput, 20 ms windows): link bytes vs payload bytes
per direction.  Under ncu (`--mode ncu`: one kernel round trip between cudaProfilerStart/Stop
for range replay) the pcie__* counters of the kernel launches themselves.

    python tools/pcie_counters.py [--mode nvml|ncu]"""
import json
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200 import chm  # noqa: E402


def sampler(handle, stop, out):
    import pynvml
    while not stop.is_set():
        tx = pynvml.nvmlDeviceGetPcieThroughput(handle, pynvml.NVML_PCIE_UTIL_TX_BYTES)  # KB/s
        rx = pynvml.nvmlDeviceGetPcieThroughput(handle, pynvml.NVML_PCIE_UTIL_RX_BYTES)
        out.append((time.perf_counter(), tx, rx))


def main():
    mode = sys.argv[sys.argv.index("--mode") + 1] if "--mode" in sys.argv else "nvml"
    n_desc, each = 16, 64 << 20
    ctx = chm.Context(device=0, host_arena_bytes=n_desc * each, swap_ctas=8, time_batches=True)
    dev = torch.device("cuda:0")
    bufs = [torch.randint(0, 256, (each,), dtype=torch.uint8, device=dev) for _ in range(n_desc)]
    descs = [(b.data_ptr(), j * each, each) for j, b in enumerate(bufs)]
    comp, s = torch.cuda.current_stream(), torch.cuda.Stream()
    if mode == "ncu":
        for flags in (chm.SWAP_KERNEL, chm.SWAP_KERNEL):  # warm, then the profiled round trip
            ctx.batch_wait(ctx.swap_out(descs, comp, s, flags), comp)
            ctx.batch_wait(ctx.swap_in(descs, comp, s, flags), comp)
        torch.cuda.synchronize()
        return
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    res = {"batch_bytes": n_desc * each, "phases": {}}
    for name, flags in (("kernel", chm.SWAP_KERNEL), ("copy_engines", chm.SWAP_CE)):
        for direction in ("d2h", "h2d"):
            fn = ctx.swap_out if direction == "d2h" else ctx.swap_in
            for _ in range(2):
                ctx.batch_wait(fn(descs, comp, s, flags), comp)
            torch.cuda.synchronize()
            samples, stop = [], threading.Event()
            th = threading.Thread(target=sampler, args=(h, stop, samples))
            th.start()
            time.sleep(0.1)
            t0 = time.perf_counter()
            batches = []
            while time.perf_counter() - t0 < 1.2:
                b = fn(descs, comp, s, flags)
                ctx.batch_wait(b, comp)
                batches.append(b)
                torch.cuda.synchronize()
            stop.set()
            th.join()
            payload = n_desc * each * len(batches) / (sum(ctx.batch_elapsed_ms(b) for b in batches) * 1e-3) / 1e9
            mid = [x for x in samples if t0 + 0.1 < x[0] < t0 + 1.1]
            tx = float(np.median([x[1] for x in mid])) * 1e3 / 1e9 if mid else None  # KB/s -> GB/s
            rx = float(np.median([x[2] for x in mid])) * 1e3 / 1e9 if mid else None
            link = tx if direction == "d2h" else rx
            res["phases"][f"{name}_{direction}"] = {
                "payload_GBps": payload, "nvml_tx_GBps": tx, "nvml_rx_GBps": rx,
                "link_over_payload": (link / payload) if link else None, "samples": len(mid)}
            print(name, direction, json.dumps(res["phases"][f"{name}_{direction}"]), flush=True)
    pynvml.nvmlShutdown()
    ctx.close()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
