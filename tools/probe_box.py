"""One-off probe of the GPU box: link, host memory, copy-engine bandwidth (context for DESIGN.md)."""
import json, os, subprocess, time
import torch

def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:  # noqa
        return str(e)

out = {}
out["nvidia_smi_pcie"] = sh("nvidia-smi -q | grep -A 12 -i 'PCI' | head -60")
out["topo"] = sh("nvidia-smi topo -m")
out["free"] = sh("free -g")
out["lscpu"] = sh("lscpu | head -30")
out["nproc"] = sh("nproc")
out["numa"] = sh("ls /sys/devices/system/node/ | grep node; cat /sys/bus/pci/devices/*/numa_node 2>/dev/null | sort | uniq -c")
bus = sh("nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader").strip()
out["gpu_bus"] = bus
if bus:
    b = bus.lower()
    if b.startswith("0000") and len(b.split(":")[0]) == 8:
        b = b[4:]
    out["gpu_numa_node"] = sh(f"cat /sys/bus/pci/devices/{b}/numa_node")
    out["gpu_link"] = sh(f"cat /sys/bus/pci/devices/{b}/current_link_speed /sys/bus/pci/devices/{b}/current_link_width /sys/bus/pci/devices/{b}/max_link_speed /sys/bus/pci/devices/{b}/max_link_width")
dev = torch.device("cuda:0")
out["mem_get_info"] = torch.cuda.mem_get_info()
res = {}
for mib in (4, 64, 256, 1024):
    n = mib << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    for name, fn in (("d2h", lambda: h.copy_(d, non_blocking=True)), ("h2d", lambda: d.copy_(h, non_blocking=True))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        res[f"{name}_{mib}MiB_GBps"] = n * reps / (s.elapsed_time(e) * 1e-3) / 1e9
    # bidirectional
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d2 = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        with torch.cuda.stream(s1):
            h.copy_(d, non_blocking=True)
        with torch.cuda.stream(s2):
            d2.copy_(h2, non_blocking=True)
    torch.cuda.synchronize()
    res[f"bidir_{mib}MiB_GBps_total"] = 2 * n * 10 / (time.perf_counter() - t0) / 1e9
out["ce_bw"] = res
t0 = time.perf_counter()
big = torch.empty(8 << 30, dtype=torch.uint8, pin_memory=True)
out["pin_8GiB_s"] = time.perf_counter() - t0
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1, default=str)
print(json.dumps(out["ce_bw"], indent=1))
