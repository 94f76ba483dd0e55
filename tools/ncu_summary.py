"""Writes a text summary of an ncu report (speed-of-light, DRAM bytes, occupancy, stall mix,
hottest SASS) for profiles/.  Usage: python tools/ncu_summary.py <rep> <out.txt> [title]"""
import csv
import io
import subprocess
import sys


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep, out, title=""):
    lines = [f"# {title or rep}", f"source: {rep}", ""]
    det = list(csv.reader(io.StringIO(ncu(rep, "--page", "details", "--csv"))))
    hdr = det[0]
    i_k = hdr.index("Kernel Name")
    i_sec, i_name, i_unit, i_val = hdr.index("Section Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    keep = {"Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
            "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy",
            "Registers Per Thread", "Dynamic Shared Memory Per Block", "Block Size", "Grid Size",
            "Warp Cycles Per Issued Instruction", "Executed Instructions", "Theoretical Occupancy"}
    if len(det) > 1:
        lines.append(f"kernel: {det[1][i_k]}")
    for r in det[1:]:
        if r[i_name] in keep:
            lines.append(f"  {r[i_sec][:34]:34s} {r[i_name]:38s} {r[i_val]:>14s} {r[i_unit]}")
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    if len(raw) > 2:
        h, u, v = raw[0], raw[1], raw[2]
        for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                     "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"):
            if name in h:
                j = h.index(name)
                lines.append(f"  raw {name:52s} {v[j]:>14s} {u[j]}")
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    if len(src) > 2:
        hdr = src[1]
        ix = {x: i for i, x in enumerate(hdr)}
        data = []
        for r in src[2:]:  # first kernel's rows only (a report with several launches repeats the header)
            if len(r) != len(hdr) or r[ix["Warp Stall Sampling (All Samples)"]] == "Warp Stall Sampling (All Samples)":
                break
            data.append(r)
        tot = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
        stalls = [x for x in hdr if x.startswith("stall_") and "Not Issued" not in x]
        agg = {x: sum(float(r[ix[x]] or 0) for r in data) for x in stalls}
        lines += ["", "stall mix (share of samples): " + ", ".join(
            f"{k[6:]} {v / max(tot, 1):.2f}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8])]
        data.sort(key=lambda r: -float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
        lines.append("hottest SASS (share of stall samples, executions, instruction):")
        for r in data[:15]:
            s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
            lines.append(f"  {s / max(tot, 1):6.3f} {float(r[ix['Instructions Executed']] or 0):10.3e}  {r[ix['Source']][:100]}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
