"""Per-CUDA-source-line instruction counts and stall samples from an ncu report
(`--print-source cuda,sass`).  Usage: python tools/ncu_lines.py <rep> <source.cu> [top]"""
import csv
import io
import subprocess
import sys


def main(rep, src, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--resolve-source-file", src], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    ix = {h: i for i, h in enumerate(hdr)}
    i_ins = hdr.index("Instructions Executed")
    i_smp = hdr.index("Warp Stall Sampling (All Samples)")
    lines = []
    for r in rows:
        if len(r) > i_ins and r[0] not in ("", "Line No") and r[0].isdigit():
            try:
                lines.append((int(r[0]), r[1], float(r[i_ins] or 0), float(r[i_smp] or 0)))
            except ValueError:
                pass
    ti = sum(x[2] for x in lines) or 1
    ts = sum(x[3] for x in lines) or 1
    print(f"total warp instructions {ti:.3e}, stall samples {ts:.0f}")
    for ln, s, ins, smp in sorted(lines, key=lambda x: -x[2])[:top]:
        print(f"{ln:5d} ins {ins / ti:6.3f} smp {smp / ts:6.3f}  {s.strip()[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
