"""Summarise an ncu --page source --print-source sass CSV: hottest instructions by stall samples
and instruction counts (run here, on the CPU box)."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = rows[2:]
    tot_s = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
    tot_i = sum(float(r[ix["Instructions Executed"]] or 0) for r in data)
    print(f"total stall samples {tot_s:.0f}, warp instructions {tot_i:.3e}")
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = {h: sum(float(r[ix[h]] or 0) for r in data) for h in stalls}
    print("stall mix:", ", ".join(f"{k[6:]}={v / max(tot_s, 1):.2f}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    data.sort(key=lambda r: -float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
    for r in data[:top]:
        s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        top_stall = max(stalls, key=lambda h: float(r[ix[h]] or 0))
        print(f"{s / max(tot_s, 1):6.3f} {float(r[ix['Instructions Executed']] or 0):10.3e} {top_stall[6:]:14s} {r[ix['Address']]:>6s} {r[ix['Source']][:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
