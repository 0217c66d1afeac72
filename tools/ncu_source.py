#!/usr/bin/env python3
"""Per-region warp-stall profile of one kernel from `ncu --page source --csv --print-source sass`.

    ncu -i rep --page source --csv --print-source sass > src.csv; python tools/ncu_source.py src.csv [bin]

Splits the SASS at BAR.SYNC instructions (the kernel's phases), prints per region the share of
stall samples, the instructions executed and the top stall reasons.
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    h = rows[1]
    data = rows[2:]
    si = h.index("Source")
    ns = h.index("Warp Stall Sampling (All Samples)")
    ie = h.index("Instructions Executed")
    stall_cols = [(i, n) for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
    regions = []
    cur = {"start": 0, "samples": 0, "inst": 0, "stalls": {}, "n": 0, "first": None}
    for k, r in enumerate(data):
        src = r[si].strip()
        if cur["first"] is None:
            cur["first"] = src[:40]
        cur["samples"] += int(r[ns] or 0)
        cur["inst"] += int(r[ie] or 0)
        cur["n"] += 1
        for i, n in stall_cols:
            v = int(r[i] or 0)
            if v:
                cur["stalls"][n[6:]] = cur["stalls"].get(n[6:], 0) + v
        if "BAR.SYNC" in src or k == len(data) - 1:
            cur["end"] = k
            regions.append(cur)
            cur = {"start": k + 1, "samples": 0, "inst": 0, "stalls": {}, "n": 0, "first": None}
    tot = sum(r["samples"] for r in regions)
    for r in regions:
        if r["samples"] < 0.005 * tot:
            continue
        top = sorted(r["stalls"].items(), key=lambda x: -x[1])[:5]
        print(f"[{r['start']:5d}-{r['end']:5d}] {100 * r['samples'] / tot:5.1f}%  inst={r['inst']:9d}  "
              + " ".join(f"{k}={100 * v / r['samples']:.0f}%" for k, v in top) + f"   | {r['first']}")


if __name__ == "__main__":
    main()
