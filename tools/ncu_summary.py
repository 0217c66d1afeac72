#!/usr/bin/env python3
"""Summarise ncu output (launch list CSV + one --set full report) into profiles/.

    python tools/ncu_summary.py --launches gpurun_out/launches.csv --report gpurun_out/prof_fused.ncu-rep \
        --tag r01 [--kernel k_fused]

Writes profiles/<tag>_launches.md (per-kernel share of the step from the cold, serialised
launch list) and profiles/<tag>_ncu_<kernel>.json/.md (duration, DRAM bytes per launch ->
roofline "traffic", issue/pipe utilisation, stall reasons, occupancy).  bench.py reads the
newest profiles/*_ncu_k_fused.json for the "traffic" field.
"""
import argparse
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    d = collections.defaultdict(list)
    unit = None
    for r in rows[hi + 1:]:
        if len(r) > vi:
            name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
            d[name].append(float(r[vi].replace(",", "")))
            unit = r[ui]
    tot = sum(sum(v) for v in d.values())
    out = []
    for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
        out.append({"kernel": k, "launches": len(v), "mean": sum(v) / len(v), "total": sum(v), "share": sum(v) / tot})
    return out, unit


def raw_metrics(rep):
    r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(r.splitlines()))
    h, units, vals = rows[0], rows[1], rows[2:]
    return h, units, vals


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--report")
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--kernel", default="k_fused")
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    if a.launches:
        rows, unit = launches(a.launches)
        lines = [f"# ncu launch list ({a.launches}): per-kernel share (cold, serialised; compare shares)", "",
                 f"| kernel | launches | mean ({unit}) | total ({unit}) | share |", "|---|---|---|---|---|"]
        for r in rows:
            lines.append(f"| {r['kernel']} | {r['launches']} | {r['mean']:.0f} | {r['total']:.0f} | {100 * r['share']:.1f}% |")
        open(os.path.join(ROOT, "profiles", f"{a.tag}_launches.md"), "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))
    if a.report:
        h, units, vals = raw_metrics(a.report)
        want = {
            "duration_ns": "gpu__time_duration.sum",
            "dram_read_bytes": "dram__bytes_read.sum",
            "dram_write_bytes": "dram__bytes_write.sum",
            "sm_cycles_active_avg": "sm__cycles_active.avg",
            "elapsed_cycles": "gpc__cycles_elapsed.max",
            "inst_executed": "smsp__inst_executed.sum",
            "ipc_active": "sm__inst_executed.avg.per_cycle_active",
            "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
            "pipe_fma_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "pipe_alu_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "pipe_lsu_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "warps_active_avg": "sm__warps_active.avg.per_cycle_active",
            "registers_per_thread": "launch__registers_per_thread",
            "dyn_smem_per_block_bytes": "launch__shared_mem_per_block_dynamic",
            "grid_size": "launch__grid_size",
            "block_size": "launch__block_size",
            "l2_hit_pct": "lts__t_sector_hit_rate.pct",
            "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        }
        results = []
        for v in vals:
            name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
            if a.kernel not in name:
                continue
            d = {"kernel": name.split("(")[0]}
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Kbyte/block": 1e3, "byte/block": 1,
                     "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}
            for k, m in want.items():
                if m in h:
                    i = h.index(m)
                    try:
                        d[k] = float(v[i].replace(",", "")) * scale.get(units[i], 1)
                    except ValueError:
                        d[k] = v[i]
            stalls = {}
            for i, n in enumerate(h):
                if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
                    try:
                        x = float(v[i].replace(",", ""))
                    except ValueError:
                        continue
                    if x > 0.02:
                        stalls[n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = x
            d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda x: -x[1]))
            if "dram_read_bytes" in d and "dram_write_bytes" in d:
                d["traffic_bytes_per_launch"] = d["dram_read_bytes"] + d["dram_write_bytes"]
            results.append(d)
        out = {"report": a.report, "kernel": a.kernel, "captures": results,
               "note": "ncu --set full --clock-control none; per-launch counters (replayed ~40x: cold caches)"}
        jp = os.path.join(ROOT, "profiles", f"{a.tag}_ncu_{a.kernel}.json")
        json.dump(out, open(jp, "w"), indent=1)
        print(json.dumps(out, indent=1)[:3000])


if __name__ == "__main__":
    sys.exit(main())
