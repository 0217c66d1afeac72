#!/usr/bin/env python3
"""Per-kernel ncu evidence (north star: "each kernel is evidenced by ncu counters: achieved HBM
GB/s against B200 peak, and bytes moved per pixel per frame against the minimal field traffic").

    python tools/ncu_evidence.py REPORT.ncu-rep --kernel REGEX --pixels N --algo-bytes B --algo-ops OPS
        --tag r02_cfg2 [--peaks MEASURED_PEAKS.json]

For every captured launch of the kernels matching REGEX: duration, DRAM bytes (read + write, per
launch and per pixel) against the algorithmic bytes per pixel, DRAM GB/s against the measured HBM
peak, FP32 lane-operations per pixel counted from the SASS source page (executed warp-level
instructions x 32, paired f32x2 ops FADD2 / FMUL2 / FFMA2 counted twice) against the algorithmic
count (predicated-on thread instructions), thread-instructions per pixel, IPC and pipe
utilisation.  Writes profiles/<tag>_<kernel>.json
and appends a row to profiles/<tag>_evidence.md.
"""
import argparse
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FP1 = {"FADD", "FMUL", "FFMA"}
FP2 = {"FADD2", "FMUL2", "FFMA2"}
RAW = {
    "duration_ns": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "sm_cycles_active_avg": "sm__cycles_active.avg",
    "elapsed_cycles": "gpc__cycles_elapsed.max",
    "inst_executed": "smsp__inst_executed.sum",
    "ipc_active": "sm__inst_executed.avg.per_cycle_active",
    "pipe_fma_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "pipe_alu_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "pipe_lsu_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "registers_per_thread": "launch__registers_per_thread",
    "grid_size": "launch__grid_size",
    "block_size": "launch__block_size",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "usecond": 1e3, "nsecond": 1,
         "ms": 1e6, "msecond": 1e6}


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def raw(rep):
    rows = list(csv.reader(ncu("-i", rep, "--page", "raw", "--csv").splitlines()))
    return rows[0], rows[1], rows[2:]


def fp_ops(rep, kname_regex):
    """(fp32 lane-ops, thread instructions) per launch from the SASS source page (predicated-on
    thread instructions; paired f32x2 ops count twice), averaged over the captured launches of
    the kernels whose name matches (template casts like "(int)7" normalised to "7")."""
    txt = ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass")
    fp, ti, nlaunch = 0, 0, 0
    header, on = None, False
    for ln in csv.reader(txt.splitlines()):
        if not ln:
            continue
        if ln[0] == "Kernel Name":
            name = re.sub(r"\((int|bool|unsigned int|long)\)", "", ln[1])
            on = re.search(kname_regex, name) is not None
            nlaunch += 1 if on else 0
            header = None
            continue
        if ln[0] == "Address":
            header = ln
            continue
        if not on or header is None or len(ln) != len(header):
            continue
        src = ln[header.index("Source")].strip()
        col = "Predicated-On Thread Instructions Executed"
        try:
            n = int(ln[header.index(col)] or 0) if col in header else 32 * int(ln[header.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        toks = src.split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        base = op.split(".")[0]
        ti += n
        if base in FP2:
            fp += 2 * n
        elif base in FP1:
            fp += n
    nlaunch = max(1, nlaunch)
    return fp / nlaunch, ti / nlaunch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--kernel", required=True, help="regex on the kernel name")
    ap.add_argument("--pixels", type=float, required=True, help="pixels one launch processes (B x H x W)")
    ap.add_argument("--algo-bytes", type=float, default=None, help="algorithmic bytes per pixel of this kernel")
    ap.add_argument("--algo-ops", type=float, default=None, help="algorithmic FP32 ops per pixel per launch")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--label", default=None)
    ap.add_argument("--name", default=None, help="json name (default: the kernel's), e.g. cfg2_k_trans")
    ap.add_argument("--peaks", default=os.path.join(ROOT, "MEASURED_PEAKS.json"))
    a = ap.parse_args()
    pk = json.load(open(a.peaks)) if os.path.exists(a.peaks) else {}
    hbm = pk.get("hbm_gbs", 6650.0)
    h, units, vals = raw(a.report)
    ki = h.index("Kernel Name")
    caps = []
    for v in vals:
        if not re.search(a.kernel, v[ki]):
            continue
        d = {"kernel": v[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")}
        for k, m in RAW.items():
            if m in h:
                i = h.index(m)
                try:
                    d[k] = float(v[i].replace(",", "")) * SCALE.get(units[i], 1)
                except ValueError:
                    pass
        caps.append(d)
    if not caps:
        print("no launches of", a.kernel, file=sys.stderr)
        return 1
    fp, ti = fp_ops(a.report, a.kernel)
    avg = {k: sum(c[k] for c in caps if k in c) / len([c for c in caps if k in c])
           for k in caps[0] if isinstance(caps[0][k], float)}
    dram = avg.get("dram_read_bytes", 0) + avg.get("dram_write_bytes", 0)
    t_s = avg["duration_ns"] * 1e-9
    out = {
        "report": os.path.basename(a.report), "kernel": caps[0]["kernel"], "label": a.label, "launches": len(caps),
        "pixels_per_launch": a.pixels, "per_launch": avg,
        "dram_bytes_per_launch": dram, "dram_bytes_per_px": dram / a.pixels,
        "algo_bytes_per_px": a.algo_bytes,
        "dram_gbs": dram / t_s / 1e9, "hbm_peak_gbs": hbm, "dram_frac_of_peak": dram / t_s / 1e9 / hbm,
        "fp32_lane_ops_per_px": fp / a.pixels, "algo_fp32_ops_per_px": a.algo_ops,
        "thread_inst_per_px": ti / a.pixels,
        "note": "ncu --set full --clock-control none (replayed, cache-flushed: cold L2; durations are "
                "serialised single launches); FP32 lane-ops from the SASS source page (FADD2/FMUL2/FFMA2 x2)",
    }
    name = a.name or re.sub(r"[^A-Za-z0-9_]+", "_", caps[0]["kernel"]).strip("_")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "profiles", f"{a.tag}_{name}.json"), "w"), indent=1)
    md = os.path.join(ROOT, "profiles", f"{a.tag}_evidence.md")
    new = not os.path.exists(md)
    with open(md, "a") as fh:
        if new:
            fh.write("| workload | kernel | launches | us (cold) | DRAM B/px | algo B/px | DRAM GB/s (frac) | "
                     "FP32 ops/px | algo ops/px | thread-inst/px | IPC | FMA pipe % | ALU pipe % |\n")
            fh.write("|---|---|---|---|---|---|---|---|---|---|---|---|---|\n")
        fh.write(f"| {a.label or a.tag} | {caps[0]['kernel']} | {len(caps)} | {avg['duration_ns'] / 1e3:.2f} | "
                 f"{dram / a.pixels:.1f} | {a.algo_bytes if a.algo_bytes is not None else '-'} | "
                 f"{dram / t_s / 1e9:.0f} ({dram / t_s / 1e9 / hbm:.3f}) | {fp / a.pixels:.0f} | "
                 f"{a.algo_ops if a.algo_ops is not None else '-'} | {ti / a.pixels:.0f} | "
                 f"{avg.get('ipc_active', 0):.2f} | {avg.get('pipe_fma_pct', 0):.0f} | {avg.get('pipe_alu_pct', 0):.0f} |\n")
    print(json.dumps(out, indent=1))
    return 0


if __name__ == "__main__":
    sys.exit(main())
