#!/usr/bin/env python3
"""Per-kernel steady-state durations of the split step on the bench workload (config 2 unless
--config): frames run as sf_predict (k_trans) and sf_update (k_upd) with CUDA events between them
on the context stream (no PDL overlap across the event), inputs from a > L2 ring.

    python tools/ktime.py [--frames 400] [--config 2] [--levels 1]
Prints one JSON line: median / mean microseconds of each kernel and of the sum."""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=400)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--ring", type=int, default=48)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2406_18031_b200 as sf
    import sfgen

    seq = sfgen.config_sequence(args.config, frames=args.ring)
    dev = torch.device("cuda", 0)
    Yd = torch.from_numpy(np.ascontiguousarray(seq.Y)).to(dev)
    Dd = torch.from_numpy(np.ascontiguousarray(seq.depth)).to(dev)
    s = torch.cuda.Stream(device=dev)
    m = sf.StructureFlow(seq.geom, seq.params, batch=1, device=0, stream=s, kernel=sf.SF_KERNEL_FUSED)
    with torch.cuda.stream(s):
        m.step(Yd[0], Dd[0])
        for k in range(1, args.ring):
            m.step(Yd[k], Dd[k])
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.frames)]
    with torch.cuda.stream(s):
        for i in range(args.frames):
            k = i % args.ring
            ev[i][0].record(s)
            m.predict()
            ev[i][1].record(s)
            m.update(Yd[k], Dd[k])
            ev[i][2].record(s)
    torch.cuda.synchronize()
    # calibration: the same event pattern around one tiny torch kernel
    x = torch.zeros(16, device=dev)
    cal = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(100)]
    with torch.cuda.stream(s):
        for c in cal:
            c[0].record(s)
            x.add_(1.0)
            c[1].record(s)
    torch.cuda.synchronize()
    tcal = [c[0].elapsed_time(c[1]) * 1e3 for c in cal[10:]]
    tp = [e[0].elapsed_time(e[1]) * 1e3 for e in ev[10:]]
    tu = [e[1].elapsed_time(e[2]) * 1e3 for e in ev[10:]]
    out = {"config": args.config, "frames": len(tp),
           "k_trans_us": {"median": statistics.median(tp), "mean": statistics.mean(tp)},
           "k_upd_us": {"median": statistics.median(tu), "mean": statistics.mean(tu)},
           "sum_median_us": statistics.median(tp) + statistics.median(tu),
           "tiny_kernel_us": statistics.median(tcal),
           "env": {k: v for k, v in os.environ.items() if k.startswith("SF_")}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
