#!/usr/bin/env python3
"""Per-kernel device times of the split step through sf_step_timed (spin-queued CUDA events) on the
bench workload; prints one JSON line {k_trans_us, k_upd_us} (means over --frames frames)."""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=100)
    ap.add_argument("--config", type=int, default=2)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2406_18031_b200 as sf
    import sfgen

    seq = sfgen.config_sequence(args.config, frames=16)
    dev = torch.device("cuda", 0)
    Yd = torch.from_numpy(np.ascontiguousarray(seq.Y)).to(dev)
    Dd = torch.from_numpy(np.ascontiguousarray(seq.depth)).to(dev)
    m = sf.StructureFlow(seq.geom, seq.params, kernel=sf.SF_KERNEL_FUSED)
    for k in range(16):
        m.step(Yd[k], Dd[k])
    torch.cuda.synchronize()
    tp, tu = [], []
    for i in range(args.frames):
        k = i % 16
        a, b = sf.sf_step_timed(m.ctx, Yd[k].data_ptr(), Dd[k].data_ptr())
        if i >= 5:
            tp.append(a * 1e3)
            tu.append(b * 1e3)
    print(json.dumps({"k_trans_us": statistics.mean(tp), "k_upd_us": statistics.mean(tu),
                      "k_trans_us_min": min(tp), "k_upd_us_min": min(tu),
                      "env": {k: v for k, v in os.environ.items() if k.startswith("SF_")}}))


if __name__ == "__main__":
    main()
