#!/usr/bin/env python3
"""Per-CTA timeline of the split step (k_trans, k_upd) on the bench workload, from a debug build
(SF_BUILD_DEBUG=1, selected with SF_LIB) with SF_DEBUG_SKIP=16384: every CTA records its entry /
exit globaltimer and SM.  Frames run back to back by sf_step on one stream (no events between the
kernels, programmatic dependent launch as in production, no CUDA graph).

    SF_LIB=ab_lib/libsf_dbg.so SF_DEBUG_SKIP=16384 python tools/cta_trace.py [--frames 24]

Prints, for the last three complete frames: each kernel's first entry / last exit relative to the
frame's k_trans first entry, the gaps between the kernels, CTA duration quantiles and the last CTAs
to finish (block x, y, SM)."""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=24)
    ap.add_argument("--ring", type=int, default=8)
    ap.add_argument("--config", type=int, default=2)
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
        m.step(Yd[0], Dd[0])  # initialisation (per-pass kernels)
        torch.cuda.synchronize()
        for k in range(1, args.frames + 1):
            m.step(Yd[k % args.ring], Dd[k % args.ring])
    torch.cuda.synchronize()
    lib = C.CDLL(sf.LIB_PATH)
    n = 4096
    buf = (C.c_ulonglong * (3 * n))()
    frames = {}
    for name, fn in (("trans", lib.sf_debug_trace_trans), ("upd", lib.sf_debug_trace_upd)):
        fn.argtypes = [C.c_int, C.c_void_p, C.c_int]
        for slot in range(4):
            assert fn(slot, buf, n) == 0
            a = np.frombuffer(buf, dtype=np.uint64).reshape(n, 3).copy()
            a = a[a[:, 1] > 0]
            frames[(name, slot)] = a
    # slot of frame f is f & 3; the fused path's first frame after init is dbg_frame 0
    last = args.frames - 1
    for f in range(last - 2, last + 1):
        sl = f & 3
        tr, up = frames[("trans", sl)], frames[("upd", sl)]
        tprev = frames[("upd", (f - 1) & 3)]
        t0 = int(tr[:, 0].min())
        rel = lambda x: (int(x) - t0) / 1e3
        print(f"frame {f}: prev k_upd last exit {rel(tprev[:, 1].max()):8.2f} us")
        for name, a in (("k_trans", tr), ("k_upd", up)):
            d = (a[:, 1].astype(np.int64) - a[:, 0].astype(np.int64)) / 1e3
            print(f"  {name:8s} CTAs {len(a):4d}  entry {rel(a[:, 0].min()):7.2f}..{rel(a[:, 0].max()):7.2f}  "
                  f"exit {rel(a[:, 1].min()):7.2f}..{rel(a[:, 1].max()):7.2f} us  dur q10/50/90/max "
                  f"{np.percentile(d, 10):.2f}/{np.median(d):.2f}/{np.percentile(d, 90):.2f}/{d.max():.2f}")
            order = np.argsort(-a[:, 1].astype(np.int64))[:6]
            tail = [(int(a[i, 2] >> 16 & 0xFFFF), int(a[i, 2] >> 32), int(a[i, 2] & 0xFFFF), round(rel(a[i, 0]), 2),
                     round(rel(a[i, 1]), 2)) for i in order]
            print(f"    last to finish (bx, by, sm, entry, exit): {tail}")
        # per-SM hand-off: entry of this kernel's CTA - exit of the previous kernel's CTA on the same SM
        for name, prev, nxt in (("k_upd(prev)->k_trans", tprev, tr), ("k_trans->k_upd", tr, up)):
            ex = {int(r[2] & 0xFFFF): int(r[1]) for r in prev}
            lat = [(int(r[0]) - ex[int(r[2] & 0xFFFF)]) / 1e3 for r in nxt if int(r[2] & 0xFFFF) in ex]
            lat = [x for x in lat if x > -50]
            if lat:
                print(f"  hand-off {name}: SMs {len(lat)}  latency q10/50/90/max {np.percentile(lat, 10):.2f}/"
                      f"{np.median(lat):.2f}/{np.percentile(lat, 90):.2f}/{max(lat):.2f} us")
        gap = rel(up[:, 0].min()) - rel(tr[:, 1].max())
        print(f"  k_upd first entry - k_trans last exit: {gap:.2f} us; frame span "
              f"{rel(up[:, 1].max()):.2f} us")


if __name__ == "__main__":
    main()
