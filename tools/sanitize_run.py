#!/usr/bin/env python3
"""Small workloads for compute-sanitizer (tools/gpu_sanitize.sh): the fused (k_trans + k_upd) and
per-pass H = 1 paths on ragged multi-CTA grids (interior, edge and corner CTAs; regions flush with
the grid border and replica cells; cp.async and TMA staging) and the pyramid (both bottom-level
updates) -- each compared with the oracle so a run is also a parity check."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2406_18031_b200 as sf
import sfgen
from sfgen import grid


def h1(kernel, H, W, frames=3):
    seq = sfgen.config_sequence(1, frames=frames, H=H, W=W)
    m = sf.StructureFlow(seq.geom, seq.params, kernel=kernel)
    o = oracle.Oracle(seq.geom, seq.params, "f32")
    for k in range(frames):
        m.step(torch.from_numpy(seq.Y[k]).cuda(), torch.from_numpy(seq.depth[k]).cuda())
        o.step(seq.Y[k], seq.depth[k])
    w, rho, yhat = m.get_fields()
    torch.cuda.synchronize()
    assert np.array_equal(w[0].cpu().numpy(), o.w) and np.array_equal(rho[0].cpu().numpy(), o.rho)
    print(f"h1 kernel={kernel} {H}x{W}: bitwise ok")


def pyramid(frames=3):
    seq = sfgen.config_sequence(1, frames=frames, H=96, W=80)
    geom = grid.gnomonic_pyramid(96, 80, seq.fov)
    m = sf.StructureFlow(geom, seq.params)
    o = oracle.PyramidOracle(geom[0], geom[1], seq.params)
    for k in range(frames):
        m.step(torch.from_numpy(seq.Y[k]).cuda(), torch.from_numpy(seq.depth[k]).cuda())
        o.step(seq.Y[k], seq.depth[k])
    w, rho, yhat = m.get_fields()
    torch.cuda.synchronize()
    assert np.array_equal(w[0].cpu().numpy(), o.w)
    print("pyramid 96x80: bitwise ok")


if __name__ == "__main__":
    which = sys.argv[1:] or ["fused", "passes", "pyramid"]
    if "fused" in which:
        h1(sf.SF_KERNEL_FUSED, 150, 130)  # W % 4 != 0: cp.async staging
        h1(sf.SF_KERNEL_FUSED, 150, 136)  # W % 4 == 0: TMA staging (racecheck does not see TMA writes)
    if "passes" in which:
        h1(sf.SF_KERNEL_PASSES, 150, 130)
    if "pyramid" in which:
        pyramid()
        os.environ["SF_UPD_LOW_PASSES"] = "1"  # the bottom-level update on the per-pass kernels
        pyramid()
        del os.environ["SF_UPD_LOW_PASSES"]
