"""The pipelined host-buffer path (sf_step_host_async + sf_wait): every frame's outputs equal
the synchronous path's and the oracle's, bit for bit."""
import numpy as np
import pytest

import oracle
import sfgen

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")]


@pytest.mark.parametrize("levels", [1, 2])
def test_async_host_frames(levels):
    import paper_2406_18031_b200 as sf
    from sfgen import grid
    F = 6
    seq = sfgen.config_sequence(1, frames=F)
    geom = seq.geom if levels == 1 else grid.gnomonic_pyramid(64, 64, seq.fov)
    m = sf.StructureFlow(geom, seq.params)
    Yp = torch.from_numpy(seq.Y.copy()).pin_memory()
    Dp = torch.from_numpy(seq.depth.copy()).pin_memory()
    outs = [(torch.empty((1, 64, 64, 3), pin_memory=True), torch.empty((1, 64, 64), pin_memory=True)) for _ in range(F)]
    for k in range(F):
        sf.sf_step_host_async(m.ctx, Yp[k].data_ptr(), Dp[k].data_ptr(), outs[k][0].data_ptr(), outs[k][1].data_ptr())
    sf.sf_wait(m.ctx)
    o = oracle.Oracle(seq.geom, seq.params) if levels == 1 else oracle.PyramidOracle(geom[0], geom[1], seq.params)
    for k in range(F):
        o.step(seq.Y[k], seq.depth[k])
        assert np.array_equal(outs[k][0][0].numpy(), o.w), f"w frame {k}"
        assert np.array_equal(outs[k][1][0].numpy(), o.rho), f"rho frame {k}"
