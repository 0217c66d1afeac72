"""GPU parity with the inertial source terms on (sf_set_motion, reading 32):
both kernels against the float32 oracle, bit for bit every frame."""
import dataclasses

import numpy as np
import pytest

import oracle
import sfgen

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")]

OMEGA = (0.004, -0.0025, 0.006)
ACCEL = (0.0005, 0.0, -0.001)


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("kernel", ["fused", "passes"])
@pytest.mark.parametrize("cid,frames", [(1, 8), (2, 3)])
def test_imu_parity(kernel, cid, frames):
    import paper_2406_18031_b200 as sf
    seq = sfgen.config_sequence(cid, frames=frames)
    p = dataclasses.replace(seq.params, omega=OMEGA, accel=ACCEL)
    kid = sf.SF_KERNEL_FUSED if kernel == "fused" else sf.SF_KERNEL_PASSES
    m = sf.StructureFlow(seq.geom, p, kernel=kid)
    o = oracle.Oracle(seq.geom, p)
    for k in range(frames):
        m.step(_dev(seq.Y[k]), _dev(seq.depth[k]))
        o.step(seq.Y[k], seq.depth[k])
        w, rho, yhat = m.get_fields()
        torch.cuda.synchronize()
        assert np.array_equal(w[0].cpu().numpy(), o.w), f"w frame {k}"
        assert np.array_equal(rho[0].cpu().numpy(), o.rho), f"rho frame {k}"
    assert sf.sf_status_flags(m.ctx)[1] == o.flags


def test_motion_off_again_is_the_plain_filter():
    import paper_2406_18031_b200 as sf
    seq = sfgen.config_sequence(1, frames=3)
    m = sf.StructureFlow(seq.geom, seq.params)
    sf.sf_set_motion(m.ctx, OMEGA, ACCEL)
    sf.sf_set_motion(m.ctx, None, None)
    o = oracle.Oracle(seq.geom, seq.params)
    for k in range(3):
        m.step(_dev(seq.Y[k]), _dev(seq.depth[k]))
        o.step(seq.Y[k], seq.depth[k])
    w, _, _ = m.get_fields()
    torch.cuda.synchronize()
    assert np.array_equal(w[0].cpu().numpy(), o.w)
