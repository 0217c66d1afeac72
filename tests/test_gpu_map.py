"""GPU parity of the Spherepix input mapping (sf_map_inputs) against the
float32 oracle (or_map_inputs): same operation order, so the mapped brightness and range agree
bit for bit (NaN = invalid at the same pixels), and the mapped inputs drive the filter to the
same state as the oracle's mapped inputs."""
import math

import numpy as np
import pytest

import oracle
import sfgen
from sfgen import grid, scene

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")]


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _cam(Hc, Wc, fov):
    f = Wc / (2 * math.tan(math.radians(fov) / 2))
    return (f, f, (Wc - 1) / 2, (Hc - 1) / 2)


def _same(a, b):
    return np.array_equal(np.isnan(a), np.isnan(b)) and np.array_equal(a[~np.isnan(a)], b[~np.isnan(b)])


@pytest.mark.parametrize("Hc,Wc,rot", [(64, 64, 0.0), (50, 90, 3.0)])
def test_map_bitwise(Hc, Wc, rot):
    import paper_2406_18031_b200 as sf
    seq = sfgen.config_sequence(1, frames=2)
    K = _cam(Hc, Wc, 66.0)
    a = math.radians(rot)
    R = np.array([[1, 0, 0], [0, math.cos(a), -math.sin(a)], [0, math.sin(a), math.cos(a)]], np.float32)
    cams = [scene.render_camera(seq.scene, Hc, Wc, K, float(k)) for k in range(2)]
    m = sf.StructureFlow(seq.geom, seq.params, batch=2)
    Yc = _dev(np.stack([c[0] for c in cams]))
    Zc = _dev(np.stack([c[1] for c in cams]))
    Y, D = m.map_inputs(Yc, Zc, K, R)
    torch.cuda.synchronize()
    for b in range(2):
        Yr, Dr = oracle.map_inputs(seq.geom, K, cams[b][0], cams[b][1], R)
        assert np.array_equal(Y[b].cpu().numpy(), Yr)
        assert _same(D[b].cpu().numpy(), Dr)


def test_map_then_filter_matches_oracle():
    """camera -> sf_map_inputs -> sf_step for 4 frames == oracle map -> oracle step, bitwise."""
    import paper_2406_18031_b200 as sf
    seq = sfgen.config_sequence(1, frames=4)
    Hc, Wc = 72, 80
    K = _cam(Hc, Wc, 64.0)
    m = sf.StructureFlow(seq.geom, seq.params)
    o = oracle.Oracle(seq.geom, seq.params)
    for k in range(4):
        Yc, Zc = scene.render_camera(seq.scene, Hc, Wc, K, float(k))
        Y, D = m.map_inputs(_dev(Yc[None]), _dev(Zc[None]), K)
        m.step(Y, D)
        Yr, Dr = oracle.map_inputs(seq.geom, K, Yc, Zc)
        o.step(Yr, Dr)
    w, rho, yhat = m.get_fields()
    torch.cuda.synchronize()
    assert np.array_equal(w[0].cpu().numpy(), o.w)
    assert np.array_equal(rho[0].cpu().numpy(), o.rho)
    assert np.array_equal(yhat[0].cpu().numpy(), o.yhat)


@pytest.mark.parametrize("mode", ["fused", "passes", "pyramid"])
def test_step_camera_matches_oracle(mode):
    """sf_step_camera (mapping fused into the H = 1 kernel's staging; map + step otherwise) ==
    oracle map -> oracle step, bit for bit, on a non-square rotated camera over 5 frames."""
    import paper_2406_18031_b200 as sf
    from sfgen import grid as G
    seq = sfgen.config_sequence(1, frames=5, H=96, W=80)
    Hc, Wc = 70, 90
    K = _cam(Hc, Wc, 70.0)
    a = math.radians(2.0)
    R = np.array([[math.cos(a), 0, math.sin(a)], [0, 1, 0], [-math.sin(a), 0, math.cos(a)]], np.float32)
    if mode == "pyramid":
        levels = G.gnomonic_pyramid(96, 80, seq.fov)
        m = sf.StructureFlow(levels, seq.params)
        o = oracle.PyramidOracle(levels[0], levels[1], seq.params)
    else:
        kid = sf.SF_KERNEL_FUSED if mode == "fused" else sf.SF_KERNEL_PASSES
        m = sf.StructureFlow(seq.geom, seq.params, kernel=kid)
        o = oracle.Oracle(seq.geom, seq.params)
    for k in range(5):
        Yc, Zc = scene.render_camera(seq.scene, Hc, Wc, K, float(k))
        Ycd, Zcd = _dev(Yc[None]), _dev(Zc[None])  # kept alive until the step has run
        sf.sf_step_camera(m.ctx, Ycd.data_ptr(), Zcd.data_ptr(), Hc, Wc, K, R.flatten())
        Yr, Dr = oracle.map_inputs(seq.geom, K, Yc, Zc, R)
        o.step(Yr, Dr)
        torch.cuda.synchronize()
        w, rho, yhat = m.get_fields()
        torch.cuda.synchronize()
        assert np.array_equal(w[0].cpu().numpy(), o.w), f"w frame {k}"
        assert np.array_equal(rho[0].cpu().numpy(), o.rho), f"rho frame {k}"
