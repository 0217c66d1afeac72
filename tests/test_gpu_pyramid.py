"""GPU parity of the H = 2 pyramid (levels = 2) against the float32
PyramidOracle, through the C-ABI: the reconstructed flow, the bottom-level inverse depth and
brightness model must agree bit for bit every frame (same arithmetic order, DESIGN.md section 4
and readings 24-30), and the sticky flags of both levels must match."""
import numpy as np
import pytest

import oracle
import sfgen
from sfgen import grid

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")]


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _run(cid, frames, H=None, W=None, kernel=None, batch=1, check_every=1):
    import paper_2406_18031_b200 as sf
    seq = sfgen.config_sequence(cid, frames=frames, H=H, W=W)
    Hh, Ww = seq.geom.shape[:2]
    levels = grid.gnomonic_pyramid(Hh, Ww, seq.fov)
    assert np.array_equal(levels[0], seq.geom)
    po = oracle.PyramidOracle(levels[0], levels[1], seq.params)
    m = sf.StructureFlow(levels, seq.params, batch=batch, kernel=sf.SF_KERNEL_AUTO if kernel is None else kernel)
    for k in range(frames):
        Y = np.stack([seq.Y[k]] * batch)
        D = np.stack([seq.depth[k]] * batch)
        m.step(_dev(Y), _dev(D))
        po.step(seq.Y[k], seq.depth[k])
        if k % check_every == 0 or k == frames - 1:
            w, rho, yhat = m.get_fields()
            torch.cuda.synchronize()
            for b in range(batch):
                assert np.array_equal(w[b].cpu().numpy(), po.w), f"w frame {k} batch {b}"
                assert np.array_equal(rho[b].cpu().numpy(), po.rho), f"rho frame {k}"
                assert np.array_equal(yhat[b].cpu().numpy(), po.yhat), f"yhat frame {k}"
    st, flags = sf.sf_status_flags(m.ctx)
    assert flags == po.flags, (flags, po.flags)
    return m, po, seq


@pytest.mark.parametrize("kernel", ["auto", "passes"])
def test_pyramid_config1_every_frame(kernel):
    import paper_2406_18031_b200 as sf
    _run(1, 10, kernel=sf.SF_KERNEL_PASSES if kernel == "passes" else None)


def test_pyramid_ragged_and_batch():
    """96 x 80 (not a multiple of any tile), max flow 2 -> top level 48 x 40, batch 2."""
    _run(1, 6, H=96, W=80, batch=2)


def test_pyramid_bench_size():
    """The bench workload's grid (512^2, max flow 8: N_1 = 8, N_2 = 4, S = [2, 4]), 4 frames."""
    _run(2, 4, check_every=3)


def test_pyramid_eval_and_unsupported():
    import paper_2406_18031_b200 as sf
    m, po, seq = _run(1, 3)
    tg, nm = m.flow_px()
    torch.cuda.synchronize()
    t_ref, n_ref = oracle.flow_px(seq.geom, po.w)
    assert np.array_equal(tg[0].cpu().numpy(), t_ref) and np.array_equal(nm[0].cpu().numpy(), n_ref)
    for call in (lambda: sf.sf_predict(m.ctx), lambda: m.get_fields(sf.SF_FIELDS_PREDICTED)):
        with pytest.raises(sf.SFError) as e:
            call()
        assert e.value.status == sf.SF_E_UNSUPPORTED
    assert sf.sf_launches_per_step(m.ctx) > 0


@pytest.mark.parametrize("max_flow,S,rule", [(11.0, 1, 0), (3.0, 3, 1)])
def test_pyramid_multi_launch_and_variants(max_flow, S, rule):
    """N1 = 11 (two bottom-level k_low launches, top N2 = 6), S1 = 1; and N1 = 3 with S1 = 3 and the
    printed dominant rule — bitwise against the pyramid oracle every frame."""
    import dataclasses

    import paper_2406_18031_b200 as sf
    seq = sfgen.config_sequence(1, frames=4, H=128, W=96)
    p = dataclasses.replace(seq.params, max_flow=max_flow, smooth_iters=S, dominant_rule=rule)
    levels = grid.gnomonic_pyramid(128, 96, seq.fov)
    po = oracle.PyramidOracle(levels[0], levels[1], p)
    m = sf.StructureFlow(levels, p)
    for k in range(4):
        m.step(_dev(seq.Y[k][None]), _dev(seq.depth[k][None]))
        po.step(seq.Y[k], seq.depth[k])
        w, rho, yhat = m.get_fields()
        torch.cuda.synchronize()
        assert np.array_equal(w[0].cpu().numpy(), po.w), f"w frame {k}"
        assert np.array_equal(rho[0].cpu().numpy(), po.rho), f"rho frame {k}"
    assert sf.sf_status_flags(m.ctx)[1] == po.flags


@pytest.mark.parametrize("cid,H,W,frames", [(1, None, None, 8), (1, 96, 80, 5), (2, None, None, 3)])
def test_pyramid_per_pass_bottom_update(cid, H, W, frames, monkeypatch):
    """The bottom-level increment update [dU] on the per-pass kernels
    (SF_UPD_LOW_PASSES=1: k_update + S x k_box, the reconstruction on the last box pass) instead
    of the default tiled k_upd (references Yhat^{k+} = Wpred.w, rho^{k+} = pred.w, the
    reconstruction in its store stage): bitwise the pyramid oracle every frame."""
    monkeypatch.setenv("SF_UPD_LOW_PASSES", "1")
    import paper_2406_18031_b200 as sf
    m, po, seq = _run(cid, frames, H=H, W=W)
    assert sf.sf_launches_per_step(m.ctx) > 0
