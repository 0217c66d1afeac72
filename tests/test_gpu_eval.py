"""GPU parity of the evaluation outputs (sf_flow_px, sf_eval) against the
float32 oracle (or_flow_px, or_eval) on a filtered config-1 state and its ground truth.

Tangent / normal flow and the per-pixel RMSE follow the same float32 operation order on both
sides: bit-identical.  The AAE cosine is computed in double with the same order on both sides;
acos itself comes from two libraries (CUDA vs glibc, each within 1-2 ulp), so the angle is
compared to 1e-10 deg.  Means are deterministic block sums vs a sequential sum: rel 1e-12."""
import math

import numpy as np
import pytest

import oracle
import sfgen

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")]


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.fixture(scope="module")
def filtered():
    import paper_2406_18031_b200 as sf
    seq = sfgen.config_sequence(1, frames=6, with_gt=True)
    m = sf.StructureFlow(seq.geom, seq.params, batch=1)
    for k in range(6):
        m.step(_dev(seq.Y[k]), _dev(seq.depth[k]))
    w, _, _ = m.get_fields()
    torch.cuda.synchronize()
    return m, seq, w[0].cpu().numpy()


def test_flow_px_bitwise(filtered):
    m, seq, w = filtered
    tg, nm = m.flow_px()
    torch.cuda.synchronize()
    t_ref, n_ref = oracle.flow_px(seq.geom, w)
    assert np.array_equal(tg[0].cpu().numpy(), t_ref)
    assert np.array_equal(nm[0].cpu().numpy(), n_ref)


def test_eval_parity(filtered):
    m, seq, w = filtered
    wgt = seq.w_gt[5].astype(np.float32)
    e = m.evaluate(_dev(wgt[None]))
    torch.cuda.synchronize()
    ref = oracle.evaluate(seq.geom, wgt, w)
    assert np.array_equal(e["rmse"][0].cpu().numpy(), ref["rmse"])
    aae = e["aae_deg"][0].cpu().numpy()
    assert np.abs(aae - ref["aae_deg"]).max() < 1e-10
    assert math.isclose(e["mean_rmse"][0], ref["mean_rmse"], rel_tol=1e-12)
    assert math.isclose(e["mean_aae_deg"][0], ref["mean_aae_deg"], rel_tol=1e-12)
    # the filter is tracking: after 6 frames the error is well below the zero-flow error
    zero = oracle.evaluate(seq.geom, wgt, np.zeros_like(wgt))
    assert ref["mean_rmse"] < zero["mean_rmse"]


def test_eval_batch_and_means_only(filtered):
    import paper_2406_18031_b200 as sf
    m, seq, _ = filtered
    wgt = np.ascontiguousarray(seq.w_gt[5].astype(np.float32))
    mb = sf.StructureFlow(seq.geom, seq.params, batch=2)
    Y = np.stack([seq.Y[0], seq.Y[1]])
    D = np.stack([seq.depth[0], seq.depth[1]])
    mb.step(_dev(Y), _dev(D))
    e = mb.evaluate(_dev(np.stack([wgt, wgt])), rasters=False)
    w, _, _ = mb.get_fields()
    torch.cuda.synchronize()
    for b in range(2):
        ref = oracle.evaluate(seq.geom, wgt, w[b].cpu().numpy())
        assert math.isclose(e["mean_rmse"][b], ref["mean_rmse"], rel_tol=1e-12)
        assert math.isclose(e["mean_aae_deg"][b], ref["mean_aae_deg"], rel_tol=1e-12)


def test_eval_fresh_context_is_state_error():
    import paper_2406_18031_b200 as sf
    seq = sfgen.config_sequence(1, frames=1)
    m = sf.StructureFlow(seq.geom, seq.params, batch=1)
    with pytest.raises(sf.SFError) as ei:
        m.flow_px()
    assert ei.value.status == sf.SF_E_STATE
