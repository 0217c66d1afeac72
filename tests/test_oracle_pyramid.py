"""Pins of the H = 2 pyramid oracle (oracle or_down2 / or_up2 /
or_predict_low / or_pyr_step, readings 24-30) against closed forms, exact special cases and
accuracy on a scene with known ground truth."""
import math

import numpy as np
import pytest

import oracle
import sfgen
from sfgen import grid
from sfgen.configs import Params

DS = 2.0 ** -8


def test_down2_closed_forms():
    """2x2 mean (reading 24): a constant stays; a dyadic ramp a j + b i + c gives the block
    centre value exactly; one invalid depth sample invalidates the coarse sample."""
    H, W = 8, 12
    ii, jj = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    Y = (0.125 * jj + 0.0625 * ii + 0.25).astype(np.float32)
    D = np.full((H, W), 3.0, np.float32)
    D[2, 3] = np.nan
    D[5, 8] = -1.0
    Y2, D2 = oracle.down2(Y, D)
    I, J = np.meshgrid(np.arange(H // 2), np.arange(W // 2), indexing="ij")
    assert np.array_equal(Y2, (0.125 * (2 * J + 0.5) + 0.0625 * (2 * I + 0.5) + 0.25).astype(np.float32))
    bad = np.zeros((H // 2, W // 2), bool)
    bad[1, 1] = bad[2, 4] = True
    assert np.isnan(D2[bad]).all() and (D2[~bad] == 3.0).all()


def test_up2_closed_forms():
    """Bilinear up-sampling (reading 25): constants are reproduced exactly; a dyadic linear field
    a I + b J is interpolated exactly at the fine pixel centres (coarse coordinate (i - 1/2) / 2)
    away from the border, and the border replicates the edge sample."""
    Hc, Wc = 6, 5
    X = np.full((Hc, Wc, 3), 0.375, np.float32)
    assert np.array_equal(oracle.up2(X), np.full((2 * Hc, 2 * Wc, 3), 0.375, np.float32))
    I, J = np.meshgrid(np.arange(Hc), np.arange(Wc), indexing="ij")
    X = np.stack([0.5 * I + 0.25 * J, -0.125 * I, 0.0625 * J], -1).astype(np.float32)
    U = oracle.up2(X)
    i, j = np.meshgrid(np.arange(2 * Hc), np.arange(2 * Wc), indexing="ij")
    ci = np.clip((i - 0.5) / 2, 0, Hc - 1)
    cj = np.clip((j - 0.5) / 2, 0, Wc - 1)
    ref = np.stack([0.5 * ci + 0.25 * cj, -0.125 * ci, 0.0625 * cj], -1)
    assert np.array_equal(U, ref.astype(np.float32))


def _flat_params(max_flow):
    return Params(max_flow=max_flow, gamma=(1.0, 1.0, 1.0, 1.0, 1.0), smooth_iters=2)


def test_predict_low_courant_one_shift():
    """FLAT grid, uniform w = (ds, 0, 0): u = 1 px/frame, N = 1, dt |u| = 1 -> the column pass is
    the exact one-pixel upwind shift of dw, rho and Yhat (replicate left border); v = 0 and
    <s, w> = 0 leave the row pass without effect; w itself stays uniform."""
    H, W = 6, 10
    g = grid.flat(H, W, DS)
    rng = np.random.default_rng(3)
    F = np.zeros((H, W, 8), np.float32)
    F[..., 0] = DS
    F[..., 3:8] = (np.round(rng.uniform(-1, 1, (H, W, 5)) * 64) / 64).astype(np.float32)
    out, flags = oracle.predict_low(g, _flat_params(1.0), F)
    assert flags == 0
    ref = F.copy()
    ref[:, 1:, 3:8] = F[:, :-1, 3:8]
    assert np.array_equal(out, ref)


def test_predict_low_pure_dilation():
    """FLAT grid, uniform w = (0, 0, c): u = v = 0, so each of the 2N passes scales w, dw and rho
    by (1 - dt sigma c) and leaves Yhat untouched (eq:img_propagation_low has no dilation)."""
    H, W, c, N = 4, 5, 0.05, 4
    g = grid.flat(H, W, DS)
    F = np.zeros((H, W, 8), np.float64)
    F[..., 2] = c
    F[..., 3:6] = [0.01, -0.02, 0.03]
    F[..., 6] = 0.4
    F[..., 7] = 0.7
    out, _ = oracle.predict_low(g, _flat_params(float(N)), F, precision="f64")
    # w_z itself is transported with its own dilation: c_{n+1} = c_n (1 - dt sigma c_n)
    cz = c
    fac = 1.0
    for _ in range(2 * N):
        fac *= 1.0 - 0.5 * cz / N
        cz *= 1.0 - 0.5 * cz / N
    assert np.allclose(out[..., 2], cz, rtol=1e-13)
    assert np.allclose(out[..., 3:7], F[..., 3:7] * fac, rtol=1e-13)
    assert np.array_equal(out[..., 7], F[..., 7])


def test_pyramid_params_rule():
    seq = sfgen.config_sequence(1, frames=1)
    g1, g2 = grid.gnomonic_pyramid(64, 64, seq.fov)
    top = oracle.pyramid_params(seq.params, g1, g2)
    assert top.max_flow == seq.params.max_flow / 2 and top.N == math.ceil(seq.params.max_flow / 2)
    assert top.smooth_iters == 4 and seq.params.smooth_iters == 2
    r = (float(g1[32, 32, 9]) / float(g2[16, 16, 9])) ** 2
    assert 0.2 < r < 0.3  # coarse pixels are twice as wide
    assert math.isclose(top.gamma[0], seq.params.gamma[0] * r, rel_tol=1e-7)


@pytest.fixture(scope="module")
def pyr_run():
    seq = sfgen.config_sequence(1, frames=40, with_gt=True)
    g1, g2 = grid.gnomonic_pyramid(64, 64, seq.fov)
    po = oracle.PyramidOracle(g1, g2, seq.params)
    p64 = oracle.PyramidOracle(g1, g2, seq.params, precision="f64")
    rmse = []
    for k in range(40):
        po.step(seq.Y[k], seq.depth[k])
        if k < 10:
            p64.step(seq.Y[k], seq.depth[k])
            if k == 9:
                drift = (np.abs(po.w - p64.w).max(), np.abs(po.rho - p64.rho).max())
                recon = oracle.up2(po.w2) + po.dw
                recon_ok = np.array_equal(po.w, recon)
        rmse.append(oracle.evaluate(seq.geom, seq.w_gt[k], po.w)["mean_rmse"])
    zero = oracle.evaluate(seq.geom, seq.w_gt[39], np.zeros((64, 64, 3), np.float32))["mean_rmse"]
    return dict(rmse=rmse, zero=zero, drift=drift, recon_ok=recon_ok)


def test_pyramid_reconstruction(pyr_run):
    """eq:hflow_reconstruction: the bottom-level flow is up(w^2) + dw, bit for bit."""
    assert pyr_run["recon_ok"]


def test_pyramid_f32_vs_f64(pyr_run):
    dw, dr = pyr_run["drift"]
    assert dw < 1e-5 and dr < 1e-5, pyr_run["drift"]


def test_pyramid_accuracy(pyr_run):
    """The two-level filter tracks the ground truth: after 40 frames the RMSE is
    below 25 % of the zero-flow error."""
    assert pyr_run["rmse"][-1] < 0.25 * pyr_run["zero"], (pyr_run["rmse"][-1], pyr_run["zero"])


def test_pyramid_increment_update_depth_term():
    """Bottom-level increment update [dU] (eq:cost_bottom; reading 28): a uniform
    inverse-depth change on a static FLAT scene is explained by the normal component of the
    increment alone -- m = ds^2 rhohat s (no rho gradient) and c_rho = ds^2 (rhohat - rho^{k+}), so
    for a dominant gamma2 dw_z = rho^{k+}/rhohat - 1 (the E_rho closed form of L572-574 applied to
    dw with prior dw^{k+} = 0).  The top level recovers the same rate, and w = up(w^2) + dw."""
    H = W = 16
    g1, g2 = grid.flat(H, W, 2.0 ** -6), grid.flat(H // 2, W // 2, 2.0 ** -5)
    p = Params(max_flow=2.0, gamma=(0.0, 1e14, 1.0, 1.0, 0.0), smooth_iters=0)
    po = oracle.PyramidOracle(g1, g2, p, precision="f64", smooth_top=0)
    Y = np.zeros((H, W), np.float32)
    po.step(Y, np.full((H, W), 2.0, np.float32))  # rho = 0.5 at both levels, w = 0
    po.step(Y, np.full((H, W), 1.6, np.float32))
    rate = 0.5 * float(np.float32(1.6)) - 1.0
    assert np.allclose(po.dw[..., 2], rate, atol=1e-6) and np.abs(po.dw[..., :2]).max() < 1e-12
    assert np.allclose(po.w2[..., 2], rate, atol=1e-6)
    assert np.allclose(po.w[..., 2], 2 * rate, atol=2e-6)
    assert np.allclose(po.rho, 1.0 / float(np.float32(1.6)), rtol=1e-14)  # gamma5 = 0: the measurement
