"""Pins of the oracle's evaluation outputs (oracle or_flow_px / or_eval):
tangent / normal flow (eq:tangent_flow, eq:normal_flow) and RMSE / AAE
(eq:RMSE_vel and the AAE of P:L726-734, reading 22), against closed forms and invariants."""
import math

import numpy as np
import pytest

import oracle
from sfgen import grid

DS = 2.0 ** -8


def _rand(shape, seed, scale=1e-3):
    return (np.random.default_rng(seed).standard_normal(shape) * scale).astype(np.float32)


def test_flow_px_flat_grid_exact():
    """FLAT grid (s = e_z, b1 = e_x, b2 = e_y, ds = 2^-8): P(s) w = (w_x, w_y, 0) exactly, so the
    tangent flow is (w_x, w_y) / ds and the normal flow w_z / ds, bit for bit."""
    g = grid.flat(16, 12, DS)
    w = _rand((16, 12, 3), 1)
    t, n = oracle.flow_px(g, w)
    assert np.array_equal(t[..., 0], w[..., 0] / np.float32(DS))
    assert np.array_equal(t[..., 1], w[..., 1] / np.float32(DS))
    assert np.array_equal(n, w[..., 2] / np.float32(DS))


@pytest.mark.parametrize("prec,tol", [("f64", 1e-12), ("f32", 2e-6)])
def test_flow_px_basis_reconstruction(prec, tol):
    """{b1, b2, s} is an orthonormal frame (b2 is Gram-Schmidt-orthogonalised against b1, both
    tangent), so w = ds (w_perp1 b1 + w_perp2 b2 + w_par s) for any w (gnomonic grid)."""
    g64 = grid.gnomonic(24, 32, 90.0, as_f64=True)
    g = g64.astype(np.float32)
    w = _rand((24, 32, 3), 2).astype(np.float64)
    t, n = oracle.flow_px(g, w, precision=prec)
    gg = g.astype(np.float64)
    s, b1, b2, ds = gg[..., 0:3], gg[..., 3:6], gg[..., 6:9], gg[..., 9:10]
    rec = ds * (t[..., 0:1] * b1 + t[..., 1:2] * b2 + n[..., None] * s)
    err = np.abs(rec - w).max() / np.abs(w).max()
    # float32 geometry is orthonormal only to ~1e-7: the f64 bound is that of the input rounding
    lim = tol if prec == "f32" else 2e-7
    assert err < lim, err


def test_flow_px_pure_normal_and_pure_tangent():
    """w = a s has no tangent flow and normal flow a/ds; w = c b1 has tangent flow (c/ds, 0)
    and no normal flow (gnomonic grid, float64 oracle, float32 input geometry)."""
    g = grid.gnomonic(16, 16, 60.0)
    gg = g.astype(np.float64)
    s, b1, ds = gg[..., 0:3], gg[..., 3:6], gg[..., 9]
    t, n = oracle.flow_px(g, 0.01 * s, precision="f64")
    assert np.abs(t).max() < 1e-12 * np.abs(n).max()
    assert np.allclose(n, 0.01 / ds, rtol=1e-12)
    t, n = oracle.flow_px(g, 0.02 * b1, precision="f64")
    assert np.allclose(t[..., 0], 0.02 / ds, rtol=1e-6)       # |b1| = 1 to float32 rounding
    assert np.abs(t[..., 1]).max() < 1e-6 * np.abs(t[..., 0]).max()
    assert np.abs(n).max() < 1e-6 * np.abs(t[..., 0]).max()


def test_rmse_closed_forms():
    """w = w_gt -> 0; w_gt - w = ds e_x on the FLAT grid -> exactly 1 px everywhere;
    translation equivariance rmse(w_gt + c, w + c) = rmse(w_gt, w) for dyadic values."""
    g = grid.flat(8, 8, DS)
    w = _rand((8, 8, 3), 3)
    e = oracle.evaluate(g, w, w)
    assert (e["rmse"] == 0).all() and e["mean_rmse"] == 0.0
    wg = w.copy()
    wg[..., 0] += np.float32(DS)
    # exact only where the shifted value is representable: use dyadic w
    wd = np.round(w * 2 ** 12).astype(np.float32) / np.float32(2 ** 12)
    wgd = wd.copy()
    wgd[..., 0] += np.float32(DS)
    e = oracle.evaluate(g, wgd, wd)
    assert np.array_equal(e["rmse"], np.ones((8, 8), np.float32))
    c = np.float32(2 ** -10)
    e2 = oracle.evaluate(g, wgd + c, wd + c)
    assert np.array_equal(e2["rmse"], e["rmse"])


def test_rmse_mean_is_pixel_mean():
    g = grid.gnomonic(20, 20, 70.0)
    wg, w = _rand((20, 20, 3), 4), _rand((20, 20, 3), 5)
    e = oracle.evaluate(g, wg, w, precision="f64")
    d = (wg.astype(np.float64) - w.astype(np.float64)) / g[..., 9:10].astype(np.float64)
    assert np.allclose(e["rmse"], np.sqrt((d * d).sum(-1)), rtol=1e-14)
    assert math.isclose(e["mean_rmse"], float(e["rmse"].mean()), rel_tol=1e-12)


def test_aae_closed_forms():
    """AAE(w, w) = 0; AAE(0, w_gt) with |w_gt/ds| = 1 is arccos(1/sqrt 2) = 45 deg; two unit
    px-flows 90 deg apart give arccos(1/2) = 60 deg; AAE is symmetric (FLAT grid)."""
    g = grid.flat(4, 4, DS)
    w = _rand((4, 4, 3), 6)
    assert oracle.evaluate(g, w, w)["aae_deg"].max() < 1e-5
    unit = np.zeros((4, 4, 3), np.float32)
    unit[..., 0] = DS
    e = oracle.evaluate(g, unit, np.zeros_like(unit))
    assert np.allclose(e["aae_deg"], 45.0, atol=1e-12)
    other = np.zeros_like(unit)
    other[..., 1] = DS
    e = oracle.evaluate(g, unit, other)
    assert np.allclose(e["aae_deg"], 60.0, atol=1e-12)
    a, b = _rand((4, 4, 3), 7), _rand((4, 4, 3), 8)
    assert np.array_equal(oracle.evaluate(g, a, b)["aae_deg"], oracle.evaluate(g, b, a)["aae_deg"])
