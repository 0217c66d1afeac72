"""Pins of the Spherepix input mapping oracle (or_map_inputs, reading 31):
a pinhole camera image resampled onto the grid, against closed forms and an independent
rendering of the same scene on the grid."""
import math

import numpy as np

import oracle
import sfgen
from sfgen import grid, scene


def _identity_camera(H, W, fov):
    f = W / (2 * math.tan(math.radians(fov) / 2))
    return (f, f, (W - 1) / 2, (H - 1) / 2)


def test_identity_camera_reproduces_grid_rendering():
    """A camera whose pixels ARE the gnomonic grid's directions: the mapped brightness equals
    the camera image, and the mapped range equals sfgen's range rendering on the grid (an
    independent path: ray casting along the grid directions)."""
    H = W = 64
    seq = sfgen.config_sequence(1, frames=1)
    g = grid.gnomonic(H, W, seq.fov)
    K = _identity_camera(H, W, seq.fov)
    Yc, Zc = scene.render_camera(seq.scene, H, W, K, 0.0)
    Y, D = oracle.map_inputs(g, K, Yc, Zc)
    assert np.abs(Y - Yc).max() < 2e-6
    assert np.nanmax(np.abs(D - seq.depth[0]) / seq.depth[0]) < 2e-6 and not np.isnan(D).any()


def test_linear_image_bilinear_exact():
    """Bilinear interpolation reproduces a linear image a j + b i + c at any sub-pixel position:
    Y_grid = a u(s) + b v(s) + c with (u, v) the f64 projection (half-resolution rotated camera)."""
    H, W = 40, 48
    g = grid.gnomonic(H, W, 70.0)
    Hc, Wc = 30, 36
    K = (30.0, 31.0, 17.5, 14.25)
    ang = math.radians(4.0)
    R = np.array([[math.cos(ang), -math.sin(ang), 0], [math.sin(ang), math.cos(ang), 0], [0, 0, 1]], np.float32)
    ii, jj = np.meshgrid(np.arange(Hc), np.arange(Wc), indexing="ij")
    Yc = (0.0078125 * jj + 0.015625 * ii + 0.25).astype(np.float32)
    Zc = np.full((Hc, Wc), 4.0, np.float32)
    Y, D = oracle.map_inputs(g, K, Yc, Zc, R)
    s = g[..., 0:3].astype(np.float64)
    t = s @ R.astype(np.float64).T
    u = K[0] * t[..., 0] / t[..., 2] + K[2]
    v = K[1] * t[..., 1] / t[..., 2] + K[3]
    inside = (u >= 0) & (u <= Wc - 1) & (v >= 0) & (v <= Hc - 1)
    ref = 0.0078125 * np.clip(u, 0, Wc - 1) + 0.015625 * np.clip(v, 0, Hc - 1) + 0.25
    assert np.abs(Y - ref).max() < 1e-5
    # fronto-parallel plane at z = 4: range lambda = 4 / t_z where the pixel footprint is hit
    foot = (u >= -0.5) & (u <= Wc - 0.5) & (v >= -0.5) & (v <= Hc - 0.5)
    assert np.allclose(D[foot], 4.0 / t[..., 2][foot], rtol=1e-6)
    assert np.isnan(D[~foot]).all() and inside.sum() > 0 and (~foot).sum() > 0


def test_invalid_depth_samples_and_behind_camera():
    H = W = 8
    g = grid.gnomonic(H, W, 60.0)
    K = _identity_camera(H, W, 60.0)
    Yc = np.full((H, W), 0.5, np.float32)
    Zc = np.full((H, W), 2.0, np.float32)
    Zc[3, 4] = np.inf
    Y, D = oracle.map_inputs(g, K, Yc, Zc)
    assert (Y == 0.5).all()
    assert np.isnan(D[3, 4]) and np.isfinite(D[0, 0])
    flip = np.diag([1.0, 1.0, -1.0]).astype(np.float32)  # camera looking backwards: nothing in front
    Y, D = oracle.map_inputs(g, K, Yc, Zc, flip)
    assert np.isnan(D).all() and (Y == 0.5).all()
