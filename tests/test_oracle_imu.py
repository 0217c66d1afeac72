"""Pins of the inertial source terms in the predictor (reading 32):
dw/dt = -(dw/ds) P w - w<s,w> - Omega x w + a_w, a_w = rho a_c - Omega x (w + Omega x s)
(eq:hflow_conservation, eq:totaldev_hflow), integrated as one explicit stage per substep."""
import dataclasses
import math

import numpy as np

import oracle
from sfgen import grid
from sfgen.configs import Params

DS = 2.0 ** -8


def _params(N, omega=None, accel=None):
    return Params(max_flow=float(N), gamma=(1.0, 1.0, 1.0, 1.0, 1.0), omega=omega, accel=accel)


def test_zero_motion_is_bitwise_the_plain_predictor():
    g = grid.gnomonic(24, 24, 70.0)
    rng = np.random.default_rng(0)
    w = (rng.standard_normal((24, 24, 3)) * 2e-3).astype(np.float32)
    rho = rng.uniform(0.1, 0.5, (24, 24)).astype(np.float32)
    outs = []
    for p in (_params(4), _params(4, (0.0, 0.0, 0.0), (0.0, 0.0, 0.0))):
        o = oracle.Oracle(g, p)
        o.set_state(w, rho, np.zeros((24, 24), np.float32))
        outs.append(o.predict())
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def test_uniform_field_discrete_closed_form():
    """FLAT grid (s = e_z), Omega = (0, 0, om) parallel to s (Omega x s = 0), a_c = (a, 0, 0),
    uniform w0 = 0 and rho0: transport and dilation vanish (uniform fields, <s,w> = w_z = 0), so
    W = w_x + i w_y follows explicit Euler on dW/dt = rho0 a - 2 i om W:
    W_N = (rho0 a / (2 i om)) (1 - (1 - 2 i om dt)^N), converging to the continuum solution."""
    om, a, rho0 = 0.0625, 0.00390625, 0.375  # float32-exact (the parameters are float32)
    g = grid.flat(6, 7, DS)
    errs = []
    for N in (2, 4, 8, 16):
        o = oracle.Oracle(g, _params(N, (0.0, 0.0, om), (a, 0.0, 0.0)), "f64")
        o.set_state(np.zeros((6, 7, 3)), np.full((6, 7), rho0), np.zeros((6, 7)))
        w, r = o.predict()
        dt = 1.0 / N
        Wn = rho0 * a / (2j * om) * (1 - (1 - 2j * om * dt) ** N)
        assert np.allclose(w[..., 0], Wn.real, rtol=1e-12, atol=1e-18)
        assert np.allclose(w[..., 1], Wn.imag, rtol=1e-12, atol=1e-18)
        assert np.all(w[..., 2] == 0) and np.all(r == rho0)
        Wc = rho0 * a / (2j * om) * (1 - np.exp(-2j * om))
        errs.append(abs(complex(w[0, 0, 0], w[0, 0, 1]) - Wc))
    # first order in dt
    assert all(errs[i + 1] < 0.6 * errs[i] for i in range(3)), errs


def test_pure_rotation_rotational_flow_is_stationary():
    """Static scene, pure camera rotation: w = w_r = -Omega x s satisfies the full PDE with zero
    time derivative (the transport term Omega x w cancels against -2 Omega x w - Omega x
    (Omega x s)).  With the inertial terms the prediction keeps it up to the upwind truncation
    error; without them it drifts by ~(Omega x w + Omega x (Omega x s)) per frame."""
    g = grid.gnomonic(48, 48, 60.0)
    s = g[..., 0:3].astype(np.float64)
    Om = np.array([0.004, -0.006, 0.01])
    w0 = -np.cross(np.broadcast_to(Om, s.shape), s)
    rho = np.full((48, 48), 0.3)
    ds = float(g[24, 24, 9])
    max_px = np.abs(w0).max() / ds
    N = max(1, math.ceil(max_px))
    errs = {}
    for imu in (True, False):
        p = _params(N, tuple(Om) if imu else None, (0.0, 0.0, 0.0) if imu else None)
        o = oracle.Oracle(g, p, "f64")
        o.set_state(w0, rho, np.zeros((48, 48)))
        w, _ = o.predict()
        errs[imu] = np.abs(w - w0)[8:-8, 8:-8].max()
    assert errs[True] < 0.1 * errs[False], errs
