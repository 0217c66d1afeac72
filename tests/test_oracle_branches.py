"""Pins of the oracle's discontinuous branches (no GPU): the advection clamp and its flags, the
tie rules of the dominant flow and of the rho one-sided difference, the one-valid-neighbour
fallback and the depth validity rule.

Each test builds a case whose expected result follows from the paper's statement alone -- an
exact pixel shift of first-order upwind transport at Courant number 1 (textbook CIR scheme),
the printed tie branch, an integer recurrence -- so that flipping any of these branches in
oracle/sf_oracle.c fails at least one assertion here (tools/oracle_mutant.sh, DESIGN.md
section 5).  Citations are PAPER.md lines (P:Lnnn).
"""
import numpy as np
import pytest

import oracle
from sfgen import grid
from sfgen.configs import Params

DS = 2.0 ** -8


def P(max_flow, **kw):
    return Params(max_flow=float(max_flow), gamma=(1.0, 1.0, 1.0, 1.0, 1.0), smooth_iters=2, **kw)


def _flat_state(H, W, wx, wy=0.0, seed=0):
    g = grid.flat(H, W, DS)
    rng = np.random.default_rng(seed)
    rho = rng.uniform(0.5, 1.0, (H, W)).astype(np.float32)
    w = np.zeros((H, W, 3), np.float32)
    w[..., 0] = wx
    w[..., 1] = wy
    return g, w, rho


# --------------------------------------------------------------------------- clamp (reading 12)
@pytest.mark.parametrize("N", [1, 2, 4, 8])
@pytest.mark.parametrize("axis", [0, 1])
def test_clamp_makes_double_flow_an_exact_N_pixel_shift(N, axis):
    """A uniform flow of 2N px/frame with max_flow = N ("maximum flow allowed", reading
    12): the dominant flow is clamped to N, so with N substeps (eq:numerical_stability)
    every pass runs at Courant number exactly 1 -- an exact N-pixel shift of rho (CIR upwind,
    P:L654-673), replicate inflow border -- and FLAG_CLAMPED is raised.  Without the clamp (or
    with a wider bound) the pass runs at Courant 2 and the shift is not exact."""
    H, W = 24, 40
    wx, wy = (2 * N * DS, 0.0) if axis == 0 else (0.0, 2 * N * DS)
    g, w, rho0 = _flat_state(H, W, wx, wy, seed=N)
    o = oracle.Oracle(g, P(N), "f32")
    o.set_state(w, rho0, np.zeros((H, W), np.float32))
    wp, rp = o.predict()
    if axis == 0:
        expect = rho0[:, np.clip(np.arange(W) - N, 0, W - 1)]
    else:
        expect = rho0[np.clip(np.arange(H) - N, 0, H - 1)]
    assert np.array_equal(rp, expect)
    assert np.array_equal(wp, w)  # uniform w is invariant under transport
    assert o.flags == oracle.FLAG_CLAMPED


def test_clamp_inactive_at_exactly_max_flow():
    """|u_hat| = max_flow is allowed (Courant 1, "<= 1"): no flag."""
    g, w, rho0 = _flat_state(8, 16, 4 * DS)
    o = oracle.Oracle(g, P(4), "f32")
    o.set_state(w, rho0, np.zeros((8, 16), np.float32))
    o.predict()
    assert o.flags == 0


@pytest.mark.parametrize("N", [1, 2, 4])
def test_literal_mode_runs_courant_two_and_flags_cfl(N):
    """clamp_advection = 0 (the paper-literal scheme): the same 2N px/frame flow is advected at
    Courant number 2, the upwind recurrence f_j <- f_j - 2 (f_j - f_{j-1}) = 2 f_{j-1} - f_j per
    pass (replicate left border), and FLAG_CFL reports the violated bound dt |u_hat| <= 1
    (eq:numerical_stability).  Integer rho keeps the recurrence exact in float32."""
    H, W = 4, 24
    g, w, _ = _flat_state(H, W, 2 * N * DS)
    rho0 = np.tile((np.arange(W) % 5).astype(np.float32), (H, 1))
    o = oracle.Oracle(g, P(N, clamp_advection=0), "f32")
    o.set_state(w, rho0, np.zeros((H, W), np.float32))
    _, rp = o.predict()
    ref = rho0.astype(np.int64)
    for _ in range(N):  # column passes; the row passes see v = 0 and <s, w> = 0
        left = ref[:, np.clip(np.arange(W) - 1, 0, W - 1)]
        ref = 2 * left - ref
    assert np.array_equal(rp, ref.astype(np.float32))
    assert o.flags == oracle.FLAG_CFL


def test_pyramid_bottom_pass_clamp():
    """The bottom-level transport (eq:hflow_propagation_low .. eq:img_propagation_low)
    clamps like the top level: w = (2 ds, 0, 0), max_flow = 1, N = 1 -> exact one-pixel shift
    of dw, rho and Yhat, FLAG_CLAMPED."""
    H, W = 6, 12
    g = grid.flat(H, W, DS)
    rng = np.random.default_rng(5)
    F = np.zeros((H, W, 8), np.float32)
    F[..., 0] = 2 * DS
    F[..., 3:8] = (np.round(rng.uniform(-1, 1, (H, W, 5)) * 64) / 64).astype(np.float32)
    out, flags = oracle.predict_low(g, P(1), F)
    ref = F.copy()
    ref[:, 1:, 3:8] = F[:, :-1, 3:8]
    assert np.array_equal(out, ref)
    assert flags == oracle.FLAG_CLAMPED
    out, flags = oracle.predict_low(g, P(1, clamp_advection=0), F)
    assert flags == oracle.FLAG_CFL
    assert not np.array_equal(out, ref)


# --------------------------------------------------------------------------- dominant-flow tie
@pytest.mark.parametrize("rule", [0, 1])
@pytest.mark.parametrize("axis", [0, 1])
def test_dominant_flow_tie_takes_the_forward_neighbour(rule, axis):
    """Converging flow u_{j-1} = +1 px, u_{j+1} = -1 px: |u_{j-1}| = |u_{j+1}|, and both the
    printed rule and the LARGEST reading take the "otherwise" branch u_{j+1}.  With
    u_hat = -1 the upwind difference is the forward one, so at Courant 1 the pixel
    takes its forward neighbour's rho exactly (N = 1)."""
    H, W = 12, 12
    g = grid.flat(H, W, DS)
    w = np.zeros((H, W, 3), np.float32)
    c = 6
    a = 0 if axis == 0 else 1
    sl_m = (slice(None), c - 1) if axis == 0 else (c - 1, slice(None))
    sl_p = (slice(None), c + 1) if axis == 0 else (c + 1, slice(None))
    w[sl_m + (a,)] = DS
    w[sl_p + (a,)] = -DS
    rho0 = np.random.default_rng(7).uniform(0.5, 1.0, (H, W)).astype(np.float32)
    o = oracle.Oracle(g, P(1, dominant_rule=rule), "f32")
    o.set_state(w, rho0, np.zeros((H, W), np.float32))
    _, rp = o.predict()
    if axis == 0:
        assert np.array_equal(rp[:, c], rho0[:, c + 1])
    else:
        assert np.array_equal(rp[c], rho0[c + 1])


# --------------------------------------------------------------------------- rho side choice
@pytest.mark.parametrize("axis", [0, 1])
def test_rho_gradient_tie_takes_forward_difference(axis):
    """A V-shaped inverse depth [1, 0.5, 1] has |D+ rho| = |D- rho| = 0.5; the printed "<="
    of eq:dominant_b1/b2 selects the forward difference D+ = +0.5 (not -0.5)."""
    H, W = 9, 9
    v = np.where(np.arange(9) % 2 == 1, 0.5, 1.0).astype(np.float32)
    rho = np.tile(v, (H, 1)) if axis == 0 else np.tile(v[:, None], (1, W))
    o = oracle.Oracle(grid.flat(H, W, 2.0 ** -6), P(2), "f32")
    _, valid, b1, b2, _ = o.invdepth_model(rho, is_inverse=True)
    assert valid.all()
    b = b1 if axis == 0 else b2
    inner = (slice(None), slice(1, -1, 2)) if axis == 0 else (slice(1, -1, 2), slice(None))
    assert np.all(b[inner] == 0.5)
    other = b2 if axis == 0 else b1
    assert np.all(other == 0)


@pytest.mark.parametrize("axis", [0, 1])
def test_one_valid_neighbour_uses_its_side(axis):
    """Quadratic inverse depth rho_j = 1/2 + j^2/64 (forward and backward differences differ),
    an invalid measurement at j = 7 (reading 14): pixel 8 has only its forward neighbour
    -> D+ = rho_9 - rho_8 = 17/64; pixel 6 only its backward one -> D- = rho_6 - rho_5 = 11/64;
    the invalid pixel itself has 0; pixels with both sides take the smaller magnitude (D-)."""
    n = 12
    v = (0.5 + np.arange(n, dtype=np.float64) ** 2 / 64).astype(np.float32)
    v[7] = np.nan
    rho = np.tile(v, (5, 1)) if axis == 0 else np.tile(v[:, None], (1, 5))
    o = oracle.Oracle(grid.flat(*rho.shape, 2.0 ** -6), P(2), "f32")
    _, valid, b1, b2, _ = o.invdepth_model(rho, is_inverse=True)
    b = b1 if axis == 0 else b2
    line = b[2] if axis == 0 else b[:, 2]
    assert not valid.flatten()[7 if axis == 0 else 7 * 5]
    assert line[8] == np.float32(17 / 64)
    assert line[6] == np.float32(11 / 64)
    assert line[7] == 0.0
    assert line[3] == np.float32(5 / 64)  # both valid: |D-| = 5/64 < |D+| = 7/64
    assert line[0] == 0.0  # replicate border: D- = 0 wins


def test_depth_validity_rule():
    """Depth lambda is valid iff finite and > 0 (eq:inv_depth rho = 1/lambda; reading 14):
    lambda = 0, negative, NaN and inf are invalid (rhohat 0, no rho fusion).  An inverse-depth input
    (input_is_inverse_depth) is valid iff finite and >= 0 (rho = 0: a point at infinity)."""
    d = np.array([[2.0, 0.0, -1.0, np.nan, np.inf, 0.5]], np.float32).repeat(3, 0)
    o = oracle.Oracle(grid.flat(3, 6, 2.0 ** -6), P(2), "f32")
    rh, valid, _, _, _ = o.invdepth_model(d)
    assert valid[0].tolist() == [True, False, False, False, False, True]
    assert rh[0].tolist() == [0.5, 0.0, 0.0, 0.0, 0.0, 2.0]
    r = np.array([[0.5, 0.0, -0.25, np.nan, np.inf, 2.0]], np.float32).repeat(3, 0)
    rh, valid, _, _, _ = o.invdepth_model(r, is_inverse=True)
    assert valid[0].tolist() == [True, True, False, False, False, True]
    assert rh[0].tolist() == [0.5, 0.0, 0.0, 0.0, 0.0, 2.0]


def test_invalid_depth_keeps_predicted_rho():
    """Where no measurement is available gamma4 = 0 and rho^{k+1} = rho^{k+}: a zero
    depth on a static zero-flow scene leaves the state's rho there untouched over frames while
    valid pixels move to the measurement."""
    H, W = 8, 8
    g = grid.flat(H, W, 2.0 ** -6)
    o = oracle.Oracle(g, P(1), "f32")
    Y = np.full((H, W), 0.5, np.float32)
    d0 = np.full((H, W), 2.0, np.float32)
    o.step(Y, d0)
    d1 = d0.copy()
    d1[3, 4] = 0.0
    d1[:, 0] = 4.0
    o.step(Y, d1)
    assert o.rho[3, 4] == np.float32(0.5)
    assert np.all(o.rho[:, 0] == np.float32(0.375))  # kappa = 1/2: (0.5 + 0.25) / 2
