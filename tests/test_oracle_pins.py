"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Each test names the pin (DESIGN.md section 5 / SURVEY.md 8(c)) and the passage it checks.
None of them re-types the oracle's formulas: they use closed forms, exact shifts,
invariants, brute-force sums and numpy's own least-squares, chosen so that a dropped
term, a wrong sign or index, or a transposed operand in the oracle fails one of them.
"""
import json
import os

import numpy as np
import pytest

import oracle
import sfgen
from sfgen import grid
from sfgen.configs import Params

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_constants.json")))


def P(max_flow=2.0, gamma=(1e3, 1e3, 1.0, 1.0, 1.0), S=2, **kw):
    return Params(max_flow=max_flow, gamma=tuple(gamma), smooth_iters=S, **kw)


# --------------------------------------------------------------------------- G1 grid
def test_G1_gnomonic_grid_invariants():
    """Spherepix invariants: unit s, tangent orthonormal basis, ds."""
    g64 = grid.gnomonic(512, 512, 90.0, as_f64=True)
    s, b1, b2, ds = grid.split(g64)
    assert np.allclose(np.linalg.norm(s, axis=-1), 1.0, atol=1e-12)
    for b in (b1, b2):
        assert np.allclose(np.linalg.norm(b, axis=-1), 1.0, atol=1e-12)
        assert np.abs(np.sum(b * s, -1)).max() < 1e-12
    assert np.abs(np.sum(b1 * b2, -1)).max() < 1e-12
    # centre pitch 2 tan(45 deg)/512 and the corner spacing of a gnomonic patch
    assert abs(ds[256, 256] - 3.906e-3) < 2e-6
    assert abs(ds[0, 0] - 1.847e-3) < 2e-6
    # b1 points to the column neighbour: <b1, s_{i,j+1}> > 0 ; b2 to the row neighbour
    assert (np.sum(b1[:, :-1] * s[:, 1:], -1) > 0).all()
    assert (np.sum(b2[:-1] * s[1:], -1) > 0).all()
    g32 = grid.gnomonic(512, 512, 90.0)
    assert g32.dtype == np.float32 and np.abs(g32 - g64).max() < 1e-7


# --------------------------------------------------------------------------- C1 zero motion
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_C1_zero_motion_invariance_bitwise(prec):
    """Zero flow, repeated identical frames: predict and update leave the state bit-identical
    for 100 frames (north_star invariant; PAPER.md L750 zero initial flow)."""
    seq = sfgen.config_sequence(1, frames=1)
    Y, D = seq.Y[0], seq.depth[0].copy()
    D[5:9, 5:9] = np.nan  # some invalid measurements too
    o = oracle.Oracle(seq.geom, seq.params, prec)
    o.step(Y, D)
    w0, r0, y0 = o.w.copy(), o.rho.copy(), o.yhat.copy()
    assert (w0 == 0).all()
    for _ in range(100):
        o.step(Y, D)
    assert np.array_equal(o.w, w0) and np.array_equal(o.rho, r0) and np.array_equal(o.yhat, y0)


# --------------------------------------------------------------------------- C2 Courant-1 shift
@pytest.mark.parametrize("N", [1, 2, 4, 8])
@pytest.mark.parametrize("direction", [(1, 0), (-1, 0), (0, 1), (0, -1), (1, 1), (-1, 1)])
def test_C2_courant_one_is_exact_pixel_shift(N, direction):
    """FLAT grid, uniform w with exactly N px/frame along an axis: first-order upwind at
    Courant number 1 is an exact shift (textbook CIR scheme).
    rho moves by exactly N pixels, inflow border replicates, w is unchanged."""
    H, W, ds = 40, 48, 2.0 ** -8
    g = grid.flat(H, W, ds)
    rng = np.random.default_rng(N)
    rho0 = rng.uniform(0.5, 1.0, size=(H, W)).astype(np.float32)
    o = oracle.Oracle(g, P(max_flow=float(N)), "f32")
    dx, dy = direction
    o.set_state(np.broadcast_to(np.array([dx * N * ds, dy * N * ds, 0.0], np.float32), (H, W, 3)), rho0,
                np.zeros((H, W), np.float32))
    w, rho = o.predict()
    jj = np.clip(np.arange(W) - dx * N, 0, W - 1)
    ii = np.clip(np.arange(H) - dy * N, 0, H - 1)
    expect = rho0[ii][:, jj]
    assert np.array_equal(rho, expect)
    assert np.array_equal(w, o.w)


# --------------------------------------------------------------------------- C3 moving front
@pytest.mark.parametrize("rule,shift", [(sfgen.configs.DOM_LARGEST, 8), (sfgen.configs.DOM_PRINTED, 0)])
def test_C3_flow_front_moves_with_dominant_flow(rule, shift):
    """1-D front u = 8 px for j < j0, 0 beyond: with the LARGEST reading
    (DESIGN reading 1) the front advances exactly 8 px in one frame; the printed formula
    (which picks the smaller neighbour) never moves it."""
    H, W, ds, N, j0 = 8, 64, 2.0 ** -8, 8, 20
    g = grid.flat(H, W, ds)
    w = np.zeros((H, W, 3), np.float32)
    w[:, :j0, 0] = N * ds
    o = oracle.Oracle(g, P(max_flow=float(N), dominant_rule=rule), "f32")
    o.set_state(w, np.ones((H, W), np.float32), np.zeros((H, W), np.float32))
    wp, _ = o.predict()
    expect = np.zeros_like(w)
    expect[:, :j0 + shift, 0] = N * ds
    assert np.array_equal(wp, expect)


# --------------------------------------------------------------------------- C4/C5 planes
def _plane_fields(g64, d, v):
    """Fronto-parallel plane z = d, camera velocity v (per frame), static scene:
    rho = s_z / d (eq:inv_depth), w = -v rho (eq:homogeneous_flow with Omega = 0, v_x = 0)."""
    s = g64[..., 0:3]
    rho = s[..., 2] / d
    return -rho[..., None] * v[None, None, :], rho


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_C4_approaching_plane_matches_closed_form(prec):
    """Camera approaching a fronto-parallel plane: after one frame of prediction the fields
    must equal the closed form at distance d - v_z.  The centre
    pixel (no tangent flow) follows the Riccati ODE w' = -w <s,w>; with the source weight
    sigma = 1/2 per pass (DESIGN reading 2) it is matched to 1e-3 relative -- the printed
    full weight per pass integrates the source twice and misses by ~3e-2."""
    H = W = 512
    g64 = grid.gnomonic(H, W, 90.0, as_f64=True)
    g = g64.astype(np.float32)
    d, vz = 5.0, 0.15
    v = np.array([0.0, 0.0, vz])
    w0, rho0 = _plane_fields(g64, d, v)
    w1, rho1 = _plane_fields(g64, d - vz, v)
    for sigma, ok in ((0.5, True), (1.0, False)):
        o = oracle.Oracle(g, P(max_flow=8.0, sigma=sigma), prec)
        o.set_state(w0.astype(o.dtype), rho0.astype(o.dtype), np.zeros((H, W), o.dtype))
        wp, rp = o.predict()
        c = (H // 2, W // 2)
        rel = abs(wp[c][2] - w1[c][2]) / abs(w1[c][2])
        assert (rel < 1e-3) == ok, (sigma, rel)
        if ok:
            m = 24
            ds = g64[m:-m, m:-m, 9]
            err_px = np.linalg.norm(wp[m:-m, m:-m] - w1[m:-m, m:-m], axis=-1) / ds
            assert err_px.max() < 0.1
            assert (np.abs(rp[m:-m, m:-m] - rho1[m:-m, m:-m]) / rho1[m:-m, m:-m]).max() < 1e-2
            # the prediction moved towards the closed form: far better than "no change"
            assert np.abs(wp - w1).max() < 0.2 * np.abs(w0 - w1).max()


def test_C5_lateral_translation_is_stationary():
    """Lateral camera motion over a fronto-parallel plane: rho = s_z/d and w = -v s_z/d do not
    change in time (the RHS of eq:hflow_conservation / eq:invdepth_conservation vanishes,
    PAPER.md L336, L347).  One predict at 8 px max flow moves them only by truncation error."""
    H = W = 512
    g64 = grid.gnomonic(H, W, 90.0, as_f64=True)
    d = 5.0
    v = np.array([0.03, -0.02, 0.0])
    w0, rho0 = _plane_fields(g64, d, v)
    o = oracle.Oracle(g64.astype(np.float32), P(max_flow=8.0), "f64")
    o.set_state(w0, rho0, np.zeros((H, W)))
    wp, rp = o.predict()
    m = 24
    ds = g64[m:-m, m:-m, 9]
    flow_px = (np.linalg.norm(w0, axis=-1)[m:-m, m:-m] / ds).max()
    assert 2.0 < flow_px < 8.0
    # first-order truncation error only: <= 1e-3 of the flow (a dropped or doubled source
    # term, or a wrong upwind side, moves the fields by >= 1e-2 of the flow)
    assert (np.linalg.norm(wp - w0, axis=-1)[m:-m, m:-m] / ds).max() < 1e-3 * flow_px
    assert (np.abs(rp - rho0)[m:-m, m:-m] / rho0[m:-m, m:-m]).max() < 1e-3
    # and the scheme does move the fields by far more with the printed source weight
    o1 = oracle.Oracle(g64.astype(np.float32), P(max_flow=8.0, sigma=1.0), "f64")
    o1.set_state(w0, rho0, np.zeros((H, W)))
    wp1, _ = o1.predict()
    assert (np.linalg.norm(wp1 - w0, axis=-1)[m:-m, m:-m] / ds).max() > 3e-3 * flow_px


# --------------------------------------------------------------------------- C6 normal flow
def test_C6_uniform_normal_flow_converges_to_continuum():
    """w = (0, 0, c) on the FLAT grid has no tangent flow, so the predictor reduces to the
    ODEs w_z' = -w_z^2, rho' = -rho w_z (eq:hflow_propagation_top / eq:invdepth_propagation_top
    with the advection term zero), whose solution at t = 1 is c/(1+c), rho0/(1+c).
    The explicit scheme converges to it at first order in dt = 1/N."""
    H, W = 6, 6
    g = grid.flat(H, W)
    c, r0 = -0.2, 0.7
    errs = []
    for N in (4, 8, 16, 32, 64):
        o = oracle.Oracle(g, P(max_flow=float(N)), "f64")
        o.set_state(np.broadcast_to(np.array([0, 0, c]), (H, W, 3)).copy(), np.full((H, W), r0), np.zeros((H, W)))
        wp, rp = o.predict()
        assert np.all(wp[..., :2] == 0)
        assert np.ptp(wp[..., 2]) == 0 and np.ptp(rp) == 0
        errs.append((abs(wp[0, 0, 2] - c / (1 + c)), abs(rp[0, 0] - r0 / (1 + c))))
    errs = np.array(errs)
    ratio = errs[:-1] / errs[1:]
    assert np.all(np.abs(ratio - 2.0) < 0.1), ratio  # first order
    assert errs[-1, 0] < 2e-3 and errs[-1, 1] < 2e-3


# --------------------------------------------------------------------------- C7 monotone
def test_C7_upwind_transport_is_monotone():
    """With <s,w> = 0 and Courant <= 1 the transport of rho is a convex combination of
    neighbours (upwind): its max does not grow and its min does not fall."""
    H, W, ds = 64, 64, 2.0 ** -8
    g = grid.flat(H, W, ds)
    rng = np.random.default_rng(7)
    jj, ii = np.meshgrid(np.arange(W), np.arange(H))
    w = np.zeros((H, W, 3), np.float32)
    w[..., 0] = (3.0 * np.sin(ii / 7.0) + 1.0 * np.cos(jj / 5.0)) * ds
    w[..., 1] = (2.5 * np.cos(jj / 9.0) - 1.0) * ds
    rho0 = rng.uniform(0.1, 1.0, (H, W)).astype(np.float32)
    o = oracle.Oracle(g, P(max_flow=4.0), "f64")
    o.set_state(w, rho0, np.zeros((H, W), np.float32))
    _, rp = o.predict()
    assert rp.max() <= rho0.max() + 1e-15 and rp.min() >= rho0.min() - 1e-15
    assert o.flags & oracle.FLAG_CLAMPED == 0


# --------------------------------------------------------------------------- M1 brightness
def _dense_weighted_ls(Y, i, j):
    """Weighted LS of eq:img_model solved directly on the 5x5 window:
    minimise sum_q G(p,q) (Y_q - beta.(q-p) - Yhat)^2 with G = g^T g, g from the golden file."""
    gg = np.array(GOLD["gaussian_g"]["value"], float) / GOLD["gaussian_g"]["divisor"]
    rows, rhs, wts = [], [], []
    for a in range(-2, 3):
        for b in range(-2, 3):
            rows.append([b, a, 1.0])  # (column offset, row offset, constant)
            rhs.append(Y[i + a, j + b])
            wts.append(gg[a + 2] * gg[b + 2])
    sw = np.sqrt(np.array(wts))
    x, *_ = np.linalg.lstsq(np.array(rows) * sw[:, None], np.array(rhs) * sw, rcond=None)
    return x  # beta1 (along j), beta2 (along i), Yhat


def test_M1_brightness_model():
    """Brightness model: exact on affine ramps, the fitted constant of an
    integer quadratic shows sum g k^2 = 1 exactly, matches a dense 25-point weighted LS, and
    the tangent lift is ghat = ds (b1 beta1 + b2 beta2) (eq:img_gradient, reading 5)."""
    H, W, ds = 40, 48, 2.0 ** -6
    o = oracle.Oracle(grid.flat(H, W, ds), P(), "f32")
    ii, jj = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    a, b, c = 0.25, -0.125, 3.0
    yh, b1, b2, gh = o.brightness_model((a * jj + b * ii + c).astype(np.float32))
    In = (slice(2, -2), slice(2, -2))
    assert np.array_equal(b1[In], np.full_like(b1[In], a)) and np.array_equal(b2[In], np.full_like(b2[In], b))
    assert np.array_equal(yh[In], (a * jj + b * ii + c)[In].astype(np.float32))
    assert np.allclose(gh[In][..., 0], ds * a, rtol=1e-6) and np.allclose(gh[In][..., 1], ds * b, rtol=1e-6)
    assert np.all(gh[..., 2] == 0)
    yh, b1, b2, _ = o.brightness_model((ii ** 2 + jj ** 2).astype(np.float32))
    assert np.array_equal(yh[In], (ii ** 2 + jj ** 2 + 2)[In].astype(np.float32))
    assert np.array_equal(b1[In], (2 * jj)[In].astype(np.float32))
    assert np.array_equal(b2[In], (2 * ii)[In].astype(np.float32))
    yh, b1, b2, _ = o.brightness_model(np.full((H, W), 0.3, np.float32))
    assert np.all(b1 == 0) and np.all(b2 == 0)
    rng = np.random.default_rng(3)
    Y = rng.uniform(0.1, 0.9, (H, W)).astype(np.float32)
    o64 = oracle.Oracle(grid.flat(H, W, ds), P(), "f64")
    yh, b1, b2, _ = o64.brightness_model(Y)
    for _ in range(50):
        i, j = rng.integers(2, H - 2), rng.integers(2, W - 2)
        x = _dense_weighted_ls(Y.astype(float), i, j)
        assert np.allclose([b1[i, j], b2[i, j], yh[i, j]], x, atol=1e-12)
    # lift on a curved grid: ghat = ds (b1 beta1 + b2 beta2), tangent to s
    gg = grid.gnomonic(32, 32, 70.0)
    og = oracle.Oracle(gg, P(), "f64")
    Yg = rng.uniform(0.1, 0.9, (32, 32)).astype(np.float32)
    _, b1, b2, gh = og.brightness_model(Yg)
    s, bb1, bb2, dsg = (x.astype(float) for x in grid.split(gg))
    expect = dsg[..., None] * (bb1 * b1[..., None] + bb2 * b2[..., None])
    assert np.allclose(gh, expect, rtol=1e-12, atol=1e-15)


# --------------------------------------------------------------------------- M2 inverse depth
def test_M2_inverse_depth_model():
    """Occlusion-aware rho gradient (eq:dominant_b1/b2): the one-sided
    difference of smaller magnitude (golden table:diff_operators), ties -> forward,
    exact on ramps, invalid depth drops out; rhohat = 1/lambda (eq:inv_depth)."""
    H, W = 12, 16
    o = oracle.Oracle(grid.flat(H, W, 2.0 ** -6), P(), "f32")
    ops = GOLD["difference_operators"]

    def apply(op, x, j, i=None):
        return sum(float(c) * x[j + int(k)] for k, c in ops[op].items())

    step = np.where(np.arange(W) < 5, 0.1, 0.9).astype(np.float32)
    rho = np.broadcast_to(step, (H, W)).copy()
    rh, valid, br1, br2, dr = o.invdepth_model(rho, is_inverse=True)
    assert valid.all() and np.array_equal(rh, rho)
    row = rh[3]
    for j in range(1, W - 1):
        fwd, bwd = apply("forward", row, j), apply("backward", row, j)
        expect = fwd if abs(fwd) <= abs(bwd) else bwd
        assert br1[3, j] == np.float32(expect)
    assert br1[3, 4] == 0.0 and br1[3, 5] == 0.0  # the step is assigned to neither side
    assert np.all(br2 == 0)
    # ramp: both sides equal -> exact gradient; depth input inverted with IEEE 1/x
    ramp = (0.5 + 0.0625 * np.arange(W, dtype=np.float32))[None].repeat(H, 0)
    rh, valid, br1, br2, _ = o.invdepth_model((1.0 / ramp).astype(np.float32), is_inverse=False)
    assert np.array_equal(rh, (np.float32(1) / (np.float32(1) / ramp)).astype(np.float32))
    assert np.allclose(br1[:, 1:-1], 0.0625, rtol=1e-6)
    # invalid depth: p invalid -> 0; neighbour invalid -> the other side
    d = np.full((H, W), 2.0, np.float32)
    d[:, 7] = np.nan
    d[:, 9] = -1.0
    rh, valid, br1, _, dr = o.invdepth_model(d)
    assert not valid[0, 7] and not valid[0, 9] and rh[0, 7] == 0 and np.all(dr[:, 7] == 0)
    assert br1[0, 8] == 0.0  # both neighbours invalid
    assert br1[0, 6] == np.float32(0.5) - np.float32(0.5)


# --------------------------------------------------------------------------- L1 LS update
def test_L1_ls_update_matches_numpy_lstsq():
    """Per-pixel update (eq:LS_update): the 3x3 LDL^T path equals
    numpy's least squares on the stacked residuals [sqrt(g1) ghat^T; sqrt(g2) m^T; sqrt(g3) I]
    w = [-sqrt(g1) cY; -sqrt(g2) crho; sqrt(g3) wp] (E_t = w - wp, reading 8) on 10^4 random
    instances, within the backward-error bound 64 cond(A) eps of the precision;
    gamma1 = gamma2 = 0 returns the prediction exactly."""
    rng = np.random.default_rng(11)
    n = 10000
    g = rng.normal(size=(n, 3)) * 10 ** rng.uniform(-3, 0, (n, 1))
    m = rng.normal(size=(n, 3)) * 10 ** rng.uniform(-3, 0, (n, 1))
    cY, cr = rng.normal(size=n) * 1e-3, rng.normal(size=n) * 1e-3
    wp = rng.normal(size=(n, 3)) * 1e-2
    gam = np.array([2e3, 5e3, 1.0])
    for prec in ("f64", "f32"):
        out = oracle.ls_solve(g, m, cY, cr, wp, gam, prec)
        dt = out.dtype
        eps = np.finfo(dt).eps
        gq, mq, cYq, crq, wpq = (x.astype(dt).astype(float) for x in (g, m, cY, cr, wp))
        worst = 0.0
        for p in range(0, n, 7):
            Amat = np.vstack([np.sqrt(gam[0]) * gq[p], np.sqrt(gam[1]) * mq[p], np.sqrt(gam[2]) * np.eye(3)])
            rhs = np.concatenate([[-np.sqrt(gam[0]) * cYq[p], -np.sqrt(gam[1]) * crq[p]], np.sqrt(gam[2]) * wpq[p]])
            x, *_ = np.linalg.lstsq(Amat, rhs, rcond=None)
            cond = np.linalg.cond(Amat.T @ Amat)
            # backward-stable 3x3 solve: error <= c * cond(A) * eps (c = 64 covers the op count and
            # the error of the f64 reference itself)
            rel = np.abs(out[p] - x).max() / max(np.abs(x).max(), 1e-30)
            worst = max(worst, rel / (cond * eps))
        assert worst < 64.0, (prec, worst)
    out = oracle.ls_solve(g, m, cY, cr, wp, np.array([0.0, 0.0, 1.0]), "f32")
    assert np.array_equal(out, wp.astype(np.float32))


# --------------------------------------------------------------------------- L2 smoothing
def test_L2_smoothing_is_iterated_5x5_box_mean():
    """'average smoothing filter of size 5x5' applied S times: equals a
    brute-force 25-term mean with replicated borders, preserves constants, is linear."""
    H, W = 20, 23
    o = oracle.Oracle(grid.flat(H, W), P(), "f64")
    rng = np.random.default_rng(5)
    x = rng.normal(size=(H, W, 3))
    y = x.copy()
    for _ in range(3):
        pad = np.pad(y, ((2, 2), (2, 2), (0, 0)), mode="edge")
        y = sum(pad[a:a + H, b:b + W] for a in range(5) for b in range(5)) / 25.0
    assert np.allclose(o.smooth(x, 3), y, rtol=1e-13, atol=1e-15)
    o32 = oracle.Oracle(grid.flat(H, W), P(), "f32")
    cst = np.full((H, W, 3), 0.3, np.float32)
    assert np.abs(o32.smooth(cst, 2) - cst).max() <= np.spacing(np.float32(0.3))
    a, b = rng.normal(size=(H, W, 3)), rng.normal(size=(H, W, 3))
    assert np.allclose(o.smooth(2 * a - b, 2), 2 * o.smooth(a, 2) - o.smooth(b, 2), atol=1e-13)


# --------------------------------------------------------------------------- L3 fusion
@pytest.mark.parametrize("g4,g5", [(1.0, 1.0), (1.0, 0.0), (3.0, 1.0)])
def test_L3_inverse_depth_fusion(g4, g5):
    """rho^{k+1} = (g4 rhohat + g5 rho^{k+})/(g4 + g5); no measurement
    -> rho^{k+} unchanged (L621)."""
    H, W = 10, 12
    o = oracle.Oracle(grid.flat(H, W), P(gamma=(0.0, 0.0, 1.0, g4, g5), S=0), "f64")
    rng = np.random.default_rng(int(g4 * 10 + g5))
    rp = rng.uniform(0.2, 1.0, (H, W))
    lam = rng.uniform(1.5, 4.0, (H, W)).astype(np.float32)
    lam[0, 0] = np.nan
    o.set_state(np.zeros((H, W, 3)), rp.copy(), np.zeros((H, W)))
    o.update(np.zeros((H, W), np.float32), lam, wp=np.zeros((H, W, 3)), rhop=rp)
    rh = 1.0 / lam.astype(float)
    expect = (g4 * rh + g5 * rp) / (g4 + g5)
    expect[0, 0] = rp[0, 0]
    assert np.allclose(o.rho, expect, rtol=1e-14)
    assert o.rho[0, 0] == rp[0, 0]


# --------------------------------------------------------------------------- U3 data terms
def test_U3_brightness_term_recovers_flow_along_gradient():
    """E_Y (eq:img_cost_top, L564): with a pure brightness constraint, the solved flow's
    component along ghat satisfies ghat.w = -ds^2 (Yhat^{k+1} - Yhat^k) in the limit of a
    dominant gamma1, and the orthogonal part keeps the prediction (aperture problem, L567)."""
    H, W, ds = 24, 24, 2.0 ** -6
    o = oracle.Oracle(grid.flat(H, W, ds), P(gamma=(1e14, 0.0, 1.0, 1.0, 1.0), S=0), "f64")
    jj = np.arange(W)[None].repeat(H, 0)
    Y0 = (0.0625 * jj).astype(np.float32)
    Y1 = (0.0625 * (jj - 0.5)).astype(np.float32)  # pattern moved +0.5 px along j (exact values)
    o.step(Y0, np.full((H, W), 2.0, np.float32))
    wp = np.zeros((H, W, 3))
    wp[..., 1] = 1e-3  # prediction orthogonal to the gradient
    o.update(Y1, np.full((H, W), 2.0, np.float32), wp=wp, rhop=o.rho.copy())
    c = (12, 12)
    # brightness constancy: u = 0.5 px  -> w_x = 0.5 ds
    # regularisation bias gamma3 / (gamma1 |ghat|^2) ~ 1e-8 relative
    assert abs(o.w[c][0] - 0.5 * ds) < 1e-7 * ds
    assert abs(o.w[c][1] - 1e-3) < 1e-12 and abs(o.w[c][2]) < 1e-12


def test_U3_depth_term_recovers_normal_flow():
    """E_rho (eq:invdepth_cost_top, L572): a uniform inverse-depth change without gradient is
    explained by the normal component alone: rhohat - rho^k + rhohat <s,w> = 0, i.e.
    <s,w> = rho^k/rhohat - 1 for a dominant gamma2 (L574: normal flow is recoverable)."""
    H, W = 16, 16
    o = oracle.Oracle(grid.flat(H, W, 2.0 ** -6), P(gamma=(0.0, 1e14, 1.0, 1.0, 0.0), S=0), "f64")
    Y = np.zeros((H, W), np.float32)
    o.step(Y, np.full((H, W), 2.0, np.float32))  # rho^k = 0.5
    o.update(Y, np.full((H, W), 1.6, np.float32), wp=np.zeros((H, W, 3)), rhop=o.rho.copy())
    rh = 1.0 / float(np.float32(1.6))
    assert abs(o.w[8, 8, 2] - (0.5 / rh - 1.0)) < 1e-6
    assert abs(o.w[8, 8, 0]) < 1e-12 and abs(o.w[8, 8, 1]) < 1e-12
    assert abs(o.rho[8, 8] - rh) < 1e-15  # g5 = 0 -> measurement


# --------------------------------------------------------------------------- drift + E1
def test_f32_vs_f64_drift_config1():
    """The float32 parity oracle stays within 1e-6 of the float64 build over config 1."""
    seq = sfgen.config_sequence(1)
    o32, _ = oracle.run_sequence(seq.geom, seq.params, seq.Y, seq.depth, "f32")
    o64, _ = oracle.run_sequence(seq.geom, seq.params, seq.Y, seq.depth, "f64")
    assert np.abs(o32.w - o64.w).max() < 1e-6
    assert np.abs(o32.rho - o64.rho).max() < 1e-6
    assert np.abs(o32.yhat - o64.yhat).max() < 1e-6


def test_E1_filter_converges_towards_ground_truth():
    """End-to-end accuracy smoke (the flow is identified and diffused,
    RMSE falls): on config 1's scene the mean endpoint error in pixels (eq:RMSE_vel) after
    40 frames is well below the error of the zero initial condition."""
    seq = sfgen.config_sequence(1, frames=40, with_gt=True)
    o, _ = oracle.run_sequence(seq.geom, seq.params, seq.Y, seq.depth, "f32")
    ds = seq.geom[..., 9][..., None]
    err = np.linalg.norm((o.w - seq.w_gt[-1]) / ds, axis=-1).mean()
    zero = np.linalg.norm(seq.w_gt[-1] / ds, axis=-1).mean()
    assert err < 0.25 * zero, (err, zero)
