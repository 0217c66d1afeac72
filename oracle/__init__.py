"""CPU oracle of the structure-flow predictor-update loop -- TEST INFRASTRUCTURE ONLY.

ctypes binding over oracle/sf_oracle.c (see its header for the algorithm, the
paper passages each function follows, and the readings).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  It shares no code with paper_2406_18031_b200/ and never
imports it; both consume inputs from sfgen/.

Precision: "f32" is the parity oracle (all values and decisions in IEEE float32),
"f64" the same algorithm in float64 (pins the f32 build's rounding drift).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import build as _build

FLAG_CLAMPED = 1
FLAG_NONFINITE = 2
FLAG_CFL = 4


class _Params(C.Structure):
    _fields_ = [("H", C.c_int32), ("W", C.c_int32), ("N", C.c_int32), ("smooth_iters", C.c_int32),
                ("dominant_rule", C.c_int32), ("clamp_advection", C.c_int32),
                ("input_is_inverse_depth", C.c_int32), ("pad", C.c_int32),
                ("max_flow", C.c_double), ("sigma", C.c_double), ("gamma", C.c_double * 5),
                ("imu", C.c_int32), ("pad2", C.c_int32), ("omega", C.c_double * 3), ("accel", C.c_double * 3)]


_LIBS: dict = {}


def _lib(prec: str):
    if prec not in _LIBS:
        path = _build.lib_path(prec)
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(_build.SRC):
            _build.build()
        lib = C.CDLL(path)
        for name in ("or_predict", "or_update", "or_step", "or_pyr_step_flat", "or_predict_low"):
            getattr(lib, name).restype = C.c_uint
        _LIBS[prec] = lib
    return _LIBS[prec]


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return a.ctypes.data_as(C.c_void_p)


def make_params(H: int, W: int, p) -> _Params:
    """p: an sfgen.Params (or any object with the same attributes)."""
    P = _Params()
    P.H, P.W, P.N = H, W, p.N
    P.smooth_iters = p.smooth_iters
    P.dominant_rule = p.dominant_rule
    P.clamp_advection = p.clamp_advection
    P.input_is_inverse_depth = p.input_is_inverse_depth
    P.max_flow = p.max_flow
    P.sigma = p.sigma
    for k in range(5):
        P.gamma[k] = p.gamma[k]
    om = getattr(p, "omega", None)
    ac = getattr(p, "accel", None)
    if om is not None or ac is not None:
        P.imu = 1
        for k in range(3):
            P.omega[k] = float(np.float32((om or (0, 0, 0))[k]))
            P.accel[k] = float(np.float32((ac or (0, 0, 0))[k]))
    return P


class Oracle:
    """State-holding wrapper: w [H][W][3], rho [H][W], yhat [H][W] in the oracle's precision."""

    def __init__(self, geom: np.ndarray, params, precision: str = "f32"):
        self.prec = precision
        self.dtype = np.float32 if precision == "f32" else np.float64
        self.lib = _lib(precision)
        geom = np.ascontiguousarray(geom, dtype=np.float32)
        self.H, self.W, _ = geom.shape
        self.params = params
        self.P = make_params(self.H, self.W, params)
        self.geo = np.empty((self.H, self.W, 10), self.dtype)
        self.lib.or_geometry(self.H, self.W, _ptr(geom), _ptr(self.geo))
        self.w = np.zeros((self.H, self.W, 3), self.dtype)
        self.rho = np.zeros((self.H, self.W), self.dtype)
        self.yhat = np.zeros((self.H, self.W), self.dtype)
        self.initialized = False
        self.flags = 0

    # -- whole-frame calls -------------------------------------------------------------
    def step(self, Y: np.ndarray, depth: np.ndarray, keep_prediction: bool = False):
        """One frame (first call = initialisation).  Returns the flags of this frame."""
        Y = np.ascontiguousarray(Y, np.float32)
        depth = np.ascontiguousarray(depth, np.float32)
        wp = rp = None
        if keep_prediction and self.initialized:
            wp = np.empty_like(self.w)
            rp = np.empty_like(self.rho)
        f = self.lib.or_step(C.byref(self.P), _ptr(self.geo), _ptr(Y), _ptr(depth), _ptr(self.w), _ptr(self.rho),
                             _ptr(self.yhat), C.c_int(0 if self.initialized else 1),
                             _ptr(wp) if wp is not None else None, _ptr(rp) if rp is not None else None)
        self.initialized = True
        self.flags |= f
        self.last_prediction = (wp, rp)
        return f

    def predict(self):
        """Return (w^{k+}, rho^{k+}) without touching the state."""
        w = self.w.copy()
        r = self.rho.copy()
        f = self.lib.or_predict(C.byref(self.P), _ptr(self.geo), _ptr(w), _ptr(r))
        self.flags |= f
        return w, r

    def update(self, Y, depth, wp=None, rhop=None):
        """Update the state from a given prediction (default: the state itself, i.e. no predict)."""
        Y = np.ascontiguousarray(Y, np.float32)
        depth = np.ascontiguousarray(depth, np.float32)
        init = not self.initialized
        if not init:
            wp = np.ascontiguousarray(self.w if wp is None else wp, self.dtype).copy()
            rhop = np.ascontiguousarray(self.rho if rhop is None else rhop, self.dtype).copy()
        f = self.lib.or_update(C.byref(self.P), _ptr(self.geo), _ptr(Y), _ptr(depth),
                               _ptr(wp) if wp is not None else None, _ptr(rhop) if rhop is not None else None,
                               _ptr(self.w), _ptr(self.rho), _ptr(self.yhat), C.c_int(1 if init else 0))
        self.initialized = True
        self.flags |= f
        return f

    def set_state(self, w, rho, yhat):
        self.w[...] = w
        self.rho[...] = rho
        self.yhat[...] = yhat
        self.initialized = True

    # -- individual steps (for the pins) -----------------------------------------------
    def brightness_model(self, Y):
        Y = np.ascontiguousarray(Y, np.float32)
        H, W = Y.shape
        out = [np.empty((H, W), self.dtype) for _ in range(3)] + [np.empty((H, W, 3), self.dtype)]
        self.lib.or_brightness_model(H, W, _ptr(Y), _ptr(self.geo), *[_ptr(o) for o in out])
        return tuple(out)  # yhat, beta1, beta2, ghat

    def invdepth_model(self, depth, is_inverse=False):
        depth = np.ascontiguousarray(depth, np.float32)
        H, W = depth.shape
        rh = np.empty((H, W), self.dtype)
        valid = np.empty((H, W), np.uint8)
        b1 = np.empty((H, W), self.dtype)
        b2 = np.empty((H, W), self.dtype)
        dr = np.empty((H, W, 3), self.dtype)
        self.lib.or_invdepth_model(H, W, _ptr(depth), C.c_int(int(is_inverse)), _ptr(self.geo), _ptr(rh),
                                   _ptr(valid), _ptr(b1), _ptr(b2), _ptr(dr))
        return rh, valid.astype(bool), b1, b2, dr

    def smooth(self, w, S):
        w = np.ascontiguousarray(w, self.dtype).copy()
        H, W, _ = w.shape
        self.lib.or_smooth(H, W, C.c_int(S), _ptr(w))
        return w


def ls_solve(g, m, cY, cr, wp, gam, precision="f32"):
    """Vectorised per-pixel 3x3 update solve (U3).  Arrays [n][3], [n][3], [n], [n], [n][3]."""
    dt = np.float32 if precision == "f32" else np.float64
    g, m, wp = (np.ascontiguousarray(x, dt) for x in (g, m, wp))
    cY, cr = (np.ascontiguousarray(x, dt) for x in (cY, cr))
    n = g.shape[0]
    out = np.empty((n, 3), dt)
    gam = np.ascontiguousarray(gam, np.float64)
    _lib(precision).or_ls_solve_batch(C.c_long(n), _ptr(g), _ptr(m), _ptr(cY), _ptr(cr), _ptr(wp), _ptr(gam),
                                      _ptr(out))
    return out


def flow_px(geom, w, precision="f32"):
    """Tangent flow [H][W][2] and normal flow [H][W] of w [H][W][3], in pixels (eq:tangent_flow,
    eq:normal_flow; reading 23)."""
    geom = np.ascontiguousarray(geom, np.float32)
    H, W, _ = geom.shape
    dt = np.float32 if precision == "f32" else np.float64
    lib = _lib(precision)
    geo = np.empty((H, W, 10), dt)
    lib.or_geometry(H, W, _ptr(geom), _ptr(geo))
    w = np.ascontiguousarray(w, dt)
    t = np.empty((H, W, 2), dt)
    nrm = np.empty((H, W), dt)
    lib.or_flow_px(C.c_long(H * W), _ptr(geom), _ptr(geo), _ptr(w), _ptr(t), _ptr(nrm))
    return t, nrm


def evaluate(geom, w_gt, w, precision="f32"):
    """Per-pixel RMSE (px/frame) and AAE (cosine and degrees) of w against w_gt, and their means
    over the pixels (eq:RMSE_vel and the AAE of P:L726-734; reading 22)."""
    geom = np.ascontiguousarray(geom, np.float32)
    H, W, _ = geom.shape
    dt = np.float32 if precision == "f32" else np.float64
    w_gt = np.ascontiguousarray(w_gt, dt)
    w = np.ascontiguousarray(w, dt)
    rmse = np.empty((H, W), dt)
    cos = np.empty((H, W), np.float64)
    deg = np.empty((H, W), np.float64)
    sums = np.zeros(2, np.float64)
    _lib(precision).or_eval(C.c_long(H * W), _ptr(geom), _ptr(w_gt), _ptr(w), _ptr(rmse), _ptr(cos), _ptr(deg),
                            _ptr(sums))
    return {"rmse": rmse, "aae_cos": cos, "aae_deg": deg, "mean_rmse": sums[0] / (H * W),
            "mean_aae_deg": sums[1] / (H * W)}


def pyramid_params(params, geom1, geom2, smooth_top: int = 4):
    """Per-level parameters of the H = 2 filter (DESIGN reading 29): the bottom level keeps
    `params`; the top level has max_flow / 2 (flows halve on the half grid), its own substep
    count ceil(max_flow / 2), smooth_top box iterations (Table 3: [2, 4]) and gains gamma1,2
    scaled by (ds1 / ds2)^2 (centre pixel separations; gains scale as ds^-2, reading 11)."""
    import copy
    top = copy.copy(params)
    top.max_flow = float(np.float32(params.max_flow) * np.float32(0.5))
    top.smooth_iters = smooth_top
    H1, W1 = geom1.shape[:2]
    H2, W2 = geom2.shape[:2]
    r = float(geom1[H1 // 2, W1 // 2, 9]) / float(geom2[H2 // 2, W2 // 2, 9])
    r2 = r * r
    g = list(params.gamma)
    top.gamma = (float(np.float32(g[0] * r2)), float(np.float32(g[1] * r2)), g[2], g[3], g[4])
    return top


class PyramidOracle:
    """H = 2 filter (or_pyr_step): top level = an H = 1 state on geom2, bottom level state
    F [H][W][8] = (w, dw, rho, Yhat).  Output flow/inverse depth: w = F[..., 0:3], rho = F[..., 6]."""

    def __init__(self, geom1, geom2, params, precision="f32", smooth_top: int = 4):
        self.prec = precision
        self.dtype = np.float32 if precision == "f32" else np.float64
        self.lib = _lib(precision)
        self.geom1 = np.ascontiguousarray(geom1, np.float32)
        self.geom2 = np.ascontiguousarray(geom2, np.float32)
        self.H, self.W = self.geom1.shape[:2]
        self.Hc, self.Wc = self.geom2.shape[:2]
        assert (self.Hc, self.Wc) == (self.H // 2, self.W // 2) and self.H % 2 == 0 and self.W % 2 == 0
        self.params_low = params
        self.params_top = pyramid_params(params, self.geom1, self.geom2, smooth_top)
        self.Plow = make_params(self.H, self.W, self.params_low)
        self.Ptop = make_params(self.Hc, self.Wc, self.params_top)
        self.geo1 = np.empty((self.H, self.W, 10), self.dtype)
        self.geo2 = np.empty((self.Hc, self.Wc, 10), self.dtype)
        self.lib.or_geometry(self.H, self.W, _ptr(self.geom1), _ptr(self.geo1))
        self.lib.or_geometry(self.Hc, self.Wc, _ptr(self.geom2), _ptr(self.geo2))
        self.w2 = np.zeros((self.Hc, self.Wc, 3), self.dtype)
        self.rho2 = np.zeros((self.Hc, self.Wc), self.dtype)
        self.yhat2 = np.zeros((self.Hc, self.Wc), self.dtype)
        self.F = np.zeros((self.H, self.W, 8), self.dtype)
        self.initialized = False
        self.flags = 0

    def step(self, Y, depth):
        Y = np.ascontiguousarray(Y, np.float32)
        depth = np.ascontiguousarray(depth, np.float32)
        self.Y2 = np.empty((self.Hc, self.Wc), np.float32)
        self.D2 = np.empty((self.Hc, self.Wc), np.float32)
        f = self.lib.or_pyr_step_flat(C.byref(self.Ptop), C.byref(self.Plow), _ptr(self.geo2), _ptr(self.geo1),
                                      _ptr(self.w2), _ptr(self.rho2), _ptr(self.yhat2), _ptr(self.F), _ptr(Y),
                                      _ptr(depth), _ptr(self.Y2), _ptr(self.D2),
                                      C.c_int(0 if self.initialized else 1))
        self.initialized = True
        self.flags |= f
        return f

    @property
    def w(self):
        return self.F[..., 0:3]

    @property
    def rho(self):
        return self.F[..., 6]

    @property
    def dw(self):
        return self.F[..., 3:6]

    @property
    def yhat(self):
        return self.F[..., 7]


def predict_low(geom, params, F, precision="f32"):
    """Bottom-level prediction alone: N substeps transporting F [H][W][8] = (w, dw, rho, Yhat) by w."""
    dt = np.float32 if precision == "f32" else np.float64
    geom = np.ascontiguousarray(geom, np.float32)
    H, W, _ = geom.shape
    lib = _lib(precision)
    geo = np.empty((H, W, 10), dt)
    lib.or_geometry(H, W, _ptr(geom), _ptr(geo))
    F = np.ascontiguousarray(F, dt).copy()
    P = make_params(H, W, params)
    f = lib.or_predict_low(C.byref(P), _ptr(geo), _ptr(F))
    return F, f


def map_inputs(geom, K, Ycam, Zcam, Rcg=None):
    """Resample a pinhole camera's brightness and z-depth ([Hc][Wc]) onto the grid (reading 31);
    K = (fx, fy, cx, cy), Rcg = grid -> camera rotation (identity by default)."""
    geom = np.ascontiguousarray(geom, np.float32)
    H, W, _ = geom.shape
    Ycam = np.ascontiguousarray(Ycam, np.float32)
    Zcam = np.ascontiguousarray(Zcam, np.float32)
    Hc, Wc = Ycam.shape
    R = np.ascontiguousarray(np.eye(3) if Rcg is None else Rcg, np.float32)
    Kf = np.ascontiguousarray(K, np.float32)
    Y = np.empty((H, W), np.float32)
    D = np.empty((H, W), np.float32)
    _lib("f32").or_map_inputs(C.c_long(H * W), _ptr(geom), _ptr(R), _ptr(Kf), Hc, Wc, _ptr(Ycam), _ptr(Zcam),
                              _ptr(Y), _ptr(D))
    return Y, D


def down2(Y, depth, is_inverse=False):
    """2 x 2 mean pyramid step of brightness and depth (reading 24)."""
    Y = np.ascontiguousarray(Y, np.float32)
    depth = np.ascontiguousarray(depth, np.float32)
    H, W = Y.shape
    Y2 = np.empty((H // 2, W // 2), np.float32)
    D2 = np.empty((H // 2, W // 2), np.float32)
    _lib("f32").or_down2(H, W, _ptr(Y), _ptr(depth), C.c_int(int(is_inverse)), _ptr(Y2), _ptr(D2))
    return Y2, D2


def up2(X, precision="f32"):
    """Bilinear 2x up-sampling of a [Hc][Wc][3] field (reading 25)."""
    dt = np.float32 if precision == "f32" else np.float64
    X = np.ascontiguousarray(X, dt)
    Hc, Wc, _ = X.shape
    out = np.empty((2 * Hc, 2 * Wc, 3), dt)
    _lib(precision).or_up2(Hc, Wc, _ptr(X), _ptr(out))
    return out


def run_sequence(geom, params, Y, depth, precision="f32", frames=None):
    """Run the filter over a sequence; returns the Oracle (final state) and the per-frame flags."""
    o = Oracle(geom, params, precision)
    F = Y.shape[0] if frames is None else frames
    flags = [o.step(Y[k], depth[k]) for k in range(F)]
    return o, flags
