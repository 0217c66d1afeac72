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
                ("max_flow", C.c_double), ("sigma", C.c_double), ("gamma", C.c_double * 5)]


_LIBS: dict = {}


def _lib(prec: str):
    if prec not in _LIBS:
        path = _build.lib_path(prec)
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(_build.SRC):
            _build.build()
        lib = C.CDLL(path)
        for name in ("or_predict", "or_update", "or_step"):
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


def run_sequence(geom, params, Y, depth, precision="f32", frames=None):
    """Run the filter over a sequence; returns the Oracle (final state) and the per-frame flags."""
    o = Oracle(geom, params, precision)
    F = Y.shape[0] if frames is None else frames
    flags = [o.step(Y[k], depth[k]) for k in range(F)]
    return o, flags
