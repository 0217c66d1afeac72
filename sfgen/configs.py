"""The BASELINE.json workloads as seeded synthetic sequences, plus run parameters.

Input recipe: GNOMONIC grids; textured planes and
spheres; camera and objects translating at constant velocity; speeds scaled so
the ground-truth tangent flow (max over the first and last frame) peaks at
0.9 x max_flow pixels unless a 2 %/frame cap on the normal rate binds first; a seeded
sub-centimetre camera jitter and random texture phases break exact symmetric ties.

Run parameters (gains etc.) are plain numbers handed identically to the oracle
and to the CUDA library.  The paper gives no gain values;
the defaults are SURVEY.md 8(c)-11's reading: gamma1 = k1/ds^2, gamma2 = k2/ds^2
(ds = centre pixel separation), gamma3 = gamma4 = gamma5 = 1.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import grid as _grid
from .scene import Plane, Scene, Sphere, Texture, pixel_flow_max, render

KAPPA1 = 2.0e3
KAPPA2 = 2.0e4

DOM_LARGEST = 0
DOM_PRINTED = 1


@dataclass
class Params:
    max_flow: float
    gamma: tuple
    smooth_iters: int = 2
    sigma: float = 0.5
    dominant_rule: int = DOM_LARGEST
    clamp_advection: int = 1
    input_is_inverse_depth: int = 0
    omega: tuple | None = None  # camera angular velocity (rad/frame) for the inertial terms (NEXT #4)
    accel: tuple | None = None  # camera linear acceleration (per frame^2)

    @property
    def N(self) -> int:
        """Substep count N = ceil(max_flow), PAPER.md L684-689 (eq:numerical_stability)."""
        return max(1, int(math.ceil(self.max_flow)))


def default_params(geom: np.ndarray, max_flow: float, smooth_iters: int = 2, **kw) -> Params:
    ds = _grid.center_ds(geom)
    g = np.array([KAPPA1 / ds ** 2, KAPPA2 / ds ** 2, 1.0, 1.0, 1.0], dtype=np.float32)
    return Params(max_flow=float(np.float32(max_flow)), gamma=tuple(float(x) for x in g),
                  smooth_iters=smooth_iters, **kw)


# ----------------------------------------------------------------------------- scenes

def _scene_plane_sphere(rng):
    objs = [
        Plane(np.array([0.0, 0.0, 6.0]), np.array([0.0, 0.0, 1.0]), Texture.random(rng, 1.5)),
        Sphere(np.array([0.6, -0.3, 4.0]), 0.8, Texture.random(rng, 2.0), np.array([-0.6, 0.2, -0.1])),
    ]
    v = np.array([1.0, 0.3, 0.25])
    return Scene(objs, rng.uniform(-0.01, 0.01, 3), v / np.linalg.norm(v))


def _scene_highspeed(rng):
    objs = [
        Plane(np.array([0.0, 1.5, 0.0]), np.array([0.0, 1.0, 0.0]), Texture.random(rng, 1.0)),
        Plane(np.array([-4.0, 0.0, 0.0]), np.array([1.0, 0.0, 0.0]), Texture.random(rng, 1.0)),
        Plane(np.array([4.0, 0.0, 0.0]), np.array([1.0, 0.0, 0.0]), Texture.random(rng, 1.0)),
        Plane(np.array([0.0, 0.0, 40.0]), np.array([0.0, 0.0, 1.0]), Texture.random(rng, 0.5)),
        Sphere(np.array([-1.0, 0.5, 8.0]), 1.0, Texture.random(rng, 2.0), np.array([0.4, 0.0, 0.2])),
        Sphere(np.array([1.5, -0.5, 12.0]), 1.5, Texture.random(rng, 2.0), np.array([-0.3, 0.1, -0.5])),
    ]
    v = np.array([0.3, 0.0, 1.0])
    return Scene(objs, rng.uniform(-0.01, 0.01, 3), v / np.linalg.norm(v))


def _scene_driving(rng):
    objs = [
        Plane(np.array([0.0, 1.5, 0.0]), np.array([0.0, 1.0, 0.0]), Texture.random(rng, 1.0)),
        Plane(np.array([-6.0, 0.0, 0.0]), np.array([1.0, 0.0, 0.0]), Texture.random(rng, 1.0)),
        Plane(np.array([6.0, 0.0, 0.0]), np.array([1.0, 0.0, 0.0]), Texture.random(rng, 1.0)),
        Plane(np.array([0.0, 0.0, 100.0]), np.array([0.0, 0.0, 1.0]), Texture.random(rng, 0.3)),
        Sphere(np.array([-2.5, 0.5, 15.0]), 1.0, Texture.random(rng, 2.0), np.array([0.0, 0.0, 0.5])),
        Sphere(np.array([2.5, 0.5, 25.0]), 1.0, Texture.random(rng, 2.0), np.array([0.0, 0.0, -0.8])),
        Sphere(np.array([0.0, 0.5, 40.0]), 1.0, Texture.random(rng, 2.0), np.array([0.2, 0.0, 0.3])),
    ]
    v = np.array([0.05, 0.0, 1.0])
    return Scene(objs, rng.uniform(-0.01, 0.01, 3), v / np.linalg.norm(v))


SCENES = {"plane_sphere": _scene_plane_sphere, "highspeed": _scene_highspeed, "driving": _scene_driving}

# BASELINE.json "configs", in order (index 0 is configs[0], the oracle-in-seconds case).
CONFIGS = {
    1: dict(H=64, W=64, fov=60.0, max_flow=2.0, frames=10, seed=1, scene="plane_sphere"),
    2: dict(H=512, W=512, fov=90.0, max_flow=8.0, frames=100, seed=2, scene="highspeed"),
    3: dict(H=1024, W=1024, fov=90.0, max_flow=16.0, frames=100, seed=3, scene="driving"),
    4: dict(H=512, W=512, fov=90.0, max_flow=8.0, frames=10, seed=100, scene="highspeed", batch=64),
    5: dict(H=8192, W=8192, fov=90.0, max_flow=8.0, frames=3, seed=5, scene="driving"),
}


@dataclass
class Sequence:
    geom: np.ndarray  # [H][W][10] float32
    Y: np.ndarray  # [F][H][W] float32
    depth: np.ndarray  # [F][H][W] float32
    w_gt: np.ndarray | None  # [F][H][W][3] float32
    params: Params
    scene: Scene
    fov: float = 0.0


MAX_NORMAL_RATE = 0.02  # |<s, w_gt>| <= 2 % depth change per frame (time to contact >= 50 frames)


def make_scene(name: str, seed: int, geom64: np.ndarray, max_flow: float, frames: int = 1,
               target: float = 0.9, subsampled: bool = False) -> Scene:
    """Scene with velocities scaled (bisection) so that, over frames 0 and F-1, the peak
    ground-truth tangent flow is target*max_flow pixels, or the peak normal rate
    |<s, w_gt>| is MAX_NORMAL_RATE per frame, whichever binds first."""
    rng = np.random.default_rng(seed)
    base = SCENES[name](rng)
    # render at reduced resolution for the scale search (per-pixel ds keeps the flow in full-res px)
    if subsampled:
        g = geom64
    else:
        step = max(1, min(geom64.shape[0], geom64.shape[1]) // 128)
        g = geom64[::step, ::step]
    def peak(a):
        sc = base.scaled(a)
        r = 0.0
        for k in sorted({0, frames - 1}):
            w = render(sc, g[..., 0:3], float(k))[2].astype(np.float64)
            normal = float(np.max(np.abs(np.sum(g[..., 0:3] * w, axis=-1))))
            r = max(r, pixel_flow_max(g, w) / (target * max_flow), normal / MAX_NORMAL_RATE)
        return r

    # frame-0 flow is linear in a; later frames grow faster (approaching objects): bisect
    hi = target * max_flow / pixel_flow_max(g, render(base, g[..., 0:3], 0.0)[2])
    lo = 0.0
    for _ in range(30):
        mid = 0.5 * (lo + hi)
        if peak(mid) > 1.0:
            hi = mid
        else:
            lo = mid
    return base.scaled(lo)


def make_sequence(H: int, W: int, fov: float, max_flow: float, frames: int, seed: int, scene: str,
                  with_gt: bool = False, smooth_iters: int = 2, **_ignored) -> Sequence:
    geom64 = _grid.gnomonic(H, W, fov, as_f64=True)
    geom = geom64.astype(np.float32)
    sc = make_scene(scene, seed, geom64, max_flow, frames)
    Ys, Ds, Ws = [], [], []
    for k in range(frames):
        y, d, w = render(sc, geom64[..., 0:3], float(k))
        Ys.append(y)
        Ds.append(d)
        if with_gt:
            Ws.append(w)
    return Sequence(geom, np.stack(Ys), np.stack(Ds), np.stack(Ws) if with_gt else None,
                    default_params(geom, max_flow, smooth_iters), sc, fov)


def band_sequence(cid: int, r0: int, r1: int, frames: int, seed: int | None = None):
    """Rows [r0, r1) of config `cid`'s sequence (same scene and speed scale as the whole grid),
    generated without the whole grid: the 8192^2 row-band config.  Returns (geom, Y, depth, params)."""
    c = dict(CONFIGS[cid])
    H, W = c["H"], c["W"]
    step = max(1, min(H, W) // 128)
    gsub = _grid.gnomonic_rows(H, W, c["fov"], 0, H, as_f64=True, col_step=step, row_step=step)
    sc = make_scene(c["scene"], c["seed"] if seed is None else seed, gsub, c["max_flow"], frames, subsampled=True)
    # row chunks keep the float64 working set small at 8192^2
    geom = np.empty((r1 - r0, W, 10), np.float32)
    Ys = np.empty((frames, r1 - r0, W), np.float32)
    Ds = np.empty((frames, r1 - r0, W), np.float32)
    for a in range(r0, r1, 256):
        b = min(r1, a + 256)
        g64 = _grid.gnomonic_rows(H, W, c["fov"], a, b, as_f64=True)
        geom[a - r0:b - r0] = g64
        for k in range(frames):
            y, d, _ = render(sc, g64[..., 0:3], float(k))
            Ys[k, a - r0:b - r0] = y
            Ds[k, a - r0:b - r0] = d
    # gains from the centre pixel of the whole grid (default_params reads the centre of the geometry)
    centre = _grid.gnomonic_rows(H, W, c["fov"], H // 2, H // 2 + 1, col_step=1)[0:1, W // 2:W // 2 + 1]
    params = default_params(centre, c["max_flow"])
    return geom, Ys, Ds, params


def config_sequence(cid: int, frames: int | None = None, H: int | None = None, W: int | None = None,
                    seed: int | None = None, with_gt: bool = False, max_flow: float | None = None) -> Sequence:
    c = dict(CONFIGS[cid])
    if max_flow is not None:
        c["max_flow"] = max_flow
    if frames is not None:
        c["frames"] = frames
    if H is not None:
        c["H"] = H
    if W is not None:
        c["W"] = W
    if seed is not None:
        c["seed"] = seed
    return make_sequence(with_gt=with_gt, **c)
