"""Seeded synthetic scenes: a small ray caster producing brightness Y, depth lambda
and ground-truth structure flow w_gt on a grid (input data, not the method).

Stand-in for the paper's Blender Urban Canyon renders (out of
scope here).  Camera and objects translate at constant velocity (the paper's
kinematic assumptions, L142-158; no rotation, so Omega = 0), textures are solid
sums of sinusoids attached to each object (brightness constancy holds exactly,
L302-308), and the ground truth is eq:homogeneous_flow (L194-198) with
Omega = 0:  w_gt = (v_x - v_c) / lambda, in radians per frame.

All geometry is float64; outputs are rounded once to float32.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Texture:
    freqs: np.ndarray  # [K][3] rad/m
    phases: np.ndarray  # [K]
    amps: np.ndarray  # [K]

    @staticmethod
    def random(rng: np.random.Generator, scale: float = 1.0, k: int = 3) -> "Texture":
        # incommensurate frequencies in random directions, wavelengths ~ 0.5 .. 3 m
        dirs = rng.normal(size=(k, 3))
        dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
        mags = rng.uniform(2.0, 9.0, size=k) * scale
        return Texture(dirs * mags[:, None], rng.uniform(0, 2 * np.pi, size=k), rng.uniform(0.5, 1.0, size=k))

    def eval(self, local: np.ndarray) -> np.ndarray:
        acc = np.zeros(local.shape[:-1])
        for f, ph, a in zip(self.freqs, self.phases, self.amps):
            acc += a * np.sin(local @ f + ph)
        return 0.5 + 0.4 * acc / np.sum(np.abs(self.amps))


@dataclass
class Plane:
    point: np.ndarray
    normal: np.ndarray
    tex: Texture
    vel: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def intersect(self, cam, d, k):
        p = self.point + k * self.vel
        n = self.normal
        den = d @ n
        with np.errstate(divide="ignore", invalid="ignore"):
            t = ((p - cam) @ n) / den
        t = np.where((np.abs(den) > 1e-12) & (t > 1e-6), t, np.inf)
        return t

    def origin(self, k):
        return self.point + k * self.vel


@dataclass
class Sphere:
    center: np.ndarray
    radius: float
    tex: Texture
    vel: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def intersect(self, cam, d, k):
        c = self.center + k * self.vel
        oc = cam - c
        b = d @ oc
        cc = oc @ oc - self.radius ** 2
        disc = b * b - cc
        with np.errstate(invalid="ignore"):
            sq = np.sqrt(np.maximum(disc, 0.0))
        t = -b - sq
        t = np.where((disc >= 0) & (t > 1e-6), t, np.inf)
        return t

    def origin(self, k):
        return self.center + k * self.vel


@dataclass
class Scene:
    objects: list
    cam_pos0: np.ndarray
    cam_vel: np.ndarray  # metres per frame
    sky_brightness: float = 0.5

    def scaled(self, a: float) -> "Scene":
        """Same scene with every velocity multiplied by a (w_gt scales by a)."""
        objs = []
        for o in self.objects:
            if isinstance(o, Plane):
                objs.append(Plane(o.point, o.normal, o.tex, o.vel * a))
            else:
                objs.append(Sphere(o.center, o.radius, o.tex, o.vel * a))
        return Scene(objs, self.cam_pos0, self.cam_vel * a, self.sky_brightness)


def render(scene: Scene, dirs: np.ndarray, k: float, row_block: int = 256):
    """Render frame k: returns (Y, depth, w_gt) float32 of shapes [H][W], [H][W], [H][W][3].

    Rays with no hit get Y = sky_brightness, depth = +inf (an invalid measurement)
    and w_gt = 0.
    """
    H, W, _ = dirs.shape
    Y = np.empty((H, W), np.float32)
    D = np.empty((H, W), np.float32)
    Wg = np.empty((H, W, 3), np.float32)
    cam = scene.cam_pos0 + k * scene.cam_vel
    for r0 in range(0, H, row_block):
        d = dirs[r0:r0 + row_block]
        best = np.full(d.shape[:-1], np.inf)
        idx = np.full(d.shape[:-1], -1, np.int32)
        for oi, o in enumerate(scene.objects):
            t = o.intersect(cam, d, k)
            m = t < best
            best = np.where(m, t, best)
            idx = np.where(m, oi, idx)
        y = np.full(best.shape, scene.sky_brightness)
        wg = np.zeros(best.shape + (3,))
        for oi, o in enumerate(scene.objects):
            m = idx == oi
            if not np.any(m):
                continue
            t = best[m]
            X = cam + t[:, None] * d[m]
            y[m] = o.tex.eval(X - o.origin(k))
            wg[m] = (o.vel - scene.cam_vel)[None, :] / t[:, None]
        Y[r0:r0 + row_block] = y
        D[r0:r0 + row_block] = best
        Wg[r0:r0 + row_block] = wg
    return Y, D, Wg


def camera_directions(Hc: int, Wc: int, K) -> np.ndarray:
    """Unit ray directions [Hc][Wc][3] (float64) of a pinhole camera with intrinsics
    K = (fx, fy, cx, cy), pixel centres at integer coordinates, looking along +z."""
    fx, fy, cx, cy = (float(x) for x in K)
    u = (np.arange(Wc, dtype=np.float64) - cx) / fx
    v = (np.arange(Hc, dtype=np.float64) - cy) / fy
    U, V = np.meshgrid(u, v)
    d = np.stack([U, V, np.ones_like(U)], -1)
    return d / np.linalg.norm(d, axis=-1, keepdims=True)


def render_camera(scene: "Scene", Hc: int, Wc: int, K, k: float):
    """Frame k as a pinhole camera sees it: brightness [Hc][Wc] and z-DEPTH [Hc][Wc] (range
    times the ray's z component; +inf where the ray hits nothing), float32."""
    d = camera_directions(Hc, Wc, K)
    Y, rng, _ = render(scene, d, k)
    Z = (rng.astype(np.float64) * d[..., 2]).astype(np.float32)
    return Y, Z


def pixel_flow_max(geom64: np.ndarray, w: np.ndarray, margin: int = 0) -> float:
    """max over pixels of the tangent flow in pixels, |(b1.w, b2.w)| / ds."""
    b1 = geom64[..., 3:6]
    b2 = geom64[..., 6:9]
    ds = geom64[..., 9]
    w = w.astype(np.float64)
    u = np.sum(b1 * w, axis=-1) / ds
    v = np.sum(b2 * w, axis=-1) / ds
    f = np.hypot(u, v)
    if margin:
        f = f[margin:-margin, margin:-margin]
    return float(np.max(f))
