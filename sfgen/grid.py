"""Spherepix-style grid geometry (input data, not the method).

The paper defers grid construction to the Spherepix data structure
(section "Spherical image data structure"): per pixel a unit
direction s_ij, a 3x2 basis B = [b1 b2] whose columns are the normalised
tangent-plane projections of the (i, j+1) and (i+1, j) neighbours (L430), and a
pixel separation Delta s_ij = ||P(s_ij) s_{i,j+1}|| (L437).  How the patch is laid
out is not given; we use a single gnomonic (perspective) patch, the reading in
SURVEY.md section 8(c)-6 / SPEC.md L39-47.

Everything here is float64 and is rounded ONCE to float32 at the end.  The
output layout (shared verbatim by the oracle and the CUDA library, both of which
derive their own working quantities from it) is

    geom[H][W][10] float32 = (s.x, s.y, s.z, b1.x, b1.y, b1.z, b2.x, b2.y, b2.z, ds)

No step of the filter's arithmetic lives in this module.
"""
from __future__ import annotations

import numpy as np

GEOM_CHANNELS = 10


def _normalize(v: np.ndarray) -> np.ndarray:
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def _tangent_project(s: np.ndarray, x: np.ndarray) -> np.ndarray:
    """P(s) x = x - s <s, x>  (eq:tmatrix)."""
    return x - s * np.sum(s * x, axis=-1, keepdims=True)


def directions_gnomonic(H: int, W: int, fov_deg: float, rows=None, cols=None) -> np.ndarray:
    """Unit directions of a gnomonic patch, square pixels, horizontal FOV = fov_deg.

    Pixel (i, j) looks through the image-plane point ((j - (W-1)/2) p, (i - (H-1)/2) p, 1)
    with pitch p = 2 tan(fov/2) / W.  The centre of the patch is the optical axis +z.
    rows / cols: optional integer index arrays (a sub-grid of the H x W patch).
    """
    if not (0.0 < fov_deg < 180.0):
        raise ValueError("fov_deg must be in (0, 180)")
    if H < 2 or W < 2:
        raise ValueError("grid must be at least 2x2")
    p = 2.0 * np.tan(np.radians(fov_deg) / 2.0) / W
    jj = np.arange(W, dtype=np.float64) if cols is None else np.asarray(cols, dtype=np.float64)
    ii = np.arange(H, dtype=np.float64) if rows is None else np.asarray(rows, dtype=np.float64)
    x = (jj - (W - 1) / 2.0) * p
    y = (ii - (H - 1) / 2.0) * p
    X, Y = np.meshgrid(x, y)
    v = np.stack([X, Y, np.ones_like(X)], axis=-1)
    return _normalize(v)


def geometry_from_directions(s: np.ndarray) -> np.ndarray:
    """Build (s, b1, b2, ds) in float64 from a [H][W][3] direction field.

    b1 = normalize(P(s) s_{i,j+1}); the last column uses -P(s) s_{i,j-1} (mirrored
    backward neighbour).  b2 = Gram-Schmidt of P(s) s_{i+1,j} against b1,
    normalised (last row mirrored).  ds = ||P(s) s_{i,j+1}||.
    """
    H, W, _ = s.shape
    nb1 = np.empty_like(s)
    nb1[:, :-1] = s[:, 1:]
    mu1 = np.empty_like(s)
    mu1[:, :-1] = _tangent_project(s[:, :-1], nb1[:, :-1])
    mu1[:, -1] = -_tangent_project(s[:, -1], s[:, -2])
    ds = np.linalg.norm(mu1, axis=-1)
    b1 = mu1 / ds[..., None]

    mu2 = np.empty_like(s)
    mu2[:-1] = _tangent_project(s[:-1], s[1:])
    mu2[-1] = -_tangent_project(s[-1], s[-2])
    mu2 = mu2 - b1 * np.sum(mu2 * b1, axis=-1, keepdims=True)
    b2 = _normalize(mu2)
    return np.concatenate([s, b1, b2, ds[..., None]], axis=-1)


def gnomonic(H: int, W: int, fov_deg: float, as_f64: bool = False) -> np.ndarray:
    """GNOMONIC grid geometry [H][W][10], float32 (or the float64 original)."""
    g = geometry_from_directions(directions_gnomonic(H, W, fov_deg))
    return g if as_f64 else g.astype(np.float32)


def gnomonic_rows(H: int, W: int, fov_deg: float, r0: int, r1: int, as_f64: bool = False,
                  col_step: int = 1, row_step: int = 1) -> np.ndarray:
    """Rows [r0, r1) (every row_step-th, every col_step-th column) of the H x W GNOMONIC grid,
    identical to gnomonic(H, W, fov)[r0:r1:row_step, ::col_step] but computed without the whole grid
    (row bands of the 8192^2 config, subsampled scale searches)."""
    rows = np.arange(r0, r1, row_step)
    cols = np.arange(0, W, col_step)
    s = directions_gnomonic(H, W, fov_deg, rows, cols)
    # neighbours: (i, j+1) (mirrored (i, j-1) on the last column) and (i+1, j) (mirrored on the last row)
    cn = np.where(cols < W - 1, cols + 1, cols - 1)
    rn = np.where(rows < H - 1, rows + 1, rows - 1)
    sc = directions_gnomonic(H, W, fov_deg, rows, cn)
    sr = directions_gnomonic(H, W, fov_deg, rn, cols)
    sign_c = np.where(cols < W - 1, 1.0, -1.0)[None, :, None]
    sign_r = np.where(rows < H - 1, 1.0, -1.0)[:, None, None]
    mu1 = sign_c * _tangent_project(s, sc)
    ds = np.linalg.norm(mu1, axis=-1)
    b1 = mu1 / ds[..., None]
    mu2 = sign_r * _tangent_project(s, sr)
    mu2 = mu2 - b1 * np.sum(mu2 * b1, axis=-1, keepdims=True)
    b2 = _normalize(mu2)
    g = np.concatenate([s, b1, b2, ds[..., None]], axis=-1)
    return g if as_f64 else g.astype(np.float32)


def gnomonic_pyramid(H: int, W: int, fov_deg: float, levels: int = 2) -> list:
    """Spherepix pyramid of a GNOMONIC patch: level h has (H / 2^(h-1)) x (W / 2^(h-1)) pixels and
    the same field of view, so a coarse pixel's direction is its 2 x 2 block centre (the image-plane
    points are affine in the pixel index).  Returns [level 1, level 2, ...] float32 geometries."""
    out = []
    for h in range(levels):
        if H % (1 << h) or W % (1 << h):
            raise ValueError("grid size must be divisible by 2^(levels-1)")
        out.append(gnomonic(H >> h, W >> h, fov_deg))
    return out


def flat(H: int, W: int, ds: float = 2.0 ** -8) -> np.ndarray:
    """FLAT test grid: s = e_z, b1 = e_x, b2 = e_y, constant ds (SURVEY 8(c) pin C2).

    Not a sphere patch: every pixel shares one tangent plane, which turns the
    filter's transport step into the textbook 2-D first-order upwind scheme.
    """
    g = np.zeros((H, W, GEOM_CHANNELS), dtype=np.float32)
    g[..., 2] = 1.0
    g[..., 3] = 1.0
    g[..., 7] = 1.0
    g[..., 9] = ds
    return g


def center_ds(geom: np.ndarray) -> float:
    H, W, _ = geom.shape
    return float(geom[H // 2, W // 2, 9])


def split(geom: np.ndarray):
    """Views (s, b1, b2, ds) of a geometry array."""
    return geom[..., 0:3], geom[..., 3:6], geom[..., 6:9], geom[..., 9]
