"""Seeded synthetic scenes for the benchmark configurations (BASELINE.json).

The reference ships no scene generator for these configurations, so this
module defines them:

* a Gaussian blob density field ``rho(x) = sum_j p_j exp(-|x-mu_j|^2 / (2 s_j^2))``
  with ``mu ~ U[-0.6, 0.6]^3``, ``s ~ U(0.05, 0.2)``, ``p ~ U(10, 50)`` drawn
  from ``np.random.default_rng(seed)`` (anisotropic per-axis ``s`` and an
  optional ground slab for the Tanks&Temples-shaped config 4);
* config 1: ``build_dense(5)`` with sigma sampled at leaf centres, then the
  reference's recursive density prune at tau = 0.1, SH ~ N(0, 0.3) drawn in
  canonical leaf order.  ``tests/golden`` pins the resulting ``.dot1`` bytes
  against the reference's own ``build_dense`` + ``prune`` + ``save_tree``;
* configs 2-5: an adaptive top-down build (below) because a dense depth-9/10
  build is 134M-1G leaves.

Everything here is host-side numpy and runs once per scene.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass
class BlobField:
    mu: np.ndarray      # (n, 3)
    s: np.ndarray       # (n, 3) per-axis widths (isotropic: equal columns)
    p: np.ndarray       # (n,)
    slab: tuple | None = None   # (z_top, thickness, density) ground slab

    @classmethod
    def make(cls, seed: int, n_blobs: int, anisotropic: bool = False, scale: float = 1.0,
             slab: tuple | None = None) -> "BlobField":
        rng = np.random.default_rng(seed)
        mu = rng.uniform(-0.6, 0.6, (n_blobs, 3)) * scale
        if anisotropic:
            s = rng.uniform(0.05, 0.2, (n_blobs, 3)) * scale
        else:
            s = np.repeat(rng.uniform(0.05, 0.2, n_blobs)[:, None], 3, axis=1) * scale
        p = rng.uniform(10.0, 50.0, n_blobs)
        return cls(mu, s, p, slab)

    def sigma_exact(self, points: np.ndarray) -> np.ndarray:
        """Density with scalar libm exp, summed blob by blob in index order.

        Bit-reproducible on any host (numpy's SIMD exp may differ in the last
        ulp between CPUs); used for the pinned config-1 scene.
        """
        pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
        out = np.zeros(pts.shape[0])
        mexp = np.frompyfunc(math.exp, 1, 1)
        for j in range(self.p.shape[0]):
            d = pts - self.mu[j]
            q = (d[:, 0] * d[:, 0]) / (2.0 * self.s[j, 0] ** 2) \
                + (d[:, 1] * d[:, 1]) / (2.0 * self.s[j, 1] ** 2) \
                + (d[:, 2] * d[:, 2]) / (2.0 * self.s[j, 2] ** 2)
            out = out + self.p[j] * mexp(-q).astype(np.float64)
        return out + self._slab(pts)

    def sigma_fast(self, points: np.ndarray) -> np.ndarray:
        """Vectorised density (numpy exp); used for the large adaptive builds."""
        pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
        out = np.zeros(pts.shape[0])
        inv = 1.0 / (2.0 * self.s ** 2)
        for j in range(self.p.shape[0]):
            d = pts - self.mu[j]
            q = d[:, 0] * d[:, 0] * inv[j, 0] + d[:, 1] * d[:, 1] * inv[j, 1] \
                + d[:, 2] * d[:, 2] * inv[j, 2]
            m = q < 40.0
            if m.any():
                out[m] += self.p[j] * np.exp(-q[m])
        return out + self._slab(pts)

    def _slab(self, pts):
        if self.slab is None:
            return 0.0
        z_top, thick, dens = self.slab
        inside = (pts[:, 2] <= z_top) & (pts[:, 2] >= z_top - thick)
        return np.where(inside, dens, 0.0)


def config1_field() -> BlobField:
    """8 isotropic blobs, seed 1 (BASELINE.json configs[0])."""
    return BlobField.make(seed=1, n_blobs=8)


def orbit_pose(radius: float, azimuth: float, elevation: float) -> np.ndarray:
    """cam_to_world for a camera on a sphere looking at the origin (z up).

    Same construction as the reference's look_at (scene_io.py:94-113):
    back = normalised(eye), right = up x back, up' = back x right.
    """
    eye = radius * np.array([math.cos(elevation) * math.cos(azimuth),
                             math.cos(elevation) * math.sin(azimuth),
                             math.sin(elevation)])
    back = eye / np.linalg.norm(eye)
    right = np.cross(np.array([0.0, 0.0, 1.0]), back)
    if np.linalg.norm(right) < 1e-9:
        right = np.cross(np.array([0.0, 1.0, 0.0]), back)
    right /= np.linalg.norm(right)
    up = np.cross(back, right)
    m = np.eye(4)
    m[:3, 0] = right
    m[:3, 1] = up
    m[:3, 2] = back
    m[:3, 3] = eye
    return m


CONFIG1_POSE = dict(radius=4.0, azimuth=0.7, elevation=0.4)
FOV_40 = 0.6981317  # camera_angle_x for a 40 degree horizontal fov


def focal_from_angle(width: int, camera_angle_x: float) -> float:
    return 0.5 * width / math.tan(0.5 * camera_angle_x)


def pinhole_rays(width: int, height: int, focal: float, cam_to_world: np.ndarray):
    """Unit world rays through pixel centres, row-major (scene_io.py:77-91)."""
    xs = (np.arange(width, dtype=np.float64) + 0.5 - 0.5 * width) / focal
    ys = -(np.arange(height, dtype=np.float64) + 0.5 - 0.5 * height) / focal
    cam = np.empty((height, width, 3), dtype=np.float64)
    cam[..., 0] = xs[None, :]
    cam[..., 1] = ys[:, None]
    cam[..., 2] = -1.0
    world = cam.reshape(-1, 3) @ cam_to_world[:3, :3].T
    world /= np.linalg.norm(world, axis=1, keepdims=True)
    origins = np.broadcast_to(cam_to_world[:3, 3], world.shape).copy()
    return origins, world
