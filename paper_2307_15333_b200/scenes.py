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


# ---------------------------------------------------------------------------
# Adaptive builds for the large configurations (torch, runs on the GPU)

def _field_torch(field: BlobField, pts):
    import torch
    mu = torch.as_tensor(field.mu, dtype=torch.float64, device=pts.device)
    inv = torch.as_tensor(1.0 / (2.0 * field.s ** 2), dtype=torch.float64, device=pts.device)
    p = torch.as_tensor(field.p, dtype=torch.float64, device=pts.device)
    out = torch.zeros(pts.shape[0], dtype=torch.float64, device=pts.device)
    for lo in range(0, mu.shape[0], 16):
        d = pts[:, None, :] - mu[None, lo:lo + 16, :]
        q = (d * d * inv[None, lo:lo + 16, :]).sum(-1)
        out += (p[None, lo:lo + 16] * torch.exp(-q)).sum(-1)
    if field.slab is not None:
        z_top, thick, dens = field.slab
        inside = (pts[:, 2] <= z_top) & (pts[:, 2] >= z_top - thick)
        out = out + inside.double() * dens
    return out


def adaptive_tree(field: BlobField, max_depth: int, basis_count: int, split_thr: float,
                  empty_thr: float = 0.05, min_depth: int = 3, half_extent: float = 1.0,
                  sh_seed: int = 0, sh_std: float = 0.3, device=None, chunk: int = 1 << 21):
    """Top-down adaptive octree over a blob field, built level by level.

    A cell at depth d < max_depth splits when d < min_depth, or when the
    density sampled at its centre and its 8 child centres spans more than
    ``split_thr * h_child`` (a finite-difference gradient bound, so refinement
    tracks the field's steep shells at every depth) and exceeds ``empty_thr``
    somewhere (refinement follows the
    field's variation, like a trained radiance field around surfaces).  Leaf
    sigma is the density at the leaf centre (build_dense's convention,
    octree.py:431-445); SH ~ N(0, sh_std) in canonical leaf order.  Returns a
    canonical ``SparseOctree`` (pool id == BFS index) on ``device``.
    """
    import torch
    from .octree import OCTANT_SIGNS, from_canonical_tensors
    dev = torch.device(device) if device is not None else (
        torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu"))
    signs = torch.as_tensor(OCTANT_SIGNS, dtype=torch.float64, device=dev)
    centers = torch.zeros(1, 3, dtype=torch.float64, device=dev)
    sig = _field_torch(field, centers)
    levels = []  # (split mask, sigma) per level
    h = half_extent
    for d in range(max_depth + 1):
        m = centers.shape[0]
        if d == max_depth or m == 0:
            levels.append((torch.zeros(m, dtype=torch.bool, device=dev), sig))
            break
        hc = h * 0.5
        split = torch.empty(m, dtype=torch.bool, device=dev)
        csig = torch.empty(m, 8, dtype=torch.float64, device=dev)
        for lo in range(0, m, chunk):
            c = centers[lo:lo + chunk]
            cc = (c[:, None, :] + hc * signs[None, :, :]).reshape(-1, 3)
            s8 = _field_torch(field, cc).reshape(-1, 8)
            csig[lo:lo + chunk] = s8
            allv = torch.cat([sig[lo:lo + chunk, None], s8], dim=1)
            mx, mn = allv.max(1).values, allv.min(1).values
            split[lo:lo + chunk] = ((mx - mn) > split_thr * hc) & (mx > empty_thr)
        if d < min_depth:
            split[:] = True
        levels.append((split, sig))
        sel = torch.nonzero(split).reshape(-1)
        centers = (centers[sel][:, None, :] + hc * signs[None, :, :]).reshape(-1, 3)
        sig = csig[sel].reshape(-1)
        h = hc
    # canonical node table
    sizes = [lv[0].shape[0] for lv in levels]
    starts = [0]
    for s_ in sizes:
        starts.append(starts[-1] + s_)
    n = starts[-1]
    node = torch.empty(n, dtype=torch.int32, device=dev)
    sigma = torch.zeros(n, dtype=torch.float32, device=dev)
    for d, (split, s_) in enumerate(levels):
        lo, hi = starts[d], starts[d + 1]
        rank = torch.cumsum(split.long(), 0) - split.long()
        idx = torch.arange(lo, hi, device=dev)
        nxt = starts[d + 1]
        node[lo:hi] = torch.where(split, (nxt + 8 * rank).int(), (~idx).int())
        sigma[lo:hi] = torch.where(split, torch.zeros_like(s_), s_).float()
    leaf = node < 0
    n_leaf = int(leaf.sum().item())
    S = pad4_(3 * basis_count)
    sh = torch.zeros(n, S, dtype=torch.float32, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(int(sh_seed))
    vals = torch.randn(n_leaf, 3 * basis_count, generator=g, device=dev, dtype=torch.float32) * sh_std
    sh[torch.nonzero(leaf).reshape(-1), :3 * basis_count] = vals
    return from_canonical_tensors((0.0, 0.0, 0.0), half_extent, basis_count, max_depth, node,
                                  sigma, sh, level_offsets=np.asarray(starts, dtype=np.int64))


def pad4_(n: int) -> int:
    return (n + 3) & ~3


def config2_scene(device=None, basis_count: int = 16):
    """BASELINE.json configs[1]/[2]: depth-9, 64-blob field, SH-3, ~2-3M leaves."""
    field = BlobField.make(seed=2, n_blobs=64)
    return adaptive_tree(field, max_depth=9, basis_count=basis_count, split_thr=CONFIG2_SPLIT_THR,
                         empty_thr=0.05, min_depth=4, sh_seed=20, device=device)


CONFIG2_SPLIT_THR = 800.0  # -> 2.62M leaves, 3.0M nodes (tools/tune_scenes.py)


def config4_field() -> BlobField:
    """BASELINE.json configs[3]: 256 anisotropic blobs over the 2x bbox plus a
    dense ground slab whose underside is the bbox floor (so only its top face
    is a density discontinuity)."""
    return BlobField.make(seed=4, n_blobs=256, anisotropic=True, scale=2.0, slab=(-1.5, 0.5, 30.0))


def config4_scene(device=None, basis_count: int = 16, split_thr: float | None = None):
    """BASELINE.json configs[3] (Tanks&Temples-shaped): depth 10 over [-2, 2]^3, SH-3, ~8M leaves."""
    return adaptive_tree(config4_field(), max_depth=10, basis_count=basis_count,
                         split_thr=CONFIG4_SPLIT_THR if split_thr is None else split_thr,
                         empty_thr=0.05, min_depth=4, half_extent=2.0, sh_seed=40, device=device)


CONFIG4_SPLIT_THR = 1000.0  # -> 8.52M leaves, 9.74M nodes (tools/tune_c4.py; 2000 stops at depth 4)


def ring_cameras(count: int, width: int, height: int, radius: float, seed: int,
                 elevation_jitter_deg: float = 15.0, camera_angle_x: float = FOV_40):
    """Cameras on a ring around the origin at +/- jittered elevation (configs[3])."""
    rng = np.random.default_rng(seed)
    focal = focal_from_angle(width, camera_angle_x)
    poses = []
    for i in range(count):
        az = 2.0 * math.pi * i / count
        el = math.radians(rng.uniform(-elevation_jitter_deg, elevation_jitter_deg))
        poses.append(orbit_pose(radius, az, el))
    return focal, poses


def hemisphere_cameras(count: int, width: int, height: int, radius: float, seed: int,
                       camera_angle_x: float = FOV_40):
    """Cameras on the upper hemisphere looking at the origin (NeRF-synthetic-shaped)."""
    rng = np.random.default_rng(seed)
    focal = focal_from_angle(width, camera_angle_x)
    poses = []
    for _ in range(count):
        az = rng.uniform(0.0, 2.0 * math.pi)
        el = math.asin(rng.uniform(0.05, 0.95))
        poses.append(orbit_pose(radius, az, el))
    return focal, poses
