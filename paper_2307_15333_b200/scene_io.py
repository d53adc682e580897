"""Cameras and the ``.dot1`` tree container.

* ``Camera`` / ``look_at`` / ``orbit_cameras`` / ``focal_from_angle`` follow
  /root/reference/pkg/src/octrf/scene_io.py:42-133 (pixel centres
  ((x+0.5-W/2)/f, -(y+0.5-H/2)/f, -1), rotated, normalised, row-major).
* ``save_tree`` / ``load_tree`` read and write the reference's byte format
  (scene_io.py:524-681): ``b"DOT1"`` + ``<III6dQ`` header (version, B,
  max_depth, lo[3], hi[3], node_count), BFS-ordered records (leaf:
  ``0x01`` + f32 sigma + f32 SH[3B]; internal: ``0x00`` + 8 x u64 child
  indices) and a CRC32 trailer verified before anything is parsed.
  Writing is vectorised from the canonical device layout; loading yields a
  canonical tree (pool id == BFS index) exactly like the reference's loader.
"""

from __future__ import annotations

import math
import struct
import zlib
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import (
    BadMagicError,
    BadVersionError,
    ChecksumError,
    ConfigError,
    InputError,
    StructureError,
    TreeFileError,
)
from .octree import VALID_BASIS_COUNTS

TREE_MAGIC = b"DOT1"
TREE_VERSION = 1
_HEADER = struct.Struct("<III6dQ")
_CRC = struct.Struct("<I")


def focal_from_angle(width: int, camera_angle_x: float) -> float:
    return 0.5 * width / math.tan(0.5 * camera_angle_x)


@dataclass(frozen=True, eq=False)
class Camera:
    """Pinhole camera looking down its local -z axis."""

    width: int
    height: int
    focal: float
    cam_to_world: np.ndarray

    def __post_init__(self) -> None:
        mat = np.asarray(self.cam_to_world, dtype=np.float64)
        if mat.shape != (4, 4):
            raise InputError(f"cam_to_world must be 4x4, got {mat.shape}")
        object.__setattr__(self, "cam_to_world", mat.copy())
        if self.width < 1 or self.height < 1:
            raise InputError("image dimensions must be positive")
        if not (math.isfinite(self.focal) and self.focal > 0):
            raise InputError(f"focal must be positive, got {self.focal}")
        rot = mat[:3, :3]
        if not np.allclose(rot @ rot.T, np.eye(3), atol=1e-4):
            raise InputError("camera rotation block is not orthonormal")

    @property
    def position(self) -> np.ndarray:
        return self.cam_to_world[:3, 3].copy()

    def rays(self):
        from .scenes import pinhole_rays
        return pinhole_rays(self.width, self.height, self.focal, self.cam_to_world)


def look_at(eye, target, up=(0.0, 0.0, 1.0)) -> np.ndarray:
    eye = np.asarray(eye, dtype=np.float64)
    back = eye - np.asarray(target, dtype=np.float64)
    norm = np.linalg.norm(back)
    if norm == 0.0:
        raise InputError("eye and target coincide")
    back /= norm
    right = np.cross(np.asarray(up, dtype=np.float64), back)
    if np.linalg.norm(right) < 1e-9:
        right = np.cross((0.0, 1.0, 0.0), back)
    right /= np.linalg.norm(right)
    true_up = np.cross(back, right)
    mat = np.eye(4)
    mat[:3, 0] = right
    mat[:3, 1] = true_up
    mat[:3, 2] = back
    mat[:3, 3] = eye
    return mat


def orbit_cameras(count: int, width: int = 256, height: int = 256, camera_angle_x: float = 0.9,
                  radius: float = 3.0, elevation: float = 0.4, target=(0.0, 0.0, 0.0)):
    if count < 1:
        raise ConfigError(f"camera count must be >= 1, got {count}")
    focal = focal_from_angle(width, camera_angle_x)
    target = np.asarray(target, dtype=np.float64)
    cams = []
    for k in range(count):
        az = 2.0 * math.pi * k / count
        eye = target + radius * np.array([math.cos(elevation) * math.cos(az),
                                          math.cos(elevation) * math.sin(az),
                                          math.sin(elevation)])
        cams.append(Camera(width, height, focal, look_at(eye, target)))
    return cams


# ---------------------------------------------------------------------------
# .dot1

def canonical_arrays(tree):
    """(node words, is_leaf, sigma rows, sh rows) in BFS order, payload of
    internal nodes zero.  Uses the device table when the tree is canonical."""
    topo = tree.topology()
    node = topo.node.detach().cpu().numpy().astype(np.int64)
    leaf = node < 0
    pid = np.where(leaf, ~node, 0)
    sig_all = tree.sigma.detach().cpu().numpy()
    sh_all = tree.sh.detach().cpu().numpy()
    sigma = np.where(leaf, sig_all[pid], 0).astype(np.float32)
    sh = np.where(leaf[:, None], sh_all[pid], 0).astype(np.float32)
    return node, leaf, sigma, sh


def tree_bytes(tree) -> bytes:
    """Serialise to the .dot1 byte string (vectorised)."""
    node, leaf, sigma, sh = canonical_arrays(tree)
    n = node.size
    B = tree.basis_count
    lo = tree.center - tree.half_extent
    hi = tree.center + tree.half_extent
    head = TREE_MAGIC + _HEADER.pack(TREE_VERSION, B, tree.max_depth, *lo, *hi, n)
    pb = 4 * (1 + 3 * B)
    size = np.where(leaf, 1 + pb, 1 + 64)
    off = np.zeros(n, dtype=np.int64)
    np.cumsum(size[:-1], out=off[1:])
    total = int(off[-1] + size[-1]) if n else 0
    buf = np.zeros(total, dtype=np.uint8)
    buf[off] = leaf.astype(np.uint8)
    li = np.nonzero(leaf)[0]
    if li.size:
        pay = np.concatenate([sigma[li, None], sh[li]], axis=1).astype("<f4")
        rows = pay.view(np.uint8).reshape(li.size, pb)
        buf[(off[li] + 1)[:, None] + np.arange(pb)] = rows
    ii = np.nonzero(~leaf)[0]
    if ii.size:
        kids = (node[ii][:, None] + np.arange(8)).astype("<u8")
        rows = kids.view(np.uint8).reshape(ii.size, 64)
        buf[(off[ii] + 1)[:, None] + np.arange(64)] = rows
    blob = head + buf.tobytes()
    return blob + _CRC.pack(zlib.crc32(blob))


def save_tree(tree, path) -> None:
    Path(path).write_bytes(tree_bytes(tree))


def load_tree(path, device=None):
    path = Path(path)
    if not path.exists():
        raise TreeFileError(f"no such tree file: {path}")
    return load_tree_bytes(path.read_bytes(), name=path.name, device=device)


def load_tree_bytes(data: bytes, name: str = "<bytes>", device=None):
    """Parse and validate a .dot1 byte string (scene_io.py:567-681)."""
    from .octree import from_canonical_arrays
    if len(data) < 4 + _HEADER.size + _CRC.size:
        raise ChecksumError(f"{name}: file too short to be a tree")
    (stored,) = _CRC.unpack_from(data, len(data) - _CRC.size)
    if zlib.crc32(data[:-_CRC.size]) != stored:
        raise ChecksumError(f"{name}: checksum mismatch")
    if data[:4] != TREE_MAGIC:
        raise BadMagicError(f"{name}: bad magic {data[:4]!r}")
    f = _HEADER.unpack_from(data, 4)
    version, B, max_depth = f[0], f[1], f[2]
    bounds = np.array(f[3:9])
    n = f[9]
    if version != TREE_VERSION:
        raise BadVersionError(f"{name}: unsupported version {version}")
    if B not in VALID_BASIS_COUNTS:
        raise StructureError(f"{name}: invalid basis count {B}")
    lo, hi = bounds[:3], bounds[3:]
    extent = hi - lo
    if not np.all(extent > 0):
        raise StructureError(f"{name}: empty bounds")
    if not np.allclose(extent, extent[0], rtol=1e-9, atol=0.0):
        raise StructureError(f"{name}: bounds are not a cube")
    if n < 1:
        raise StructureError(f"{name}: no nodes")
    body = len(data) - 4 - _HEADER.size - _CRC.size
    pb = 4 * (1 + 3 * B)
    if n * min(1 + pb, 1 + 64) > body:
        raise StructureError(f"{name}: node count exceeds file size")
    start = 4 + _HEADER.size
    end = len(data) - _CRC.size
    # record offsets: sequential scan of the 1-byte tags
    offs = np.empty(n, dtype=np.int64)
    tags = np.empty(n, dtype=np.uint8)
    off = start
    for i in range(n):
        if off >= end:
            raise StructureError(f"{name}: record stream truncated")
        t = data[off]
        if t > 1:
            raise StructureError(f"{name}: unknown record tag {t}")
        offs[i] = off + 1
        tags[i] = t
        off += 1 + (pb if t else 64)
        if off > end:
            raise StructureError(f"{name}: record stream truncated")
    if off != end:
        raise StructureError(f"{name}: trailing bytes after records")
    raw = np.frombuffer(data, dtype=np.uint8)
    li = np.nonzero(tags == 1)[0]
    ii = np.nonzero(tags == 0)[0]
    pay = raw[offs[li][:, None] + np.arange(pb)].copy().view("<f4").reshape(li.size, 1 + 3 * B)
    kids = np.full((n, 8), -1, dtype=np.int64)
    if ii.size:
        k = raw[offs[ii][:, None] + np.arange(64)].copy().view("<u8").reshape(ii.size, 8)
        if ((k == 0) | (k >= n)).any():
            raise StructureError(f"{name}: child index out of range")
        kids[ii] = k.astype(np.int64)
    sig = pay[:, 0]
    if not np.all(np.isfinite(sig)) or np.any(sig < 0):
        raise StructureError(f"{name}: leaf density out of range")
    if not np.all(np.isfinite(pay[:, 1:])):
        raise StructureError(f"{name}: non-finite SH coefficient")
    refs = np.zeros(n, dtype=np.int64)
    if ii.size:
        np.add.at(refs, kids[ii].reshape(-1), 1)
    if np.any(refs[1:] != 1):
        raise StructureError(f"{name}: nodes must be referenced exactly once")
    # BFS from record 0 -> canonical order (pool id == BFS index)
    new_index = np.full(n, -1, dtype=np.int64)
    order_parts = []
    frontier = np.array([0], dtype=np.int64)
    assigned, depth = 0, 0
    while frontier.size:
        order_parts.append(frontier)
        new_index[frontier] = np.arange(assigned, assigned + frontier.size)
        assigned += frontier.size
        inner = frontier[tags[frontier] == 0]
        if inner.size and depth >= max_depth:
            raise StructureError(f"{name}: node deeper than max_depth")
        frontier = kids[inner].reshape(-1)
        depth += 1
    if assigned != n:
        raise StructureError(f"{name}: unreachable nodes present")
    order = np.concatenate(order_parts)
    leaf_o = tags[order] == 1
    node = np.where(leaf_o, ~np.arange(n), new_index[np.maximum(kids[order, 0], 0)]).astype(np.int32)
    sigma = np.zeros(n, dtype=np.float32)
    sh = np.zeros((n, 3 * B), dtype=np.float32)
    row_of = np.full(n, -1, dtype=np.int64)
    row_of[li] = np.arange(li.size)
    lrows = row_of[order[leaf_o]]
    sigma[leaf_o] = pay[lrows, 0]
    sh[leaf_o] = pay[lrows, 1:]
    center = (lo + hi) / 2.0
    half = float(extent[0] / 2.0)
    return from_canonical_arrays(center, half, B, max_depth, node, sigma, sh, device=device)
