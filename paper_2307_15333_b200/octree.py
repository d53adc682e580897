"""Sparse octree: the reference's pooled-array API over a device-resident tree.

Mirrors ``octrf.octree.SparseOctree`` (/root/reference/pkg/src/octrf/octree.py:71-450):
pooled node ids with the root at slot 0, a LIFO free list, half-open cells
``[c-h, c+h)``, octant bits x -> 1, y -> 2, z -> 4, split copies the payload,
merge averages it in fp64 and rounds once to f32, ``generation`` bumps on
every structural mutation.

B200 layout.  The payload lives on the GPU: ``sigma`` is a float32 tensor
``[capacity]`` and ``sh`` a float32 ``[capacity, 3B]`` view of a row-padded
``[capacity, pad4(3B)]`` store (16-byte rows for vector loads).  Topology has
two representations, each rebuilt lazily from the other:

* the host pool (numpy ``_child/_parent/_depth/_leaf/_alive/_center`` + free
  list), exactly the reference's, used by the single-edit API;
* the canonical device node table (``int32`` per node in BFS order, leaf
  words ``~pool_id``; see include/dot_b200.h), which the kernels traverse.

Device refine (``calibrate``) and ``load_tree`` produce a canonical tree
directly (pool id == BFS index, free list empty) without touching the host
pool; the host arrays are materialised only if a host API asks for them.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field
from typing import Callable, Sequence, Union

import numpy as np
import torch

from .errors import (
    ConfigError,
    DepthCapError,
    HandleError,
    OutOfBoundsError,
    PreconditionError,
    StructureError,
)

INVALID = -1
VALID_BASIS_COUNTS = (1, 4, 9, 16)
OCTANT_SIGNS = np.array(
    [[(1.0 if o & 1 else -1.0), (1.0 if o & 2 else -1.0), (1.0 if o & 4 else -1.0)]
     for o in range(8)], dtype=np.float64)


def pad4(n: int) -> int:
    return (n + 3) & ~3


def default_device() -> torch.device:
    return torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")


@dataclass
class LeafPayload:
    """Raw density and 3*B channel-major SH coefficients (octree.py:43-57)."""

    sigma: float
    sh: np.ndarray

    def copy(self) -> "LeafPayload":
        return LeafPayload(float(self.sigma), np.array(self.sh, dtype=np.float32))


@dataclass
class TreeStats:
    leaf_count: int
    internal_count: int
    depth_histogram: dict = field(default_factory=dict)
    payload_bytes: int = 0


InitSource = Union[LeafPayload, Callable[[np.ndarray], tuple], int]


@dataclass
class DeviceTopology:
    """Canonical node table of one tree generation."""

    generation: int
    node: torch.Tensor                 # int32 [n_nodes], device
    pool_id: torch.Tensor | None       # int32 [n_nodes] pool id per canonical node, None = identity
    level_offsets: np.ndarray          # int64 [levels + 1], BFS level boundaries
    locate: torch.Tensor | None = None  # int32 [8^L] locate table (dot_locate_build)
    locate_level: int = -1             # -1 = not built yet, 0 = not used
    locate_extra: dict = field(default_factory=dict)  # level -> table, for callers asking another level

    @property
    def n_nodes(self) -> int:
        return int(self.node.shape[0])


def locate_level_default() -> int:
    """Level of the traversal locate table of the render paths (env
    DOT_LOCATE_LEVEL, 0 = off): 7 (2 MB) -- coherent camera rays reuse its
    entries from L1 (200-view render: level 4..8 = 30.95 / 30.84 / 30.72 /
    30.75 / 30.97 ms)."""
    return int(os.environ.get("DOT_LOCATE_LEVEL", "7"))


def locate_level_train() -> int:
    """Locate-table level of the training backward (env DOT_TRAIN_LOCATE_LEVEL).
    The render's level 7 (2 MB, the same table): with the 80-register
    backward, level 9 (512 MB, one load per depth-9 leaf) no longer pays --
    step 2.43 ms with level 7 vs 2.44 with level 9 (the backward equal, the
    optimizer faster without the 512 MB table churning L2) -- and it saves
    512 MB per tree generation."""
    return int(os.environ.get("DOT_TRAIN_LOCATE_LEVEL", "7"))


class SparseOctree:
    """Pooled-array octree over a world cube (reference API, device payload)."""

    def __init__(self, center: Sequence[float], half_extent: float, basis_count: int,
                 max_depth: int = 10, capacity: int = 64, device=None):
        if basis_count not in VALID_BASIS_COUNTS:
            raise ConfigError(f"basis_count must be one of {VALID_BASIS_COUNTS}, got {basis_count}")
        if max_depth < 0:
            raise ConfigError(f"max_depth must be >= 0, got {max_depth}")
        if not (half_extent > 0 and math.isfinite(half_extent)):
            raise ConfigError(f"half_extent must be positive, got {half_extent}")
        self.basis_count = int(basis_count)
        self.max_depth = int(max_depth)
        self.center = np.asarray(center, dtype=np.float64).reshape(3).copy()
        self.half_extent = float(half_extent)
        self.generation = 0
        self.device = torch.device(device) if device is not None else default_device()
        cap = max(int(capacity), 8)
        self._hp = _empty_pool(cap)
        self._free: list[int] = list(range(cap - 1, 0, -1))
        self._sigma = torch.zeros(cap, dtype=torch.float32, device=self.device)
        self._sh_store = torch.zeros(cap, self.sh_stride, dtype=torch.float32, device=self.device)
        self._hp["alive"][0] = 1
        self._hp["leaf"][0] = 1
        self._hp["center"][0] = self.center
        self.leaf_count = 1
        self.internal_count = 0
        self._topo: DeviceTopology | None = None

    # ------------------------------------------------------------------
    # Payload and layout

    @property
    def sh_stride(self) -> int:
        return pad4(3 * self.basis_count)

    @property
    def sigma(self) -> torch.Tensor:
        return self._sigma

    @sigma.setter
    def sigma(self, value):
        self._sigma.copy_(torch.as_tensor(value, dtype=torch.float32).reshape(self._sigma.shape))

    @property
    def sh(self) -> torch.Tensor:
        nsh = 3 * self.basis_count
        return self._sh_store if nsh == self.sh_stride else self._sh_store[:, :nsh]

    @sh.setter
    def sh(self, value):
        self.sh.copy_(torch.as_tensor(value, dtype=torch.float32).reshape(self.sh.shape))

    @property
    def capacity(self) -> int:
        return int(self._sigma.shape[0])

    @property
    def root(self) -> int:
        return 0

    def half_at(self, depth: int) -> float:
        return self.half_extent * 2.0 ** (-int(depth))

    def half_table(self) -> np.ndarray:
        return self.half_extent * 2.0 ** (-np.arange(self.max_depth + 1, dtype=np.float64))

    # ------------------------------------------------------------------
    # Host pool (lazy)

    def _host(self) -> dict:
        if self._hp is None:
            self._hp = _pool_from_canonical(self)
            self._free = []
        return self._hp

    @property
    def _child(self) -> np.ndarray:
        return self._host()["child"]

    @property
    def _parent(self) -> np.ndarray:
        return self._host()["parent"]

    @property
    def _depth(self) -> np.ndarray:
        return self._host()["depth"]

    @property
    def _leaf(self) -> np.ndarray:
        return self._host()["leaf"]

    @property
    def _alive(self) -> np.ndarray:
        return self._host()["alive"]

    @property
    def _center(self) -> np.ndarray:
        return self._host()["center"]

    # ------------------------------------------------------------------
    # Device topology (lazy)

    def topology(self) -> DeviceTopology:
        """Canonical node table for the current generation (rebuilt if stale)."""
        if self._topo is not None and self._topo.generation == self.generation:
            return self._topo
        order, new_index, offsets = level_order(self)
        leaf = self._leaf[order] == 1
        first = np.where(leaf, 0, new_index[self._child[order, 0]])
        node = np.where(leaf, ~order, first).astype(np.int32)
        identity = bool(np.array_equal(order, np.arange(order.size)))
        pool = None if identity else torch.from_numpy(order.astype(np.int32)).to(self.device)
        self._topo = DeviceTopology(self.generation, torch.from_numpy(node).to(self.device), pool,
                                    offsets)
        return self._topo

    def _set_canonical(self, node: torch.Tensor, sigma: torch.Tensor, sh_store: torch.Tensor,
                       leaf_count: int, level_offsets: np.ndarray | None = None) -> None:
        """Adopt a canonical device tree (pool id == BFS index); host pool goes lazy."""
        self._sigma = sigma
        self._sh_store = sh_store
        self.leaf_count = int(leaf_count)
        self.internal_count = int(node.shape[0]) - self.leaf_count
        self.generation += 1
        if level_offsets is None:
            level_offsets = _level_offsets_from_node(node)
        self._topo = DeviceTopology(self.generation, node, None, level_offsets)
        self._hp = None
        self._free = []

    def tree_view(self, locate: bool = True, locate_level: int | None = None):
        """C-ABI ``dot_tree_view`` of the current generation (+ keepalive).
        ``locate=False`` (refine) skips building the traversal locate table;
        ``locate_level`` asks for a table of that level instead of the
        default one (each built once per generation)."""
        from ._lib import DotTreeView
        if self.device.type != "cuda":
            raise ConfigError("the tree payload is not on a CUDA device; the B200 kernels "
                              "have no CPU fallback")
        topo = self.topology()
        v = DotTreeView()
        v.node = topo.node.data_ptr()
        v.n_nodes = topo.n_nodes
        v.sigma = self._sigma.data_ptr()
        v.sh = self._sh_store.data_ptr()
        v.capacity = self.capacity
        v.basis_count = self.basis_count
        v.sh_stride = self.sh_stride
        for k in range(3):
            v.center[k] = float(self.center[k])
        v.half_extent = self.half_extent
        v.max_depth = self.max_depth
        v.locate_level = 0
        v.locate = None
        if locate:
            self._attach_locate(v, topo)
            if locate_level is not None and v.locate_level > 0:
                self._attach_locate_level(v, topo, locate_level)
        return v, topo

    def _attach_locate(self, v, topo: DeviceTopology) -> None:
        """Locate table of this generation (built once, lazily): replaces the
        first L node loads of every traversal descent by one table load; used
        only for dyadic roots, where it is exact (dot_b200.h)."""
        from . import _lib
        if topo.locate_level < 0:
            topo.locate_level = 0
            want = locate_level_default()
            deepest = len(topo.level_offsets) - 2
            lib = _lib.load()
            if want > 0 and 0 < deepest <= 21 and lib.dot_locate_supported(ctypes.byref(v)):
                lv = min(want, deepest)
                table = torch.empty(1 << (3 * lv), dtype=torch.int32, device=self.device)
                _lib.call("dot_locate_build", ctypes.byref(v), lv, _lib.ptr(table), _lib.stream_ptr())
                topo.locate, topo.locate_level = table, lv
        if topo.locate_level > 0 and _lib.load().dot_locate_supported(ctypes.byref(v)):
            v.locate_level = topo.locate_level
            v.locate = topo.locate.data_ptr()

    def _attach_locate_level(self, v, topo: DeviceTopology, level: int) -> None:
        """Swap in a table of another level (same exactness conditions as the
        default one, which was checked when it was built)."""
        from . import _lib
        deepest = len(topo.level_offsets) - 2
        lv = min(int(level), deepest, 9)
        if lv <= 0 or lv == topo.locate_level:
            return
        table = topo.locate_extra.get(lv)
        if table is None:
            table = torch.empty(1 << (3 * lv), dtype=torch.int32, device=self.device)
            _lib.call("dot_locate_build", ctypes.byref(v), lv, _lib.ptr(table), _lib.stream_ptr())
            topo.locate_extra[lv] = table
        v.locate_level = lv
        v.locate = table.data_ptr()

    # ------------------------------------------------------------------
    # Queries (octree.py:115-181)

    def is_live(self, node: int) -> bool:
        return 0 <= node < self.capacity and bool(self._alive[node])

    def is_leaf(self, node: int) -> bool:
        self._check_live(node)
        return bool(self._leaf[node])

    def node_depth(self, node: int) -> int:
        self._check_live(node)
        return int(self._depth[node])

    def node_center(self, node: int) -> np.ndarray:
        self._check_live(node)
        return self._center[node].copy()

    def children(self, node: int) -> np.ndarray:
        self._check_live(node)
        if self._leaf[node]:
            raise PreconditionError(f"node {node} is a leaf, has no children")
        return self._child[node].copy()

    def parent(self, node: int) -> int:
        self._check_live(node)
        return int(self._parent[node])

    def payload(self, node: int) -> LeafPayload:
        self._check_live(node)
        if not self._leaf[node]:
            raise PreconditionError(f"node {node} is internal, has no payload")
        return LeafPayload(float(self._sigma[node]), self.sh[node].detach().cpu().numpy().copy())

    def set_payload(self, node: int, payload: LeafPayload) -> None:
        self._check_live(node)
        if not self._leaf[node]:
            raise PreconditionError(f"node {node} is internal, has no payload")
        sh = np.asarray(payload.sh, dtype=np.float32).reshape(-1)
        if sh.shape[0] != 3 * self.basis_count:
            raise ConfigError(f"sh length {sh.shape[0]} != 3*B={3 * self.basis_count}")
        if not (math.isfinite(payload.sigma) and np.isfinite(sh).all()):
            raise ConfigError("payload values must be finite")
        self._sigma[node] = float(np.float32(payload.sigma))
        self.sh[node] = torch.from_numpy(sh).to(self.device)

    def leaf_ids(self) -> np.ndarray:
        hp = self._host()
        return np.nonzero((hp["alive"] == 1) & (hp["leaf"] == 1))[0].astype(np.int64)

    def internal_ids(self) -> np.ndarray:
        hp = self._host()
        return np.nonzero((hp["alive"] == 1) & (hp["leaf"] == 0))[0].astype(np.int64)

    def _check_live(self, node: int) -> None:
        if not self.is_live(node):
            raise HandleError(f"node id {node} does not resolve to a live node")

    # ------------------------------------------------------------------
    # Mutation (octree.py:186-304) -- host topology, device payload

    def _grow(self, extra: int) -> None:
        hp = self._host()
        old = self.capacity
        new = max(old * 2, old + extra)
        grown = _empty_pool(new)
        for k, v in hp.items():
            grown[k][:old] = v
        self._hp = grown
        sig = torch.zeros(new, dtype=torch.float32, device=self.device)
        sig[:old] = self._sigma
        sh = torch.zeros(new, self.sh_stride, dtype=torch.float32, device=self.device)
        sh[:old] = self._sh_store
        self._sigma, self._sh_store = sig, sh
        self._free.extend(range(new - 1, old - 1, -1))

    def _alloc(self) -> int:
        if not self._free:
            self._grow(8)
        return self._free.pop()

    def split_leaf(self, leaf: int) -> np.ndarray:
        """Replace a leaf with 8 children carrying exact payload copies."""
        self._check_live(leaf)
        hp = self._host()
        if not hp["leaf"][leaf]:
            raise PreconditionError(f"split target {leaf} is not a leaf")
        depth = int(hp["depth"][leaf])
        if depth >= self.max_depth:
            raise DepthCapError(f"leaf {leaf} already at max_depth {self.max_depth}")
        ids = np.array([self._alloc() for _ in range(8)], dtype=np.int64)
        hp = self._hp
        child_half = self.half_at(depth) * 0.5
        hp["alive"][ids] = 1
        hp["leaf"][ids] = 1
        hp["parent"][ids] = leaf
        hp["depth"][ids] = depth + 1
        hp["center"][ids] = hp["center"][leaf] + child_half * OCTANT_SIGNS
        hp["leaf"][leaf] = 0
        hp["child"][leaf] = ids
        tid = torch.from_numpy(ids).to(self.device)
        self._sigma[tid] = self._sigma[leaf].clone()
        self._sh_store[tid] = self._sh_store[leaf].clone()
        self._sigma[leaf] = 0.0
        self._sh_store[leaf] = 0.0
        self.leaf_count += 7
        self.internal_count += 1
        self.generation += 1
        return ids

    def _merge_payload(self, parents: np.ndarray, kids: np.ndarray) -> None:
        # numpy orders: sigma (P,8) last-axis mean -> pairwise; sh (P,8,3B)
        # middle-axis mean -> sequential (octree.py:284-285).
        tk = torch.from_numpy(kids).to(self.device)
        tp = torch.from_numpy(parents).to(self.device)
        s = self._sigma[tk].double()
        ssum = ((s[:, 0] + s[:, 1]) + (s[:, 2] + s[:, 3])) + ((s[:, 4] + s[:, 5]) + (s[:, 6] + s[:, 7]))
        h = self._sh_store[tk].double()
        hsum = h[:, 0]
        for k in range(1, 8):
            hsum = hsum + h[:, k]
        self._sigma[tp] = (ssum / 8.0).float()
        self._sh_store[tp] = (hsum / 8.0).float()

    def merge_children(self, parent: int) -> int:
        """Collapse 8 leaf children into the parent, averaging payloads."""
        self._check_live(parent)
        hp = self._host()
        if hp["leaf"][parent]:
            raise PreconditionError(f"merge target {parent} is a leaf")
        kids = hp["child"][parent].copy()
        if not hp["leaf"][kids].all():
            raise PreconditionError(f"node {parent} has internal children; merge bottom-up first")
        self._merge_payload(np.array([parent]), kids[None, :])
        for c in kids:
            self._release(int(c))
        hp["leaf"][parent] = 1
        hp["child"][parent] = INVALID
        self.leaf_count -= 7
        self.internal_count -= 1
        self.generation += 1
        return parent

    def _release(self, node: int) -> None:
        hp = self._hp
        hp["alive"][node] = 0
        hp["leaf"][node] = 0
        hp["parent"][node] = INVALID
        hp["child"][node] = INVALID
        self._free.append(node)

    def merge_children_many(self, parents: np.ndarray) -> None:
        """Vectorized merge of many disjoint parents (all children leaves)."""
        parents = np.asarray(parents, dtype=np.int64)
        if parents.size == 0:
            return
        hp = self._host()
        kids = hp["child"][parents]
        if not (hp["alive"][parents].all() and (hp["leaf"][parents] == 0).all()
                and hp["leaf"][kids.reshape(-1)].all()):
            raise PreconditionError("batch merge preconditions violated")
        self._merge_payload(parents, kids)
        flat = kids.reshape(-1)
        hp["alive"][flat] = 0
        hp["leaf"][flat] = 0
        hp["parent"][flat] = INVALID
        hp["child"][flat] = INVALID
        self._free.extend(int(c) for c in flat)
        hp["leaf"][parents] = 1
        hp["child"][parents] = INVALID
        self.leaf_count -= 7 * parents.size
        self.internal_count -= parents.size
        self.generation += 1

    def split_leaf_many(self, leaves: np.ndarray) -> np.ndarray:
        leaves = np.asarray(leaves, dtype=np.int64)
        out = np.empty((leaves.size, 8), dtype=np.int64)
        for i, leaf in enumerate(leaves):
            out[i] = self.split_leaf(int(leaf))
        return out

    # ------------------------------------------------------------------
    # Addressing / inspection (octree.py:309-388)

    def locate(self, point: Sequence[float]) -> tuple:
        p = np.asarray(point, dtype=np.float64).reshape(3)
        lo = self.center - self.half_extent
        hi = self.center + self.half_extent
        if not ((p >= lo).all() and (p < hi).all()):
            raise OutOfBoundsError(f"point {p.tolist()} outside half-open bounds")
        hp = self._host()
        node = 0
        while not hp["leaf"][node]:
            c = hp["center"][node]
            octant = int(p[0] >= c[0]) | (int(p[1] >= c[1]) << 1) | (int(p[2] >= c[2]) << 2)
            node = int(hp["child"][node, octant])
        return node, hp["center"][node].copy(), self.half_at(int(hp["depth"][node]))

    def stats(self) -> TreeStats:
        leaves = self.leaf_ids()
        depths = self._depth[leaves]
        hist = {int(d): int(n) for d, n in zip(*np.unique(depths, return_counts=True))}
        return TreeStats(int(self.leaf_count), int(self.internal_count), hist,
                         int(leaves.size) * 4 * (1 + 3 * self.basis_count))

    def validate(self) -> None:
        """Structural invariants (octree.py:338-388); raises StructureError."""
        hp = self._host()
        alive = np.nonzero(hp["alive"] == 1)[0]
        leaves = alive[hp["leaf"][alive] == 1]
        internals = alive[hp["leaf"][alive] == 0]
        if leaves.size != self.leaf_count or internals.size != self.internal_count:
            raise StructureError("node counters disagree with alive flags")
        if leaves.size != 7 * internals.size + 1:
            raise StructureError(f"L = 7I + 1 violated: L={leaves.size} I={internals.size}")
        if not hp["alive"][0]:
            raise StructureError("root slot 0 is dead")
        seen = np.zeros(self.capacity, dtype=bool)
        seen[0] = True
        frontier = np.array([0], dtype=np.int64)
        count = 1
        while frontier.size:
            inner = frontier[hp["leaf"][frontier] == 0]
            if inner.size == 0:
                break
            flat = hp["child"][inner].reshape(-1)
            if (flat < 0).any() or (flat >= self.capacity).any():
                raise StructureError("child index out of range")
            if not hp["alive"][flat].all():
                raise StructureError("internal node points at a dead child")
            if seen[flat].any():
                raise StructureError("node reachable through two parents")
            if not (hp["parent"][flat] == np.repeat(inner, 8)).all():
                raise StructureError("parent back-pointer mismatch")
            if not (hp["depth"][flat] == np.repeat(hp["depth"][inner] + 1, 8)).all():
                raise StructureError("child depth != parent depth + 1")
            halves = self.half_extent * 2.0 ** (-hp["depth"][flat].astype(np.float64))
            expect = (np.repeat(hp["center"][inner], 8, axis=0)
                      + halves[:, None] * np.tile(OCTANT_SIGNS, (inner.size, 1)))
            if not np.array_equal(expect, hp["center"][flat]):
                raise StructureError("child centers off the octant grid")
            seen[flat] = True
            count += flat.size
            frontier = flat
        if count != alive.size:
            raise StructureError("live nodes unreachable from root")
        if (hp["depth"][leaves] > self.max_depth).any():
            raise StructureError("leaf deeper than max_depth")
        sig = self._sigma.detach().cpu().numpy()[leaves]
        sh = self.sh.detach().cpu().numpy()[leaves]
        if not (np.isfinite(sig).all() and np.isfinite(sh).all()):
            raise StructureError("non-finite payload")
        if (sig < 0).any():
            raise StructureError("negative density")


# ---------------------------------------------------------------------------
# Pool helpers

def _empty_pool(cap: int) -> dict:
    return {
        "child": np.full((cap, 8), INVALID, dtype=np.int64),
        "parent": np.full(cap, INVALID, dtype=np.int64),
        "depth": np.zeros(cap, dtype=np.int32),
        "leaf": np.zeros(cap, dtype=np.uint8),
        "alive": np.zeros(cap, dtype=np.uint8),
        "center": np.zeros((cap, 3), dtype=np.float64),
    }


def level_order(tree: SparseOctree):
    """Live node ids in BFS order, old->new map, and level offsets
    (scene_io.py:529-541, the reference's only canonical order)."""
    hp = tree._host()
    new_index = np.full(tree.capacity, -1, dtype=np.int64)
    parts = []
    offsets = [0]
    frontier = np.array([0], dtype=np.int64)
    assigned = 0
    while frontier.size:
        parts.append(frontier)
        new_index[frontier] = np.arange(assigned, assigned + frontier.size)
        assigned += frontier.size
        offsets.append(assigned)
        internal = frontier[hp["leaf"][frontier] == 0]
        frontier = hp["child"][internal].reshape(-1)
    return np.concatenate(parts), new_index, np.asarray(offsets, dtype=np.int64)


def _level_offsets_from_node(node: torch.Tensor) -> np.ndarray:
    w = node.detach().cpu().numpy()
    offsets = [0]
    lo, hi = 0, 1
    while lo < hi:
        offsets.append(hi)
        n_int = int((w[lo:hi] >= 0).sum())
        lo, hi = hi, hi + 8 * n_int
    return np.asarray(offsets, dtype=np.int64)


def _pool_from_canonical(tree: SparseOctree) -> dict:
    """Host pool arrays of a canonical tree (pool id == BFS index)."""
    topo = tree._topo
    w = topo.node.detach().cpu().numpy().astype(np.int64)
    n = w.size
    cap = tree.capacity
    hp = _empty_pool(cap)
    internal = np.nonzero(w >= 0)[0]
    hp["alive"][:n] = 1
    hp["leaf"][:n] = (w < 0).astype(np.uint8)
    kids = w[internal][:, None] + np.arange(8)
    hp["child"][internal] = kids
    hp["parent"][kids.reshape(-1)] = np.repeat(internal, 8)
    hp["center"][0] = tree.center
    off = topo.level_offsets
    for d in range(len(off) - 1):
        lo, hi = off[d], off[d + 1]
        hp["depth"][lo:hi] = d
        inner = np.arange(lo, hi)[w[lo:hi] >= 0]
        if inner.size:
            child_half = tree.half_at(d) * 0.5
            k = hp["child"][inner].reshape(-1)
            hp["center"][k] = (np.repeat(hp["center"][inner], 8, axis=0)
                               + child_half * np.tile(OCTANT_SIGNS, (inner.size, 1)))
    return hp


# ---------------------------------------------------------------------------
# Builders

def build_dense(depth: int, center: Sequence[float], half_extent: float, basis_count: int,
                init: InitSource, max_depth: int = 10, device=None) -> SparseOctree:
    """Complete octree of uniform leaf depth (octree.py:391-450).

    ``init``: a LeafPayload for every leaf, a callable mapping (N, 3) leaf
    centres to (sigma[N], sh[N, 3B]), or an int seed (sigma ~ U[0,1),
    sh ~ N(0, 0.5), same streams as the reference).  The result is already
    canonical (pool id == BFS index).
    """
    if not (0 <= depth <= max_depth):
        raise ConfigError(f"depth {depth} outside [0, max_depth={max_depth}]")
    n_total = (8 ** (depth + 1) - 1) // 7
    tree = SparseOctree(center, half_extent, basis_count, max_depth=max_depth,
                        capacity=n_total, device=device)
    hp = tree._hp
    if depth > 0:
        tree._free.clear()
        offsets = [(8 ** k - 1) // 7 for k in range(depth + 2)]
        centers = tree.center[None, :]
        for k in range(depth + 1):
            lo, hi = offsets[k], offsets[k + 1]
            if k > 0:
                child_half = tree.half_at(k - 1) * 0.5
                n_parents = centers.shape[0]
                centers = (np.repeat(centers, 8, axis=0)
                           + child_half * np.tile(OCTANT_SIGNS, (n_parents, 1)))
                hp["parent"][lo:hi] = np.repeat(np.arange(offsets[k - 1], lo, dtype=np.int64), 8)
            hp["alive"][lo:hi] = 1
            hp["depth"][lo:hi] = k
            hp["center"][lo:hi] = centers
            if k < depth:
                base = offsets[k + 1] + 8 * np.arange(hi - lo, dtype=np.int64)
                hp["child"][lo:hi] = base[:, None] + np.arange(8, dtype=np.int64)
                hp["leaf"][lo:hi] = 0
            else:
                hp["leaf"][lo:hi] = 1
        tree.leaf_count = 8 ** depth
        tree.internal_count = (8 ** depth - 1) // 7
    leaves = (np.arange(n_total - 8 ** depth, n_total, dtype=np.int64) if depth > 0
              else np.array([0], dtype=np.int64))
    centers = hp["center"][leaves]
    nsh = 3 * basis_count
    if isinstance(init, LeafPayload):
        sh = np.asarray(init.sh, dtype=np.float32).reshape(-1)
        if sh.shape[0] != nsh:
            raise ConfigError(f"init sh length {sh.shape[0]} != 3*B={nsh}")
        sig = np.full(leaves.size, np.float32(init.sigma), dtype=np.float32)
        shv = np.broadcast_to(sh, (leaves.size, nsh))
    elif callable(init):
        sig, shv = init(centers)
        sig = np.asarray(sig, dtype=np.float32).reshape(-1)
        shv = np.asarray(shv, dtype=np.float32).reshape(len(leaves), nsh)
        if sig.shape[0] != leaves.size:
            raise ConfigError("init callback returned wrong-length sigma")
    else:
        rng = np.random.default_rng(int(init))
        sig = rng.uniform(0.0, 1.0, leaves.size).astype(np.float32)
        shv = rng.normal(0.0, 0.5, (leaves.size, nsh)).astype(np.float32)
    tl = torch.from_numpy(leaves).to(tree.device)
    tree._sigma[tl] = torch.from_numpy(np.ascontiguousarray(sig)).to(tree.device)
    tree.sh[tl] = torch.from_numpy(np.ascontiguousarray(shv)).to(tree.device)
    return tree


def from_pool_arrays(arrays: dict, device=None) -> SparseOctree:
    """Rebuild a tree from the reference's pool state (``child``, ``parent``,
    ``depth``, ``leaf``, ``alive``, ``center``, ``sigma``, ``sh``, ``free``,
    ``root_center``, ``half_extent``, ``basis_count``, ``max_depth``), keeping
    its exact slot ids and free list."""
    tree = SparseOctree(arrays["root_center"], float(arrays["half_extent"]),
                        int(arrays["basis_count"]), max_depth=int(arrays["max_depth"]),
                        capacity=8, device=device)
    cap = int(np.asarray(arrays["sigma"]).shape[0])
    hp = _empty_pool(cap)
    for k in hp:
        hp[k][:] = np.asarray(arrays[k]).astype(hp[k].dtype)
    tree._hp = hp
    tree._free = [int(x) for x in np.asarray(arrays["free"]).reshape(-1)]
    tree._sigma = torch.from_numpy(np.ascontiguousarray(arrays["sigma"], dtype=np.float32)).to(tree.device)
    store = torch.zeros(cap, tree.sh_stride, dtype=torch.float32, device=tree.device)
    nsh = 3 * tree.basis_count
    store[:, :nsh] = torch.from_numpy(
        np.ascontiguousarray(arrays["sh"], dtype=np.float32).reshape(cap, nsh)).to(tree.device)
    tree._sh_store = store
    tree.leaf_count = int(((hp["alive"] == 1) & (hp["leaf"] == 1)).sum())
    tree.internal_count = int(((hp["alive"] == 1) & (hp["leaf"] == 0)).sum())
    return tree


def from_canonical_tensors(center, half_extent, basis_count, max_depth, node: torch.Tensor,
                           sigma: torch.Tensor, sh_store: torch.Tensor,
                           level_offsets: np.ndarray | None = None) -> SparseOctree:
    """Adopt device tensors of a canonical tree (node words, sigma, padded SH store)."""
    tree = SparseOctree(center, half_extent, basis_count, max_depth=max_depth, capacity=8,
                        device=node.device)
    tree._set_canonical(node, sigma, sh_store, int((node < 0).sum().item()), level_offsets)
    tree.generation = 0
    tree._topo.generation = 0
    return tree


def from_canonical_arrays(center, half_extent, basis_count, max_depth, node: np.ndarray,
                          sigma: np.ndarray, sh: np.ndarray, device=None) -> SparseOctree:
    """Tree from canonical BFS arrays (node words with leaf word = ~index,
    payload rows in BFS order).  No host pool is built."""
    tree = SparseOctree(center, half_extent, basis_count, max_depth=max_depth, capacity=8,
                        device=device)
    n = int(node.shape[0])
    S = tree.sh_stride
    store = torch.zeros(n, S, dtype=torch.float32, device=tree.device)
    store[:, :3 * basis_count] = torch.from_numpy(
        np.ascontiguousarray(sh, dtype=np.float32).reshape(n, 3 * basis_count)).to(tree.device)
    sig = torch.from_numpy(np.ascontiguousarray(sigma, dtype=np.float32).reshape(n)).to(tree.device)
    tnode = torch.from_numpy(np.ascontiguousarray(node, dtype=np.int32)).to(tree.device)
    tree.generation = -1
    tree._set_canonical(tnode, sig, store, int((node < 0).sum()))
    tree.generation = 0
    tree._topo.generation = 0
    return tree
