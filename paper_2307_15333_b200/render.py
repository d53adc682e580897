"""Differentiable volume rendering over the octree -- the drop-in boundary.

Same functions, argument meaning and error behaviour as the reference's
``octrf.render`` (/root/reference/pkg/src/octrf/render.py:105-241); the work
runs in the sm_100a kernels of ``libdot_b200.so`` (no CPU fallback):

* ``segment_batch`` / ``traverse``  -> ``dot_trace_count`` + ``dot_trace_fill``
* ``render_rays`` / ``render_ray`` / ``render_image`` -> ``dot_render_fwd``
* ``render_and_backprop`` -> ``dot_render_bwd`` (loss, leaf gradients,
  per-leaf signal and the touched set in one fused kernel)

Array conventions: numpy inputs give numpy float64 outputs like the
reference (one H2D copy in, one D2H copy out).  torch tensors give torch
outputs on the tree's device with no host synchronisation (float32 colours
and gradients, float64 signal); host torch tensors are copied with
``non_blocking`` so pinned buffers overlap.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import InputError
from .octree import SparseOctree, locate_level_train

EPS_T = 1e-4  # early-termination transmittance threshold (render.py:23)
UNIT_TOL = 1e-6
COHERENT_MIN_RAYS = 1 << 14  # below this a key sort costs more than it saves
WARP_SCHED = os.environ.get("DOT_WARP_SCHED", "1") == "1"
SCHED_MAX_RAYS = 1 << 30
# warps per chunk of the cost-ordered launch (dot_sched_order_costs), env
# DOT_COST_CHUNK overrides.  Measured: a 2^20-ray configs[1] batch packs best
# with single warps (chunks of 2 / 4: +2 / +5 % backward); a 2^21-ray batch
# of the larger configs[3] scene wants chunks of 16 warps (single warps +2 %:
# neighbouring warps share L2 lines of the 1.9 GB payload).
COST_CHUNK_ENV = os.environ.get("DOT_COST_CHUNK")


def cost_chunk(n: int) -> int:
    if COST_CHUNK_ENV:
        return int(COST_CHUNK_ENV)
    return 1 if n <= (1 << 20) else 16


def _sched_table(tree) -> torch.Tensor:
    """Learned per-key-bucket warp cost table of this tree object (u16,
    2^24 coarse + 2^27 fine entries = 288 MB, survives refines: it only
    orders launches)."""
    t = getattr(tree, "_sched_table", None)
    if t is None or t.device != tree.device:
        t = torch.zeros((1 << 24) + (1 << 27), dtype=torch.int16, device=tree.device)
        tree._sched_table = t
        tree._sched_written = None  # event after the last dot_sched_update
        tree._sched_read = None     # event after the last side-stream dot_sched_order
    return t


def _sched_order(tree, sorted_keys: torch.Tensor, n: int, stream) -> torch.Tensor:
    """dot_sched_order on ``stream``; ordered after the table's last update
    and recorded as its latest reader (see render_and_backprop's update)."""
    table = _sched_table(tree)
    cur = torch.cuda.current_stream(tree.device)
    if stream is not cur and tree._sched_written is not None:
        stream.wait_event(tree._sched_written)
    warp_order = torch.empty((n + 31) // 32, dtype=torch.int32, device=tree.device)
    _lib.call("dot_sched_order", _lib.ptr(sorted_keys), n, _lib.ptr(table), _lib.ptr(warp_order),
              _lib.stream_ptr(stream))
    if stream is not cur:
        ev = torch.cuda.Event()
        ev.record(stream)
        tree._sched_read = ev
    return warp_order


@dataclass
class Ray:
    origin: np.ndarray
    dir: np.ndarray
    t_near: float = 0.0
    t_far: float = math.inf

    def __post_init__(self):
        self.origin = np.asarray(self.origin, dtype=np.float64).reshape(3)
        self.dir = np.asarray(self.dir, dtype=np.float64).reshape(3)
        if abs(float(np.linalg.norm(self.dir)) - 1.0) > UNIT_TOL:
            raise InputError("ray direction must be a unit vector")
        if not self.t_near < self.t_far:
            raise InputError(f"t_near {self.t_near} must be < t_far {self.t_far}")


@dataclass
class RaySegmentList:
    """Ordered (leaf, t_entry, delta) triples; consecutive segments abut."""

    leaf: np.ndarray
    t_entry: np.ndarray
    delta: np.ndarray

    def __len__(self) -> int:
        return int(self.leaf.shape[0])


@dataclass
class RenderOutput:
    rgb: np.ndarray
    per_segment_Q: np.ndarray
    transmittance_final: float


class GradBuffer:
    """Loss gradients for every leaf touched by the batch (render.py:63-78).

    ``dsigma`` [capacity] and ``dsh`` [capacity, 3B] are dense by node id;
    ``touched`` lists the touched leaf ids ascending; ``touched_mask`` is the
    u8 mask the kernels write (kept on device for the optimizer).

    For numpy callers (``host=True``) the device buffers are kept and the
    float64 numpy views the reference returns are made on first attribute
    access, so a caller that hands the gradients straight to
    ``rmsprop_step`` (the reference's train_epoch pattern, optim.py:147-150)
    never copies them to the host.
    """

    def __init__(self, dsigma, dsh, touched_mask, generation, dsh_store=None, host=False):
        self.generation = generation
        self.dsh_store = dsh_store  # padded [capacity, pad4(3B)] device store
        self._host = bool(host)
        self._dev = {"dsigma": dsigma, "dsh": dsh, "touched_mask": touched_mask}
        self._np = {}
        self._touched = None

    def _get(self, name):
        if not self._host:
            return self._dev[name]
        if name not in self._np:
            t = self._dev[name]
            a = t.detach().cpu().numpy()
            self._np[name] = a if name == "touched_mask" else a.astype(np.float64)
        return self._np[name]

    def _set(self, name, value):
        self._dev[name] = value
        self._np.pop(name, None)

    dsigma = property(lambda self: self._get("dsigma"), lambda self, v: self._set("dsigma", v))
    dsh = property(lambda self: self._get("dsh"), lambda self, v: self._set("dsh", v))
    touched_mask = property(lambda self: self._get("touched_mask"),
                            lambda self, v: self._set("touched_mask", v))

    def device_tensors(self):
        """(dsigma, dsh, touched_mask) as they live on the device (torch
        tensors; numpy arrays for a GradBuffer built from host data)."""
        return self._dev["dsigma"], self._dev["dsh"], self._dev["touched_mask"]

    @property
    def touched(self):
        if self._touched is None:
            m = self.touched_mask
            if isinstance(m, np.ndarray):
                self._touched = np.nonzero(m)[0].astype(np.int64)
            else:
                self._touched = torch.nonzero(m).reshape(-1)
        return self._touched

    @touched.setter
    def touched(self, value):
        self._touched = value

    def get(self, leaf: int):
        return float(self.dsigma[leaf]), self.dsh[leaf].copy() if isinstance(self.dsh, np.ndarray) \
            else self.dsh[leaf].clone()


# ---------------------------------------------------------------------------
# input / output plumbing

class _IO:
    """Tracks whether the caller handed us numpy, host torch or device torch."""

    def __init__(self, tree: SparseOctree, like):
        self.tree = tree
        self.numpy = not isinstance(like, torch.Tensor)
        self.host_torch = isinstance(like, torch.Tensor) and like.device.type != "cuda"

    def rays(self, x, name: str) -> torch.Tensor:
        dev = self.tree.device
        if isinstance(x, torch.Tensor):
            t = x.reshape(-1, 3)
            if t.dtype != torch.float64:
                t = t.double()
            return t.to(dev, non_blocking=True).contiguous()
        a = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, 3)
        return torch.from_numpy(a).to(dev, non_blocking=True)

    def out(self, t: torch.Tensor, dtype=np.float64):
        if self.numpy:
            return t.detach().cpu().numpy().astype(dtype, copy=False)
        if self.host_torch:
            return t.to("cpu", non_blocking=False)
        return t


def _on_device(x, dev: torch.device) -> bool:
    """Tensor (or device) ``x`` is on ``dev`` (a device without an index matches any index)."""
    xd = x if isinstance(x, torch.device) else x.device
    return xd.type == dev.type and (dev.index is None or xd.index is None or xd.index == dev.index)


def _check_out(name: str, x, dtype, tree) -> None:
    """A caller-provided per-leaf output: contiguous [capacity] of ``dtype`` on the tree's device."""
    if x is not None and (not isinstance(x, torch.Tensor) or x.dtype != dtype or not _on_device(x, tree.device)
                          or x.numel() != tree.capacity or not x.is_contiguous()):
        raise InputError(f"{name} must be a contiguous {dtype} [capacity] tensor on {tree.device}")


def _background(bg) -> np.ndarray:
    b = np.asarray(bg, dtype=np.float64)
    if b.ndim == 0:
        b = np.full(3, float(b))
    return np.ascontiguousarray(b.reshape(3))


def _bg_ptr(bg: np.ndarray):
    return bg.ctypes.data_as(_lib.c_void_p)


# ---------------------------------------------------------------------------
# API

def segment_batch(tree: SparseOctree, origins, dirs, t_near: float = 0.0, t_far: float = math.inf):
    """Segment many rays at once; returns (offsets, leaf, t_entry, delta).

    Leaf ids and f64 t/delta are bit-identical to the reference's
    count/fill kernels (_kernels.py:161-182)."""
    io = _IO(tree, origins)
    o = io.rays(origins, "origins")
    d = io.rays(dirs, "dirs")
    n = o.shape[0]
    if d.shape[0] != n:
        raise InputError(f"batch length mismatch: {n} origins, {d.shape[0]} dirs")
    view, _topo = tree.tree_view()
    dev = tree.device
    counts = torch.empty(n, dtype=torch.int64, device=dev)
    s = _lib.stream_ptr()
    _lib.call("dot_trace_count", _lib.ctypes.byref(view), _lib.ptr(o), _lib.ptr(d), n,
              float(t_near), float(t_far), _lib.ptr(counts), s)
    offsets = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=offsets[1:])
    total = int(offsets[-1].item()) if n else 0
    seg_leaf = torch.empty(total, dtype=torch.int64, device=dev)
    seg_t = torch.empty(total, dtype=torch.float64, device=dev)
    seg_delta = torch.empty(total, dtype=torch.float64, device=dev)
    _lib.call("dot_trace_fill", _lib.ctypes.byref(view), _lib.ptr(o), _lib.ptr(d), n,
              float(t_near), float(t_far), _lib.ptr(offsets), _lib.ptr(seg_leaf), _lib.ptr(seg_t),
              _lib.ptr(seg_delta), s)
    return (io.out(offsets, np.int64), io.out(seg_leaf, np.int64), io.out(seg_t),
            io.out(seg_delta))


def traverse(tree: SparseOctree, ray: Ray) -> RaySegmentList:
    """Exact leaf-boundary segmentation of one ray (render.py:127-131)."""
    _, leaf, t, d = segment_batch(tree, ray.origin[None, :], ray.dir[None, :], ray.t_near, ray.t_far)
    return RaySegmentList(leaf, t, d)


def render_rays(tree: SparseOctree, origins, dirs, background, early_stop_eps: float = EPS_T,
                t_near: float = 0.0, t_far: float = math.inf, return_aux: bool = False,
                return_depth: bool = False):
    """Composite a batch of rays (render.py:134-152).

    return_aux adds (T_final, weight sum); return_depth appends the expected
    termination depth sum_i T_i Q_i (t_i + delta_i/2) (not in the reference).
    """
    io = _IO(tree, origins)
    o = io.rays(origins, "origins")
    d = io.rays(dirs, "dirs")
    n = o.shape[0]
    if d.shape[0] != n:
        raise InputError(f"batch length mismatch: {n} origins, {d.shape[0]} dirs")
    dev = tree.device
    rgb = torch.empty(n, 3, dtype=torch.float32, device=dev)
    tfin = torch.empty(n, dtype=torch.float32, device=dev) if return_aux else None
    wsum = torch.empty(n, dtype=torch.float32, device=dev) if return_aux else None
    depth = torch.empty(n, dtype=torch.float32, device=dev) if return_depth else None
    bg = _background(background)
    view, _topo = tree.tree_view()
    _lib.call("dot_render_fwd", _lib.ctypes.byref(view), _lib.ptr(o), _lib.ptr(d), n, _bg_ptr(bg),
              float(early_stop_eps), float(t_near), float(t_far), _lib.ptr(rgb), _lib.ptr(tfin),
              _lib.ptr(wsum), _lib.ptr(depth), _lib.stream_ptr())
    out = [io.out(rgb)]
    if return_aux:
        out += [io.out(tfin), io.out(wsum)]
    if return_depth:
        out.append(io.out(depth))
    return out[0] if len(out) == 1 else tuple(out)


def render_ray(tree: SparseOctree, ray: Ray, background, early_stop_eps: float = EPS_T) -> RenderOutput:
    """One ray: rgb, per-segment Q (zero past the cut) and final T (render.py:155-172)."""
    segs = traverse(tree, ray)
    rgb, tfin, _ = render_rays(tree, ray.origin[None, :], ray.dir[None, :], background,
                               early_stop_eps, ray.t_near, ray.t_far, return_aux=True)
    sig = tree.sigma.detach().cpu().numpy()[segs.leaf].astype(np.float64)
    alpha = np.exp(-sig * segs.delta)
    q = 1.0 - alpha
    if early_stop_eps > 0.0 and len(segs):
        trans = np.cumprod(alpha)
        cut = np.nonzero(trans < early_stop_eps)[0]
        if cut.size:
            q[int(cut[0]) + 1:] = 0.0
    return RenderOutput(rgb=rgb[0], per_segment_Q=q, transmittance_final=float(tfin[0]))


@dataclass
class BackpropWorkspace:
    """Reusable per-leaf output buffers for repeated render_and_backprop calls."""

    dsigma: torch.Tensor
    dsh_store: torch.Tensor
    signal: torch.Tensor
    touched: torch.Tensor
    loss: torch.Tensor

    @classmethod
    def for_tree(cls, tree: SparseOctree) -> "BackpropWorkspace":
        cap, dev = tree.capacity, tree.device
        return cls(torch.zeros(cap, dtype=torch.float32, device=dev),
                   torch.zeros(cap, tree.sh_stride, dtype=torch.float32, device=dev),
                   torch.zeros(cap, dtype=torch.float64, device=dev),
                   torch.zeros(cap, dtype=torch.uint8, device=dev),
                   torch.zeros(1, dtype=torch.float64, device=dev))

    def zero_(self) -> None:
        for t in (self.dsigma, self.dsh_store, self.signal, self.touched, self.loss):
            t.zero_()


@dataclass
class RayPlan:
    """A batch's coherence order: the kernel's ray index (the caller's
    ray_index composed with the key sort) and the sorted 31-bit keys (which
    also index the warp-schedule table; None for plans from a ``PoolRank``)."""

    n: int
    idx: torch.Tensor
    sorted_keys: "torch.Tensor | None"
    event: "torch.cuda.Event | None" = None
    warp_order: "torch.Tensor | None" = None  # launch order, when computed with the plan
    costs: "torch.Tensor | None" = None       # the per-ray cost column the order came from (refreshed after the backward)

    def wait(self, stream=None) -> None:
        if self.event is not None:
            (stream or torch.cuda.current_stream()).wait_event(self.event)


# All 31 key bits are sorted: dropping the finest 7 (3 radix passes instead
# of 4) made the backward 3.5 % slower (coarser coherence).
PLAN_SORT_BEGIN_BIT = int(os.environ.get("DOT_PLAN_SORT_BEGIN_BIT", "0"))


def pool_keys(tree: SparseOctree, origins: torch.Tensor, dirs: torch.Tensor) -> torch.Tensor:
    """31-bit coherence keys of every ray of a resident pool (dot_ray_keys32),
    computed once so that ``plan_batch(..., keys=)`` gathers 4 B per ray
    instead of re-reading each ray's 48 bytes at random.  Keys only order
    the work: stale keys (rays edited afterwards) cost speed, never
    correctness."""
    n = int(origins.shape[0])
    keys = torch.empty(n, dtype=torch.int32, device=tree.device)
    view, _topo = tree.tree_view()
    _lib.call("dot_ray_keys32", _lib.ctypes.byref(view), _lib.ptr(origins), _lib.ptr(dirs), n, None, n,
              _lib.ptr(keys), _lib.stream_ptr())
    return keys


class PoolRank:
    """A resident ray pool ranked by its coherence keys (``pool_rank``):
    ``rank[ray]`` = the ray's position in key order, ``order`` its inverse
    (int32 each, 8 B per pool ray).  ``plan_batch(..., rank=)`` then orders a
    batch of pool rays without a sort (``dot_plan_ranked``: a one-bit-per-
    position counting sort over a pool-sized bitmap).

    Fastest layout: the pool's arrays stored in key order once
    (``permute``), so a plan's output positions ARE the rays (no gather);
    ``in_key_order()`` is the rank for that permuted pool (callers keep
    their own ray ids; ``positions(ids)`` maps them), ``identity(n)`` the
    rank for callers that sample positions directly.  Like ``pool_keys`` it
    only orders work: stale ranks cost speed, never correctness.  The plan
    workspace belongs to this object; plans through it are ordered across
    streams by an event."""

    def __init__(self, rank: torch.Tensor | None, order: torch.Tensor | None, n_pool: int | None = None,
                 device=None):
        for t in (rank, order):
            if t is not None and t.dtype != torch.int32:
                raise InputError("rank / order must be int32 tensors of the pool's length")
        if rank is not None and order is not None and rank.shape != order.shape:
            raise InputError("rank / order must have the pool's length")
        ref = rank if rank is not None else order
        self.rank = None if rank is None else rank.contiguous()
        self.order = None if order is None else order.contiguous()
        self.n_pool = int(ref.shape[0]) if ref is not None else int(n_pool)
        self.device = ref.device if ref is not None else torch.device(device)
        self._ws = None
        self._ready = None  # event after the last plan that used the workspace

    @classmethod
    def identity(cls, n_pool: int, device) -> "PoolRank":
        """For a pool already stored in key order whose callers pass key
        positions as ray indices."""
        return cls(None, None, n_pool, device)

    def in_key_order(self) -> "PoolRank":
        """The rank of this pool after ``permute``: caller ids still map
        through ``rank``, plan outputs are positions in the permuted arrays."""
        return PoolRank(self.rank, None, self.n_pool, self.device)

    def permute(self, *tensors):
        """The pool's per-ray arrays in key order (row i = the ray at
        position i); new tensors, the inputs are untouched."""
        if self.order is None:
            raise InputError("permute needs the rank's order (pool_rank output)")
        idx = self.order.long()
        return tuple(None if t is None else t[idx] for t in tensors)

    def positions(self, ray_ids: torch.Tensor) -> torch.Tensor:
        """Key positions of caller ray ids (identity without a rank)."""
        ids = torch.as_tensor(ray_ids, device=self.device).reshape(-1).to(torch.int64)
        return ids if self.rank is None else self.rank[ids].to(torch.int64)

    def tensors(self):
        return tuple(t for t in (self.rank, self.order) if t is not None)

    def workspace(self, n: int, stream, mode: int) -> torch.Tensor:
        need = int(_lib.load().dot_plan_ranked_workspace(self.n_pool, n, mode))
        if self._ready is not None:
            stream.wait_event(self._ready)
        if self._ws is None or self._ws.numel() < need:
            with torch.cuda.stream(stream):  # zeroed where it is used
                self._ws = torch.zeros(need, dtype=torch.uint8, device=self.device)
        return self._ws

    def done(self, stream) -> None:
        self._ready = torch.cuda.Event()
        self._ready.record(stream)


def pool_rank(tree: SparseOctree, origins: torch.Tensor, dirs: torch.Tensor, bits: int | None = None) -> PoolRank:
    """Rank a resident pool once by its coherence keys for
    ``plan_batch(..., rank=)``: ``bits`` 62 (origin Morton 3 x 10 bits, then
    octahedral direction 2 x 16 bits, ``dot_ray_keys``) or 31 (the
    ``pool_keys`` keys, ties in pool order)."""
    bits = int(os.environ.get("DOT_RANK_BITS", "62")) if bits is None else bits
    if bits not in (31, 62):
        raise InputError(f"pool_rank: bits must be 31 or 62, got {bits}")
    n = int(origins.shape[0])
    if n >= 1 << 31:
        raise InputError("pool_rank: a pool must have < 2^31 rays")
    dev = tree.device
    if bits == 31:
        order = torch.argsort(pool_keys(tree, origins, dirs), stable=True)
    else:
        keys = torch.empty(n, dtype=torch.int64, device=dev)
        view, _topo = tree.tree_view()
        _lib.call("dot_ray_keys", _lib.ctypes.byref(view), _lib.ptr(origins), _lib.ptr(dirs), n, _lib.ptr(keys),
                  _lib.stream_ptr())
        order = torch.argsort(keys)  # keys < 2^62: the signed order is the key order
        del keys
    rank = torch.empty(n, dtype=torch.int32, device=dev)
    rank.scatter_(0, order, torch.arange(n, dtype=torch.int32, device=dev))
    return PoolRank(rank, order.to(torch.int32))


def ray_costs(tree: SparseOctree, origins: torch.Tensor, dirs: torch.Tensor, early_stop_eps: float = EPS_T,
              t_near: float = 0.0, t_far: float = math.inf) -> torch.Tensor:
    """Per-ray schedule cost of a ray pool (``dot_ray_costs``: composited +
    post-cut / 2 segments, int16 [n], device): the first-epoch prediction of
    each ray's share of a backward warp.  Pass it to ``plan_batch(costs=)``;
    every backward then refreshes the entries of the rays it processed with
    its own counts, so later epochs schedule from the previous visit.  Order
    only: stale or zero costs cost speed, never correctness."""
    n = int(origins.shape[0])
    cost = torch.zeros(n, dtype=torch.int16, device=tree.device)
    view, _topo = tree.tree_view(locate_level=locate_level_train())
    _lib.call("dot_ray_costs", _lib.ctypes.byref(view), _lib.ptr(origins), _lib.ptr(dirs), n, None, n,
              float(early_stop_eps), float(t_near), float(t_far), _lib.ptr(cost), _lib.stream_ptr())
    return cost


def plan_batch(tree: SparseOctree, origins: torch.Tensor, dirs: torch.Tensor, ray_index=None,
               stream=None, wait_current: bool = True, keys: torch.Tensor | None = None,
               costs: torch.Tensor | None = None, rank: PoolRank | None = None,
               ids: torch.Tensor | None = None, out: tuple | None = None) -> RayPlan:
    """Coherence order of a batch (origin / octahedral-direction Morton keys,
    dot_ray_keys32 + a radix sort).  Depends only on the rays, so it can run
    on a side stream (``stream``) ahead of the step that consumes it; the
    returned plan carries an event the consumer waits on.  ``wait_current``
    orders the side stream after the work queued so far on the current stream
    (off when the rays were produced on ``stream`` itself).  ``keys``: the
    pool's precomputed keys (``pool_keys``), gathered by ``ray_index``.
    ``costs`` (int16 per ray of the arrays, e.g. ``ray_costs``): launch the
    backward's warps longest first by these per-ray costs
    (``dot_sched_order_costs``) instead of the learned key-bucket table; the
    backward writes its fresh counts back into ``costs``.  ``rank``
    (``pool_rank``): order a batch of pool rays by the pool's 62-bit key rank
    without a sort (``dot_plan_ranked``, one cooperative launch that also
    builds the warp order from ``costs`` and regroups the rays by cost inside
    128-ray windows, so each warp holds rays of similar length); the plan
    then carries no keys, so its warp order comes only from ``costs``.
    ``ids`` (with ``rank``): the rays of ``origins`` / ``dirs`` ARE the batch
    (a staged batch) and ``ids`` their ids in the ranked dataset; the plan
    orders the batch's slots (``costs``: one entry per slot).  ``out``
    (ranked plans): preallocated (int64 [n] index, int32 [ceil(n / 32)] warp
    order) the plan writes into -- no allocation on the plan's path (e.g. per
    staging slot)."""
    idx = None if ray_index is None else torch.as_tensor(ray_index, device=tree.device).reshape(-1).to(torch.int64)
    n = int(idx.shape[0]) if idx is not None else int(origins.shape[0])
    n_pool = int(origins.shape[0])
    if costs is not None and (not isinstance(costs, torch.Tensor) or costs.dtype != torch.int16
                              or not _on_device(costs, tree.device) or costs.numel() != n_pool
                              or not costs.is_contiguous()):
        raise InputError(f"costs must be a contiguous int16 tensor with one entry per ray ({n_pool}) "
                         f"on {tree.device}")
    mode = None
    if ids is not None:
        if rank is None or idx is not None:
            raise InputError("plan_batch(ids=) needs rank= and no ray_index (the arrays are the batch)")
        idx = torch.as_tensor(ids, device=tree.device).reshape(-1).to(torch.int64)
        n = int(idx.shape[0])
        if n != n_pool:
            raise InputError(f"ids has {n} entries for a batch of {n_pool} rays")
        mode = 2  # DOT_PLAN_SLOTS
    if rank is not None:
        if idx is None:
            raise InputError("plan_batch(rank=) orders batches of a pool: pass ray_index (or ids=)")
        if keys is not None:
            raise InputError("plan_batch: pass keys= or rank=, not both")
        if not isinstance(rank, PoolRank) or not _on_device(rank.device, tree.device) or \
                (mode is None and rank.n_pool != n_pool):
            raise InputError(f"rank must be a PoolRank of this pool ({n_pool} rays) on {tree.device}")
        if mode is None:
            mode = 0 if rank.order is None else 1  # DOT_PLAN_POSITIONS / DOT_PLAN_POOL_RAYS
    view, _topo = tree.tree_view()
    cur = torch.cuda.current_stream(tree.device)
    s = stream or cur
    if s is not cur:
        if wait_current:
            s.wait_stream(cur)  # inputs produced on the current stream
        # the inputs (and the index temporary made above) are read on the side
        # stream: keep the allocator from recycling them before it is done
        for t in (idx, origins, dirs, keys, costs) + (rank.tensors() if rank is not None else ()):
            if t is not None:
                t.record_stream(s)
    with torch.cuda.stream(s):
        ranked_order = None
        if rank is not None:
            if out is not None:
                order, ranked_order = out[0][:n], out[1][:(n + 31) // 32]
                if order.dtype != torch.int64 or ranked_order.dtype != torch.int32 or order.numel() < n \
                        or ranked_order.numel() < (n + 31) // 32:
                    raise InputError("plan_batch(out=): int64 [n] index and int32 [ceil(n / 32)] warp order")
            else:
                order = torch.empty(n, dtype=torch.int64, device=tree.device)
            ws = rank.workspace(n, s, mode)
            if costs is not None and WARP_SCHED and 0 < n <= SCHED_MAX_RAYS:
                # the warp launch order in the same launch
                if out is None:
                    ranked_order = torch.empty((n + 31) // 32, dtype=torch.int32, device=tree.device)
            else:
                ranked_order = None
            _lib.call("dot_plan_ranked", _lib.ptr(rank.rank), _lib.ptr(rank.order), rank.n_pool, _lib.ptr(idx), n,
                      mode, _lib.ptr(costs if ranked_order is not None else None), cost_chunk(n),
                      _lib.ptr(ranked_order), _lib.ptr(ws), ws.numel(), _lib.ptr(order), _lib.stream_ptr(s))
            rank.done(s)
            idx, sorted_keys = order, None
        elif keys is not None:
            if idx is not None:
                pk = keys
                keys = torch.empty(n, dtype=torch.int32, device=tree.device)
                _lib.call("dot_gather_keys", _lib.ptr(pk), int(pk.shape[0]), _lib.ptr(idx), n, _lib.ptr(keys),
                          _lib.stream_ptr(s))
        else:
            keys = torch.empty(n, dtype=torch.int32, device=tree.device)
            _lib.call("dot_ray_keys32", _lib.ctypes.byref(view), _lib.ptr(origins), _lib.ptr(dirs), n_pool,
                      _lib.ptr(idx), n, _lib.ptr(keys), _lib.stream_ptr(s))
        if rank is None:
            # one radix sort carrying the ray index: the sorted values are the
            # kernel's ray_index directly
            sorted_keys = torch.empty_like(keys)
            order = torch.empty(n, dtype=torch.int64, device=tree.device)
            _lib.call("dot_plan_sort", _lib.ptr(keys), _lib.ptr(idx), n, PLAN_SORT_BEGIN_BIT,
                      _lib.ptr(sorted_keys), _lib.ptr(order), _lib.stream_ptr(s))
            idx = order
        # the warp launch order too, off the critical path: from the rays'
        # costs when given, else the learned table as of its last update
        warp_order = ranked_order
        if warp_order is None and WARP_SCHED and 0 < n <= SCHED_MAX_RAYS:
            if costs is not None:
                warp_order = torch.empty((n + 31) // 32, dtype=torch.int32, device=tree.device)
                _lib.call("dot_sched_order_costs", _lib.ptr(costs), int(costs.shape[0]), _lib.ptr(idx), n, cost_chunk(n),
                          _lib.ptr(warp_order), _lib.stream_ptr(s))
            elif sorted_keys is not None:
                warp_order = _sched_order(tree, sorted_keys, n, s)
        ev = None
        if s is not cur:
            ev = torch.cuda.Event()
            ev.record(s)
            for t in (idx, sorted_keys, warp_order):
                if t is not None:
                    t.record_stream(cur)
    return RayPlan(n, idx, sorted_keys, ev, warp_order, costs if warp_order is not None else None)


def render_and_backprop(tree: SparseOctree, origins, dirs, targets, background,
                        early_stop_eps: float = EPS_T, t_near: float = 0.0,
                        t_far: float = math.inf, grad_scale: float | None = None,
                        workspace: BackpropWorkspace | None = None, accumulate: bool = False,
                        return_rgb: bool = False, kernel_events=None, kernel_flags: int = 0,
                        coherent: bool = True, deterministic: bool = False, ray_index=None,
                        plan: "RayPlan | None" = None, weight_sum=None, weight_max=None):
    """Batch MSE loss, analytic leaf gradients and per-leaf signal (render.py:175-225).

    Returns (loss, GradBuffer, signal).  ``grad_scale`` defaults to the
    reference's 2/n; a ray-sharded caller passes 2/n_global so per-rank
    partial gradients sum to the full-batch gradient.  With numpy inputs the
    loss is a Python float and gradients are float64 numpy arrays; with torch
    inputs everything stays on the device (loss is a 0-d tensor).

    ``ray_index`` (device int64 tensor, optional; not in the reference) makes
    the batch ``origins[ray_index]`` etc. -- e.g. a random slice of a
    resident ray pool -- read in place by the kernel instead of gathered.
    ``coherent`` reorders the batch internally (origin / direction Morton
    keys) so each warp walks neighbouring cells; results are sums over rays.

    ``plan`` (``plan_batch``, optional): the batch's coherence order computed
    ahead of time -- e.g. on a side stream while the previous step runs.

    ``deterministic=True`` reduces every leaf's contributions in the
    reference's order (scatter_kernel: rays in batch order, f64 sums) via
    per-segment records + a radix sort (``dot_render_bwd_sorted``): results
    are bit-identical from run to run and the signal equals the reference's
    bit for bit.  It synchronises once per call and is slower than the
    default (warp-cooperative atomic) reduction.

    ``weight_sum`` / ``weight_max`` (device f64 [capacity] tensors, optional;
    not in the reference): accumulate per leaf the sum / max of the
    compositing weight T_i Q_i of its composited segments (the north star's
    "max/sum compositing weight" signal; atomic path only).  An index in
    ``ray_index`` outside the arrays skips that ray and makes the loss NaN.
    """
    io = _IO(tree, origins)
    o = io.rays(origins, "origins")
    d = io.rays(dirs, "dirs")
    t = io.rays(targets, "targets")
    if ray_index is not None:
        idx = torch.as_tensor(ray_index, device=tree.device).reshape(-1).to(torch.int64)
        if o.shape[0] != d.shape[0] or o.shape[0] != t.shape[0]:
            raise InputError("origins, dirs and targets must have the same length")
        if deterministic:  # the reference order is the batch order: materialise it
            o, d, t, idx = o[idx], d[idx], t[idx], None
    else:
        idx = None
    n = int(idx.shape[0]) if idx is not None else o.shape[0]
    if idx is None and (t.shape[0] != n or d.shape[0] != n):
        raise InputError(f"batch length mismatch: {n} origins, {d.shape[0]} dirs, "
                         f"{t.shape[0]} targets")
    n_pool = int(o.shape[0])
    _check_out("weight_sum", weight_sum, torch.float64, tree)
    _check_out("weight_max", weight_max, torch.float64, tree)
    if deterministic and (weight_sum is not None or weight_max is not None):
        raise InputError("weight_sum / weight_max are not available with deterministic=True")
    ws = workspace if workspace is not None else BackpropWorkspace.for_tree(tree)
    if ws.dsigma.shape[0] != tree.capacity:
        raise InputError("workspace capacity does not match the tree")
    if workspace is not None and not accumulate:
        ws.zero_()
    if return_rgb and idx is not None:
        raise InputError("return_rgb is not available with ray_index")
    rgb = torch.empty(n, 3, dtype=torch.float32, device=tree.device) if return_rgb else None
    warp_order = ray_used = sorted_keys = None
    if n:
        gs = 2.0 / n if grad_scale is None else float(grad_scale)
        bg = _background(background)
        view, _topo = tree.tree_view(locate_level=locate_level_train())
        plan_costs = None
        if plan is not None:
            if plan.n != n:
                raise InputError(f"ray plan is for {plan.n} rays, batch has {n}")
            plan.wait()
            idx, sorted_keys, warp_order, plan_costs = plan.idx, plan.sorted_keys, plan.warp_order, plan.costs
        elif coherent and n >= COHERENT_MIN_RAYS:
            p = plan_batch(tree, o, d, idx)
            idx, sorted_keys, warp_order = p.idx, p.sorted_keys, p.warp_order
        if plan_costs is not None:
            pass  # the backward writes each ray's fresh cost straight into the column
        elif sorted_keys is not None and WARP_SCHED and n <= SCHED_MAX_RAYS:
            # launch the warps whose key buckets were costliest last time first
            if warp_order is None:
                warp_order = _sched_order(tree, sorted_keys, n, torch.cuda.current_stream(tree.device))
            ray_used = torch.empty(n, dtype=torch.int16, device=tree.device)
        if kernel_events is not None:
            kernel_events[0].record()
        if deterministic:
            if rgb is not None:
                raise InputError("return_rgb is not available with deterministic=True")
            _lib.call("dot_render_bwd_sorted", _lib.ctypes.byref(view), _lib.ptr(o), _lib.ptr(d),
                      _lib.ptr(t), _lib.ptr(idx), _lib.ptr(warp_order), _lib.ptr(ray_used), n,
                      _bg_ptr(bg), float(early_stop_eps),
                      float(t_near), float(t_far), gs, _lib.ptr(ws.dsigma), _lib.ptr(ws.dsh_store),
                      tree.sh_stride, _lib.ptr(ws.signal), _lib.ptr(ws.touched), _lib.ptr(ws.loss),
                      _lib.stream_ptr())
        else:
            _lib.call("dot_render_bwd", _lib.ctypes.byref(view), _lib.ptr(o), _lib.ptr(d), _lib.ptr(t), n_pool,
                      _lib.ptr(idx), _lib.ptr(warp_order), _lib.ptr(ray_used), _lib.ptr(plan_costs), n, _bg_ptr(bg),
                      float(early_stop_eps), float(t_near), float(t_far), gs, _lib.ptr(ws.dsigma),
                      _lib.ptr(ws.dsh_store), tree.sh_stride, _lib.ptr(ws.signal), _lib.ptr(ws.touched),
                      _lib.ptr(ws.loss), _lib.ptr(rgb), _lib.ptr(weight_sum), _lib.ptr(weight_max),
                      int(kernel_flags), _lib.stream_ptr())
        if kernel_events is not None:
            kernel_events[1].record()
        if ray_used is not None:
            # write the table only after every side-stream reader queued so far
            table = _sched_table(tree)
            cur = torch.cuda.current_stream(tree.device)
            if tree._sched_read is not None:
                cur.wait_event(tree._sched_read)
            _lib.call("dot_sched_update", _lib.ptr(sorted_keys), _lib.ptr(ray_used), n,
                      _lib.ptr(table), _lib.stream_ptr())
            ev = torch.cuda.Event()
            ev.record(cur)
            tree._sched_written = ev
    nsh = 3 * tree.basis_count
    dsh = ws.dsh_store if nsh == tree.sh_stride else ws.dsh_store[:, :nsh]
    if io.numpy:
        loss = float(ws.loss.item()) / n if n else 0.0
        # the float64 numpy gradients are made on first access (GradBuffer);
        # a caller-owned workspace may be overwritten by its next call: copy now
        grads = GradBuffer(ws.dsigma, dsh, ws.touched, tree.generation, ws.dsh_store, host=True)
        if workspace is not None:
            grads.dsigma, grads.dsh, grads.touched_mask  # noqa: B018 (materialise)
            grads._dev = {"dsigma": grads.dsigma, "dsh": grads.dsh, "touched_mask": grads.touched_mask}
            grads.dsh_store = None
        out = (loss, grads, ws.signal.cpu().numpy())
        if return_rgb:
            out = out + (rgb.cpu().numpy().astype(np.float64),)
        return out
    loss = ws.loss[0] / max(n, 1)
    grads = GradBuffer(ws.dsigma, dsh, ws.touched, tree.generation, ws.dsh_store)
    out = (loss, grads, ws.signal)
    if return_rgb:
        out = out + (rgb,)
    return out


def signal_pass(tree: SparseOctree, origins, dirs, early_stop_eps: float = EPS_T, t_near: float = 0.0,
                t_far: float = math.inf, ray_index=None, buffer=None, signal=None, weight_sum=None,
                weight_max=None, touched=None, coherent: bool = True, plan: "RayPlan | None" = None):
    """Training signal without gradients (``dot_signal_fwd``): per leaf the
    sum over the batch's composited segments of Q = 1 - exp(-sigma delta) --
    exactly the ``signal`` output of ``render_and_backprop`` (render.py:
    175-225, _kernels.py:337) that ``SignalBuffer.accumulate`` consumes
    (signals.py:58-69) -- at the cost of a traversal and one sigma gather
    per segment (no SH rows, no gradient reductions), for calibration-only
    passes.

    Accumulates (+=) into ``buffer.accumulator`` (a ``SignalBuffer``; its
    ray count is bumped like ``accumulate``) or into ``signal`` (device f64
    [capacity]); with neither, a fresh zeroed array is returned.  Optional
    ``weight_sum`` / ``weight_max`` (f64 [capacity]) collect the sum / max
    of the compositing weight T_i Q_i, ``touched`` (u8 [capacity]) marks
    every traversed leaf (post-cut included).  numpy inputs give a numpy
    signal; torch inputs stay on the device (no synchronisation).  ``plan``
    (``plan_batch``, optional): the batch's order computed ahead, e.g. from a
    ranked pool with its cost column (key order regrouped by cost)."""
    io = _IO(tree, origins)
    o = io.rays(origins, "origins")
    d = io.rays(dirs, "dirs")
    n_pool = int(o.shape[0])
    if d.shape[0] != n_pool:
        raise InputError(f"batch length mismatch: {n_pool} origins, {d.shape[0]} dirs")
    idx = None
    if ray_index is not None:
        if not isinstance(ray_index, torch.Tensor):  # host indices: reject bad ones before any work
            ri = np.asarray(ray_index).reshape(-1)
            if ri.size and (ri.min() < 0 or ri.max() >= n_pool):
                raise InputError(f"ray_index entries outside [0, {n_pool})")
        idx = torch.as_tensor(ray_index, device=tree.device).reshape(-1).to(torch.int64)
    n = int(idx.shape[0]) if idx is not None else n_pool
    cap, dev = tree.capacity, tree.device
    if buffer is not None:
        buffer.check_fresh()
        signal = buffer.accumulator
    elif signal is None:
        signal = torch.zeros(cap, dtype=torch.float64, device=dev)
    for name, x, dt in (("signal", signal, torch.float64), ("weight_sum", weight_sum, torch.float64),
                        ("weight_max", weight_max, torch.float64), ("touched", touched, torch.uint8)):
        _check_out(name, x, dt, tree)
    if n:
        if plan is not None:
            if plan.n != n:
                raise InputError(f"ray plan is for {plan.n} rays, batch has {n}")
            plan.wait()
            idx = plan.idx
            if plan.warp_order is not None and n % 32 == 0:
                # the signal kernel walks its rays in array order (128-ray
                # blocks): materialise the plan's longest-first warp order
                idx = idx.view(n // 32, 32)[plan.warp_order.long()].reshape(-1)
        elif coherent and n >= COHERENT_MIN_RAYS:
            idx = plan_batch(tree, o, d, idx).idx
        view, _topo = tree.tree_view(locate_level=locate_level_train())
        invalid = torch.zeros(1, dtype=torch.int64, device=dev)
        _lib.call("dot_signal_fwd", _lib.ctypes.byref(view), _lib.ptr(o), _lib.ptr(d), n_pool, _lib.ptr(idx), n,
                  float(early_stop_eps), float(t_near), float(t_far), _lib.ptr(signal), _lib.ptr(weight_sum),
                  _lib.ptr(weight_max), _lib.ptr(touched), _lib.ptr(invalid), _lib.stream_ptr())
        if io.numpy and int(invalid.item()):
            raise InputError(f"{int(invalid.item())} ray_index entries outside [0, {n_pool})")
    if buffer is not None:
        buffer.epoch_rays += n
    return io.out(signal) if io.numpy else signal


def render_view(tree: SparseOctree, camera, background, early_stop_eps: float = EPS_T,
                return_aux: bool = False):
    """Render a pinhole ``Camera`` with in-kernel ray generation (8x4-pixel
    warp tiles, no ray arrays); returns a device tensor [H, W, 3] (f32), plus
    (T_final, depth) [H, W] with return_aux."""
    dev = tree.device
    H, W = int(camera.height), int(camera.width)
    rgb = torch.empty(H, W, 3, dtype=torch.float32, device=dev)
    tfin = torch.empty(H, W, dtype=torch.float32, device=dev) if return_aux else None
    depth = torch.empty(H, W, dtype=torch.float32, device=dev) if return_aux else None
    m = np.ascontiguousarray(camera.cam_to_world, dtype=np.float64).reshape(4, 4)
    bg = _background(background)
    view, _topo = tree.tree_view()
    _lib.call("dot_render_camera", _lib.ctypes.byref(view), m.ctypes.data_as(_lib.c_void_p),
              float(camera.focal), W, H, _bg_ptr(bg), float(early_stop_eps), _lib.ptr(rgb),
              _lib.ptr(tfin), _lib.ptr(depth), _lib.stream_ptr())
    return (rgb, tfin, depth) if return_aux else rgb


def render_views(tree: SparseOctree, cameras, background, early_stop_eps: float = EPS_T,
                 return_aux: bool = False):
    """Render many pinhole cameras of one resolution in a single launch
    (in-kernel rays, 8x4-pixel warp tiles); returns [V, H, W, 3] f32 on the
    device (+ (T_final, depth) [V, H, W] with return_aux).  Same pixels as
    ``render_view`` per camera."""
    cams = list(cameras)
    dev = tree.device
    V = len(cams)
    if V == 0:
        raise InputError("no cameras")
    H, W = int(cams[0].height), int(cams[0].width)
    if any(int(c.height) != H or int(c.width) != W for c in cams):
        raise InputError("render_views needs cameras of one resolution")
    rgb = torch.empty(V, H, W, 3, dtype=torch.float32, device=dev)
    tfin = torch.empty(V, H, W, dtype=torch.float32, device=dev) if return_aux else None
    depth = torch.empty(V, H, W, dtype=torch.float32, device=dev) if return_aux else None
    m = np.ascontiguousarray(np.stack([np.asarray(c.cam_to_world, dtype=np.float64).reshape(4, 4)
                                       for c in cams]))
    f = np.ascontiguousarray([float(c.focal) for c in cams], dtype=np.float64)
    bg = _background(background)
    view, _topo = tree.tree_view()
    _lib.call("dot_render_cameras", _lib.ctypes.byref(view), m.ctypes.data_as(_lib.c_void_p),
              f.ctypes.data_as(_lib.c_void_p), V, W, H, _bg_ptr(bg), float(early_stop_eps),
              _lib.ptr(rgb), _lib.ptr(tfin), _lib.ptr(depth), _lib.stream_ptr())
    return (rgb, tfin, depth) if return_aux else rgb


def render_image(tree: SparseOctree, camera, background, worker_count: int | None = None,
                 early_stop_eps: float = EPS_T, chunk: int = 65536,
                 exact_rays: bool = True) -> np.ndarray:
    """H x W x 3 float64 image (render.py:228-241).

    By default renders ``camera.rays()`` -- the very same f64 rays as the
    reference, so images (and ``heldout_psnr``) match it within the float
    tolerance.  ``exact_rays=False`` renders pinhole cameras
    (``cam_to_world``/``focal``) with in-kernel rays (``render_view``): no
    host ray build or copy, but directions can differ from numpy's matmul in
    the last ulp.  ``worker_count`` and ``chunk`` are accepted for API
    compatibility; results never depend on them."""
    if not exact_rays and all(hasattr(camera, a) for a in ("cam_to_world", "focal")):
        return render_view(tree, camera, background, early_stop_eps).double().cpu().numpy()
    origins, dirs = camera.rays()
    rgb = render_rays(tree, origins, dirs, background, early_stop_eps)
    return np.asarray(rgb).reshape(camera.height, camera.width, 3)
