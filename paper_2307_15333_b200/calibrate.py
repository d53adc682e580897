"""Signal-guided structural calibration (DOT refine) on the device.

Same API and selection rules as ``octrf.calibrate``
(/root/reference/pkg/src/octrf/calibrate.py:22-249); the pass itself runs
in ``dot_refine_plan_create`` / ``dot_refine_apply`` (csrc/refine.cu):
prune (one-shot or recursive), sample on the post-prune topology, and a
canonical BFS rebuild of the tree in one go.

Id spaces.  The reference mutates its pool in place (LIFO slot reuse) and
its report's events carry pool ids.  Here the refined tree is written
canonically (pool id == BFS index, capacity == node count).  Report events
are therefore ("merge", old parent id, old kid ids) and ("split", old leaf
id, new kid ids); ``report.remap`` carries the device-side old->new mapping
that ``RmsPropState.remap`` consumes.  Compare topologies after
canonicalisation (``save_tree`` bytes), as SURVEY.md section 0.3 prescribes.
"""

from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ConfigError
from .signals import SignalBuffer, SignalTarget

K_KEPT, K_MERGED, K_NEWCHILD, K_SPLITPARENT = 0, 1, 2, 3


@dataclass
class CalibrationConfig:
    tau: float = 1.0
    gamma: float = 0.01
    recursive: bool = False
    sample_threshold: float | None = None
    check_invariants: bool = False

    def __post_init__(self):
        if self.tau < 0:
            raise ConfigError(f"tau must be >= 0, got {self.tau}")
        if not 0.0 <= self.gamma <= 1.0:
            raise ConfigError(f"gamma must be in [0, 1], got {self.gamma}")
        if self.sample_threshold is not None and self.sample_threshold < 0:
            raise ConfigError("sample_threshold must be >= 0")


@dataclass
class RefineRemap:
    """Device-side description of one refine: for every new canonical node,
    the old canonical node it comes from and how (K_* codes), plus the merge
    rounds needed to average per-leaf state the way the reference does."""

    old_node: torch.Tensor          # int32 [n_old] old canonical node table
    old_pool_id: torch.Tensor | None  # int32 [n_old] pool ids (None = identity)
    src_index: torch.Tensor         # int64 [n_new]
    src_kind: torch.Tensor          # uint8 [n_new]
    merge_round: torch.Tensor       # int32 [n_old]: prune round that merged the node, 0 = none
    rounds: int


class CalibrationReport:
    """calibrate.py:45-68.  ``events`` is materialised on first access from
    the device-side ``remap`` (merge rounds, split sources, the new node
    table), so a report nobody reads the events of costs no host work."""

    def __init__(self, leaves_before: int, leaves_after: int, merges_applied: int, splits_applied: int,
                 recursion_rounds: int, events: list | None = None, remap: "RefineRemap | None" = None,
                 new_node: torch.Tensor | None = None):
        self.leaves_before = leaves_before
        self.leaves_after = leaves_after
        self.merges_applied = merges_applied
        self.splits_applied = splits_applied
        self.recursion_rounds = recursion_rounds
        self.remap = remap
        self._new_node = new_node
        self._events = events

    @property
    def events(self) -> list:
        if self._events is None:
            self._events = _events_from_remap(self.remap, self._new_node)
        return self._events

    @events.setter
    def events(self, value):
        self._events = value

    def __repr__(self) -> str:
        return (f"CalibrationReport(leaves_before={self.leaves_before}, leaves_after={self.leaves_after}, "
                f"merges_applied={self.merges_applied}, splits_applied={self.splits_applied}, "
                f"recursion_rounds={self.recursion_rounds})")

    def to_json(self) -> str:
        return json.dumps({
            "leaves_before": self.leaves_before,
            "leaves_after": self.leaves_after,
            "merges_applied": self.merges_applied,
            "splits_applied": self.splits_applied,
            "recursion_rounds": self.recursion_rounds,
        })


class _Plan:
    """RAII wrapper of a dot_refine_plan."""

    def __init__(self, tree, acc, use_sigma, tau, gamma, recursive, threshold):
        self.tree = tree
        self.view, self.topo = tree.tree_view(locate=False)
        self.acc = acc
        stats = _lib.DotRefineStats()
        handle = ctypes.c_void_p()
        off = np.ascontiguousarray(self.topo.level_offsets, dtype=np.int64)
        _lib.call("dot_refine_plan_create", ctypes.byref(self.view), _lib.ptr(self.topo.pool_id),
                  _lib.ptr(acc), int(use_sigma), float(tau), float(gamma), int(recursive),
                  int(threshold is not None), float(threshold or 0.0),
                  off.ctypes.data_as(ctypes.c_void_p), int(off.size), ctypes.byref(handle),
                  ctypes.byref(stats), _lib.stream_ptr())
        self.handle = handle
        self.stats = stats
        self._lists = None

    def _fetch_lists(self):
        if self._lists is None:
            mp, nm, sl, ns, mr = (ctypes.POINTER(ctypes.c_int64)(), ctypes.c_int64(),
                                  ctypes.POINTER(ctypes.c_int64)(), ctypes.c_int64(),
                                  ctypes.POINTER(ctypes.c_int32)())
            _lib.call("dot_refine_plan_lists", self.handle, ctypes.byref(mp), ctypes.byref(nm),
                      ctypes.byref(sl), ctypes.byref(ns), ctypes.byref(mr), _lib.stream_ptr())
            self._lists = (
                np.ctypeslib.as_array(mp, (nm.value,)).copy() if nm.value else np.empty(0, np.int64),
                np.ctypeslib.as_array(mr, (nm.value,)).copy() if nm.value else np.empty(0, np.int32),
                np.ctypeslib.as_array(sl, (ns.value,)).copy() if ns.value else np.empty(0, np.int64))
        return self._lists

    @property
    def merge_parents(self):
        return self._fetch_lists()[0]

    @property
    def merge_round(self):
        return self._fetch_lists()[1]

    @property
    def split_leaves(self):
        return self._fetch_lists()[2]

    def pool_ids(self, canon: np.ndarray) -> np.ndarray:
        if self.topo.pool_id is None:
            return canon.astype(np.int64)
        return self.topo.pool_id.cpu().numpy()[canon].astype(np.int64)

    def apply(self) -> RefineRemap:
        tree = self.tree
        n_new = int(self.stats.n_new_nodes)
        dev = tree.device
        new_node = torch.empty(n_new, dtype=torch.int32, device=dev)
        new_sigma = torch.empty(n_new, dtype=torch.float32, device=dev)
        new_sh = torch.empty(n_new, tree.sh_stride, dtype=torch.float32, device=dev)
        src_index = torch.empty(n_new, dtype=torch.int64, device=dev)
        src_kind = torch.empty(n_new, dtype=torch.uint8, device=dev)
        max_levels = 64
        offs = np.zeros(max_levels + 1, dtype=np.int64)
        nlev = ctypes.c_int32()
        _lib.call("dot_refine_apply", self.handle, ctypes.byref(self.view), _lib.ptr(new_node),
                  _lib.ptr(new_sigma), _lib.ptr(new_sh), _lib.ptr(src_index), _lib.ptr(src_kind),
                  offs.ctypes.data_as(ctypes.c_void_p), max_levels, ctypes.byref(nlev),
                  _lib.stream_ptr())
        mround = torch.empty(self.topo.n_nodes, dtype=torch.int32, device=dev)
        _lib.call("dot_refine_plan_merge_rounds", self.handle, _lib.ptr(mround), _lib.stream_ptr())
        remap = RefineRemap(self.topo.node, self.topo.pool_id, src_index, src_kind, mround,
                            int(self.stats.recursion_rounds))
        tree._set_canonical(new_node, new_sigma, new_sh, int(self.stats.leaves_after),
                            offs[:nlev.value + 1].copy())
        return remap

    def close(self):
        if self.handle:
            _lib.load().dot_refine_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _acc_for(buffer: SignalBuffer, acc=None):
    use_sigma = buffer.target is SignalTarget.DENSITY_SIGMA
    a = buffer.accumulator if acc is None else acc
    a = torch.as_tensor(a, dtype=torch.float64).to(buffer.tree.device).contiguous()
    return a, use_sigma


def _events_from_remap(remap: RefineRemap | None, new_node: torch.Tensor | None) -> list:
    """Reference-style event list (calibrate.py:45-68), vectorised: merges
    ("merge", parent, kids) by (round, pool id) with old pool ids, then splits
    ("split", leaf, kids) by ascending pool id with the new canonical ids of
    the 8 children (the refined tree is canonical, see module docstring)."""
    if remap is None:
        return []
    node_old = remap.old_node.cpu().numpy().astype(np.int64)
    pool = (remap.old_pool_id.cpu().numpy().astype(np.int64) if remap.old_pool_id is not None
            else np.arange(node_old.size, dtype=np.int64))
    mr = remap.merge_round.cpu().numpy()
    p = np.nonzero(mr)[0]
    p = p[np.lexsort((pool[p], mr[p]))]
    mk = pool[node_old[p][:, None] + np.arange(8)]
    ev = [("merge", a, tuple(b)) for a, b in zip(pool[p].tolist(), mk.tolist())]
    kind = remap.src_kind.cpu().numpy()
    sp = np.nonzero(kind == K_SPLITPARENT)[0]
    if sp.size:
        leaf = pool[remap.src_index.cpu().numpy()[sp]]
        first = new_node.cpu().numpy().astype(np.int64)[sp]
        o = np.argsort(leaf, kind="stable")
        kids = first[o][:, None] + np.arange(8)
        ev += [("split", a, tuple(b)) for a, b in zip(leaf[o].tolist(), kids.tolist())]
    return ev


def _run(tree, buffer, tau, gamma, recursive, threshold, apply=True, acc=None, events=True,
         lists=False):
    a, use_sigma = _acc_for(buffer, acc)
    plan = _Plan(tree, a, use_sigma, tau, gamma, recursive, threshold)
    try:
        st = plan.stats
        if lists:
            plan._fetch_lists()  # before apply: the lists describe the old tree
        remap = plan.apply() if apply else None
        new_node = tree.topology().node if apply else None
        report = CalibrationReport(int(st.leaves_before), int(st.leaves_after),
                                   int(st.merges_applied), int(st.splits_applied),
                                   int(st.recursion_rounds), None if events else [], remap, new_node)
        return report, plan
    finally:
        plan.close()


def select_prune(tree, buffer: SignalBuffer, tau: float) -> np.ndarray:
    """Parents of all-leaf sibling sets whose signals all sit <= tau (ascending ids)."""
    buffer.check_fresh()
    if tau < 0:
        raise ConfigError(f"tau must be >= 0, got {tau}")
    _, plan = _run(tree, buffer, tau, 0.0, 0, None, apply=False, events=False, lists=True)
    return np.sort(plan.pool_ids(plan.merge_parents))


def prune(tree, buffer: SignalBuffer, tau: float, recursive: bool = False) -> CalibrationReport:
    """Merge every selected sibling set; optionally repeat to a fixed point."""
    buffer.check_fresh()
    if tau < 0:
        raise ConfigError(f"tau must be >= 0, got {tau}")
    report, _ = _run(tree, buffer, tau, 0.0, 1 if recursive else 0, None)
    return report


def select_sample(tree, buffer: SignalBuffer, gamma: float, threshold=None) -> np.ndarray:
    """The hottest ceil(gamma*L) leaves (ties -> smaller id), or all above threshold."""
    buffer.check_fresh()
    if not 0.0 <= gamma <= 1.0:
        raise ConfigError(f"gamma must be in [0, 1], got {gamma}")
    _, plan = _run(tree, buffer, 0.0, gamma, -1, threshold, apply=False, events=False,
                   lists=True)
    return np.sort(plan.pool_ids(plan.split_leaves))


def sample(tree, buffer: SignalBuffer, gamma: float, threshold=None) -> CalibrationReport:
    """Split every selected leaf; payload copies keep renders unchanged."""
    buffer.check_fresh()
    if not 0.0 <= gamma <= 1.0:
        raise ConfigError(f"gamma must be in [0, 1], got {gamma}")
    report, _ = _run(tree, buffer, 0.0, gamma, -1, threshold)
    return report


def calibrate(tree, buffer: SignalBuffer, config: CalibrationConfig,
              events: bool = True) -> CalibrationReport:
    """One calibration event: prune, sample on the post-prune topology, reset.

    ``report.events`` is built lazily on first access (``events=False``
    returns an empty list instead)."""
    buffer.check_fresh()
    gamma = config.gamma if (config.sample_threshold is not None or config.gamma > 0.0) else 0.0
    report, _ = _run(tree, buffer, config.tau, gamma, 1 if config.recursive else 0,
                     config.sample_threshold, events=events)
    if config.check_invariants:
        tree.validate()
    buffer.reset()
    return report
