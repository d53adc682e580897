"""ctypes binding of the C ABI in ``include/dot_b200.h`` (libdot_b200.so).

The extension is mandatory: there is no CPU fallback.  If the library is
missing or fails to load, every entry point raises immediately.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ConfigError, InputError, OctrfError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdot_b200.so")
# experiment builds only (tools/): another in-tree build of the same ABI
_LIB_OVERRIDE = os.environ.get("DOT_LIB_PATH")

DOT_OK, DOT_BAD_ARG, DOT_OOM, DOT_CUDA_ERR, DOT_NO_DEVICE = range(5)
ABI_VERSION = 12

c_void_p = ctypes.c_void_p
c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int32
c_f64 = ctypes.c_double


class DotTreeView(ctypes.Structure):
    _fields_ = [
        ("node", c_void_p), ("n_nodes", c_i64), ("sigma", c_void_p), ("sh", c_void_p),
        ("capacity", c_i64), ("basis_count", c_i32), ("sh_stride", c_i32),
        ("center", c_f64 * 3), ("half_extent", c_f64), ("max_depth", c_i32),
        ("locate_level", c_i32), ("locate", c_void_p),
    ]


MAX_PEERS = 8


class DotPeerRows(ctypes.Structure):
    _fields_ = [
        ("sigma", c_void_p * MAX_PEERS), ("sh", c_void_p * MAX_PEERS),
        ("grad_sigma", c_void_p * MAX_PEERS), ("grad_sh", c_void_p * MAX_PEERS),
        ("touched", c_void_p * MAX_PEERS), ("world", c_i32), ("rank", c_i32),
    ]


class DotRefineStats(ctypes.Structure):
    _fields_ = [
        ("leaves_before", c_i64), ("leaves_after", c_i64), ("merges_applied", c_i64),
        ("splits_applied", c_i64), ("recursion_rounds", c_i64), ("n_new_nodes", c_i64),
    ]


# name -> (restype, argtypes); every symbol declared in include/dot_b200.h
_SIGNATURES = {
    "dot_abi_version": (c_i32, []),
    "dot_last_error": (ctypes.c_char_p, []),
    "dot_device_check": (c_i32, []),
    "dot_exp_ref_host": (None, [c_void_p, c_void_p, c_i64]),
    "dot_exp_ref_device": (c_i32, [c_void_p, c_void_p, c_i64, c_void_p]),
    "dot_locate_supported": (c_i32, [c_void_p]),
    "dot_locate_build": (c_i32, [c_void_p, c_i32, c_void_p, c_void_p]),
    "dot_trace_count": (c_i32, [c_void_p, c_void_p, c_void_p, c_i64, c_f64, c_f64, c_void_p, c_void_p]),
    "dot_trace_fill": (c_i32, [c_void_p, c_void_p, c_void_p, c_i64, c_f64, c_f64, c_void_p, c_void_p,
                               c_void_p, c_void_p, c_void_p]),
    "dot_render_fwd": (c_i32, [c_void_p, c_void_p, c_void_p, c_i64, c_void_p, c_f64, c_f64, c_f64,
                               c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "dot_render_camera": (c_i32, [c_void_p, c_void_p, c_f64, c_i32, c_i32, c_void_p, c_f64, c_void_p,
                                  c_void_p, c_void_p, c_void_p]),
    "dot_render_cameras": (c_i32, [c_void_p, c_void_p, c_void_p, c_i32, c_i32, c_i32, c_void_p, c_f64, c_void_p,
                                   c_void_p, c_void_p, c_void_p]),
    "dot_render_bwd": (c_i32, [c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_void_p, c_void_p, c_void_p,
                               c_void_p, c_i64,
                               c_void_p, c_f64, c_f64, c_f64, c_f64, c_void_p, c_void_p, c_i32, c_void_p,
                               c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_i32, c_void_p]),
    "dot_signal_fwd": (c_i32, [c_void_p, c_void_p, c_void_p, c_i64, c_void_p, c_i64, c_f64, c_f64, c_f64,
                               c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "dot_render_bwd_sorted": (c_i32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                      c_i64, c_void_p,
                                      c_f64, c_f64, c_f64, c_f64, c_void_p, c_void_p, c_i32, c_void_p,
                                      c_void_p, c_void_p, c_void_p]),
    "dot_sched_order": (c_i32, [c_void_p, c_i64, c_void_p, c_void_p, c_void_p]),
    "dot_sched_update": (c_i32, [c_void_p, c_void_p, c_i64, c_void_p, c_void_p]),
    "dot_sched_order_costs": (c_i32, [c_void_p, c_i64, c_void_p, c_i64, c_i32, c_void_p, c_void_p]),
    "dot_ray_costs": (c_i32, [c_void_p, c_void_p, c_void_p, c_i64, c_void_p, c_i64, c_f64, c_f64, c_f64,
                              c_void_p, c_void_p]),
    "dot_ray_keys": (c_i32, [c_void_p, c_void_p, c_void_p, c_i64, c_void_p, c_void_p]),
    "dot_ray_keys32": (c_i32, [c_void_p, c_void_p, c_void_p, c_i64, c_void_p, c_i64, c_void_p, c_void_p]),
    "dot_gather_keys": (c_i32, [c_void_p, c_i64, c_void_p, c_i64, c_void_p, c_void_p]),
    "dot_plan_sort": (c_i32, [c_void_p, c_void_p, c_i64, c_i32, c_void_p, c_void_p, c_void_p]),
    "dot_plan_ranked_workspace": (c_i64, [c_i64, c_i64, c_i32]),
    "dot_plan_ranked": (c_i32, [c_void_p, c_void_p, c_i64, c_void_p, c_i64, c_i32, c_void_p, c_i32, c_void_p,
                                c_void_p, c_i64, c_void_p, c_void_p]),
    "dot_ray_stats":(c_i32, [c_void_p, c_void_p, c_void_p, c_i64, c_f64, c_void_p, c_void_p]),
    "dot_refine_plan_create": (c_i32, [c_void_p, c_void_p, c_void_p, c_i32, c_f64, c_f64, c_i32, c_i32,
                                       c_f64, c_void_p, c_i32, c_void_p, c_void_p, c_void_p]),
    "dot_refine_plan_lists": (c_i32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                      c_void_p]),
    "dot_refine_apply": (c_i32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                 c_void_p, c_i32, c_void_p, c_void_p]),
    "dot_refine_plan_merge_rounds": (c_i32, [c_void_p, c_void_p, c_void_p]),
    "dot_refine_plan_destroy": (None, [c_void_p]),
    "dot_rmsprop_step_peers": (c_i32, [c_void_p, c_i32, c_i32, c_i32, c_void_p, c_void_p, c_i64, c_i64, c_f64,
                                       c_f64, c_f64, c_f64, c_i32, c_void_p]),
    "dot_rmsprop_step": (c_i32, [c_void_p, c_void_p, c_i32, c_i32, c_void_p, c_void_p, c_void_p,
                                 c_void_p, c_i32, c_void_p, c_i64, c_f64, c_f64, c_f64, c_f64,
                                 c_i32, c_void_p]),
    "dot_rmsprop_step_sparse": (c_i32, [c_void_p, c_void_p, c_i32, c_i32, c_void_p, c_void_p, c_void_p,
                                        c_void_p, c_i32, c_void_p, c_i64, c_f64, c_f64, c_f64, c_f64,
                                        c_i32, c_void_p]),
    "dot_rmsprop_step_f32state": (c_i32, [c_void_p, c_void_p, c_i32, c_i32, c_void_p, c_void_p, c_void_p,
                                          c_void_p, c_i32, c_void_p, c_i64, c_f64, c_f64, c_f64, c_f64,
                                          c_i32, c_void_p]),
}

_lib = None
_lock = threading.Lock()


class ExtensionError(OctrfError):
    """The CUDA extension is missing, failed to load, or a CUDA call failed."""


def load(path: str | None = None):
    """Load libdot_b200.so (raises ExtensionError if absent -- no fallback)."""
    global _lib
    path = path or _LIB_OVERRIDE or LIB_PATH
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ExtensionError(
                f"{path} is missing; build it with `python -m paper_2307_15333_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.dot_abi_version() != ABI_VERSION:
            raise ExtensionError(f"{path} has ABI {lib.dot_abi_version()}, expected {ABI_VERSION}; "
                                 "rebuild it with `python -m paper_2307_15333_b200.build`")
        _lib = lib
        return lib


def symbols():
    return list(_SIGNATURES)


def check(status: int, what: str = "") -> None:
    if status == DOT_OK:
        return
    msg = load().dot_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status == DOT_BAD_ARG:
        raise InputError(text)
    if status == DOT_OOM:
        raise MemoryError(text)
    raise ExtensionError(text)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def ptr(t) -> int:
    """Device pointer of a torch tensor (0 for None)."""
    return 0 if t is None else int(t.data_ptr())


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


__all__ = ["DotTreeView", "DotPeerRows", "DotRefineStats", "ExtensionError", "load", "check", "call", "ptr",
           "stream_ptr", "symbols", "LIB_PATH", "ConfigError"]
