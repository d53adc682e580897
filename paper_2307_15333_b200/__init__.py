"""B200-native Dynamic PlenOctree (DOT, arXiv 2307.15333) hot path.

Drop-in for the reference package ``octrf``'s render / backward / signal /
refine path: same public names, argument meaning and errors, backed by the
sm_100a kernels in ``libdot_b200.so`` (C ABI: include/dot_b200.h).

Exports resolve lazily so ``import paper_2307_15333_b200`` stays cheap and
host-only helpers (scenes, .dot1 IO) work without loading the extension.
"""

from importlib import import_module

__version__ = "0.1.0"

_EXPORTS = {
    "SparseOctree": "octree", "LeafPayload": "octree", "TreeStats": "octree",
    "build_dense": "octree", "INVALID": "octree", "level_order": "octree",
    "EPS_T": "render", "Ray": "render", "RaySegmentList": "render", "RenderOutput": "render",
    "GradBuffer": "render", "segment_batch": "render", "traverse": "render",
    "render_rays": "render", "render_ray": "render", "render_and_backprop": "render",
    "render_image": "render", "BackpropWorkspace": "render", "signal_pass": "render",
    "render_view": "render", "render_views": "render", "plan_batch": "render",
    "pool_keys": "render", "pool_rank": "render", "PoolRank": "render", "ray_costs": "render",
    "SignalTarget": "signals", "SignalBuffer": "signals", "signal_value": "signals",
    "signal_values": "signals",
    "CalibrationConfig": "calibrate", "CalibrationReport": "calibrate", "calibrate": "calibrate",
    "prune": "calibrate", "sample": "calibrate", "select_prune": "calibrate",
    "select_sample": "calibrate",
    "RmsPropState": "optim", "rmsprop_step": "optim", "TrainConfig": "optim",
    "train_epoch": "optim", "train": "optim", "train_step": "optim", "StepWorkspace": "optim",
    "heldout_psnr": "optim", "write_history": "optim", "ResidentRays": "optim",
    "Camera": "scene_io", "look_at": "scene_io", "orbit_cameras": "scene_io",
    "save_tree": "scene_io", "load_tree": "scene_io",
    "RayBatchStager": "staging", "LossReader": "staging",
    "eval_sh_basis": "sh", "eval_sh_basis_many": "sh", "decode_color": "sh", "sh_from_rgb": "sh",
}

__all__ = sorted(_EXPORTS) + ["errors", "__version__"]


def __getattr__(name):
    if name == "errors":
        return import_module(".errors", __name__)
    mod = _EXPORTS.get(name)
    if mod is None:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
    value = getattr(import_module(f".{mod}", __name__), name)
    globals()[name] = value
    return value
