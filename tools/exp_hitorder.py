"""Experiment: order the training batch by the Morton code of each ray's
expected termination point (from a forward render with depth) instead of the
(origin, direction) coherence key, and time the backward kernel only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_15333_b200 import scenes  # noqa: E402
from paper_2307_15333_b200.render import BackpropWorkspace, render_and_backprop, render_rays  # noqa: E402


def spread(v):
    v = v & 0x3FF
    v = (v | (v << 16)) & 0x030000FF
    v = (v | (v << 8)) & 0x0300F00F
    v = (v | (v << 4)) & 0x030C30C3
    v = (v | (v << 2)) & 0x09249249
    return v


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


dev = torch.device("cuda")
tree = scenes.config2_scene(device=dev)
o_all, d_all, t_all = bench.build_training_pool(tree, dev)
g = torch.Generator(device=dev)
g.manual_seed(7)
idx = torch.randperm(o_all.shape[0], generator=g, device=dev)[: 1 << 20]
o, d, t = o_all[idx].contiguous(), d_all[idx].contiguous(), t_all[idx].contiguous()
ws = BackpropWorkspace.for_tree(tree)
ms = timeit(lambda: render_and_backprop(tree, o, d, t, 1.0, 1e-4, workspace=ws))
print(f"coherence key (in API, incl. sort): {ms:.3f} ms")
_, tf, _, dep = render_rays(tree, o, d, 1.0, 1e-4, return_aux=True, return_depth=True)
w = (1.0 - tf.double()).clamp(min=1e-6)
hit = o + d * (dep.double() / w)[:, None]
for bits, name in ((10, "hit10"), (7, "hit7"), (5, "hit5")):
    q = ((hit + 1.0) / 2.0).clamp(0, 0.999999) * (1 << bits)
    q = q.long()
    key = spread(q[:, 0]) | (spread(q[:, 1]) << 1) | (spread(q[:, 2]) << 2)
    perm = torch.argsort(key)
    oo, dd, tt = o[perm].contiguous(), d[perm].contiguous(), t[perm].contiguous()
    ms = timeit(lambda: render_and_backprop(tree, oo, dd, tt, 1.0, 1e-4, workspace=ws, coherent=False))
    print(f"{name} order (pre-sorted, kernel only): {ms:.3f} ms")
# reference: coherence order pre-sorted, kernel only
keys = torch.empty(o.shape[0], dtype=torch.int32, device=dev)
from paper_2307_15333_b200 import _lib  # noqa: E402
view, _ = tree.tree_view()
_lib.call("dot_ray_keys32", _lib.ctypes.byref(view), _lib.ptr(o), _lib.ptr(d), 0, o.shape[0], _lib.ptr(keys),
          _lib.stream_ptr())
perm = torch.argsort(keys)
oo, dd, tt = o[perm].contiguous(), d[perm].contiguous(), t[perm].contiguous()
ms = timeit(lambda: render_and_backprop(tree, oo, dd, tt, 1.0, 1e-4, workspace=ws, coherent=False))
print(f"coherence order (pre-sorted, kernel only): {ms:.3f} ms")
