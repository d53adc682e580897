"""Micro-benchmark of the sparse RMSProp update on the configs[1] training
state: one real backward fills the gradients / touched mask, then
rmsprop_step (consume=False, so the gradients persist) is timed alone."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_15333_b200 import scenes  # noqa: E402
from paper_2307_15333_b200.optim import RmsPropState, rmsprop_step  # noqa: E402
from paper_2307_15333_b200.render import BackpropWorkspace, render_and_backprop  # noqa: E402

dev = torch.device("cuda")
tree = scenes.config2_scene(device=dev)
o_all, d_all, t_all = bench.build_training_pool(tree, dev)
g = torch.Generator(device=dev)
g.manual_seed(7)
idx = torch.randperm(o_all.shape[0], generator=g, device=dev)[: 1 << 20]
ws = BackpropWorkspace.for_tree(tree)
_loss, grads, _sig = render_and_backprop(tree, o_all, d_all, t_all, 1.0, 1e-4, workspace=ws, ray_index=idx)
state = RmsPropState(tree)
touched = int(torch.as_tensor(grads.touched_mask).sum())
for _ in range(3):
    rmsprop_step(tree, grads, state)
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        rmsprop_step(tree, grads, state)
    b.record()
    torch.cuda.synchronize()
    best = min(best, a.elapsed_time(b) / 10)
row = 4 + 4 + 8 + 3 * tree.basis_count * (4 + 4 + 8)
gb = touched * row * 2 / 1e9  # read + write of g, theta, v per touched row
print(f"{os.environ.get('VARIANT', '')}: {best * 1e3:.1f} us, touched {touched} of {tree.capacity} rows, "
      f"{gb / (best / 1e3):.0f} GB/s (g read+write, theta rw, v rw)")
