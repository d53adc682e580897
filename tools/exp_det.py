"""Time the deterministic backward on the config-2 batch (profile range)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2307_15333_b200 import scenes
from paper_2307_15333_b200.render import BackpropWorkspace, render_and_backprop
dev = torch.device("cuda")
tree = scenes.config2_scene(device=dev)
o_all, d_all, t_all = bench.build_training_pool(tree, dev)
g = torch.Generator(device=dev); g.manual_seed(7)
idx = torch.randperm(o_all.shape[0], generator=g, device=dev)[: 1 << 20]
o, d, t = o_all[idx].contiguous(), d_all[idx].contiguous(), t_all[idx].contiguous()
ws = BackpropWorkspace.for_tree(tree)
for _ in range(3):
    render_and_backprop(tree, o, d, t, 1.0, 1e-4, workspace=ws, deterministic=True)
torch.cuda.synchronize()
torch.cuda.profiler.start()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
render_and_backprop(tree, o, d, t, 1.0, 1e-4, workspace=ws, deterministic=True)
b.record()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("det ms", a.elapsed_time(b))
