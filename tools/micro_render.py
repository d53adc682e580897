"""Micro-benchmark of the configs[2] render: 200 800x800 hemisphere views in
one render_views launch (in-kernel rays), CUDA events, best of 3."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_15333_b200 import scenes  # noqa: E402
from paper_2307_15333_b200.render import render_views  # noqa: E402
from paper_2307_15333_b200.scene_io import Camera  # noqa: E402

dev = torch.device("cuda")
tree = scenes.config2_scene(device=dev)
focal, poses = scenes.hemisphere_cameras(200, bench.W, bench.H, bench.RADIUS, seed=4)
cams = [Camera(bench.W, bench.H, focal, p) for p in poses]
for _ in range(3):
    render_views(tree, cams, bench.BG, bench.EPS)
torch.cuda.synchronize()
best = 1e9
for _ in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    render_views(tree, cams, bench.BG, bench.EPS)
    b.record()
    torch.cuda.synchronize()
    best = min(best, a.elapsed_time(b))
print(f"{os.environ.get('VARIANT', '')}: {best:.3f} ms / 200 views, {bench.W * bench.H * 200 / best / 1e6:.3e} rays/s")
