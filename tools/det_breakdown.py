"""Kernel breakdown of one deterministic backward (dot_render_bwd_sorted) on
a configs[1] 2^20-ray batch: torch.profiler kernel durations and the wall
time of the call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_15333_b200 import scenes  # noqa: E402
from paper_2307_15333_b200.render import BackpropWorkspace, render_and_backprop  # noqa: E402


def main():
    dev = torch.device("cuda")
    tree = scenes.config2_scene(device=dev)
    o, d, t = bench.build_training_pool(tree, dev)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    idx = torch.randperm(o.shape[0], generator=g, device=dev)[: 1 << 20]
    ob, db, tb = o[idx].contiguous(), d[idx].contiguous(), t[idx].contiguous()
    ws = BackpropWorkspace.for_tree(tree)
    for _ in range(2):
        render_and_backprop(tree, ob, db, tb, 1.0, 1e-4, workspace=ws, deterministic=True)
    torch.cuda.synchronize()
    c = time.perf_counter()
    for _ in range(3):
        render_and_backprop(tree, ob, db, tb, 1.0, 1e-4, workspace=ws, deterministic=True)
    torch.cuda.synchronize()
    print(f"wall per call {1e3 * (time.perf_counter() - c) / 3:.3f} ms")
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        render_and_backprop(tree, ob, db, tb, 1.0, 1e-4, workspace=ws, deterministic=True)
        torch.cuda.synchronize()
    tot = {}
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            tot[e.name[:70]] = tot.get(e.name[:70], 0.0) + e.device_time_total
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:14]:
        print(f"{v:9.1f} us  {k}")


if __name__ == "__main__":
    main()
