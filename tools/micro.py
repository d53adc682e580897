"""Micro-benchmarks of the hot kernels on the config-2 scene (CUDA events).

    python tools/micro.py [--batch 20] [--order morton]
Prints ms per call for render_fwd on the training batch and for the backward
(dot_render_bwd flags: 0 default warp-cooperative scatter, 32768 per-lane
REDs, 8192 / 16384 timing diagnostics; "det" = deterministic sorted path)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_15333_b200 import scenes  # noqa: E402
from paper_2307_15333_b200.render import BackpropWorkspace, render_and_backprop, render_rays  # noqa: E402


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=20)
    ap.add_argument("--order", default="random")
    ap.add_argument("--flags", default="0,1,32768,det")
    args = ap.parse_args()
    dev = torch.device("cuda")
    tree = scenes.config2_scene(device=dev)
    o_all, d_all, t_all = bench.build_training_pool(tree, dev)
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    idx = torch.randperm(o_all.shape[0], generator=g, device=dev)[: 1 << args.batch]
    if args.order == "morton":
        idx = idx[torch.argsort(bench.morton_key(idx))]
    elif args.order == "raster":
        idx = idx.sort().values
    o, d, t = o_all[idx].contiguous(), d_all[idx].contiguous(), t_all[idx].contiguous()
    n = o.shape[0]
    print(f"rays {n}, order {args.order}, leaves {tree.leaf_count}")
    ms = timeit(lambda: render_rays(tree, o, d, 1.0, 1e-4))
    print(f"render_fwd           {ms:7.3f} ms   {n / ms / 1e3:8.1f} Mrays/s")
    fo, fd = bench.view_rays_torch(*scenes.hemisphere_cameras(1, 800, 800, 4.03, seed=4)[0:1],
                                   scenes.hemisphere_cameras(1, 800, 800, 4.03, seed=4)[1][0], dev)
    ms = timeit(lambda: render_rays(tree, fo, fd, 1.0, 1e-4))
    print(f"render_fwd full view {ms:7.3f} ms   {fo.shape[0] / ms / 1e3:8.1f} Mrays/s")
    ws = BackpropWorkspace.for_tree(tree)
    for f in args.flags.split(","):
        if f == "det":
            fn = lambda: render_and_backprop(tree, o, d, t, 1.0, 1e-4, workspace=ws, deterministic=True)
        else:
            fn = lambda: render_and_backprop(tree, o, d, t, 1.0, 1e-4, workspace=ws, kernel_flags=int(f))
        ms = timeit(fn)
        print(f"bwd flags={f:<5s}      {ms:7.3f} ms   {n / ms / 1e3:8.1f} Mrays/s")


if __name__ == "__main__":
    main()
