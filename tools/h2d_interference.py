"""Does a concurrent host->device copy slow the backward?  The backward on a
resident, ranked, cost-regrouped 2^20-ray batch timed alone and while a side
stream copies pinned host buffers (the staged loop's ~80 MB per step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_15333_b200 import scenes  # noqa: E402
from paper_2307_15333_b200.render import BackpropWorkspace, PoolRank, plan_batch, pool_rank, ray_costs, \
    render_and_backprop  # noqa: E402


def main():
    dev = torch.device("cuda")
    tree = scenes.config2_scene(device=dev)
    o, d, t = bench.build_training_pool(tree, dev)
    pr = pool_rank(tree, o, d)
    costs = ray_costs(tree, o, d)
    o, d, t, costs = pr.permute(o, d, t, costs)
    ident = PoolRank.identity(o.shape[0], dev)
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    idxs = [torch.randperm(o.shape[0], generator=g, device=dev)[: 1 << 20] for _ in range(6)]
    plans = [plan_batch(tree, o, d, i, rank=ident, costs=costs) for i in idxs]
    host = torch.empty(80 << 20, dtype=torch.uint8).pin_memory()
    devbuf = torch.empty(80 << 20, dtype=torch.uint8, device=dev)
    side = torch.cuda.Stream()
    ws = BackpropWorkspace.for_tree(tree)
    for busy in (False, True, False, True):
        ts = []
        for rep in range(2):
            for i, p in zip(idxs, plans):
                if busy:
                    with torch.cuda.stream(side):
                        for _ in range(2):
                            devbuf.copy_(host, non_blocking=True)
                ev = [torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)]
                ws.zero_()
                render_and_backprop(tree, o, d, t, 1.0, 1e-4, workspace=ws, accumulate=True, ray_index=i, plan=p,
                                    kernel_events=ev)
                torch.cuda.synchronize()
                ts.append(ev[0].elapsed_time(ev[1]))
        print(f"{'with H2D' if busy else 'alone':9s} backward {np.mean(ts[6:]):.3f} ms")


if __name__ == "__main__":
    main()
