"""Backward time when rays are re-sorted by cost inside windows of G
consecutive rays of the key-ordered batch (warps of similar-cost rays,
still spatially near), warps launched longest first.  Kernel time only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_15333_b200 import _lib, scenes  # noqa: E402
from paper_2307_15333_b200.render import BackpropWorkspace, PoolRank, plan_batch, pool_rank, ray_costs  # noqa: E402


def main():
    dev = torch.device("cuda")
    tree = scenes.config2_scene(device=dev)
    o, d, t = bench.build_training_pool(tree, dev)
    pr = pool_rank(tree, o, d)
    costs = ray_costs(tree, o, d)
    o, d, t, costs = pr.permute(o, d, t, costs)
    n_pool = o.shape[0]
    ident = PoolRank.identity(n_pool, dev)
    view, _ = tree.tree_view(locate_level=7)
    bg = np.ones(3)
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    plans = [plan_batch(tree, o, d, torch.randperm(n_pool, generator=g, device=dev)[: 1 << 20], rank=ident).idx
             for _ in range(8)]

    def run(idx):
        n = idx.shape[0]
        wo = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
        _lib.call("dot_sched_order_costs", _lib.ptr(costs), n_pool, _lib.ptr(idx), n, 1, _lib.ptr(wo),
                  _lib.stream_ptr())
        ws = BackpropWorkspace.for_tree(tree)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.call("dot_render_bwd", _lib.ctypes.byref(view), _lib.ptr(o), _lib.ptr(d), _lib.ptr(t), n_pool,
                  _lib.ptr(idx), _lib.ptr(wo), None, None, n, bg.ctypes.data_as(_lib.c_void_p), 1e-4, 0.0,
                  float("inf"), 2.0 / n, _lib.ptr(ws.dsigma), _lib.ptr(ws.dsh_store), tree.sh_stride,
                  _lib.ptr(ws.signal), _lib.ptr(ws.touched), _lib.ptr(ws.loss), None, None, None, 0,
                  _lib.stream_ptr())
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    buckets = int(os.environ.get("BUCKETS", "0"))  # > 0: sort by a log-scale cost bucket instead of the cost
    for G in [int(x) for x in os.environ.get("WINDOWS", "32,64,128,256,512,1024").split(",")]:
        times = []
        for rep in range(2):
            for idx in plans:
                n = idx.shape[0]
                m = n // G * G  # a ragged tail keeps its order
                c = costs[idx[:m]].view(-1, G)
                if buckets:
                    c = torch.clamp((torch.log2(c.float() + 1.0) * (buckets / 10.0)).long(), max=buckets - 1)
                order = c.argsort(dim=1, descending=True, stable=True)
                j = (order + torch.arange(0, m, G, device=dev).view(-1, 1)).reshape(m)
                times.append(run(torch.cat([idx[:m][j], idx[m:]]).contiguous()))
        print(f"window {G:5d}: backward {np.mean(times[8:]):.3f} ms")


if __name__ == "__main__":
    main()
