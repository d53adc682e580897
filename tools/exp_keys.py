"""Coherence-key resolution vs backward time: the production 31-bit keys vs
the 62-bit keys of dot_ray_keys (origin 10 bits per axis, octahedral
direction 16 x 16 bits), both with the cost-ordered launch.  Kernel time
only (CUDA events around dot_render_bwd), mean of 8 random 2^20-ray batches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_15333_b200 import _lib, scenes  # noqa: E402
from paper_2307_15333_b200.render import BackpropWorkspace, plan_batch, pool_keys, ray_costs  # noqa: E402


def main():
    dev = torch.device("cuda")
    tree = scenes.config2_scene(device=dev)
    o, d, t = bench.build_training_pool(tree, dev)
    n_pool = o.shape[0]
    k32 = pool_keys(tree, o, d)
    view, _ = tree.tree_view(locate_level=7)
    k64 = torch.empty(n_pool, dtype=torch.int64, device=dev)
    _lib.call("dot_ray_keys", _lib.ctypes.byref(view), _lib.ptr(o), _lib.ptr(d), n_pool, _lib.ptr(k64),
              _lib.stream_ptr())
    costs = ray_costs(tree, o, d)
    bg = np.ones(3)
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    batches = [torch.randperm(n_pool, generator=g, device=dev)[: 1 << 20] for _ in range(8)]

    def run(idx_sorted, flags=0):
        n = idx_sorted.shape[0]
        wo = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
        _lib.call("dot_sched_order_costs", _lib.ptr(costs), n_pool, _lib.ptr(idx_sorted), n, 1, _lib.ptr(wo),
                  _lib.stream_ptr())
        ws = BackpropWorkspace.for_tree(tree)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.call("dot_render_bwd", _lib.ctypes.byref(view), _lib.ptr(o), _lib.ptr(d), _lib.ptr(t), n_pool,
                  _lib.ptr(idx_sorted), _lib.ptr(wo), None, None, n, bg.ctypes.data_as(_lib.c_void_p), 1e-4, 0.0,
                  float("inf"), 2.0 / n, _lib.ptr(ws.dsigma), _lib.ptr(ws.dsh_store), tree.sh_stride,
                  _lib.ptr(ws.signal), _lib.ptr(ws.touched), _lib.ptr(ws.loss), None, None, None, flags,
                  _lib.stream_ptr())
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    flags = [int(f) for f in os.environ.get("FLAGS", "").split(",") if f]
    if flags:
        plans = [plan_batch(tree, o, d, idx, keys=k32).idx for idx in batches]
        for f in [0] + flags:
            times = [run(p, f) for p in plans + plans]
            print(f"flags {f:6d} backward {np.mean(times[8:]):.3f} ms")
        return
    for name, fn in (
            ("31-bit (production)", lambda idx: plan_batch(tree, o, d, idx, keys=k32).idx),
            ("62-bit", lambda idx: idx[torch.sort(k64[idx]).indices]),
            ("62-bit, top 40", lambda idx: idx[torch.sort(k64[idx] >> 22).indices]),
            ("62-bit, top 48", lambda idx: idx[torch.sort(k64[idx] >> 14).indices])):
        times = []
        for rep in range(2):
            for idx in batches:
                times.append(run(fn(idx)))
        print(f"{name:22s} backward {np.mean(times[8:]):.3f} ms")


if __name__ == "__main__":
    main()
