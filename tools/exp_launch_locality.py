"""Does spatial locality between concurrently resident warps matter?  One
2^20-ray batch planned as in the bench (ranked pool, regrouped windows),
its backward launched in different warp orders, kernel time only:
  plan       the plan kernel's own order (exact warp cost; equal costs in
             atomic arrival order)
  stable     exact warp cost descending, key order inside equal costs
  bucket k   k log-scale buckets per octave of the warp cost, key order
             inside a bucket (coarser = longer key-ordered runs, fewer
             warps of different scene regions resident together)
  key        key order, no cost order (the locality extreme)."""
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
    plans = [plan_batch(tree, o, d, torch.randperm(n_pool, generator=g, device=dev)[: 1 << 20], rank=ident,
                        costs=costs) for _ in range(6)]
    ws = BackpropWorkspace.for_tree(tree)

    def run(idx, wo):
        n = idx.shape[0]
        ws.zero_()
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

    def orders(p):
        n = p.idx.shape[0]
        nb = n // 32
        wc = costs[p.idx[: nb * 32]].view(nb, 32).to(torch.int64).amax(1)
        out = {"plan": p.warp_order}
        out["stable"] = torch.argsort(-wc, stable=True)
        for k in (3, 2, 1):
            bk = torch.floor(torch.log2(wc.double() + 1.0) * k).to(torch.int64)
            out[f"bucket {k}"] = torch.argsort(-bk, stable=True)
        out["key"] = torch.arange(nb, device=dev)
        return {k: v.to(torch.int32).contiguous() for k, v in out.items()}

    res = {}
    for rep in range(3):
        for p in plans:
            for name, wo in orders(p).items():
                ms = run(p.idx, wo)
                if rep:
                    res.setdefault(name, []).append(ms)
    for name, v in res.items():
        print(f"{name:10s}: backward {np.mean(v):.4f} ms (min {np.min(v):.4f})")


if __name__ == "__main__":
    main()
