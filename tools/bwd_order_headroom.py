"""Headroom of the backward's warp launch order (diagnostic build with the
per-block timeline): one 2^20-ray batch in its coherence order, launched
(a) in the learned-schedule order, (b) by each warp's exact cost
(max over its rays of the composited + post-cut/2 count the kernel reports),
(c) by each warp's measured duration from run (a) -- the upper bound of any
cost-ordered launch.  Prints the kernel span of each.  RANKED=1: the
batch planned as in the bench (ranked pool, cost-regrouped windows)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_15333_b200 import _lib, scenes  # noqa: E402
from paper_2307_15333_b200.render import (BackpropWorkspace, PoolRank, plan_batch, pool_rank, ray_costs,
                                          render_and_backprop)  # noqa: E402


def timeline(nb):
    buf = np.zeros(2 * nb, dtype=np.uint64)
    _lib.load().dot_diag_timeline(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int(nb))
    t0, t1 = buf[0::2].astype(np.float64), buf[1::2].astype(np.float64)
    base = t0.min()
    return (t0 - base) / 1e3, (t1 - base) / 1e3


def main():
    dev = torch.device("cuda")
    tree = scenes.config2_scene(device=dev)
    o, d, t = bench.build_training_pool(tree, dev)
    g = torch.Generator(device=dev)
    for k in range(4):
        g.manual_seed(100 + k)
        idx = torch.randperm(o.shape[0], generator=g, device=dev)[: 1 << 20]
        render_and_backprop(tree, o, d, t, 1.0, ray_index=idx, workspace=BackpropWorkspace.for_tree(tree))
    g.manual_seed(999)
    if os.environ.get("RANKED"):  # the bench's plan: ranked pool in key order, regrouped windows
        pr = pool_rank(tree, o, d)
        costs = ray_costs(tree, o, d)
        o, d, t, costs = pr.permute(o, d, t, costs)
        idx = torch.randperm(o.shape[0], generator=g, device=dev)[: 1 << 20]
        p = plan_batch(tree, o, d, idx, rank=PoolRank.identity(o.shape[0], dev), costs=costs)
    else:
        idx = torch.randperm(o.shape[0], generator=g, device=dev)[: 1 << 20]
        p = plan_batch(tree, o, d, idx)
    n = p.n
    nb = n // 32
    view, _ = tree.tree_view(locate_level=7)
    bg = np.ones(3)
    used = torch.zeros(n, dtype=torch.int16, device=dev)

    def run(order):
        ws = BackpropWorkspace.for_tree(tree)
        spans = []
        for _ in range(3):
            ws.zero_()
            _lib.call("dot_render_bwd", _lib.ctypes.byref(view), _lib.ptr(o), _lib.ptr(d), _lib.ptr(t), o.shape[0],
                      _lib.ptr(p.idx), _lib.ptr(order), _lib.ptr(used), None, n, bg.ctypes.data_as(_lib.c_void_p), 1e-4,
                      0.0, float("inf"), 2.0 / n, _lib.ptr(ws.dsigma), _lib.ptr(ws.dsh_store), tree.sh_stride,
                      _lib.ptr(ws.signal), _lib.ptr(ws.touched), _lib.ptr(ws.loss), None, None, None, 0,
                      _lib.stream_ptr())
            torch.cuda.synchronize()
            t0, t1 = timeline(nb)
            spans.append(t1.max())
        return min(spans), t0, t1

    span_a, t0, t1 = run(p.warp_order)
    order_a = p.warp_order.cpu().numpy()
    dur = np.empty(nb)
    dur[order_a] = (t1 - t0)  # block b ran warp order_a[b]
    cost = used.cpu().numpy().astype(np.int64).reshape(nb, 32).max(1)
    for name, key in (("exact cost", cost), ("measured duration", dur)):
        for chunk in (1, 16):
            nc = nb // chunk
            ck = key[: nc * chunk].reshape(nc, chunk).max(1)
            co = np.argsort(-ck, kind="stable")
            order = (co[:, None] * chunk + np.arange(chunk)).reshape(-1).astype(np.int32)
            span, _, _ = run(torch.from_numpy(order).to(dev))
            print(f"{name:18s} chunk {chunk:3d}: span {span:7.0f} us")
    print(f"learned schedule        : span {span_a:7.0f} us")
    print(f"ideal packing bound     : {dur.sum() / 2960:7.0f} us (sum of warp durations / ~2960 resident warps)")


if __name__ == "__main__":
    main()
