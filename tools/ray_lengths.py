"""Distribution of per-ray work on the configs[1] training batch: traversed
segments (dot_trace_count), composited segments (ray_used of the backward),
and the per-warp maxima in the kernel's coherence order (what bounds a
warp's duration and the wave tail)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_15333_b200 import _lib, scenes  # noqa: E402
from paper_2307_15333_b200.render import BackpropWorkspace, plan_batch  # noqa: E402


def main():
    dev = torch.device("cuda")
    tree = scenes.config2_scene(device=dev)
    o, d, t = bench.build_training_pool(tree, dev)
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    idx = torch.randperm(o.shape[0], generator=g, device=dev)[: 1 << 20]
    p = plan_batch(tree, o, d, idx)
    n = p.n
    oo, dd = o[p.idx].contiguous(), d[p.idx].contiguous()
    view, _ = tree.tree_view()
    counts = torch.empty(n, dtype=torch.int64, device=dev)
    _lib.call("dot_trace_count", _lib.ctypes.byref(view), _lib.ptr(oo), _lib.ptr(dd), n, 0.0, float("inf"),
              _lib.ptr(counts), _lib.stream_ptr())
    ws = BackpropWorkspace.for_tree(tree)
    used = torch.zeros(n, dtype=torch.int16, device=dev)
    bg = np.ones(3)
    vt, _ = tree.tree_view(locate_level=9)
    _lib.call("dot_render_bwd", _lib.ctypes.byref(vt), _lib.ptr(o), _lib.ptr(d), _lib.ptr(t), o.shape[0],
              _lib.ptr(p.idx), None, _lib.ptr(used), None, n, bg.ctypes.data_as(_lib.c_void_p), 1e-4, 0.0, float("inf"),
              2.0 / n, _lib.ptr(ws.dsigma), _lib.ptr(ws.dsh_store), tree.sh_stride, _lib.ptr(ws.signal),
              _lib.ptr(ws.touched), _lib.ptr(ws.loss), None, None, None, 0, _lib.stream_ptr())
    c = counts.cpu().numpy()
    u = used.cpu().numpy().astype(np.int64)
    post = c - u
    q = [50, 90, 99, 99.9, 99.99, 100]
    print("traversed  ", dict(zip(q, np.percentile(c, q).round(1))), "mean", c.mean())
    print("composited ", dict(zip(q, np.percentile(u, q).round(1))), "mean", u.mean())
    print("post-cut   ", dict(zip(q, np.percentile(post, q).round(1))), "mean", post.mean())
    wm = c[: n // 32 * 32].reshape(-1, 32).max(1)
    wu = u[: n // 32 * 32].reshape(-1, 32).max(1)
    wsum = c[: n // 32 * 32].reshape(-1, 32).sum(1)
    print("warp max traversed ", dict(zip(q, np.percentile(wm, q).round(1))), "mean", wm.mean())
    print("warp max composited", dict(zip(q, np.percentile(wu, q).round(1))), "mean", wu.mean())
    print("lane efficiency (sum/32max) traversed", wsum.sum() / (32 * wm.sum()))
    top = np.argsort(c)[-5:]
    for r in top:
        print("long ray", r, "traversed", c[r], "composited", u[r], "o", oo[r].tolist(), "d", dd[r].tolist())


if __name__ == "__main__":
    main()
