"""Experiment: how well does a table of past per-warp costs, keyed by the top
bits of the coherence key, predict the next batch's per-warp cost?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2307_15333_b200 import scenes, _lib
from paper_2307_15333_b200.render import BackpropWorkspace, render_and_backprop
dev = torch.device("cuda")
tree = scenes.config2_scene(device=dev)
o_all, d_all, t_all = bench.build_training_pool(tree, dev)
g = torch.Generator(device=dev); g.manual_seed(7)
perm = torch.randperm(o_all.shape[0], generator=g, device=dev)
ws = BackpropWorkspace.for_tree(tree)
view, _ = tree.tree_view()
def batch(k):
    idx = perm[k << 20:(k + 1) << 20]
    o, d, t = o_all[idx].contiguous(), d_all[idx].contiguous(), t_all[idx].contiguous()
    keys = torch.empty(o.shape[0], dtype=torch.int32, device=dev)
    _lib.call("dot_ray_keys32", _lib.ctypes.byref(view), _lib.ptr(o), _lib.ptr(d), 0, o.shape[0], _lib.ptr(keys), _lib.stream_ptr())
    p = torch.argsort(keys)
    o, d, t, keys = o[p].contiguous(), d[p].contiguous(), t[p].contiguous(), keys[p]
    _, _, _, rgb = render_and_backprop(tree, o, d, t, 1.0, 1e-4, workspace=ws, coherent=False, return_rgb=True, kernel_flags=2048)
    used = rgb.reshape(-1)[0::3][: o.shape[0]].cpu().numpy()
    return keys.cpu().numpy().astype(np.int64), used
for bits in (16, 20, 24):
    tab = {}
    for k in range(4):
        keys, used = batch(k)
        wkey = keys[0::32] >> (31 - bits)
        wmax = used.reshape(-1, 32).max(1)
        if k >= 1:
            pred = np.array([tab.get(int(x), np.nan) for x in wkey])
            ok = ~np.isnan(pred)
            from scipy.stats import spearmanr
            rho = spearmanr(pred[ok], wmax[ok]).correlation
            print(f"bits {bits} step {k}: coverage {ok.mean():.2f} spearman {rho:.3f}")
        for x, m in zip(wkey, wmax):
            tab[int(x)] = max(tab.get(int(x), 0), m) if False else 0.5 * tab.get(int(x), m) + 0.5 * m
