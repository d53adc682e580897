import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2307_15333_b200 import scenes, _lib
from paper_2307_15333_b200 import render as R
dev = torch.device("cuda")
tree = scenes.config2_scene(device=dev)
o_all, d_all, t_all = bench.build_training_pool(tree, dev)
g = torch.Generator(device=dev); g.manual_seed(7)
idx = torch.randperm(o_all.shape[0], generator=g, device=dev)[: 1 << 20]
o, d, t = o_all[idx].contiguous(), d_all[idx].contiguous(), t_all[idx].contiguous()
ws = R.BackpropWorkspace.for_tree(tree)
for _ in range(3):
    R.render_and_backprop(tree, o, d, t, 1.0, 1e-4, workspace=ws)
torch.cuda.synchronize()
tab = R._sched_table(tree)
print("table nonzero", int((tab != 0).sum()), "max", int(tab.max()))
view, _ = tree.tree_view()
keys = torch.empty(o.shape[0], dtype=torch.int32, device=dev)
_lib.call("dot_ray_keys32", _lib.ctypes.byref(view), _lib.ptr(o), _lib.ptr(d), 0, o.shape[0], _lib.ptr(keys), _lib.stream_ptr())
sk, perm = torch.sort(keys)
wo = torch.empty((o.shape[0] + 31) // 32, dtype=torch.int32, device=dev)
_lib.call("dot_sched_order", _lib.ptr(sk), o.shape[0], _lib.ptr(tab), _lib.ptr(wo), _lib.stream_ptr())
w = wo.cpu().numpy()
print("order is perm:", np.array_equal(np.sort(w), np.arange(len(w))), "identity:", np.array_equal(w, np.arange(len(w))), w[:10], w[-5:])
b = (sk[::32].to(torch.int64) & 0x7FFFFFFF) >> 7
c = tab[b].cpu().numpy().astype(np.int64) & 0xFFFF
print("warp predicted cost: first 10 in order", c[w[:10]], "last", c[w[-10:]], "mean", c.mean(), "max", c.max())

def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

oo, dd, tt = o[perm].contiguous(), d[perm].contiguous(), t[perm].contiguous()
n = oo.shape[0]
ru = torch.empty(n, dtype=torch.int16, device=dev)
bgv = np.ones(3)
def bwd(order):
    _lib.call("dot_render_bwd", _lib.ctypes.byref(view), _lib.ptr(oo), _lib.ptr(dd), _lib.ptr(tt), 0, _lib.ptr(order), _lib.ptr(ru), n,
              bgv.ctypes.data_as(_lib.c_void_p), 1e-4, 0.0, float("inf"), 2.0 / n, _lib.ptr(ws.dsigma), _lib.ptr(ws.dsh_store),
              tree.sh_stride, _lib.ptr(ws.signal), _lib.ptr(ws.touched), _lib.ptr(ws.loss), 0, 0, _lib.stream_ptr())
print("identity order  %.3f ms" % timeit(lambda: bwd(None)))
print("table order     %.3f ms" % timeit(lambda: bwd(wo)))
used = ru.cpu().numpy().astype(np.int64) & 0xFFFF
wmax = np.zeros(len(w), np.int64)
wmax[: n // 32] = used[: (n // 32) * 32].reshape(-1, 32).max(1)
for ch in (16,):
    nc = len(w) // ch
    cm = wmax[: nc * ch].reshape(nc, ch).max(1)
    corder = np.concatenate([np.arange(c * ch, (c + 1) * ch) for c in np.argsort(-cm, kind="stable")] + [np.arange(nc * ch, len(w))]).astype(np.int32)
    co = torch.from_numpy(corder).to(dev)
    print(f"exact-used chunk-{ch} order %.3f ms" % timeit(lambda: bwd(co)))
