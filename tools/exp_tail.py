import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2307_15333_b200 import scenes
from paper_2307_15333_b200.render import BackpropWorkspace, render_and_backprop
dev = torch.device("cuda")
tree = scenes.config2_scene(device=dev)
o_all, d_all, t_all = bench.build_training_pool(tree, dev)
g = torch.Generator(device=dev); g.manual_seed(7)
idx = torch.randperm(o_all.shape[0], generator=g, device=dev)[: 1 << 20]
ws = BackpropWorkspace.for_tree(tree)
o, d, t = o_all[idx].contiguous(), d_all[idx].contiguous(), t_all[idx].contiguous()
for _ in range(3):
    out = render_and_backprop(tree, o, d, t, 1.0, 1e-4, workspace=ws, return_rgb=True, kernel_flags=2048)
torch.cuda.synchronize()
rgb = out[3]
ts = rgb.reshape(-1).view(torch.int64)[: 4 * ((o.shape[0] + 31) // 32)].reshape(-1, 4).cpu().numpy()
t0, t1, sm, maxu = ts[:, 0], ts[:, 1], ts[:, 2], ts[:, 3]
span = t1.max() - t0.min()
print("kernel span us", span / 1e3, "warps", len(t0))
dur = (t1 - t0) / 1e3
print("warp dur us: mean %.1f p50 %.1f p90 %.1f p99 %.1f max %.1f" % (dur.mean(), np.median(dur), np.percentile(dur, 90), np.percentile(dur, 99), dur.max()))
# active warps over time
tt = np.linspace(t0.min(), t1.max(), 41)
act = [int(((t0 <= x) & (t1 > x)).sum()) for x in tt[:-1]]
print("active warps over time (40 bins):", act)
print("mean active", np.mean(act), "of", 148 * 32)
# when does the last warp start
print("last start at %.1f%% of span" % (100 * (t0.max() - t0.min()) / span))
print("corr(maxu, dur)", np.corrcoef(maxu, dur)[0, 1], "maxu mean", maxu.mean())

# ideal LPT: launch warps in descending measured duration (same batch, same order of rays)
import ctypes
from paper_2307_15333_b200 import _lib
lib = _lib.load()
order = torch.from_numpy(np.argsort(-dur, kind="stable").astype(np.int32)).to(dev)
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
# the API sorts by coherence key internally: replicate its order so warp ids match
keys = torch.empty(o.shape[0], dtype=torch.int32, device=dev)
view, _ = tree.tree_view()
_lib.call("dot_ray_keys32", _lib.ctypes.byref(view), _lib.ptr(o), _lib.ptr(d), 0, o.shape[0], _lib.ptr(keys), _lib.stream_ptr())
perm = torch.argsort(keys)
oo, dd, tt = o[perm].contiguous(), d[perm].contiguous(), t[perm].contiguous()
base = timeit(lambda: render_and_backprop(tree, oo, dd, tt, 1.0, 1e-4, workspace=ws, coherent=False))
lib.dot_exp_set_warp_order(ctypes.c_void_p(order.data_ptr()))
lpt = timeit(lambda: render_and_backprop(tree, oo, dd, tt, 1.0, 1e-4, workspace=ws, coherent=False))
# coarse LPT: keep chunks of 64 consecutive warps together, order chunks by max duration
ch = 64
nw = len(dur)
cd = np.array([dur[i:i + ch].max() for i in range(0, nw, ch)])
corder = np.concatenate([np.arange(c * ch, min((c + 1) * ch, nw)) for c in np.argsort(-cd, kind="stable")]).astype(np.int32)
corder_t = torch.from_numpy(corder).to(dev)
lib.dot_exp_set_warp_order(ctypes.c_void_p(corder_t.data_ptr()))
lpt64 = timeit(lambda: render_and_backprop(tree, oo, dd, tt, 1.0, 1e-4, workspace=ws, coherent=False))
lib.dot_exp_set_warp_order(None)
print(f"kernel-only coherent order {base:.3f} ms, ideal LPT {lpt:.3f} ms, chunk-64 LPT {lpt64:.3f} ms")
