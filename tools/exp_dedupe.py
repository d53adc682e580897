"""Experiment: how often do lanes of a warp sit in the same leaf at the same
step of the walk (the dedupe a __match_any_sync aggregation of gradient REDs
could exploit)?  Batch in the training plan order (config2 scene)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_15333_b200 import scenes  # noqa: E402
from paper_2307_15333_b200.render import plan_batch, segment_batch  # noqa: E402

dev = torch.device("cuda")
tree = scenes.config2_scene(device=dev)
o_all, d_all, t_all = bench.build_training_pool(tree, dev)
g = torch.Generator(device=dev)
g.manual_seed(7)
idx = torch.randperm(o_all.shape[0], generator=g, device=dev)[: 1 << 18]
o, d = o_all[idx].contiguous(), d_all[idx].contiguous()
plan = plan_batch(tree, o, d)
o, d = o[plan.idx].contiguous(), d[plan.idx].contiguous()
off, leaf, t, dl = segment_batch(tree, o, d)
cnt = off[1:] - off[:-1]
n = o.shape[0]
for cap in (16, 32, 64, 100000):
    c = cnt.clamp(max=cap)
    S = int(c.max())
    M = torch.full((n, S), -1, dtype=torch.int64, device=dev)
    pos = torch.arange(S, device=dev)[None, :]
    valid = pos < c[:, None]
    src = (off[:-1, None] + pos).clamp(max=leaf.shape[0] - 1)
    M[valid] = leaf[src[valid]]
    W = M.view(n // 32, 32, S).transpose(1, 2)  # warp, step, lane
    s, _ = torch.sort(W, dim=2)
    act = (s >= 0).sum().item()
    uniq = ((s[:, :, 1:] != s[:, :, :-1]) & (s[:, :, 1:] >= 0)).sum().item() + (s[:, :, 0] >= 0).sum().item()
    # window: same leaf anywhere in the warp's whole (capped) walk
    Wl = M.view(n // 32, 32 * S)
    sl, _ = torch.sort(Wl, dim=1)
    uw = ((sl[:, 1:] != sl[:, :-1]) & (sl[:, 1:] >= 0)).sum().item() + (sl[:, 0] >= 0).sum().item()
    print(f"first {cap} segs: active {act}, unique per step {uniq} ({uniq / act:.3f}), "
          f"unique per warp {uw} ({uw / act:.3f})")
