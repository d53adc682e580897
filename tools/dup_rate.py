"""How often do lanes of one backward warp scatter into the same leaf in the
same pass-2 step?  (Upper bound on what merging equal-leaf rows inside a
warp round could save in SH-gradient reductions.)  Coherence-ordered 2^20
batch of the configs[1] pool; the first 2^17 rays in plan order."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_15333_b200 import scenes  # noqa: E402
from paper_2307_15333_b200.render import plan_batch, pool_keys, segment_batch  # noqa: E402


def main():
    dev = torch.device("cuda")
    tree = scenes.config2_scene(device=dev)
    o, d, t = bench.build_training_pool(tree, dev)
    k32 = pool_keys(tree, o, d)
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    idx = torch.randperm(o.shape[0], generator=g, device=dev)[: 1 << 20]
    pidx = plan_batch(tree, o, d, idx, keys=k32).idx
    sigma = tree.sigma.double()
    for start in (0, 1 << 19):
        sel = pidx[start:start + (1 << 17)]
        off, leaf, _, dl = segment_batch(tree, o[sel].contiguous(), d[sel].contiguous())
        a = torch.exp(-sigma[leaf] * dl)
        n = sel.shape[0]
        ray = torch.repeat_interleave(torch.arange(n, device=dev), off[1:] - off[:-1])
        # transmittance before each segment (per-ray exclusive cumprod)
        la = torch.log(a.clamp_min(1e-300))
        cs = torch.cumsum(la, 0)
        base = torch.cat([torch.zeros(1, device=dev, dtype=cs.dtype), cs])[off[:-1]][ray]
        tb = torch.exp(cs - la - base)
        comp = tb >= 1e-4  # composited (the segment that crosses eps is included)
        live = comp & (a < 1.0)
        step = torch.arange(leaf.shape[0], device=dev) - off[:-1][ray]
        warp = ray // 32
        sel_l = live.nonzero().squeeze(1)
        key_round = warp[sel_l] * 4096 + step[sel_l]
        rows = sel_l.shape[0]
        rounds = torch.unique(key_round).shape[0]
        distinct = torch.unique(key_round * (1 << 27) + leaf[sel_l]).shape[0]
        # pairs (round) -> any duplicate count, and per-warp window (all steps)
        distinct_warp = torch.unique(warp[sel_l] * (1 << 27) + leaf[sel_l]).shape[0]
        print(f"rays {start}..: rows {rows} rounds {rounds} lanes/round {rows / rounds:.1f}  "
              f"distinct (round,leaf) {distinct} -> {distinct / rows:.3f} of rows;  "
              f"distinct (warp,leaf) {distinct_warp / rows:.3f}")


if __name__ == "__main__":
    main()
